#!/bin/bash
# usage (GPU box): bash tools/round_artifacts.sh TAG -- the round's committed evidence into
# gpurun_out/: bench lines per config, the reference arm, the GPU test log, the ncu launch
# list of the default bench command and one ncu --set full capture of the layer kernel.
tag=${1:-r02}
o=gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > $o/${tag}_gputest.log 2>&1; tail -1 $o/${tag}_gputest.log
for c in c2 c3 c1; do
  timeout 900 python bench.py --config $c > $o/${tag}_bench_$c.json 2> $o/${tag}_bench_$c.err; echo "$c rc=$?"
done
timeout 1200 python bench.py --config c5 > $o/${tag}_bench_c5_1gpu.json 2> $o/${tag}_bench_c5.err; echo "c5 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $o/${tag}_bench_reference.json 2> $o/${tag}_bench_reference.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:louver_layer_v9 -c 300 --csv \
  --log-file $o/${tag}_launches.csv python bench.py --steps 8 --warmup 4 --no-cpu-baseline > $o/${tag}_launches_bench.log 2>&1
echo "launches rc=$?"
WHICH=query REPS=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:louver_layer_v9 -s 1 -c 1 \
  -o $o/${tag}_layer_full python tools/profile_layer.py > $o/${tag}_ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py $o/${tag}_layer_full.ncu-rep > $o/${tag}_layer_v9_ncu_full.txt 2>&1
timeout 600 python tools/trace_bench.py > $o/${tag}_trace.txt 2>&1; echo "trace rc=$?"
