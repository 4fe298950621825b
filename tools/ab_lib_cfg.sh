#!/bin/bash
# usage: tools/ab_lib_cfg.sh CONFIG [rounds] -- A/B of liblouver_b200_before.so vs _after.so on one bench config (GPU box)
for i in $(seq ${2:-2}); do
  for v in before after; do
    cp paper_2605_06763_b200/liblouver_b200_$v.so paper_2605_06763_b200/liblouver_b200.so
    echo -n "$v "; python bench.py --config $1 --steps 200 --warmup 5 --no-cpu-baseline --no-dense-lib 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],3), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value'],2))"
  done
done
cp paper_2605_06763_b200/liblouver_b200_after.so paper_2605_06763_b200/liblouver_b200.so
