#!/bin/bash
# usage: tools/ab.sh [runs] -- prints value/frac of a short C2 bench per run (GPU box)
runs=${1:-2}
for i in $(seq $runs); do
  python bench.py --steps 300 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],3), 'frac', round(d['roofline']['frac'],4), 'dense', round(d['dense']['us_per_layer'],1), 'mhz', d['clocks']['sm_mhz'])"
done
