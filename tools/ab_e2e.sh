#!/bin/bash
# usage: tools/ab_e2e.sh [runs] -- e2e (host buffers, lv_query_layers) of a short C2 bench with
# copy-engine transfers (LV_LAYERS_MAPPED=0) and mapped host buffers (default) (GPU box)
for i in $(seq ${1:-2}); do
  for m in 0 1; do
    echo -n "mapped=$m "
    LV_LAYERS_MAPPED=$m python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-dense-lib 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],3), 'e2e', round(d['e2e']['value'],3))"
  done
done
