#!/bin/bash
# usage: tools/ab_c1.sh VAR "v1 v2 ..." [rounds] -- C1 bench value per setting of env VAR (GPU box)
var=$1; vals=$2
for i in $(seq ${3:-2}); do
  for v in $vals; do
    echo -n "$var=$v "
    env $var=$v python bench.py --config c1 --steps 300 --warmup 5 --no-cpu-baseline --no-dense-lib 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],3), 'mhz', d['clocks']['sm_mhz'])"
  done
done
