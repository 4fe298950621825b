#!/bin/bash
# usage: tools/ab_env.sh VAR "v1 v2 ..." [rounds] -- C2 bench value per setting of env VAR, interleaved (GPU box)
var=$1; vals=$2
for i in $(seq ${3:-2}); do
  for v in $vals; do
    echo -n "$var=$v "; env $var=$v bash tools/ab.sh 1
  done
done
