#!/bin/bash
# usage: tools/ab_lib.sh [rounds] -- A/B of liblouver_b200_before.so vs _after.so on the C2 bench (GPU box)
for i in $(seq ${1:-2}); do
  for v in before after; do
    cp paper_2605_06763_b200/liblouver_b200_$v.so paper_2605_06763_b200/liblouver_b200.so
    echo -n "$v "; bash tools/ab.sh 1
  done
done
cp paper_2605_06763_b200/liblouver_b200_after.so paper_2605_06763_b200/liblouver_b200.so
