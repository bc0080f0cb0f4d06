#!/bin/bash
# A/B of plan env switches: ENVS="A;B" over OPS (op:cells), with an oracle check.
OUT=${OUT:-gpurun_out/envab}
mkdir -p $OUT
IFS=';' read -ra EV <<< "${ENVS:-X=0}"
{
for spec in ${OPS:-hs_n8:4096}; do
  op=${spec%%:*}; n=${spec##*:}
  for e in "${EV[@]}"; do
    echo "== $op $n [$e]"
    env $e timeout 600 python tools/prof_q.py --op $op --cells $n --iters 4 --check ${CHECK:-6} 2>&1 | grep -E "iter 3|check"
  done
done
} > $OUT/envab.txt 2>&1
cat $OUT/envab.txt
