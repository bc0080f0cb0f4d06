#!/bin/bash
# N=L=16: units per CTA x R rings (teams) at one cell per tile (SPLITM)
OUT=${OUT:-gpurun_out/n16}
mkdir -p $OUT
{
for env in "X=0" "BFQ_CELLS=1 BFQ_UNITS=6 BFQ_TEAMS=2" "BFQ_CELLS=1 BFQ_UNITS=5 BFQ_TEAMS=2" ${EXTRA_ENVS}; do
  echo "== hs_n16 16384 [$env]"
  env $env BFQ_PLAN_STATS=1 timeout 400 python tools/prof_q.py --op hs_n16 --cells 16384 --iters 4 --check 3 2>&1 | grep -E "^plan|^\{|iter 3|check|err|Error|error"
done
} > $OUT/units.txt 2>&1
cat $OUT/units.txt
