#!/bin/bash
# N=L=16 plan-knob sweep: one line of ENVS (separated by ';') per run
OUT=${OUT:-gpurun_out/n16}
mkdir -p $OUT
IFS=';' read -ra ES <<< "${ENVS:-X=0;BFQ_UNITS=5;BFQ_PACK_WORK=1;BFQ_UNIT_BALANCE=1;BFQ_TILE_CHUNK=8;BFQ_TILE_CHUNK=32}"
{
for env in "${ES[@]}"; do
  echo "== ${OP:-hs_n16} ${CELLS:-16384} [$env]"
  env $env BFQ_PLAN_STATS=1 timeout 400 python tools/prof_q.py --op ${OP:-hs_n16} --cells ${CELLS:-16384} --iters 4 --check 3 2>&1 | grep -E "^plan|^\{|iter 3|check|err|Error|error"
done
} > $OUT/${NAME:-units}.txt 2>&1
cat $OUT/${NAME:-units}.txt
