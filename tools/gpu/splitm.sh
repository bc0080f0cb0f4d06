#!/bin/bash
OUT=${OUT:-gpurun_out/splitm}
mkdir -p $OUT
{
echo "== checked SPLITM hs_n16"
BFQ_LIB=checked BFQ_CELLS=1 timeout 900 python tools/checked_run.py --ops hs_n16 --cells 5 2>&1 | tail -5
for env in "X=0" "BFQ_CELLS=1" "BFQ_CELLS=1 BFQ_UNITS=5" "BFQ_CELLS=1 BFQ_UNITS=6" "BFQ_CELLS=1 BFQ_UNITS=7" "BFQ_CELLS=1 BFQ_UNITS=4 BFQ_TEAMS=1" "BFQ_TILE_CHUNK=16" "BFQ_CELLS=1 BFQ_TILE_CHUNK=16"; do
  echo "== hs_n16 16384 [$env]"
  env $env BFQ_PLAN_STATS=1 timeout 300 python tools/prof_q.py --op hs_n16 --cells 16384 --iters 3 2>&1 | grep -E "^plan|^\{|iter 2"
done
} > $OUT/splitm.txt 2>&1
cat $OUT/splitm.txt
