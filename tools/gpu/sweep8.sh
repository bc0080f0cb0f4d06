#!/bin/bash
# Plan-knob sweep for configs 2 and 4 (env overrides of the tiling choice).
OUT=${OUT:-gpurun_out/sweep}
mkdir -p $OUT
run() { # op cells env...
  local op=$1 n=$2; shift 2
  echo "== $op $n [$*]"
  env "$@" timeout 200 python tools/prof_q.py --op $op --cells $n --iters 4 2>&1 | grep -E "^\{|iter 3"
}
{
for n in 4096 65536; do
  run hs_n8 $n X=0
  run hs_n8 $n BFQ_ONE_CTA=1
  run hs_n8 $n BFQ_TEAMS=2
  run hs_n8 $n BFQ_TEAMS=3
  run hs_n8 $n BFQ_CELLS=4
  run hs_n8 $n BFQ_NO_X1_CELLS8=1
  run hs_n8 $n BFQ_TILE_CHUNK=16
  run hs_n8 $n BFQ_TILE_CHUNK=256
  run hs_n8 $n BFQ_NO_DIAG=1
  run hs_n8 $n BFQ_NO_ROW_REORDER=1
done
for n in 2048 16384; do
  run hs_n16 $n X=0
  run hs_n16 $n BFQ_TEAMS=1
  run hs_n16 $n BFQ_TEAMS=2
  run hs_n16 $n BFQ_UNITS=4
  run hs_n16 $n BFQ_TILE_CHUNK=16
  run hs_n16 $n BFQ_NO_DIAG=1
done
} > $OUT/sweep.txt 2>&1
cat $OUT/sweep.txt
