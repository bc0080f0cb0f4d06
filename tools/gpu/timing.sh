#!/bin/bash
# Timing experiments on libbfq_timing.so (-DBFQ_PHASE_CLOCKS): each BFQ_DEBUG
# switch removes one piece of work (results wrong; timing only).
#   0 baseline | 8 phase clocks | 1 skip stage 1 | 2 skip stage 2 | 4 no R-ring wait
#   16 table rows always L1 hits | 64 no Phi stores | 128 no g scaling
OUT=${OUT:-gpurun_out/timing}
mkdir -p $OUT
for spec in ${OPS:-hs_n12:8192 hs_n8:8192 hs_n16:2048}; do
  op=${spec%%:*}; n=${spec##*:}
  for dbg in ${DBGS:-0 8 1 2 4 16 64 128}; do
    echo "== $op BFQ_DEBUG=$dbg"
    BFQ_LIB=timing BFQ_DEBUG=$dbg timeout 300 python tools/prof_q.py --op $op --cells $n --iters 4 2>&1 | tail -3
  done
done > $OUT/timing.txt 2>&1
cat $OUT/timing.txt
