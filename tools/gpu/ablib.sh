#!/bin/bash
# Same-box A/B of two builds: tools/gpu/libbfq_prev.so (another revision, via
# BFQ_AB_LIB) against the current libbfq.so, alternating, over OPS (op:cells).
OUT=${OUT:-gpurun_out/ablib}
mkdir -p $OUT
{
for spec in ${OPS:-hs_n12:65536}; do
  op=${spec%%:*}; n=${spec##*:}
  for rep in 1 2; do
    for lib in prev cur; do
      echo "== $op $n $lib #$rep"
      if [ $lib = prev ]; then export BFQ_AB_LIB=$PWD/tools/gpu/libbfq_prev.so; else unset BFQ_AB_LIB; fi
      timeout 600 python tools/prof_q.py --op $op --cells $n --iters 4 --check ${CHECK:-1} 2>&1 | grep -E "iter 3|check"
    done
  done
done
} > $OUT/ab.txt 2>&1
cat $OUT/ab.txt
