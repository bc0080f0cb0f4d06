#!/bin/bash
# A/B of the exp library variant (-DBFQ_EXPERIMENT) against the timing build.
OUT=${OUT:-gpurun_out/ab}
mkdir -p $OUT
{
for spec in ${OPS:-hs_n8:4096 hs_n8:65536 hs_n16:16384}; do
  op=${spec%%:*}; n=${spec##*:}
  for lib in timing exp; do
    echo "== $op $n BFQ_LIB=$lib $ENVX"
    env $ENVX BFQ_LIB=$lib timeout 600 python tools/prof_q.py --op $op --cells $n --iters 4 --check ${CHECK:-6} 2>&1 | grep -E "iter 3|check"
  done
done
} > $OUT/ab.txt 2>&1
cat $OUT/ab.txt
