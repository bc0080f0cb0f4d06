#!/bin/bash
# compute-sanitizer evidence (racecheck, synccheck, memcheck) on small batches
# of the Q kernels: the pair-split kernel at N=L=4 (generic 5-point tile) and
# N=L=12 (headline instantiation), the N=L=8 X1 kernel, and the single-warp
# fallback kernel (BFQ_KERNEL=1).  Outputs in gpurun_out/sanitize_*.log.
OUT=gpurun_out
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool op cells [env]
  local tool=$1 op=$2 cells=$3 tag=$4; shift 4
  env "$@" timeout 900 $CS --tool $tool --error-exitcode 7 python tools/sanitize_q.py --op $op --cells $cells \
    > $OUT/sanitize_${tool}_${op}${tag}.log 2>&1
  echo "$tool $op $cells $tag rc=$?" | tee -a $OUT/sanitize_summary.txt
}
: > $OUT/sanitize_summary.txt
for tool in ${TOOLS:-racecheck synccheck memcheck}; do
  run $tool hs_n4 9 ""
  run $tool hs_n8 9 ""
  run $tool hs_n12 5 ""
  run $tool hs_n4 9 _k1 BFQ_KERNEL=1
done
