# Rebuild libbfq.so with per-phase cycle counters / stage-skip switches and
# time each stage alone (GPU box).  BFQ_DEBUG: 8 phase clocks, 1 skip stage 1,
# 2 skip stage 2 (results wrong in the skip modes: timing only).
set -e
cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -shared -DBFQ_PHASE_CLOCKS -I include -o paper_2605_28475_b200/libbfq.so 2>/dev/null paper_2605_28475_b200/csrc/bfq_cuda.cu paper_2605_28475_b200/csrc/bfq_plan.cpp paper_2605_28475_b200/csrc/bfr_build.cu paper_2605_28475_b200/csrc/bfq_project.cu
for op in ${OPS:-hs_n12 hs_n8 mm_n10}; do
  for dbg in ${DBGS:-0 8 1 2}; do
    echo "== $op BFQ_DEBUG=$dbg"
    BFQ_DEBUG=$dbg python tools/prof_q.py --op $op --cells 8192 --iters 3 2>&1 | tail -3
  done
done > gpurun_out/phase_clocks.txt 2>&1
