# Rebuild libbfq.so with per-phase cycle counters and print the phase shares (GPU box).
set -e
cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -shared -DBFQ_PHASE_CLOCKS -I include -o paper_2605_28475_b200/libbfq.so 2>/dev/null paper_2605_28475_b200/csrc/bfq_cuda.cu paper_2605_28475_b200/csrc/bfq_plan.cpp paper_2605_28475_b200/csrc/bfr_build.cu
for op in synth_n16 hs_n12; do BFQ_DEBUG=8 python tools/prof_q.py --op $op --cells 4096 --iters 2 2>&1 | tail -3; done > gpurun_out/phase_clocks.txt
