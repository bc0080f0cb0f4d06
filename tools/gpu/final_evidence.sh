#!/bin/bash
# Everything profiles/r02_* was collected from, in one GPU call:
#   gpurun --timeout 3300 -- 'bash tools/gpu/final_evidence.sh'   then   python tools/collect_evidence.py r02
# GPU tests, smoke, every bench line (+ the reference arm), the ncu launch list of the default bench
# command, ncu --set full of the headline Q kernel, of the folded projection kernel and of the
# N=L=16 / 10 / 8 Q kernels, the DRAM traffic of one launch at the bench size, the live-reference
# drop-in latency.
CONFIGS="${CONFIGS:-hs8 hs16 mm10 rk4 proj12 proj8 rbuild12}" bash tools/gpu/r02_evidence.sh > gpurun_out/ev_run.log 2>&1
OUT=gpurun_out/pp TESTS=0 PCONFIGS="" bash tools/gpu/proj_prof.sh > gpurun_out/pp_run.log 2>&1
PROFS="${PROFS:-hs_n16:1024 mm_n10:4096 hs_n8:8192}" bash tools/gpu/r02_prof.sh > gpurun_out/prof_run.log 2>&1
timeout 600 python tools/dropin_latency.py > gpurun_out/ev/dropin_latency.json 2> gpurun_out/ev/dropin_latency.err
tail -3 gpurun_out/ev/pytest_gpu.log
