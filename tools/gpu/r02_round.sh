#!/bin/bash
# GPU tests + the live-reference drop-in latency + bench lines (BENCHES as in bench_set.sh)
OUT=${OUT:-gpurun_out/round}
mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python tools/dropin_latency.py > $OUT/dropin_latency.json 2> $OUT/dropin_latency.err
OUT=$OUT TESTS=0 bash tools/gpu/bench_set.sh
