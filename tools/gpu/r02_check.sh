#!/bin/bash
# Round-2 GPU check in one call: GPU tests, smoke, the default bench line, config 2,
# and one compute-sanitizer probe.  Outputs under gpurun_out/r02/.
OUT=${OUT:-gpurun_out/r02}
mkdir -p $OUT
nvidia-smi > $OUT/nvidia_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1; echo "build rc=$?" >> $OUT/build.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 600 python bench.py --config hs8 > $OUT/bench_hs8.json 2> $OUT/bench_hs8.err
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --error-exitcode 7 python tools/sanitize_q.py --op hs_n4 --cells 9 > $OUT/sanitize_probe.log 2>&1; echo "rc=$?" >> $OUT/sanitize_probe.log
ls -la $OUT
