#!/bin/bash
# One GPU call: build, the GPU test suite, the default bench line and config 2.
OUT=${OUT:-gpurun_out/run}

mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 600 python bench.py --config hs8 > $OUT/bench_hs8.json 2> $OUT/bench_hs8.err
