#!/bin/bash
# One GPU call: tests, bench (plain), ncu launch list of the same bench command,
# ncu --set full of one Q launch.  Outputs in gpurun_out/.
set -x
OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
python bench.py --steps 5 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
BENCHSMALL="python bench.py --steps 2 --warmup 1 --cells 4096 --no-cpu --e2e-steps 0"
$BENCHSMALL > $OUT/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/launches.csv $BENCHSMALL > $OUT/ncu_launches.log 2>&1
python tools/prof_q.py --op hs_n12 --cells 2048 > $OUT/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bfq_q_kernel -s 2 -c 1 -o $OUT/prof_hs12 python tools/prof_q.py --op hs_n12 --cells 2048 > $OUT/ncu_hs12.log 2>&1
