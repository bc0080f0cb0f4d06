#!/bin/bash
# All BASELINE configs that have an operator in operators/ (one GPU call), plus the R-build lines.
OUT=gpurun_out
python bench.py --steps 5 --warmup 3 > $OUT/bench_hs12.json 2> $OUT/bench_hs12.err
python bench.py --config hs8 --steps 10 --warmup 3 > $OUT/bench_hs8.json 2> $OUT/bench_hs8.err
python bench.py --config hs8 --cells 65536 --steps 5 --warmup 3 --no-cpu > $OUT/bench_hs8_64k.json 2>> $OUT/bench_hs8.err
python bench.py --config mm10 --steps 5 --warmup 3 > $OUT/bench_mm10.json 2> $OUT/bench_mm10.err
python bench.py --config rk4 --steps 20 --warmup 3 --no-cpu > $OUT/bench_rk4.json 2> $OUT/bench_rk4.err
python bench.py --config hs16 --steps 3 --warmup 3 --no-cpu > $OUT/bench_hs16.json 2> $OUT/bench_hs16.err
if [ -f operators/synth_n16.bfct ]; then python bench.py --config syn16 --steps 3 --warmup 3 --no-cpu > $OUT/bench_syn16.json 2> $OUT/bench_syn16.err; fi
python bench.py --config rbuild12 --steps 3 --warmup 3 > $OUT/bench_rbuild12.json 2> $OUT/bench_rbuild12.err
python bench.py --config rbuild16 --steps 2 --warmup 3 --no-cpu > $OUT/bench_rbuild16.json 2> $OUT/bench_rbuild16.err
python bench.py --impl reference --steps 1 --warmup 0 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
