#!/bin/bash
# All BASELINE configs that have an operator in operators/ (one GPU call).
OUT=gpurun_out
python bench.py --steps 5 --warmup 3 > $OUT/bench_hs12.json 2> $OUT/bench_hs12.err
python bench.py --config hs8 --steps 10 --warmup 3 > $OUT/bench_hs8.json 2> $OUT/bench_hs8.err
python bench.py --config hs8 --cells 65536 --steps 5 --warmup 3 --no-cpu > $OUT/bench_hs8_64k.json 2>> $OUT/bench_hs8.err
python bench.py --config mm10 --steps 5 --warmup 3 > $OUT/bench_mm10.json 2> $OUT/bench_mm10.err
python bench.py --config rk4 --steps 20 --warmup 3 --no-cpu > $OUT/bench_rk4.json 2> $OUT/bench_rk4.err
if [ -f operators/hs_n16.bfct ]; then python bench.py --config hs16 --steps 3 --warmup 3 > $OUT/bench_hs16.json 2> $OUT/bench_hs16.err; fi
if [ -f operators/synth_n16.bfct ]; then python bench.py --config syn16 --steps 3 --warmup 3 --no-cpu > $OUT/bench_syn16.json 2> $OUT/bench_syn16.err; fi
