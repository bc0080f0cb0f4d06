#!/bin/bash
# Round-end evidence in one GPU call (outputs in gpurun_out/, summarised on the box):
# tests, smoke, every bench line, the ncu launch list of the DEFAULT bench
# command, and one ncu --set full capture of the headline kernel.
OUT=gpurun_out
mkdir -p $OUT /tmp/ncurep
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for c in ${CONFIGS:-hs8 mm10 hs16 rk4 rbuild12}; do
  timeout 900 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 1200 ncu --target-processes application-only --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_default.csv \
   python bench.py > $OUT/ncu_launches.log 2>&1
timeout 300 python tools/prof_q.py --op hs_n12 --cells 2048 > $OUT/prof_hs_n12.log 2>&1 && \
timeout 900 ncu --target-processes application-only --set full --clock-control none --import-source on -k regex:bfq_q_kernel -s 2 -c 1 \
   -o /tmp/ncurep/prof_hs_n12 python tools/prof_q.py --op hs_n12 --cells 2048 > $OUT/ncu_hs_n12.log 2>&1
if [ -f /tmp/ncurep/prof_hs_n12.ncu-rep ]; then
  python tools/ncu_summary.py /tmp/ncurep/prof_hs_n12.ncu-rep > $OUT/ncu_sum_hs_n12.txt 2>&1
  python tools/ncu_cluster_stalls.py /tmp/ncurep/prof_hs_n12.ncu-rep >> $OUT/ncu_sum_hs_n12.txt 2>&1
  ncu -i /tmp/ncurep/prof_hs_n12.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $OUT/src_hs_n12.csv.gz
fi
ls -la $OUT
