#!/bin/bash
# Round-2 evidence in one GPU call: GPU tests, smoke, every bench line (incl. the
# reference arm), the ncu launch list of the DEFAULT bench command, and one
# ncu --set full capture of the headline kernel.  Outputs in gpurun_out/ev/.
OUT=${OUT:-gpurun_out/ev}
mkdir -p $OUT /tmp/ncurep
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for c in ${CONFIGS:-hs8 hs16 mm10 rk4 proj12 rbuild12}; do
  timeout 900 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 1200 ncu -f --target-processes application-only --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file $OUT/launches_default.csv python bench.py > $OUT/ncu_launches.log 2>&1
timeout 300 python tools/prof_q.py --op hs_n12 --cells 2048 > $OUT/prof_hs_n12.log 2>&1 && \
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:bfq_q_kernel -s 2 -c 1 \
   -o /tmp/ncurep/ev_hs_n12 python tools/prof_q.py --op hs_n12 --cells 2048 > $OUT/ncu_hs_n12.log 2>&1
if [ -f /tmp/ncurep/ev_hs_n12.ncu-rep ]; then
  python tools/ncu_summary.py /tmp/ncurep/ev_hs_n12.ncu-rep > $OUT/ncu_sum_hs_n12.txt 2>&1
  python tools/ncu_cluster_stalls.py /tmp/ncurep/ev_hs_n12.ncu-rep >> $OUT/ncu_sum_hs_n12.txt 2>&1
  ncu -i /tmp/ncurep/ev_hs_n12.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $OUT/src_hs_n12.csv.gz
fi
# DRAM traffic of one launch at the bench size (65,536 cells) for the roofline's traffic key
timeout 900 ncu -f --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
   -k regex:bfq_q_kernel -s 3 -c 1 --csv python tools/prof_q.py --op hs_n12 --cells 65536 --iters 4 > $OUT/ncu_traffic_hs12.csv 2>&1
ls -la $OUT
