#!/bin/bash
# ncu evidence only (see round_profile.sh): launch list of the default bench
# command and one --set full capture of the headline kernel, summarised here.
OUT=gpurun_out
mkdir -p $OUT /tmp/ncurep
timeout 1200 ncu --target-processes application-only --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file $OUT/launches_default.csv python bench.py > $OUT/ncu_launches.log 2>&1; echo "rc=$?" >> $OUT/ncu_launches.log
timeout 300 python tools/prof_q.py --op hs_n12 --cells 2048 > $OUT/prof_hs_n12.log 2>&1 && \
timeout 900 ncu --target-processes application-only --set full --clock-control none --import-source on -k regex:bfq_q_kernel -s 2 -c 1 \
   -o /tmp/ncurep/prof_hs_n12 python tools/prof_q.py --op hs_n12 --cells 2048 > $OUT/ncu_hs_n12.log 2>&1
if [ -f /tmp/ncurep/prof_hs_n12.ncu-rep ]; then
  python tools/ncu_summary.py /tmp/ncurep/prof_hs_n12.ncu-rep > $OUT/ncu_sum_hs_n12.txt 2>&1
  python tools/ncu_cluster_stalls.py /tmp/ncurep/prof_hs_n12.ncu-rep >> $OUT/ncu_sum_hs_n12.txt 2>&1
fi
