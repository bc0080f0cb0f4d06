#!/bin/bash
# ncu --set full of one Q launch per config, with source-level SASS metrics
# (per-instruction shared wavefronts vs ideal, stalls); reports summarised on the box.
OUT=${OUT:-gpurun_out/prof}
mkdir -p $OUT /tmp/ncurep
PROFS=${PROFS:-"hs_n8:8192 hs_n12:2048 hs_n16:1024"}
for spec in $PROFS; do
  op=${spec%%:*}; n=${spec##*:}
  tag=${TAG:-}$op
  timeout 300 python tools/prof_q.py --op $op --cells $n > $OUT/prof_$tag.log 2>&1 && \
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:bfq_q_kernel -s 2 -c 1 \
     -o /tmp/ncurep/prof_$tag python tools/prof_q.py --op $op --cells $n > $OUT/ncu_$tag.log 2>&1
  if [ -f /tmp/ncurep/prof_$tag.ncu-rep ]; then
    python tools/ncu_summary.py /tmp/ncurep/prof_$tag.ncu-rep > $OUT/ncu_sum_$tag.txt 2>&1
    python tools/ncu_cluster_stalls.py /tmp/ncurep/prof_$tag.ncu-rep >> $OUT/ncu_sum_$tag.txt 2>&1
    ncu -i /tmp/ncurep/prof_$tag.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $OUT/src_$tag.csv.gz
    ncu -i /tmp/ncurep/prof_$tag.ncu-rep --page raw --csv 2>/dev/null | gzip > $OUT/raw_$tag.csv.gz
  fi
done
ls -la $OUT
