#!/bin/bash
# One GPU call: bench lines for every Q config + ncu --set full of one Q
# launch per config; reports summarised on the box (gpurun_out/ <= 64 MiB).
OUT=gpurun_out
mkdir -p $OUT /tmp/ncurep
CONFIGS=${CONFIGS:-"hs12 hs8 mm10 hs16 rk4"}
PROFS=${PROFS:-"hs_n8:8192 mm_n10:8192 hs_n16:1024"}
for c in $CONFIGS; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
for spec in $PROFS; do
  op=${spec%%:*}; n=${spec##*:}
  timeout 300 python tools/prof_q.py --op $op --cells $n > $OUT/prof_$op.log 2>&1 && \
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:bfq_q_kernel -s 2 -c 1 \
     -o /tmp/ncurep/prof_$op python tools/prof_q.py --op $op --cells $n > $OUT/ncu_$op.log 2>&1
  if [ -f /tmp/ncurep/prof_$op.ncu-rep ]; then
    python tools/ncu_summary.py /tmp/ncurep/prof_$op.ncu-rep > $OUT/ncu_sum_$op.txt 2>&1
    python tools/ncu_cluster_stalls.py /tmp/ncurep/prof_$op.ncu-rep >> $OUT/ncu_sum_$op.txt 2>&1
    ncu -i /tmp/ncurep/prof_$op.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $OUT/src_$op.csv.gz
    ncu -i /tmp/ncurep/prof_$op.ncu-rep --page raw --csv 2>/dev/null | gzip > $OUT/raw_$op.csv.gz
  fi
done
ls -la $OUT
