OUT=gpurun_out
python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1
for spec in hs_n12:65536 mm_n10:32768 hs_n8:32768 hs_n16:16384; do
  op=${spec%%:*}; n=${spec##*:}
  echo "== $op $n" >> $OUT/q.txt
  timeout 300 python tools/prof_q.py --op $op --cells $n --iters 3 2>&1 | grep -v "^iter 0" | tail -2 >> $OUT/q.txt
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:bfq_q_kernel -s 1 -c 1 python tools/prof_q.py --op $op --cells $n --iters 2 2>&1 | grep -E "dram__|gpu__time" >> $OUT/q.txt
done
