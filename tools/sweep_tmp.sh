OUT=gpurun_out/q.txt; : > $OUT
python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1
for spec in hs_n12:65536 hs_n16:16384 mm_n10:32768 hs_n8:4096; do
  op=${spec%%:*}; n=${spec##*:}
  echo "== $op $n" >> $OUT
  timeout 300 python tools/prof_q.py --op $op --cells $n --iters 4 2>&1 | grep -E "^\{|^iter 3" | cut -c1-250 >> $OUT
done
