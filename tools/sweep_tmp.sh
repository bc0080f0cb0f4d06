OUT=gpurun_out/sweep4.txt; : > $OUT
python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1
for op in hs_n8 mm_n10 hs_n4; do
 for env in "" "BFQ_ONE_CTA=1" "BFQ_TEAMS=2"; do
  echo "== $op [$env]" >> $OUT
  env $env timeout 120 python tools/prof_q.py --op $op --cells 32768 --iters 3 2>&1 | grep -v "^iter 0" | tail -2 >> $OUT
 done
done
