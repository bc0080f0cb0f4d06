OUT=gpurun_out/sweep2.txt; : > $OUT
for env in "" "BFQ_TEAMS=2" "BFQ_STAGES=1 BFQ_TEAMS=3"; do
 for op in hs_n12; do
  echo "== $op [$env]" >> $OUT
  env $env timeout 120 python tools/prof_q.py --op $op --cells 16384 --iters 3 2>&1 | grep -v "^iter 0" | tail -3 >> $OUT
 done
done
