OUT=gpurun_out/sweep5.txt; : > $OUT
for env in "" "BFQ_KERNEL=1" "BFQ_ONE_CTA=1 BFQ_TEAMS=2" "BFQ_TEAMS=2" "BFQ_TEAMS=3" "BFQ_NO_X1_CELLS8=1"; do
  echo "== hs_n8 [$env]" >> $OUT
  env $env timeout 120 python tools/prof_q.py --op hs_n8 --cells 4096 --iters 5 2>&1 | grep -E "^\{|^iter 4" >> $OUT
done
