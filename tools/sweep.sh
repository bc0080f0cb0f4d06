# Plan-knob sweep (GPU box): env overrides of the tiling choice per operator.
OUT=gpurun_out/sweep.txt
: > $OUT
for op in ${OPS:-hs_n12 mm_n10 hs_n8}; do
  for env in "" "BFQ_CELLS=2" "BFQ_CELLS=2 BFQ_TEAMS=2" "BFQ_STAGES=2 BFQ_TEAMS=2" "BFQ_TEAMS=1" "BFQ_NO_DIAG=1" $EXTRA; do
    echo "== $op [$env]" >> $OUT
    env $env timeout 120 python tools/prof_q.py --op $op --cells 16384 --iters 3 2>&1 | tail -2 >> $OUT
  done
done
