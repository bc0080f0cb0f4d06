OUT=gpurun_out/hostchunk2.txt; : > $OUT
for ch in 256 512 1024; do
  echo "== hs12 chunk $ch" >> $OUT
  BFQ_HOST_CHUNK=$ch timeout 600 python bench.py --no-cpu --steps 3 --warmup 3 --e2e-steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']))" >> $OUT
done
for ch in 128 256 512; do
  for c in hs8 mm10; do
  echo "== $c chunk $ch" >> $OUT
  BFQ_HOST_CHUNK=$ch timeout 600 python bench.py --config $c --no-cpu --steps 3 --warmup 3 --e2e-steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']))" >> $OUT
  done
done
