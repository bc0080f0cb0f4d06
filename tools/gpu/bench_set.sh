#!/bin/bash
# GPU tests (optional) + a set of bench lines.  BENCHES="name:args;name:args"
OUT=${OUT:-gpurun_out/set}
mkdir -p $OUT
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
fi
IFS=';' read -ra BS <<< "${BENCHES:-hs12:--config hs12}"
for b in "${BS[@]}"; do
  name=${b%%:*}; args=${b#*:}
  timeout 900 python bench.py $args > $OUT/bench_$name.json 2> $OUT/bench_$name.err
done
python - <<'PY' > $OUT/summary.txt
import glob, json, os
out = os.environ.get("OUT", "gpurun_out/set")
for f in sorted(glob.glob(out + "/bench_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d.get("roofline", {})
        p = d.get("parity") or {}
        print(f"{os.path.basename(f):28s} {d['value']:14.1f} {d['unit']} frac {r.get('frac', 0):.3f} exec {r.get('exec_frac', 0):.3f} "
              f"parity {p.get('max_rel_err')} ({p.get('cells')}) clocks {d.get('clocks', {}).get('sm_mhz')}")
    except Exception as e:
        print(f, "ERR", e)
PY
cat $OUT/summary.txt
tail -3 $OUT/pytest_gpu.log 2>/dev/null
