#!/bin/bash
# Projection kernel iteration: GPU tests, the two bench lines, one ncu capture of the v2 kernel.
OUT=${OUT:-gpurun_out/pp}
mkdir -p $OUT /tmp/ncurep
if [ "${TESTS:-1}" = "1" ]; then
  timeout 600 python -m pytest tests/test_gpu_project_general.py tests/test_gpu_project.py -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
fi
for c in ${PCONFIGS:-proj12 proj8}; do timeout 600 python bench.py --config $c --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err; done
if [ "${NCU:-1}" = "1" ]; then
  timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:k_project -s 1 -c 1 -o /tmp/ncurep/pp \
    python tools/prof_proj.py --cells 1024 ${PARGS:-} > $OUT/ncu.log 2>&1
  python tools/ncu_summary.py /tmp/ncurep/pp.ncu-rep > $OUT/sum.txt 2>&1
  cp /tmp/ncurep/pp.ncu-rep $OUT/
fi
tail -2 $OUT/pytest.log 2>/dev/null
python - <<'PY'
import json, os, glob
out = os.environ.get("OUT", "gpurun_out/pp")
for f in sorted(glob.glob(out + "/bench_proj*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1]); r = d["roofline"]
        print(f, round(d["value"]), "cells/s", round(r["achieved"]), "GB/s frac", round(r["frac"], 3), "fp64", round(r["fp64_frac"], 3), "parity", d["parity"]["max_rel_err"])
    except Exception as e:
        print(f, "ERR", e, open(f.replace(".json", ".err")).read()[-500:])
PY
cat $OUT/sum.txt 2>/dev/null
