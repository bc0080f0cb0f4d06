#!/bin/bash
OUT=${OUT:-gpurun_out/proj}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_project_general.py -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for c in ${PCONFIGS:-proj12 proj8}; do timeout 600 python bench.py --config $c --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err; done
tail -3 $OUT/pytest.log
python - <<'PY'
import json, os, glob
out = os.environ.get("OUT", "gpurun_out/proj")
for f in sorted(glob.glob(out + "/bench_proj*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1]); r = d["roofline"]
        print(f, round(d["value"]), "cells/s", round(r["achieved"]), "GB/s frac", round(r["frac"], 3), "fp64", round(r["fp64_frac"], 3), "parity", d["parity"]["max_rel_err"])
    except Exception as e:
        print(f, "ERR", e, open(f.replace(".json", ".err")).read()[-500:])
PY
