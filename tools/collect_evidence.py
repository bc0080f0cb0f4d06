"""Copy the outputs of tools/gpu/r02_evidence.sh (gpurun_out/ev, pp, prof) into profiles/ under the
round's names and print the one-line summary of every bench line."""
import collections
import csv
import io
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R = sys.argv[1] if len(sys.argv) > 1 else "r02"
ev, pp, prof = (os.path.join(ROOT, "gpurun_out", d) for d in ("ev", "pp", "prof"))
out = os.path.join(ROOT, "profiles")


def cp(src, dst):
    if os.path.exists(src):
        shutil.copy(src, os.path.join(out, dst))


for f in sorted(os.listdir(ev)):
    if f.startswith("bench_") and f.endswith(".json"):
        name = f[6:-5]
        cp(os.path.join(ev, f), f"{R}_bench_{'hs12' if name == 'default' else name}.json")
        try:
            d = json.loads(open(os.path.join(ev, f)).read().strip().splitlines()[-1])
            r, p = d.get("roofline") or {}, d.get("parity") or {}
            print(f"{name:10s} {d['value']:12.1f} {d['unit']:11s} frac {r.get('frac')} exec {r.get('exec_frac')} useful "
                  f"{r.get('useful_frac')} parity {p.get('max_rel_err')} ({p.get('cells')}) e2e "
                  f"{(d.get('e2e') or {}).get('value')} cpu {(d.get('cpu_baseline') or {}).get('value')}")
        except Exception as e:  # noqa: BLE001
            print(name, "ERR", e)
cp(os.path.join(ev, "pytest_gpu.log"), f"{R}_pytest_gpu.log")
cp(os.path.join(ev, "smoke.log"), f"{R}_smoke.log")
cp(os.path.join(ev, "launches_default.csv"), f"{R}_launches_default.csv")
cp(os.path.join(ev, "ncu_traffic_hs12.csv"), f"{R}_ncu_traffic_hs12.csv")
cp(os.path.join(ev, "dropin_latency.json"), f"{R}_dropin_latency.json")
cp(os.path.join(pp, "sum.txt"), f"{R}_ncu_project_fold_proj12.txt")
for src, dst in ((os.path.join(ev, "ncu_sum_hs_n12.txt"), f"{R}_ncu_hs12_final.txt"),
                 (os.path.join(prof, "ncu_sum_hs_n16.txt"), f"{R}_ncu_hs_n16.txt"),
                 (os.path.join(prof, "ncu_sum_mm_n10.txt"), f"{R}_ncu_mm_n10.txt"),
                 (os.path.join(prof, "ncu_sum_hs_n8.txt"), f"{R}_ncu_hs_n8.txt")):
    if os.path.exists(src):
        txt = open(src).read()
        if "Traceback" in txt:
            txt = txt[:txt.index("Traceback")]
        open(os.path.join(out, dst), "w").write(txt)
lc = os.path.join(ev, "launches_default.csv")
if os.path.exists(lc):
    rows = [l for l in open(lc) if l.startswith('"')]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for x in csv.DictReader(io.StringIO("".join(rows))):
        if x.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v, u = float(x["Metric Value"].replace(",", "")), x["Metric Unit"]
        ms = v / 1e6 if u.startswith("n") else v / 1e3 if u.startswith("u") else v if u.startswith("m") else v * 1e3
        agg[x["Kernel Name"]][0] += 1
        agg[x["Kernel Name"]][1] += ms
    tot = sum(v[1] for v in agg.values())
    lines = ["# ncu --metrics gpu__time_duration.sum --clock-control none of the DEFAULT bench command (python bench.py)",
             "# per-launch times are cold-cache and serialised: the SHARE of the step is what compares with bench.py"]
    lines += [f"{100 * v[1] / tot:6.2f}% {v[0]:5d} launches {v[1]:10.3f} ms  {k[:80]}"
              for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])]
    open(os.path.join(out, f"{R}_launches_summary.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[2:5]))
