"""GPU R-tensor build vs the reference-built operator caches (R after corrections)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_28475_b200 import rbuild  # noqa: E402
from paper_2605_28475_b200.operator import load_cache  # noqa: E402

names = sys.argv[1:] or ["hs_n2", "hs_n4", "mm_n4", "hs_k4l6", "mm_k4l6", "hs_n8", "mm_n10", "hs_n12"]
for name in names:
    path = os.path.join(ROOT, "operators", name + ".bfct")
    if not os.path.exists(path):
        print(name, "missing")
        continue
    ref = load_cache(path)
    g = rbuild.GridSpec(*ref.r.grid)
    t = time.time()
    r = rbuild.assemble_r_tensor(ref.cfg, g)
    r = rbuild.apply_detailed_balance(rbuild.apply_conservation(r))
    wall = time.time() - t
    st = rbuild.last_stats()
    err = np.abs(r.values - ref.r.values).max() / np.abs(ref.r.values).max()
    tf = 2 * st["contract_macs"] / st["ms_contract"] / 1e9 if st["ms_contract"] else 0
    d = np.abs(r.values - ref.r.values) / np.abs(ref.r.values).max()
    worst = np.unravel_index(d.argmax(), d.shape)
    if len(sys.argv) > 1:
        print(f"  by k1: {[float(f'{d[k].max():.1e}') for k in range(d.shape[0])]}  argmax (k,a,b,tau) {worst} "
              f"{ref.r.channels.triplets[worst[3]]}")
        np.save(os.path.join(ROOT, "gpurun_out", f"r_{name}_tau{worst[3]}.npy"), r.values[..., worst[3]])
    print(f"{name}: rel_linf {err:.3e}  wall {wall:.2f}s  device {st['ms_total']:.1f} ms  "
          f"contract {st['ms_contract']:.1f} ms ({tf:.2f} exec TF/s, alg {2*st['alg_macs']/1e12:.3f} TFLOP)  "
          f"points {st['n_points']}", flush=True)
