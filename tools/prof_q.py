"""Minimal driver for ncu: a few Q(f,f) launches on one config (no CPU legs)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2605_28475_b200 import engine, inputs  # noqa: E402
from paper_2605_28475_b200.operator import load_cache  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--op", default="hs_n8")
ap.add_argument("--cells", type=int, default=8192)
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--bilinear", action="store_true")
ap.add_argument("--check", type=int, default=0, help="compare this many cells with the CPU oracle")
a = ap.parse_args()
path = os.path.join(ROOT, "operators", a.op + ".bfct")
if os.path.exists(path):
    op = load_cache(path)
else:  # hs_n16 is not shipped: assemble it on the GPU (bfr_assemble)
    from paper_2605_28475_b200 import rbuild
    from paper_2605_28475_b200.operator import SpectralConfig
    n = int(a.op.split("_n")[1])
    op = rbuild.build_operator(SpectralConfig(n, n, 0.0 if a.op.startswith("mm") else 1.0))
cells = inputs.perturbed_maxwellians(op.cfg.n_k, op.cfg.l_max, a.cells, seed=1)
f = torch.from_numpy(cells).cuda()
f3 = f.clone() if a.bilinear else None
plan = engine.plan_for(op)
print(plan.info)
q = torch.empty_like(f)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(a.iters):
    ev0.record()
    engine.evaluate_batch(plan, f, f3, out=q)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    print(f"iter {i}: {ms:.3f} ms  {a.cells / ms * 1e3:.0f} cells/s  "
          f"{plan.flops_per_cell * a.cells / ms / 1e9:.2f} alg TFLOP/s  "
          f"{2 * plan.info['exec_macs_per_cell'] * a.cells / ms / 1e9:.2f} exec TFLOP/s")

if os.environ.get("BFQ_DEBUG", "0") != "0" and int(os.environ["BFQ_DEBUG"]) & 8:
    import ctypes
    from paper_2605_28475_b200 import _lib
    lib = _lib.lib()
    buf = (ctypes.c_ulonglong * 8)()
    lib.bfq_debug_phase_clocks(buf)
    if plan.info["warps_per_cta"] in (8, 16) and os.environ.get("BFQ_KERNEL", "2") == "2":  # pair-split kernel
        names = ["stage1", "bar1", "wait R", "stage2", "bar2", "total"]
        n = max(buf[6], 1)
    else:
        names = ["stage1+flush", "wait R", "stage2", "refill", "total"]
        n = max(buf[5], 1)
    tot = buf[len(names) - 1]
    print("phase cycles per warp (avg over %d warps):" % n, {k: round(buf[j] / n) for j, k in enumerate(names)})
    print("shares:", {k: round(100.0 * buf[j] / max(tot, 1), 1) for j, k in enumerate(names[:-1])})

if a.check:
    import numpy as np

    from oracle import q_oracle

    oop = q_oracle.OracleOperator.from_operator(op)
    ws = q_oracle.angular_workspace(oop)
    qh = q.cpu().numpy()
    idx = np.unique(np.linspace(0, a.cells - 1, a.check).round().astype(int))
    c3 = f3.cpu().numpy() if f3 is not None else cells
    errs = [q_oracle.rel_err(qh[i], q_oracle.q_angular_first(oop, cells[i], c3[i] if a.bilinear else None,
                                                             workspace=ws)) for i in idx]
    print(f"check: {len(idx)} cells, max rel err {max(errs):.3e}", "OK" if max(errs) <= 1e-12 else "FAIL")

