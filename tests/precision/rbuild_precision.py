"""Accuracy study of the R-tensor build at N=L=12 (test infrastructure).

The reference evaluates the gain integrand's radial polynomial as a monomial
expansion (kinematic.py:458-471), an alternating sum whose terms exceed the
result by ~1e3 at k1 = 12, so its fp64 rounding is amplified.  This script
measures, for selected channels, the relative l-inf distance between

  ref  -- the R stored by the reference's `boltzfact build` (operators/hs_n12.bfct)
  f64  -- the CPU oracle (numpy restatement of the reference, fp64)
  ld   -- the same with the gain integrand in long double (64-bit mantissa)
  gpu  -- the GPU build (an rbuild dump: gpurun_out/rdump_hs_n12.npz, made by
          tools/rbuild_dump.py hs_n12 on the box)

Usage:  python tests/precision/rbuild_precision.py [tau ...]   (~1.5 min/channel pair)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import r_oracle  # noqa: E402
from paper_2605_28475_b200.operator import load_cache  # noqa: E402

OPNAME = os.environ.get("BFR_PRECISION_OP", "hs_n12")
op = load_cache(os.path.join(ROOT, "operators", OPNAME + ".bfct"))
cfg = op.cfg
mx = np.abs(op.r.values).max()
dump = os.path.join(ROOT, "gpurun_out", f"rdump_{OPNAME}.npz")
gpu = np.load(dump)["r"] if os.path.exists(dump) else None
taus = [int(t) for t in sys.argv[1:]] or [567, 579]
for tau in taus:
    res = {}
    for prec in ("f64", "ld"):
        res[prec] = r_oracle.assemble_r(cfg.k_max, cfg.l_max, cfg.gamma, grid=op.r.grid[:7], only=[tau],
                                        precision=prec)[..., tau]
    res["ref"] = op.r.values[..., tau]
    one = os.path.join(ROOT, "gpurun_out", f"r_{OPNAME}_tau{tau}.npy")
    if gpu is not None:
        res["gpu"] = gpu[..., tau]
    elif os.path.exists(one):
        res["gpu"] = np.load(one)
    names = list(res)
    print(f"tau={tau} {op.r.channels.triplets[tau]}  (relative to max|R| over all channels)")
    for i, a in enumerate(names):
        for b in names[i + 1:]:
            d = np.abs(res[a] - res[b])
            print(f"  {a:>3} vs {b:<3}: {d.max() / mx:.3e}   k1={d.shape[0] - 1} row {d[-1].max() / mx:.3e}   "
                  f"k1<=8 {d[:9].max() / mx:.3e}", flush=True)
