"""Per-call latency of the drop-in through the LIVE reference package.

    python tools/dropin_latency.py [--ops hs_n8,hs_n12,mm_n10] [--calls 30]

Imports the unmodified reference from baseline/_ref, registers the "gpu"
strategy into its contraction.STRATEGIES, and times one-cell calls of the
reference's own ``evaluate(op, c, "gpu")`` (host numpy in, host numpy out:
H2D, one Q launch, D2H, sync) against ``evaluate(op, c)`` on the CPU, plus
one step of ``harness.rk4_integrate(..., strategy="gpu")`` (4 calls).
Prints one JSON line per operator.
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))

import numpy as np  # noqa: E402

from boltzfact import basis, cache, contraction, harness  # noqa: E402
from paper_2605_28475_b200 import engine, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ops", default="hs_n8,hs_n12,mm_n10")
ap.add_argument("--calls", type=int, default=30)
a = ap.parse_args()
assert engine.register_with_reference(contraction)
try:
    from threadpoolctl import threadpool_limits
    limit = threadpool_limits(limits=1)  # the reference's per-cell CPU path, one core
except ImportError:  # pragma: no cover
    limit = None
for name in a.ops.split(","):
    op = cache.load_cache(os.path.join(ROOT, "operators", name + ".bfct"))
    cfg = op.cfg
    c = basis.CoefficientField(inputs.perturbed_maxwellians(cfg.n_k, cfg.l_max, 1, seed=5)[0].copy(), cfg)
    contraction.evaluate(op, c, "gpu")  # plan build + first launch
    lat = []
    for _ in range(a.calls):
        t0 = time.perf_counter()
        q = contraction.evaluate(op, c, "gpu")
        lat.append(time.perf_counter() - t0)
    t0 = time.perf_counter()
    ref = contraction.evaluate(op, c)
    cpu_s = time.perf_counter() - t0
    err = float(np.max(np.abs(q.values - ref.values)) / np.max(np.abs(ref.values)))
    t0 = time.perf_counter()
    tr = harness.rk4_integrate(op, c, 0.001, 1, strategy="gpu")
    rk4_s = time.perf_counter() - t0
    print(json.dumps({
        "operator": name, "n_k": cfg.n_k, "l_max": cfg.l_max,
        "gpu_call_ms": {"median": 1e3 * statistics.median(lat), "min": 1e3 * min(lat), "max": 1e3 * max(lat),
                        "calls": len(lat)},
        "cpu_reference_call_ms": 1e3 * cpu_s, "speedup_per_call": cpu_s / statistics.median(lat),
        "rel_err_vs_reference": err, "rk4_step_gpu_ms": 1e3 * rk4_s, "rk4_moment_drift": tr.moment_drift(),
        "path": "boltzfact.contraction.evaluate(op, c, 'gpu') -> engine.q_gpu (H2D, bfq_eval, D2H, sync)",
    }), flush=True)
