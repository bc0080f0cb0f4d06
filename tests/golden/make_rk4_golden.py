"""Build container only: the reference's own RK4 trajectory for config 5
(Maxwell molecules N=L=10, bimodal cells, dt = 0.01, 1,000 steps), recorded
every 100 steps, for the GPU trajectory test (tests/test_gpu_rk4.py).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_rk4_golden.py

Runs boltzfact.harness.rk4_integrate (harness.py:79-120) with its default
strategy on operators/mm_n10.bfct (built by the reference CLI) -- about 6 min
per cell on one core."""
import os
import sys

import numpy as np
from threadpoolctl import threadpool_limits

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from boltzfact import basis, cache, harness  # noqa: E402

from paper_2605_28475_b200 import inputs  # noqa: E402

CELLS = (3, 11)  # of inputs.bimodal(..., 16, seed=2026)
op = cache.load_cache(os.path.join(ROOT, "operators", "mm_n10.bfct"))
cfg = op.cfg
c0 = inputs.bimodal(cfg.k_max + 1, cfg.l_max, 16, seed=2026)
snaps, times = [], None
with threadpool_limits(limits=2):
    for i in CELLS:
        tr = harness.rk4_integrate(op, basis.CoefficientField(c0[i].copy(), cfg), 0.01, 1000, record_every=100)
        snaps.append(tr.coeffs)
        times = tr.times
        print(f"cell {i}: moment drift {tr.moment_drift():.3e}", flush=True)
np.savez_compressed(os.path.join(ROOT, "tests", "golden", "rk4_mm_n10.npz"), cells=np.array(CELLS), seed=2026,
                    n_cells=16, dt=0.01, n_steps=1000, times=times, snapshots=np.stack(snaps, axis=1))
