"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container (the reference is importable there, read-only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

For every operator cache under ``operators/`` it stores seeded input cells and
the reference's own ``evaluate(op, c)`` (default strategy ``angular_first``,
contraction.py:327-340) plus a bilinear ``q_angular_first(op, c1, c2)`` pair.
It also stores reference ``basis.project`` outputs for drifting Maxwellians
(pins the analytic input generator) and the closed-form Maxwell relaxation
rates of ``pkg/tests/oracles.py:59-72``.  The fixtures are small ``.npz``
files; the GPU box never needs the reference.
"""

from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(REPO))

from boltzfact import cache as ref_cache  # noqa: E402
from boltzfact.basis import CoefficientField, SpectralConfig, project  # noqa: E402
from boltzfact.contraction import evaluate, linearize, q_angular_first, q_naive  # noqa: E402

sys.path.insert(0, "/root/reference/pkg/tests")
from oracles import maxwell_eigenvalue_ref  # noqa: E402

from paper_2605_28475_b200 import inputs  # noqa: E402

OUT = Path(__file__).resolve().parent

# operator file -> (#uniform cells, #perturbed-Maxwellian cells)
CASES = {
    "hs_n2": (4, 2),
    "mm_n4": (4, 4),
    "hs_n4": (4, 4),
    "mm_k4l6": (3, 2),
    "hs_k4l6": (3, 2),
    "hs_n8": (3, 3),
    "mm_n10": (2, 2),
    "hs_n12": (2, 2),
    "hs_n16": (1, 2),
}


def one(name: str, n_uni: int, n_pm: int) -> None:
    path = REPO / "operators" / f"{name}.bfct"
    if not path.exists():
        print(f"skip {name}: no operator file")
        return
    op = ref_cache.load_cache(path)
    cfg = op.cfg
    cells = np.concatenate([
        inputs.uniform_fields(cfg.n_k, cfg.l_max, n_uni, seed=1000 + cfg.l_max),
        inputs.perturbed_maxwellians(cfg.n_k, cfg.l_max, n_pm, seed=2000 + cfg.l_max),
    ])
    if name.startswith("mm_n4"):
        cells = np.concatenate([cells, inputs.maxwell_config1(cfg.n_k, cfg.l_max, seed=1, n_cells=2)])
    q = np.stack([evaluate(op, CoefficientField(c.copy(), cfg)).values for c in cells])
    qn = np.stack([q_naive(op, CoefficientField(c.copy(), cfg)).values for c in cells[:1]])
    c1 = inputs.uniform_fields(cfg.n_k, cfg.l_max, 1, seed=11)[0]
    c2 = inputs.uniform_fields(cfg.n_k, cfg.l_max, 1, seed=12)[0]
    q12 = q_angular_first(op, CoefficientField(c1, cfg), CoefficientField(c2, cfg)).values
    extra = {}
    if cfg.n_dof <= 300:  # reference linearize (contraction.py:343-369) at equilibrium and a perturbed state
        extra["jac_eq"] = linearize(op, CoefficientField.equilibrium(cfg))
        extra["jac_c"] = cells[n_uni]
        extra["jac_pm"] = linearize(op, CoefficientField(cells[n_uni].copy(), cfg))
    np.savez_compressed(OUT / f"{name}.npz", cells=cells, q=q, q_naive0=qn, c1=c1, c2=c2, q12=q12,
                        k_max=cfg.k_max, l_max=cfg.l_max, gamma=cfg.gamma, **extra)
    print(f"{name}: {cells.shape[0]} cells, max|Q| {np.abs(q).max():.3e}")


def projections() -> None:
    rows = []
    for (k_max, l_max) in ((4, 4), (8, 8)):
        cfg = SpectralConfig(k_max, l_max, 1.0)
        for u, t in (((0.1, -0.2, 0.25), 0.9), ((0.0, 0.0, 0.0), 1.0), ((0.3, 0.3, -0.3), 1.2),
                     ((1.2, 0.4, -0.7), 1.0)):
            u = np.array(u)
            f = lambda p, u=u, t=t: (2 * math.pi * t) ** -1.5 * np.exp(-((p - u) ** 2).sum(1) / (2 * t))  # noqa: E731
            rows.append((k_max, l_max, u, t, project(f, cfg, 64).values))
    np.savez_compressed(OUT / "project.npz",
                        **{f"c{i}": r[4] for i, r in enumerate(rows)},
                        meta=np.array([[r[0], r[1], *r[2], r[3]] for r in rows]))
    rates = np.array([[k, l, maxwell_eigenvalue_ref(k, l)] for k in range(6) for l in range(8)])
    np.savez_compressed(OUT / "maxwell_rates.npz", rates=rates)
    print("projections + Maxwell rates written")


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        if n in CASES:
            one(n, *CASES[n])
    if not sys.argv[1:]:
        projections()
