"""Golden vectors of the GENERAL projection: the live reference's
basis.project(f, cfg, order) (basis.py:262-299) for the test functions of
project_funcs.py at the CASES sizes.  Run in the build container, where the
reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_project_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

from boltzfact.basis import SpectralConfig, project  # noqa: E402

from project_funcs import CASES, FUNCS  # noqa: E402

out = {}
for k, l, order in CASES:
    cfg = SpectralConfig(k, l, 1.0)
    for name, f in FUNCS.items():
        out[f"{name}_k{k}_l{l}_o{order}"] = project(f, cfg, order).values
np.savez_compressed(os.path.join(HERE, "project_general.npz"), **out)
print("wrote", len(out), "projections")
