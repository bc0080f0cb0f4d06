"""Dump GPU R + half-plane integrals for one operator (diagnostics)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_28475_b200 import rbuild  # noqa: E402
from paper_2605_28475_b200.operator import load_cache  # noqa: E402

name = sys.argv[1]
ref = load_cache(os.path.join(ROOT, "operators", name + ".bfct"))
r, halves = rbuild.assemble_r_tensor(ref.cfg, rbuild.GridSpec(*ref.r.grid), return_halves=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"rdump_{name}.npz"), r=r.values, halves=halves)
print("saved", rbuild.last_stats())
