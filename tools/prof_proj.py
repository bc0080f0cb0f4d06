"""Minimal driver for ncu: a few general-projection launches (bfq_project_samples)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2605_28475_b200 import project as gproject  # noqa: E402
from paper_2605_28475_b200.operator import SpectralConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=12, help="N = L")
ap.add_argument("--order", type=int, default=64)
ap.add_argument("--cells", type=int, default=1024)
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
cfg = SpectralConfig(a.n, a.n, 1.0)
pj = gproject.Projector(cfg, a.order)
g = torch.Generator(device="cuda").manual_seed(1)
samples = torch.rand((a.cells, pj.n_points), dtype=torch.float64, device="cuda", generator=g)
out = torch.empty((a.cells, cfg.n_k, cfg.n_q), dtype=torch.float64, device="cuda")
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(a.iters):
    ev0.record()
    pj.project(samples, out)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    print(f"iter {i}: {ms:.3f} ms  {a.cells / ms * 1e3:.0f} cells/s  {pj.bytes_per_cell * a.cells / ms / 1e6:.0f} GB/s")
