"""Golden R tensors from the REFERENCE's own assembler (kinematic.assemble_r_tensor).

Run in the build container (reference importable, read-only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_rtensor_golden.py

Writes ``rtensor_quadconv.npz``: the raw (uncorrected) R at N=L=4 for the pads
of the reference's ``quadconv`` validation suite (cli.py:292-310: pads
0,2,4,8,16,32 against pad 64), for gamma = 1 and gamma = 0, plus one
kernel_scale = 0.5 case.  The operator caches in ``operators/`` pin the
corrected R at larger N.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np
from boltzfact.basis import SpectralConfig
from boltzfact.kinematic import assemble_r_tensor
from boltzfact.quadrature import grid_sizes

OUT = Path(__file__).resolve().parent
PADS = (0, 2, 4, 8, 16, 32, 64)

if __name__ == "__main__":
    out = {}
    for gamma in (1.0, 0.0):
        cfg = SpectralConfig(4, 4, gamma)
        for pad in PADS:
            g = grid_sizes(4, 4, pad, pad)
            out[f"g{int(gamma)}_pad{pad}"] = assemble_r_tensor(cfg, g).values
            out[f"g{int(gamma)}_pad{pad}_grid"] = np.array(g.as_tuple())
            print(gamma, pad, flush=True)
    cfg = SpectralConfig(3, 2, 0.5)
    g = grid_sizes(3, 2, 4, 6)
    out["k3l2_g05_ks05"] = assemble_r_tensor(cfg, g, kernel_scale=0.5).values
    out["k3l2_g05_ks05_grid"] = np.array(g.as_tuple())
    np.savez_compressed(OUT / "rtensor_quadconv.npz", **out)
    print("written")
