"""CPU oracle for the general projection -- TEST INFRASTRUCTURE ONLY.

Only ``tests/`` and ``bench.py``'s CPU-baseline leg may import this module.
It restates the reference's ``basis.project`` (basis.py:262-299) on samples
already taken on its product grid: the same two einsums, in the same order,
as the reference performs after calling f --

    ang[v, q]  = sum_{t,p} f[v,t,p] Y[q,t,p] w_t w_p     (basis.py:291-292)
    c[k, q]    = sum_v rad[k,q,v] ang[v,q] r_w[v]         (basis.py:294-298)

with Y the real spherical harmonic table (_real_sph_table, basis.py:244-258)
and rad the radial functions (radial_eval_all, basis.py:126-132).  Parity is
pinned by tests/test_project_general.py against tests/golden/
project_general.npz (the live reference's outputs).
"""

from __future__ import annotations

import math

import numpy as np
from scipy.special import lpmv


class ProjectionOracle:
    def __init__(self, k_max: int, l_max: int, grid):
        """``grid`` = (v, r_w, cos_t, w_t, phi, w_p) of basis.project (:272-282)."""
        self.n_k, self.l_max = k_max + 1, l_max
        v, self.r_w, cos_t, self.w_t, phi, self.w_p = grid
        n_q = (l_max + 1) ** 2
        y = np.empty((n_q, cos_t.size, phi.size))
        for l in range(l_max + 1):
            for m in range(l + 1):
                norm = math.exp(0.5 * (math.log((2 * l + 1) / (4.0 * math.pi))
                                       + math.lgamma(l - m + 1.0) - math.lgamma(l + m + 1.0)))
                th = norm * lpmv(m, l, cos_t)
                if m == 0:
                    y[l * l + l] = th[:, None]
                else:
                    s = (-1.0) ** m * math.sqrt(2.0)
                    y[l * l + l + m] = s * th[:, None] * np.cos(m * phi)
                    y[l * l + l - m] = s * th[:, None] * np.sin(m * phi)
        self.ylm = y
        rad = np.empty((self.n_k, n_q, v.size))
        x = 0.5 * v * v
        for l in range(l_max + 1):
            a = l + 0.5
            lag = np.empty((self.n_k, v.size))
            lag[0] = 1.0
            if self.n_k > 1:
                lag[1] = 1.0 + a - x
            for k in range(1, self.n_k - 1):
                lag[k + 1] = ((2 * k + a + 1 - x) * lag[k] - (k + a) * lag[k - 1]) / (k + 1)
            norms = np.array([math.exp(0.5 * (1.5 * math.log(2.0 * math.pi) + math.lgamma(k + 1.0)
                                               - (l + 0.5) * math.log(2.0) - math.lgamma(k + l + 1.5)))
                              for k in range(self.n_k)])
            phis = norms[:, None] * v**l * lag
            for m in range(-l, l + 1):
                rad[:, l * l + l + m, :] = phis
        self.rad = rad
        self.shape = (v.size, cos_t.size, phi.size)

    def project(self, samples: np.ndarray) -> np.ndarray:
        fv = np.asarray(samples, dtype=float).reshape(self.shape)
        ang = np.einsum("vtp,qtp,t,p->vq", fv, self.ylm, self.w_t, self.w_p)
        return np.einsum("kqv,vq,v->kq", self.rad, ang, self.r_w)
