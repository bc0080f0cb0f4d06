"""Velocity-space test functions for the general projection parity
(basis.project, basis.py:262-299): deterministic, non-Maxwellian, evaluated on
(n, 3) point arrays.  Shared by make_project_golden.py (run against the live
reference) and the tests."""

import numpy as np

NORM = (2.0 * np.pi) ** -1.5


def aniso_poly(pts):
    """Maxwellian times an anisotropic polynomial (stress, heat-flux-like terms)."""
    vx, vy, vz = pts[:, 0], pts[:, 1], pts[:, 2]
    r2 = vx * vx + vy * vy + vz * vz
    return NORM * np.exp(-0.5 * r2) * (1.0 + 0.3 * vx * vy - 0.2 * vz**3 + 0.05 * vx * vx - 0.01 * r2 * vz)


def bimodal_t(pts):
    """Two drifting Maxwellians with different temperatures and weights."""
    a = pts - np.array([0.7, -0.2, 0.4])
    b = pts - np.array([-0.5, 0.3, -0.6])
    fa = (2.0 * np.pi * 0.8) ** -1.5 * np.exp(-np.sum(a * a, axis=1) / 1.6)
    fb = (2.0 * np.pi * 1.3) ** -1.5 * np.exp(-np.sum(b * b, axis=1) / 2.6)
    return 0.6 * fa + 0.4 * fb


def quartic(pts):
    """Non-Gaussian tail with a non-polynomial angular modulation."""
    d = pts - np.array([0.2, 0.1, -0.3])
    r2 = np.sum(d * d, axis=1)
    return 0.05 * np.exp(-0.125 * r2 * r2) * (1.0 + 0.1 * np.sin(pts[:, 0]) * np.cos(0.5 * pts[:, 2]))


FUNCS = {"aniso_poly": aniso_poly, "bimodal_t": bimodal_t, "quartic": quartic}
CASES = [(4, 4, 16), (8, 8, 32), (12, 12, 64)]  # (k_max, l_max, radial quadrature order)
