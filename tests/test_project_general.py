"""General projection (basis.project, basis.py:262-299), host side: the grid,
the sample points and the kernel's weight tables (paper_2605_28475_b200/
project.py) are pinned against the live reference's outputs stored in
tests/golden/project_general.npz -- the same contraction the GPU kernel
performs, done here with numpy on the tables -- and against the reference's
quadrature / point construction when the reference is importable."""

import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, reference_available

sys.path.insert(0, GOLDEN)
from project_funcs import CASES, FUNCS  # noqa: E402

from paper_2605_28475_b200 import project as gproject  # noqa: E402
from paper_2605_28475_b200.operator import SpectralConfig  # noqa: E402

GOLD = np.load(os.path.join(GOLDEN, "project_general.npz"))


def host_projection(samples, cfg, order):
    """The kernel's contraction on the host: azimuthal, polar, radial sums."""
    phi_tab, theta_tab, radial_tab, (n_v, n_t, n_p) = gproject.projection_tables(cfg, order)
    f = samples.reshape(n_v, n_t, n_p)
    g = np.einsum("vtp,cp->vtc", f, phi_tab)
    out = np.empty((cfg.n_k, cfg.n_q))
    for l in range(cfg.l_max + 1):
        for m in range(-l, l + 1):
            col = 0 if m == 0 else (2 * -m - 1 if m < 0 else 2 * m)
            a = g[:, :, col] @ theta_tab[l * (l + 1) // 2 + abs(m)]  # (n_v,)
            out[:, l * l + l + m] = radial_tab[l] @ a
    return out


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("name", sorted(FUNCS))
def test_tables_reproduce_reference_project(case, name):
    k, l, order = case
    cfg = SpectralConfig(k, l, 1.0)
    pts = gproject.project_points(cfg, order)
    got = host_projection(FUNCS[name](pts), cfg, order)
    ref = GOLD[f"{name}_k{k}_l{l}_o{order}"]
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_order_validation():
    with pytest.raises(ValueError):
        gproject.projection_grid(4, 0)
    with pytest.raises(ValueError):
        gproject.project(lambda p: np.ones(len(p)), SpectralConfig(2, 2), 0)


@pytest.mark.skipif(not reference_available(), reason="reference not importable")
def test_points_and_rules_match_reference(reference):
    from boltzfact import quadrature

    cfg = SpectralConfig(6, 5, 1.0)
    v, r_w, cos_t, w_t, phi, w_p = gproject.projection_grid(cfg.l_max, 20)
    ggl = quadrature.gauss_laguerre_gen(20, 0.5)
    assert np.allclose(v, np.sqrt(2.0 * ggl.nodes), rtol=0, atol=1e-14)
    gl = quadrature.gauss_legendre(20)
    assert np.array_equal(cos_t, gl.nodes) or np.allclose(cos_t, gl.nodes, rtol=0, atol=1e-15)
    tp = quadrature.trapezoid_periodic(41)
    assert np.array_equal(phi, tp.nodes) and np.array_equal(w_p, tp.weights)
    pts = gproject.project_points(cfg, 20)
    assert pts.shape == (20 * 20 * 41, 3)


@pytest.mark.parametrize("case", CASES)
def test_projection_oracle_matches_reference(case):
    """oracle/project_oracle.py (bench's CPU baseline) against the live reference."""
    from oracle.project_oracle import ProjectionOracle

    k, l, order = case
    cfg = SpectralConfig(k, l, 1.0)
    orc = ProjectionOracle(k, l, gproject.projection_grid(l, order))
    pts = gproject.project_points(cfg, order)
    for name, f in FUNCS.items():
        ref = GOLD[f"{name}_k{k}_l{l}_o{order}"]
        assert np.max(np.abs(orc.project(f(pts)) - ref)) <= 1e-14 * np.max(np.abs(ref))
