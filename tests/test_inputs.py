"""Seeded input generator: pinned to the reference's basis.project."""

import math
import os

import numpy as np

from conftest import GOLDEN
from paper_2605_28475_b200 import inputs


def test_maxwellian_projection_matches_reference_project():
    d = np.load(os.path.join(GOLDEN, "project.npz"))
    meta = d["meta"]
    for i, (k_max, l_max, ux, uy, uz, t) in enumerate(meta):
        ref = d[f"c{i}"]
        mine = inputs.project_maxwellians(int(k_max) + 1, int(l_max), np.array([[ux, uy, uz]]), np.array([t]))[0]
        # the reference's own order-64 product quadrature is accurate to ~1e-13
        assert np.abs(mine - ref).max() < 5e-13


def test_projection_live_against_reference(reference):
    from boltzfact.basis import SpectralConfig, project

    cfg = SpectralConfig(3, 5, 1.0)
    u, t = np.array([0.25, -0.1, 0.05]), 1.1
    f = lambda p: (2 * math.pi * t) ** -1.5 * np.exp(-((p - u) ** 2).sum(1) / (2 * t))  # noqa: E731
    ref = project(f, cfg, 64).values
    mine = inputs.project_maxwellians(cfg.n_k, cfg.l_max, u[None], np.array([t]))[0]
    assert np.abs(mine - ref).max() < 5e-13


def test_block_seeding_is_shard_independent():
    full = inputs.perturbed_maxwellians(5, 4, 3000, seed=7)
    part = inputs.perturbed_maxwellians(5, 4, 1100, seed=7, start=1500)
    assert np.array_equal(full[1500:2600], part)
    b_full = inputs.bimodal(5, 4, 2100, seed=3)
    assert np.array_equal(b_full[1024:2100], inputs.bimodal(5, 4, 1076, seed=3, start=1024))


def test_generator_invariants():
    c = inputs.perturbed_maxwellians(7, 6, 64, seed=1)
    assert np.all(np.isfinite(c))
    # mass of a projected Maxwellian is exactly its density (1) up to quadrature
    assert np.abs(c[:, 0, 0] - 1.0).max() < 1e-12
    c1 = inputs.maxwell_config1(5, 4, seed=2, n_cells=3)
    assert np.all(c1[:, 0, 0] == 1.0) and np.all(c1[:, 0, 1:4] == 0.0) and np.all(c1[:, 1, 0] == 0.0)
    b = inputs.bimodal(5, 4, 8, seed=1)
    odd = [q for q in range(25) if int(math.isqrt(q)) % 2 == 1]
    assert np.abs(b[:, :, odd]).max() < 1e-15  # symmetric pair: odd l vanish
