"""R-tensor build: the CPU oracle against the reference's R, and the host-side
tables of the GPU build (grid sizes, 3-j symbols, Gaunt table, cache writer)."""

import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_op
from oracle import r_oracle
from paper_2605_28475_b200 import rbuild
from paper_2605_28475_b200.operator import SpectralConfig, load_cache, save_cache

SMALL = ["hs_n2", "hs_n4", "mm_n4"]
ALL_OPS = ["hs_n2", "hs_n4", "mm_n4", "hs_k4l6", "mm_k4l6", "hs_n8", "mm_n10", "hs_n12"]


def rel_linf(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


@pytest.mark.parametrize("name", SMALL)
def test_oracle_matches_reference_r(name):
    """kinematic.py restatement == the R stored by `boltzfact build` (after corrections)."""
    op = load_op(name)
    cfg = op.cfg
    r = r_oracle.assemble_r(cfg.k_max, cfg.l_max, cfg.gamma, grid=op.r.grid[:7])
    assert rel_linf(r, op.r.values) < 2e-15


def test_oracle_matches_reference_raw_r_golden():
    """Raw (uncorrected) R of the reference's quadconv suite pads, incl. kernel_scale."""
    path = os.path.join(GOLDEN, "rtensor_quadconv.npz")
    if not os.path.exists(path):
        pytest.skip("rtensor golden not generated")
    d = np.load(path)
    for key in ("g1_pad0", "g0_pad8", "k3l2_g05_ks05"):
        grid = tuple(int(x) for x in d[key + "_grid"])
        k, l, gam, ks = (3, 2, 0.5, 0.5) if key.startswith("k3") else (4, 4, float(key[1]), 1.0)
        r = r_oracle.assemble_r(k, l, gam, grid=grid[:7], kernel_scale=ks, conservation=False,
                                detailed_balance=False)
        assert rel_linf(r, d[key]) < 2e-15, key


@pytest.mark.parametrize("name", ALL_OPS)
def test_grid_sizes_match_caches(name):
    op = load_op(name)
    g = rbuild.grid_sizes(op.cfg.k_max, op.cfg.l_max)
    assert g.as_tuple() == tuple(op.r.grid)
    assert r_oracle.grid_sizes(op.cfg.k_max, op.cfg.l_max) == tuple(op.r.grid[:7])


def test_check_grid_rejects_under_resolved():
    g = rbuild.grid_sizes(4, 4, 0, 0)
    rbuild.check_grid(g, 4, 4)
    bad = rbuild.GridSpec(g.n_e - 1, *g.as_tuple()[1:])
    with pytest.raises(ValueError, match="n_e"):
        rbuild.check_grid(bad, 4, 4)
    with pytest.raises(ValueError):
        rbuild.grid_sizes(4, 4, -1, 0)


def test_wigner3j_known_values_and_symmetries():
    # (1 1 0; 0 0 0) = -1/sqrt(3); (2 2 2; 0 0 0) = -sqrt(2/35)
    assert rbuild.wigner3j(1, 1, 0, 0, 0, 0) == pytest.approx(-1 / math.sqrt(3), abs=2e-16)
    assert rbuild.wigner3j(2, 2, 2, 0, 0, 0) == pytest.approx(-math.sqrt(2 / 35), abs=1e-16)
    assert rbuild.wigner3j(1, 1, 1, 0, 0, 0) == 0.0
    rng = np.random.default_rng(3)
    for _ in range(200):
        l1, l2 = (int(x) for x in rng.integers(0, 9, 2))
        l3 = int(rng.integers(abs(l1 - l2), l1 + l2 + 1))
        m1 = int(rng.integers(-l1, l1 + 1))
        m2 = int(rng.integers(-l2, l2 + 1))
        m3 = -m1 - m2
        v = rbuild.wigner3j(l1, l2, l3, m1, m2, m3)
        assert v == r_oracle.wigner3j(l1, l2, l3, m1, m2, m3) or abs(v - r_oracle.wigner3j(
            l1, l2, l3, m1, m2, m3)) < 1e-16
        sign = -1.0 if (l1 + l2 + l3) % 2 else 1.0
        assert rbuild.wigner3j(l2, l1, l3, m2, m1, m3) == sign * v
        assert rbuild.wigner3j(l1, l2, l3, -m1, -m2, -m3) == sign * v


@pytest.mark.parametrize("name", ["hs_n2", "hs_n4", "hs_k4l6", "hs_n8"])
def test_gaunt_table_bitwise_equal_to_reference(name):
    op = load_op(name)
    coo = rbuild.build_gaunt_coo(op.cfg.l_max)
    for col in ("q1", "q2", "q3", "tau", "slice_starts", "slice_tau", "slice_q1"):
        assert np.array_equal(getattr(coo, col), getattr(op.g, col)), col
    assert np.array_equal(coo.g, op.g.g)
    assert coo.channels.triplets == op.g.channels.triplets


def test_channels_and_structural_counts():
    # test_acceptance.py:37,46-56: N_T = 42 at L = 4; N_G at L = 4 / 8
    assert rbuild.enumerate_channels(4).n_t == 42
    assert rbuild.build_gaunt_coo(4).n_g == 1158
    assert rbuild.build_gaunt_coo(8).n_g == 23621


@pytest.mark.parametrize("name", ["hs_n2", "hs_n4", "hs_k4l6"])
def test_save_cache_roundtrip_is_bytewise(tmp_path, name):
    src = os.path.join(os.path.dirname(os.path.dirname(__file__)), "operators", name + ".bfct")
    op = load_op(name)
    out = tmp_path / "x.bfct"
    n = save_cache(out, op)
    assert n == os.path.getsize(out)
    assert out.read_bytes() == open(src, "rb").read()
    again = load_cache(out)
    assert np.array_equal(again.r.values, op.r.values)


def test_null_space_corrections_host_side():
    from paper_2605_28475_b200.operator import RTensor

    op = load_op("hs_n4")

    raw = RTensor(np.ones_like(op.r.values), op.r.channels, 1.0, op.r.grid)
    c = rbuild.apply_conservation(raw)
    assert c.conservation_applied and c.max_zeroed == 1.0
    for t, (l1, _, _) in enumerate(op.r.channels.triplets):
        assert np.all(c.values[0, :, :, t] == 0.0) == (l1 <= 1)
        assert np.all(c.values[1, :, :, t] == 0.0) == (l1 == 0)
    b = rbuild.apply_detailed_balance(c)
    t0 = op.r.channels.tau(0, 0, 0) - 1
    assert b.detailed_balance_applied and np.all(b.values[:, 0, 0, t0] == 0.0)
    assert np.array_equal(rbuild.apply_conservation(c).values, c.values)  # idempotent


def test_gpu_build_without_library_fails_loudly(monkeypatch):
    from paper_2605_28475_b200 import _lib

    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/libbfq.so")
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(_lib.EngineUnavailable):
        rbuild.assemble_r_tensor(SpectralConfig(2, 2, 1.0))


def test_gpu_rtensor_type_flows_through_reference_build(reference, tmp_path, monkeypatch):
    """register_with_reference swaps the reference's assemble_r_tensor; the
    RTensor we return satisfies the reference's corrections, FactorizedOperator
    and save_cache/load_cache (GPU call stubbed with the reference's own R)."""
    import boltzfact.cache as rcache
    import boltzfact.contraction as rcon
    import boltzfact.kinematic as rkin

    from paper_2605_28475_b200.operator import RTensor

    ref = load_op("hs_n4")
    raw = r_oracle.assemble_r(4, 4, 1.0, conservation=False, detailed_balance=False)

    def fake_assemble(cfg, grid=None, *, kernel_scale=1.0, threads=1, device=0, return_halves=False):
        g = grid or rbuild.grid_sizes(cfg.k_max, cfg.l_max)
        return RTensor(raw.copy(), rbuild.enumerate_channels(cfg.l_max), float(cfg.gamma), g)

    monkeypatch.setattr(rbuild, "assemble_r_tensor", fake_assemble)
    monkeypatch.setattr(rkin, "assemble_r_tensor", rkin.assemble_r_tensor)
    monkeypatch.setattr(rcon, "assemble_r_tensor", rcon.assemble_r_tensor)
    assert rbuild.register_with_reference(rkin, rcon)
    assert rcon.assemble_r_tensor is fake_assemble
    from boltzfact.basis import SpectralConfig as RCfg

    op = rcon.build_operator(RCfg(4, 4, 1.0))
    assert np.abs(op.r.values - ref.r.values).max() / np.abs(ref.r.values).max() < 2e-15
    assert op.r.conservation_applied and op.r.detailed_balance_applied
    path = tmp_path / "x.bfct"
    rcache.save_cache(path, op)
    back = rcache.load_cache(path)
    assert np.array_equal(back.r.values, op.r.values)
