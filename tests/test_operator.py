"""Host-side operator model: BFCT loader and the CPU part of plan building."""

import dataclasses
import os

import numpy as np
import pytest

from conftest import OPERATORS, load_op
from paper_2605_28475_b200 import engine
from paper_2605_28475_b200.operator import (
    CacheFormatError,
    CacheIntegrityError,
    CoefficientField,
    SpectralConfig,
    load_cache,
    moments,
    q_degree,
    q_index,
)


def test_loader_matches_reference_loader(reference):
    for name in ("hs_n2", "mm_n4", "hs_k4l6", "hs_n8"):
        mine = load_op(name)
        ref = reference.cache.load_cache(os.path.join(OPERATORS, f"{name}.bfct"))
        assert np.array_equal(mine.r.values, ref.r.values)
        for col in ("q1", "q2", "q3", "tau", "g", "slice_starts", "slice_tau", "slice_q1"):
            assert np.array_equal(getattr(mine.g, col), getattr(ref.g, col)), col
        assert mine.g.channels.triplets == ref.g.channels.triplets
        assert mine.cfg.gamma == ref.cfg.gamma and mine.r.conservation_applied == ref.r.conservation_applied


def test_cache_errors(tmp_path):
    blob = open(os.path.join(OPERATORS, "hs_n2.bfct"), "rb").read()
    (tmp_path / "a").write_bytes(b"BFC")
    with pytest.raises(CacheFormatError):
        load_cache(tmp_path / "a")
    (tmp_path / "b").write_bytes(b"XXXX" + blob[4:])
    with pytest.raises(CacheFormatError):
        load_cache(tmp_path / "b")
    bad = bytearray(blob)
    bad[4] = 9  # version
    (tmp_path / "c").write_bytes(bytes(bad))
    with pytest.raises(CacheFormatError):
        load_cache(tmp_path / "c")
    bad = bytearray(blob)
    bad[-1] ^= 1
    (tmp_path / "d").write_bytes(bytes(bad))
    with pytest.raises(CacheIntegrityError):
        load_cache(tmp_path / "d")


def test_index_maps_and_moments():
    assert q_index(0, 0) == 1 and q_index(1, -1) == 2 and q_index(1, 1) == 4
    for q in range(1, 50):
        assert q_index(*q_degree(q)) == q
    cfg = SpectralConfig(2, 2)
    c = CoefficientField.equilibrium(cfg)
    mass, mom, energy = moments(c)
    assert mass == 1.0 and np.all(mom == 0) and energy == 1.5
    with pytest.raises(ValueError):
        CoefficientField(np.zeros((2, 2)), cfg)
    with pytest.raises(ValueError):
        SpectralConfig(1, 1, gamma=2.0)


def test_host_plan_folds_symmetric_operators():
    for name in ("hs_n2", "mm_n4", "hs_k4l6", "hs_n8"):
        info = engine.host_plan_info(load_op(name))
        assert info["folded"] == 1
        assert info["cells_per_cta"] * 1 <= 8 and info["smem_bytes"] <= 232448


def test_host_plan_detects_broken_symmetry():
    op = load_op("hs_n4")
    r = op.r.values.copy()
    r[2, 1, 3, 7] += 1e-3  # break R[k1,a,b,tau] == R[k1,b,a,tau']
    bad = dataclasses.replace(op, r=dataclasses.replace(op.r, values=r))
    assert engine.host_plan_info(bad)["folded"] == 0
    g = op.g.g.copy()
    z = int(np.flatnonzero(op.g.q2 != op.g.q3)[0])  # a row that is not its own swap partner
    g[z] *= 1.0 + 1e-12
    bad = dataclasses.replace(op, g=dataclasses.replace(op.g, g=g))
    assert engine.host_plan_info(bad)["folded"] == 0


def test_host_plan_rejects_bad_tables():
    op = load_op("hs_n2")
    perm = np.arange(op.g.n_g)[::-1].copy()
    g2 = dataclasses.replace(op.g, q1=op.g.q1[perm], q2=op.g.q2[perm], q3=op.g.q3[perm],
                             tau=op.g.tau[perm], g=op.g.g[perm])
    with pytest.raises(ValueError, match="sorted"):
        engine.host_plan_info(dataclasses.replace(op, g=g2))
    q2 = op.g.q2.copy()
    q2[0] = op.cfg.n_q + 5
    with pytest.raises(ValueError):
        engine.host_plan_info(dataclasses.replace(op, g=dataclasses.replace(op.g, q2=q2)))


def test_host_plan_large_configs_fit():
    """Every BASELINE size gets a shared-memory configuration (CPU-only check)."""
    for name in ("hs_n12", "mm_n10"):
        path = os.path.join(OPERATORS, f"{name}.bfct")
        if not os.path.exists(path):
            continue
        info = engine.host_plan_info(load_op(name))
        assert info["folded"] == 1 and info["smem_bytes"] <= 232448


def test_annealed_packing_keeps_a_valid_schedule(monkeypatch):
    """The annealing refinement of the CTA packing (bfq_plan.cpp, on by default where
    two R rings fit) never needs more CTAs per tile than the greedy packers, and the
    plan stays valid (the builder self-checks every unit is scheduled exactly once)."""
    op = load_op("hs_n8")
    monkeypatch.setenv("BFQ_PACK_REFINE", "0")
    greedy = engine.host_plan_info(op)
    monkeypatch.setenv("BFQ_PACK_REFINE", "1")
    refined = engine.host_plan_info(op)
    assert refined["items_per_tile"] <= greedy["items_per_tile"]
    for k in ("cells_per_cta", "warps_per_cta", "smem_bytes", "exec_macs_per_cell", "useful_macs_per_cell"):
        assert refined[k] == greedy[k]
