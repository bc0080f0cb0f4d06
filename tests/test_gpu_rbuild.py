"""GPU R-tensor build (bfr_assemble) against the reference's own R tensors.

Parity bar: relative l-inf error
max|R_gpu - R_ref| / max|R_ref| <= 1e-12 -- the reference's `quadconv`
criterion (cli.py:292-310) -- for every operator up to N=L=10.  At N=L=12 the
reference's own fp64 rounding in its monomial radial expansion
(kinematic.py:458-471) reaches 1.1e-12 at k1 = 12 (measured against an
extended-precision restatement, tests/precision/rbuild_precision.py); the GPU
build carries that expansion in compensated arithmetic and is held to 2e-12
there.  At N=L=16 (k1 up to 16) two fp64 evaluations of the reference algorithm
already differ by ~1e-10 (reference vs its numpy restatement 8.1e-11, vs long
double 1.2e-10, profiles/r01_rbuild_precision.txt); the GPU build is at 2.2e-10
and held to 4e-10.
"""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN, golden, load_op
from paper_2605_28475_b200 import engine, rbuild
from paper_2605_28475_b200.operator import (
    CoefficientField,
    RTensor,
    SpectralConfig,
    load_cache,
    moments,
    save_cache,
)

pytestmark = pytest.mark.gpu

BARS = {"hs_n2": 1e-12, "hs_n4": 1e-12, "mm_n4": 1e-12, "hs_k4l6": 1e-12, "mm_k4l6": 1e-12,
        "hs_n8": 1e-12, "mm_n10": 1e-12, "hs_n12": 2e-12, "hs_n16": 4e-10}


def rel_linf(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


def corrected(r):
    return rbuild.apply_detailed_balance(rbuild.apply_conservation(r))


@pytest.mark.parametrize("name", list(BARS))
def test_r_matches_reference_cache(name):
    ref = load_op(name)
    r = corrected(rbuild.assemble_r_tensor(ref.cfg, rbuild.GridSpec(*ref.r.grid)))
    err = rel_linf(r.values, ref.r.values)
    assert err <= BARS[name], f"{name}: rel l-inf {err:.3e}"
    # the corrected slots are exact zeros, as in the reference
    t0 = ref.r.channels.tau(0, 0, 0) - 1
    assert np.all(r.values[:, 0, 0, t0] == 0.0)
    for t, (l1, _, _) in enumerate(ref.r.channels.triplets):
        if l1 <= 1:
            assert np.all(r.values[0, :, :, t] == 0.0)
    st = rbuild.last_stats()
    assert st["ms_total"] > 0 and st["contract_macs"] > 0


def _quadconv():
    path = os.path.join(GOLDEN, "rtensor_quadconv.npz")
    if not os.path.exists(path):
        pytest.skip("rtensor golden not generated")
    return np.load(path)


@pytest.mark.parametrize("gamma", [1, 0])
def test_raw_r_matches_reference_at_every_quadconv_pad(gamma):
    """Raw (uncorrected) R of assemble_r_tensor for the reference's quadconv pads."""
    d = _quadconv()
    cfg = SpectralConfig(4, 4, float(gamma))
    for pad in (0, 2, 4, 8, 16, 32, 64):
        grid = rbuild.GridSpec(*(int(x) for x in d[f"g{gamma}_pad{pad}_grid"]))
        r = rbuild.assemble_r_tensor(cfg, grid)
        assert rel_linf(r.values, d[f"g{gamma}_pad{pad}"]) <= 1e-13, pad


@pytest.mark.parametrize("gamma", [1, 0])
def test_quadconv_suite(gamma):
    """cli.py:292-310: monotone decay of the pad error vs pad 64 and pad-32 below 1e-12."""
    cfg = SpectralConfig(4, 4, float(gamma))
    ref = rbuild.assemble_r_tensor(cfg, rbuild.grid_sizes(4, 4, 64, 64)).values
    scale = np.abs(ref).max()
    errs = [float(np.abs(rbuild.assemble_r_tensor(cfg, rbuild.grid_sizes(4, 4, p, p)).values - ref).max()
                  / scale) for p in (0, 2, 4, 8, 16, 32)]
    assert all(b < a for a, b in zip(errs, errs[1:])), errs
    assert errs[-1] < 1e-12, errs


def test_kernel_scale_and_gamma_half():
    d = _quadconv()
    grid = rbuild.GridSpec(*(int(x) for x in d["k3l2_g05_ks05_grid"]))
    r = rbuild.assemble_r_tensor(SpectralConfig(3, 2, 0.5), grid, kernel_scale=0.5)
    assert rel_linf(r.values, d["k3l2_g05_ks05"]) <= 1e-13
    r1 = rbuild.assemble_r_tensor(SpectralConfig(3, 2, 0.5), grid, kernel_scale=1.0)
    assert rel_linf(0.5 * r1.values, r.values) <= 1e-15


def test_slot_symmetry_is_exact():
    """R[k,a,b,(l1,l2,l3)] == R[k,b,a,(l1,l3,l2)] bitwise (kinematic.py:559-569)."""
    ref = load_op("hs_n8")
    r = rbuild.assemble_r_tensor(ref.cfg, rbuild.GridSpec(*ref.r.grid))
    ch = r.channels
    for t, (l1, l2, l3) in enumerate(ch.triplets):
        s = ch.tau(l1, l3, l2) - 1
        assert np.array_equal(r.values[..., t], r.values[..., s].transpose(0, 2, 1))


def test_build_operator_drives_q_to_reference_golden(tmp_path):
    """build_operator on the GPU -> Q(f,f) on the GPU == the reference's evaluate()."""
    for name in ("hs_n4", "mm_n4", "hs_k4l6"):
        ref = load_op(name)
        op = rbuild.build_operator(ref.cfg)
        assert op.r.conservation_applied and op.r.detailed_balance_applied
        assert op.r.max_zeroed > 0.0
        g = golden(name)
        q = engine.evaluate_batch(op, torch.from_numpy(g["cells"]).cuda()).cpu().numpy()
        for qi, qr in zip(q, g["q"]):
            assert np.abs(qi - qr).max() / np.abs(qr).max() <= 1e-12
            mass, mom, en = moments(CoefficientField(qi, ref.cfg))
            assert mass == 0.0 and np.all(mom == 0.0) and en == 0.0
        eq = CoefficientField.equilibrium(ref.cfg)
        assert np.abs(engine.evaluate(op, eq, "gpu").values).max() == 0.0
        # the cache written from the GPU build reads back identically
        path = tmp_path / f"{name}.bfct"
        save_cache(path, op)
        back = load_cache(path)
        assert np.array_equal(back.r.values, op.r.values) and np.array_equal(back.g.g, op.g.g)


def test_rejects_unsupported_sizes():
    with pytest.raises(ValueError):
        rbuild.assemble_r_tensor(SpectralConfig(17, 2, 1.0))  # n_k > 17
    with pytest.raises(ValueError):
        rbuild.assemble_r_tensor(SpectralConfig(4, 4, 1.0), rbuild.GridSpec(3, 3, 3, 3, 3, 3, 3, 0, 0))


def test_rtensor_type_is_reference_compatible():
    r = rbuild.assemble_r_tensor(SpectralConfig(2, 2, 1.0))
    assert isinstance(r, RTensor) and r.values.shape == (3, 3, 3, r.channels.n_t)
    assert r.values.flags.c_contiguous and r.max_zeroed == 0.0


def test_build_is_bitwise_deterministic():
    """Fixed-order split reduction: two assemblies of the same operator are identical."""
    ref = load_op("hs_n8")
    g = rbuild.GridSpec(*ref.r.grid)
    a = rbuild.assemble_r_tensor(ref.cfg, g).values
    b = rbuild.assemble_r_tensor(ref.cfg, g).values
    assert np.array_equal(a, b)
