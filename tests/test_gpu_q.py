"""GPU parity of the Q(f,f) engine (sm_100a kernels through the C ABI).

Bar: per-cell max|Q_gpu - Q_ref| / max|Q_ref| <= 1e-12 (the reference's own
metric, test_contraction.py:63-65 / cli.py:380-383); invariant slots and
Q(eq), Q(0) bitwise 0.0 (test_acceptance.py:73-92).
"""

import os
import types

import numpy as np
import pytest

from conftest import OPERATORS, golden, golden_names, load_op
from oracle import q_oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2605_28475_b200 import engine, inputs  # noqa: E402
from paper_2605_28475_b200.operator import (  # noqa: E402
    CacheFormatError,
    CacheIntegrityError,
    CoefficientField,
    moments,
)

TOL = 1e-12


def gpu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run(op, cells, cells3=None):
    out = engine.evaluate_batch(op, gpu(cells), None if cells3 is None else gpu(cells3))
    return out.cpu().numpy()


def assert_invariants_zero(q):
    assert np.all(q[:, 0, 0] == 0.0)
    if q.shape[2] > 1:
        assert np.all(q[:, 0, 1:4] == 0.0)
    if q.shape[1] > 1:
        assert np.all(q[:, 1, 0] == 0.0)


@pytest.mark.parametrize("name", golden_names())
def test_golden_parity(name):
    op, d = load_op(name), golden(name)
    q = run(op, d["cells"])
    for i in range(q.shape[0]):
        assert q_oracle.rel_err(q[i], d["q"][i]) <= TOL, (name, i)
    assert_invariants_zero(q)
    q12 = run(op, d["c1"][None], d["c2"][None])[0]
    assert q_oracle.rel_err(q12, d["q12"]) <= TOL


@pytest.mark.parametrize("name", ["hs_n2", "mm_n4", "hs_k4l6", "hs_n8"])
def test_batch_vs_oracle_and_invariants(name):
    op = load_op(name)
    cfg = op.cfg
    cells = np.concatenate([
        inputs.perturbed_maxwellians(cfg.n_k, cfg.l_max, 37, seed=3),
        inputs.uniform_fields(cfg.n_k, cfg.l_max, 11, seed=4),
    ])
    q = run(op, cells)
    oop = q_oracle.OracleOperator.from_operator(op)
    for i in list(range(0, cells.shape[0], 5)) + [cells.shape[0] - 1]:
        assert q_oracle.rel_err(q[i], q_oracle.q_angular_first(oop, cells[i])) <= TOL, i
    assert_invariants_zero(q)
    for i in range(q.shape[0]):
        mass, mom, energy = moments(CoefficientField(q[i], cfg))
        assert mass == 0.0 and np.all(mom == 0.0) and energy == 0.0


@pytest.mark.parametrize("name", ["hs_n2", "hs_n4", "hs_n8"])
def test_equilibrium_and_zero_map_to_zero(name):
    op = load_op(name)
    cfg = op.cfg
    cells = np.zeros((10, cfg.n_k, cfg.n_q))
    cells[:5, 0, 0] = 1.0
    q = run(op, cells)
    assert np.abs(q).max() == 0.0
    q = run(op, cells, cells[::-1].copy())  # bilinear path: Q(eq, 0), Q(0, eq)
    assert np.abs(q).max() == 0.0


@pytest.mark.parametrize("name", ["hs_n2", "hs_k4l6", "hs_n8"])
def test_bilinearity_and_symmetric_paths_agree(name):
    op = load_op(name)
    cfg = op.cfg
    c1 = inputs.uniform_fields(cfg.n_k, cfg.l_max, 9, seed=21)
    c2 = inputs.uniform_fields(cfg.n_k, cfg.l_max, 9, seed=22)
    base = run(op, c1, c2)
    left = run(op, 2.5 * c1, c2)
    right = run(op, c1, 2.5 * c2)
    for i in range(base.shape[0]):  # max-norm relative, the reference's metric
        assert q_oracle.rel_err(left[i], 2.5 * base[i]) <= 1e-13
        assert q_oracle.rel_err(right[i], 2.5 * base[i]) <= 1e-13
    # folded Q(f,f) vs the unfolded bilinear kernel with f3 a distinct copy of f
    sym = run(op, c1)
    full = run(op, c1, c1.copy())
    for i in range(sym.shape[0]):
        assert q_oracle.rel_err(sym[i], full[i]) <= 1e-13


@pytest.mark.parametrize("n", [0, 1, 3, 7, 8, 9, 17, 31])
def test_ragged_batches_are_position_independent(n):
    op = load_op("hs_n4")
    cfg = op.cfg
    cells = inputs.perturbed_maxwellians(cfg.n_k, cfg.l_max, 40, seed=8)
    big = run(op, cells)
    if n == 0:
        out = engine.evaluate_batch(op, gpu(cells[:0]))
        assert out.shape == (0, cfg.n_k, cfg.n_q)
        return
    small = run(op, cells[:n])
    assert np.array_equal(small, big[:n])
    shifted = run(op, cells[3:3 + n])
    assert np.array_equal(shifted, big[3:3 + n])


def test_deterministic():
    op = load_op("hs_n8")
    cfg = op.cfg
    cells = inputs.perturbed_maxwellians(cfg.n_k, cfg.l_max, 64, seed=9)
    assert np.array_equal(run(op, cells), run(op, cells))


def test_maxwell_linearized_diagonal_matches_closed_form():
    """test_contraction.py:156-167: the linearised Maxwell operator at
    equilibrium is diagonal with the closed-form rates (oracles.py:59-72)."""
    op = load_op("mm_k4l6")
    cfg = op.cfg
    rates = {(int(k), int(l)): v for k, l, v in golden("maxwell_rates")["rates"]}
    modes = [(k, l) for k in range(cfg.n_k) for l in range(cfg.l_max + 1)]
    eq = np.zeros((len(modes), cfg.n_k, cfg.n_q))
    eq[:, 0, 0] = 1.0
    e = np.zeros_like(eq)
    for i, (k, l) in enumerate(modes):
        e[i, k, l * l + l] = 1.0
    lin = run(op, eq, e) + run(op, e, eq)  # J e = Q(eq, e) + Q(e, eq)
    for i, (k, l) in enumerate(modes):
        assert abs(lin[i, k, l * l + l] - rates[(k, l)]) <= 1e-11, (k, l)


def test_config1_closed_form_rates():
    """Config 1 (N=L=4 Maxwell): Q[k,q(l,m)] = lambda_kl c[k,q(l,m)] for 2k+l <= 3."""
    op = load_op("mm_n4")
    cfg = op.cfg
    rates = {(int(k), int(l)): v for k, l, v in golden("maxwell_rates")["rates"]}
    cells = inputs.maxwell_config1(cfg.n_k, cfg.l_max, seed=1, n_cells=4)
    q = run(op, cells)
    scale = np.abs(q).max()
    for k in range(cfg.n_k):
        for l in range(cfg.l_max + 1):
            if 2 * k + l > 3:
                continue
            for m in range(-l, l + 1):
                qq = l * l + l + m
                expect = rates[(k, l)] * cells[:, k, qq] if (k, l) not in ((0, 0), (0, 1), (1, 0)) else 0.0
                assert np.all(np.abs(q[:, k, qq] - expect) <= 1e-12 * scale), (k, l, m)


def test_reference_strategy_dropin():
    op = load_op("hs_n4")
    d = golden("hs_n4")
    stats = engine.ContractionStats()
    c = CoefficientField(d["cells"][0].copy(), op.cfg)
    q = engine.evaluate(op, c, "gpu", stats=stats)
    assert isinstance(q, CoefficientField)
    assert q_oracle.rel_err(q.values, d["q"][0]) <= TOL
    n_k = op.cfg.n_k
    assert stats.flops == op.g.n_g * n_k**2 + op.n_s * n_k**3 and stats.n_calls == 1
    with pytest.raises(ValueError):
        engine.evaluate(op, c, "nope")

    class FakeContraction:  # the reference's module-level dict (contraction.py:320-324)
        STRATEGIES = {}

    assert engine.register_with_reference(FakeContraction)
    got = FakeContraction.STRATEGIES["gpu"](op, c, CoefficientField(d["c2"], op.cfg))
    assert q_oracle.rel_err(got.values, run(op, d["cells"][:1], d["c2"][None])[0]) == 0.0


def test_input_validation():
    op = load_op("hs_n4")
    cfg = op.cfg
    with pytest.raises(ValueError):
        engine.evaluate_batch(op, torch.zeros((2, cfg.n_k, cfg.n_q), dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        engine.evaluate_batch(op, torch.zeros((2, cfg.n_k + 1, cfg.n_q), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        engine.evaluate_batch(op, torch.zeros((2, cfg.n_q, cfg.n_k), dtype=torch.float64, device="cuda").transpose(1, 2))
    with pytest.raises(ValueError):
        engine.evaluate_batch(op, gpu(np.zeros((cfg.n_k, cfg.n_q))))
    with pytest.raises(ValueError):
        engine.q_gpu(op, CoefficientField(np.zeros((cfg.n_k, cfg.n_q)), cfg),
                     types.SimpleNamespace(values=np.zeros((1, 1))))


def test_unsorted_operator_rejected():
    import dataclasses

    op = load_op("hs_n2")
    perm = np.arange(op.g.n_g)[::-1].copy()
    g2 = dataclasses.replace(op.g, q1=op.g.q1[perm], q2=op.g.q2[perm], q3=op.g.q3[perm],
                             tau=op.g.tau[perm], g=op.g.g[perm])
    bad = dataclasses.replace(op, g=g2)
    with pytest.raises(ValueError):
        engine.GpuPlan.from_operator(bad)


def test_native_bfct_loader(tmp_path):
    path = os.path.join(OPERATORS, "hs_n4.bfct")
    plan = engine.GpuPlan.from_bfct(path)
    op = load_op("hs_n4")
    cells = inputs.perturbed_maxwellians(op.cfg.n_k, op.cfg.l_max, 20, seed=2)
    assert np.array_equal(run(plan, cells), run(op, cells))
    blob = bytearray(open(path, "rb").read())
    blob[100] ^= 0xFF
    (tmp_path / "bad.bfct").write_bytes(bytes(blob))
    with pytest.raises(CacheIntegrityError):
        engine.GpuPlan.from_bfct(tmp_path / "bad.bfct")
    blob = bytearray(open(path, "rb").read())
    blob[0:4] = b"XXXX"
    (tmp_path / "magic.bfct").write_bytes(bytes(blob))
    with pytest.raises(CacheFormatError):
        engine.GpuPlan.from_bfct(tmp_path / "magic.bfct")
    (tmp_path / "short.bfct").write_bytes(b"BFCT")
    with pytest.raises(CacheFormatError):
        engine.GpuPlan.from_bfct(tmp_path / "short.bfct")


def test_host_buffer_path_matches_device_path():
    op = load_op("hs_n8")
    cfg = op.cfg
    cells = inputs.perturbed_maxwellians(cfg.n_k, cfg.l_max, 4100, seed=12)
    dev = run(op, cells)
    host = engine.evaluate_host(op, cells)
    assert np.array_equal(host, dev)
    c2 = inputs.uniform_fields(cfg.n_k, cfg.l_max, 33, seed=1)
    assert np.array_equal(engine.evaluate_host(op, cells[:33], c2), run(op, cells[:33], c2))


def test_hs12_headline_operator():
    """Config 3 operator: golden cells, plus a 2048-cell batch checked against
    the oracle on a stratified subset and bitwise invariants everywhere."""
    op = load_op("hs_n12")
    cfg = op.cfg
    cells = inputs.perturbed_maxwellians(cfg.n_k, cfg.l_max, 2048, seed=33)
    q = run(op, cells)
    assert_invariants_zero(q)
    oop = q_oracle.OracleOperator.from_operator(op)
    ws = q_oracle.angular_workspace(oop)
    for i in (0, 1, 511, 1024, 2047):
        ref = q_oracle.q_angular_first(oop, cells[i], workspace=ws)
        assert q_oracle.rel_err(q[i], ref) <= TOL, i


@pytest.mark.parametrize("name", ["hs_n2", "mm_n4", "mm_k4l6", "hs_k4l6"])
def test_linearize_matches_reference(name):
    """Batched GPU Jacobian vs the reference's linearize (contraction.py:343-369)."""
    op, d = load_op(name), golden(name)
    if "jac_eq" not in d:
        pytest.skip("no reference Jacobian in the golden file")
    cfg = op.cfg
    eq = CoefficientField.equilibrium(cfg)
    j_eq = engine.linearize(op, eq)
    assert q_oracle.rel_err(j_eq, d["jac_eq"]) <= 1e-12
    j_pm = engine.linearize(op, CoefficientField(d["jac_c"].copy(), cfg))
    assert q_oracle.rel_err(j_pm, d["jac_pm"]) <= 1e-12
    # structure at equilibrium (test_contraction.py:133-147): block-diagonal in q, 5 invariants
    blocks = j_eq.reshape(cfg.n_k, cfg.n_q, cfg.n_k, cfg.n_q).copy()
    for qq in range(cfg.n_q):
        blocks[:, qq, :, qq] = 0.0
    assert np.abs(blocks).max() == 0.0
    if name == "hs_k4l6":
        lam = np.linalg.eigvals(j_eq)
        assert int(np.sum(np.abs(lam) < 1e-12)) == 5


def test_n16_path_synthetic_operator():
    """N=L=16 (config-4 shape: n_k = 17, three 8x8 tiles per axis) on the
    synthetic-R operator, against the oracle on two cells."""
    if not os.path.exists(os.path.join(OPERATORS, "synth_n16.bfct")):
        pytest.skip("synthetic N=L=16 operator not present")
    op = load_op("synth_n16")
    cfg = op.cfg
    cells = inputs.perturbed_maxwellians(cfg.n_k, cfg.l_max, 9, seed=16)
    q = run(op, cells)
    assert_invariants_zero(q)
    oop = q_oracle.OracleOperator.from_operator(op)
    for i in (0, 8):
        assert q_oracle.rel_err(q[i], q_oracle.q_angular_first(oop, cells[i])) <= TOL, i
    q12 = run(op, cells[:3], cells[3:6])  # bilinear path at n_k = 17
    assert q_oracle.rel_err(q12[1], q_oracle.q_angular_first(oop, cells[1], cells[4])) <= TOL


def test_n16_config4_on_gpu_built_operator():
    """Config 4 (hard spheres N=L=16, n_k = 17: two DMMA tiles + the DFMA X1
    row/column per axis, DUAL row groups) with the real Gaunt table and an R
    tensor assembled on this GPU (bfr_assemble) -- the reference's own N=16
    cache is a multi-hour CPU build that is not always shipped.
      * kernel parity: GPU Q vs the oracle on the SAME operator, 1e-12;
      * end-to-end parity vs the reference's evaluate() goldens (tests/golden/
        hs_n16.npz, reference operator): bounded by the GPU-built R's distance
        to the reference R (<= 4e-10 relative, test_gpu_rbuild.py BARS), which
        the high-k rows amplify to 2.1e-9 in Q (measured), so the bar here is
        5e-9 -- the 1e-12 bar against the reference's own N=16 operator is
        test_golden_parity[hs_n16], run whenever operators/hs_n16.bfct is shipped;
      * invariant slots bitwise zero; bilinear path against its golden."""
    from paper_2605_28475_b200 import rbuild
    from paper_2605_28475_b200.operator import SpectralConfig

    d = golden("hs_n16")
    op = rbuild.build_operator(SpectralConfig(16, 16, 1.0))
    cells = d["cells"]
    q = run(op, cells)
    assert_invariants_zero(q)
    oop = q_oracle.OracleOperator.from_operator(op)
    assert q_oracle.rel_err(q[0], q_oracle.q_angular_first(oop, cells[0])) <= TOL
    for i in range(cells.shape[0]):
        assert q_oracle.rel_err(q[i], d["q"][i]) <= 5e-9, i
    q12 = run(op, d["c1"][None], d["c2"][None])[0]
    assert q_oracle.rel_err(q12, q_oracle.q_angular_first(oop, d["c1"], d["c2"])) <= TOL
    assert q_oracle.rel_err(q12, d["q12"]) <= 5e-9


def test_output_overlapping_input_is_rejected():
    """CTAs of a tile still read its cells while others write Q, so
    in-place / overlapping outputs are refused (wrapper and C ABI)."""
    from paper_2605_28475_b200 import _lib

    op = load_op("hs_n4")
    cfg = op.cfg
    f = gpu(inputs.perturbed_maxwellians(cfg.n_k, cfg.l_max, 16, seed=2))
    with pytest.raises(ValueError, match="overlap"):
        engine.evaluate_batch(op, f, out=f)
    big = torch.zeros((17, cfg.n_k, cfg.n_q), dtype=torch.float64, device="cuda")
    big[:16] = f
    with pytest.raises(ValueError, match="overlap"):
        engine.evaluate_batch(op, big[:16], out=big[1:])
    f3 = f.clone()
    with pytest.raises(ValueError, match="overlap"):
        engine.evaluate_batch(op, f, f3, out=f3)
    plan = engine.plan_for(op)
    lib = _lib.lib()
    st = torch.cuda.current_stream().cuda_stream
    assert lib.bfq_eval(plan.handle, f.data_ptr(), None, f.data_ptr() + 8 * cfg.n_dof, 16, st) == _lib.BFQ_EINVAL
    assert b"overlap" in lib.bfq_last_error()
    h = np.zeros((16, cfg.n_k, cfg.n_q))
    assert lib.bfq_eval_host(plan.handle, h.ctypes.data, None, h.ctypes.data, 16) == _lib.BFQ_EINVAL
    # disjoint buffers still work, and the result did not change
    out = engine.evaluate_batch(op, f)
    assert np.array_equal(out.cpu().numpy(), run(op, f.cpu().numpy()))


def test_host_path_pinned_and_pageable_agree():
    """bfq_eval_host: pinned buffers are copied asynchronously, pageable ones
    staged through the plan's pinned chunks; both equal the device path."""
    op = load_op("hs_n8")
    cfg = op.cfg
    cells = inputs.perturbed_maxwellians(cfg.n_k, cfg.l_max, 1000, seed=13)
    dev = run(op, cells)
    pageable = engine.evaluate_host(op, cells)
    assert np.array_equal(pageable, dev)
    from paper_2605_28475_b200 import _lib

    hin = torch.from_numpy(cells).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    _lib.check(_lib.lib().bfq_eval_host(engine.plan_for(op).handle, hin.data_ptr(), None, hout.data_ptr(), 1000))
    assert np.array_equal(hout.numpy(), dev)
    # mixed: pinned input, pageable output
    out = np.empty_like(cells)
    _lib.check(_lib.lib().bfq_eval_host(engine.plan_for(op).handle, hin.data_ptr(), None, out.ctypes.data, 1000))
    assert np.array_equal(out, dev)
