"""GPU-resident RK4 (config 5 driver) against an oracle RK4 on the CPU.

Reference semantics: harness.rk4_integrate (harness.py:79-120), invariants
exactly conserved (moment_drift() == 0.0, test_harness.py:22-26), divergence
raises RuntimeError (harness.py:103-107).
"""

import numpy as np
import pytest

from conftest import load_op
from oracle import q_oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2605_28475_b200 import harness, inputs  # noqa: E402
from paper_2605_28475_b200.operator import CoefficientField  # noqa: E402


def oracle_rk4_step(oop, y, dt):
    rhs = lambda v: q_oracle.q_angular_first(oop, v)  # noqa: E731
    k1 = rhs(y)
    k2 = rhs(y + 0.5 * dt * k1)
    k3 = rhs(y + 0.5 * dt * k2)
    k4 = rhs(y + dt * k3)
    return y + (dt / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)


def oracle_rk4(op, y, dt, n):
    oop = q_oracle.OracleOperator.from_operator(op)
    rhs = lambda v: q_oracle.q_angular_first(oop, v)  # noqa: E731
    for _ in range(n):
        k1 = rhs(y)
        k2 = rhs(y + 0.5 * dt * k1)
        k3 = rhs(y + 0.5 * dt * k2)
        k4 = rhs(y + dt * k3)
        y = y + (dt / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
    return y


@pytest.mark.parametrize("name,n_steps", [("mm_n4", 20), ("mm_k4l6", 10)])
def test_rk4_matches_oracle_and_conserves(name, n_steps):
    op = load_op(name)
    cfg = op.cfg
    c0 = inputs.bimodal(cfg.n_k, cfg.l_max, 6, seed=5)
    tr = harness.rk4_integrate_batch(op, c0, 0.01, n_steps, record_every=5, watch=[0, 5])
    assert tr.moment_drift() == 0.0
    for j, cell in enumerate([0, 5]):
        ref = oracle_rk4(op, c0[cell], 0.01, n_steps)
        assert q_oracle.rel_err(tr.snapshots[-1, j], ref) <= 1e-12
    fin = tr.final.cpu().numpy()
    assert np.array_equal(fin[[0, 5]], tr.snapshots[-1])


def test_rk4_single_cell_dropin():
    op = load_op("mm_n4")
    c = CoefficientField(inputs.bimodal(op.cfg.n_k, op.cfg.l_max, 1, seed=2)[0], op.cfg)
    tr = harness.rk4_integrate(op, c, 0.01, 6, record_every=2)
    assert tr.coeffs.shape == (4, op.cfg.n_k, op.cfg.n_q) and np.allclose(tr.times, [0, 0.02, 0.04, 0.06])
    assert tr.moment_drift() == 0.0
    assert q_oracle.rel_err(tr.coeffs[-1], oracle_rk4(op, c.values, 0.01, 6)) <= 1e-12
    with pytest.raises(ValueError):
        harness.rk4_integrate(op, c, -1.0, 3)


def test_rk4_divergence_raises():
    op = load_op("hs_n4")
    c0 = inputs.perturbed_maxwellians(op.cfg.n_k, op.cfg.l_max, 4, seed=1)
    c0[2] *= 1e150
    with pytest.raises(RuntimeError, match="diverged"):
        harness.rk4_integrate_batch(op, c0, 1.0, 3)
    # the exact first non-finite step, as the reference reports it
    # (harness.py:103-107): cell 2 scaled by 1e20 overflows in step 2 (oracle RK4)
    c0 = inputs.perturbed_maxwellians(op.cfg.n_k, op.cfg.l_max, 4, seed=1)
    c0[2] *= 1e20
    oop = q_oracle.OracleOperator.from_operator(op)
    y, first = c0[2].copy(), None
    with np.errstate(all="ignore"):
        for step in range(1, 8):
            y = oracle_rk4_step(oop, y, 1.0)
            if not np.all(np.isfinite(y)):
                first = step
                break
    assert first == 2
    with pytest.raises(RuntimeError, match=f"diverged at step {first} "):
        harness.rk4_integrate_batch(op, c0, 1.0, 7, record_every=5)


def test_rk4_config5_operator():
    """Config 5 (Maxwell N=L=10, bimodal): a short GPU trajectory vs the oracle."""
    op = load_op("mm_n10")
    cfg = op.cfg
    c0 = inputs.bimodal(cfg.n_k, cfg.l_max, 64, seed=7)
    tr = harness.rk4_integrate_batch(op, c0, 0.01, 3, record_every=3, watch=[17])
    assert tr.moment_drift() == 0.0
    assert q_oracle.rel_err(tr.snapshots[-1, 0], oracle_rk4(op, c0[17], 0.01, 3)) <= 1e-12


def test_rk4_config5_full_trajectory_matches_reference():
    """Config 5 as BASELINE.json states it: Maxwell molecules N=L=10, bimodal
    cells, RK4 dt = 0.01 for 1,000 steps.  Two cells of a 16-cell batch are
    compared at every 100th step with the reference's own rk4_integrate
    trajectory (tests/golden/make_rk4_golden.py, harness.py:79-120); the
    invariants of every cell stay bitwise constant."""
    import os

    from conftest import GOLDEN

    path = os.path.join(GOLDEN, "rk4_mm_n10.npz")
    if not os.path.exists(path):
        pytest.skip("reference RK4 trajectory not generated")
    d = np.load(path)
    op = load_op("mm_n10")
    cfg = op.cfg
    c0 = inputs.bimodal(cfg.n_k, cfg.l_max, int(d["n_cells"]), seed=int(d["seed"]))
    watch = [int(i) for i in d["cells"]]
    tr = harness.rk4_integrate_batch(op, c0, float(d["dt"]), int(d["n_steps"]), record_every=100, watch=watch)
    assert tr.moment_drift() == 0.0
    assert np.allclose(tr.times, d["times"])
    ref = d["snapshots"]  # (records, cells, n_k, n_q)
    assert tr.snapshots.shape == ref.shape
    for r in range(ref.shape[0]):
        for j in range(len(watch)):
            assert q_oracle.rel_err(tr.snapshots[r, j], ref[r, j]) <= 1e-12, (r, j)


def test_fused_rk4_equals_unfused_bitwise(tmp_path):
    """the fused step (stage arguments, weighted sum and the new
    state formed in the Q epilogues, 4 launches, BFQ_RK4_FUSED=1) equals the
    default unfused sequence (Q launches + elementwise stage kernels) bit for bit."""
    import os
    import subprocess
    import sys

    from conftest import ROOT

    script = tmp_path / "rk4_run.py"
    script.write_text(
        "import os, sys\n"
        f"sys.path.insert(0, {ROOT!r})\n"
        "import numpy as np, torch\n"
        "from paper_2605_28475_b200 import harness, inputs\n"
        "from paper_2605_28475_b200.operator import load_cache\n"
        f"op = load_cache(os.path.join({ROOT!r}, 'operators', sys.argv[1] + '.bfct'))\n"
        "c0 = inputs.bimodal(op.cfg.n_k, op.cfg.l_max, 37, seed=11)\n"
        "tr = harness.rk4_integrate_batch(op, c0, 0.01, 7, record_every=1, watch=np.arange(37))\n"
        "np.save(sys.argv[2], np.concatenate([tr.snapshots.ravel(), tr.final.cpu().numpy().ravel()]))\n")
    outs = {}
    for name in ("mm_n4", "hs_n8", "mm_n10"):
        for mode in ("fused", "unfused"):
            env = dict(os.environ)
            env.pop("BFQ_RK4_FUSED", None)
            if mode == "fused":
                env["BFQ_RK4_FUSED"] = "1"
            path = tmp_path / f"{name}_{mode}.npy"
            res = subprocess.run([sys.executable, str(script), name, str(path)], env=env, capture_output=True,
                                 text=True, timeout=600)
            assert res.returncode == 0, res.stderr[-3000:]
            outs[(name, mode)] = np.load(path)
        assert np.array_equal(outs[(name, "fused")], outs[(name, "unfused")]), name
