"""The drop-in exercised through the LIVE reference package (not a stand-in):
the unmodified ``boltzfact`` installed into ``baseline/_ref`` (pip --target of
the reference) travels to the GPU box with the snapshot.
``engine.register_with_reference`` installs the "gpu" strategy into the
reference's own ``contraction.STRATEGIES`` (contraction.py:320-324); then

* the reference's ``evaluate(op, c, "gpu")`` (contraction.py:327-340) on the
  reference's own ``load_cache`` operator must match its ``evaluate(op, c)``
  (angular_first on the CPU) to 1e-12 with the invariant slots exactly 0, and
* the reference's ``harness.rk4_integrate(..., strategy="gpu")``
  (harness.py:79-120) must follow its CPU trajectory to 1e-12 with
  ``moment_drift() == 0.0``.

Skipped when baseline/_ref is absent (the install is git-ignored)."""

import os
import sys

import numpy as np
import pytest

from conftest import OPERATORS, ROOT

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

REF = os.path.join(ROOT, "baseline", "_ref")
if not os.path.isdir(os.path.join(REF, "boltzfact")):
    pytest.skip("baseline/_ref (the installed reference) not present", allow_module_level=True)
if REF not in sys.path:
    sys.path.insert(0, REF)

from boltzfact import basis, cache, contraction, harness  # noqa: E402

from paper_2605_28475_b200 import engine, inputs  # noqa: E402


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.fixture(scope="module")
def registered():
    assert engine.register_with_reference(contraction)
    assert contraction.STRATEGIES["gpu"] is engine.q_gpu
    return contraction


@pytest.mark.parametrize("name", ["hs_n4", "hs_n8", "mm_n10"])
def test_reference_evaluate_gpu_strategy(registered, name):
    op = cache.load_cache(os.path.join(OPERATORS, f"{name}.bfct"))  # the reference's own loader
    cfg = op.cfg
    cells = inputs.perturbed_maxwellians(cfg.n_k, cfg.l_max, 3, seed=11)
    for v in cells:
        c = basis.CoefficientField(v.copy(), cfg)
        stats = contraction.ContractionStats()
        q = contraction.evaluate(op, c, "gpu", stats=stats)
        ref = contraction.evaluate(op, c)  # angular_first, CPU
        assert isinstance(q, basis.CoefficientField)
        assert _rel(q.values, ref.values) <= 1e-12
        assert np.all(q.values[0, :4] == 0.0) and q.values[1, 0] == 0.0
        mass, mom, energy = basis.moments(q)
        assert mass == 0.0 and np.all(np.asarray(mom) == 0.0) and energy == 0.0
        assert stats.n_calls == 1 and stats.flops == op.g.n_g * cfg.n_k**2 + op.n_s * cfg.n_k**3
    with pytest.raises(ValueError):
        contraction.evaluate(op, basis.CoefficientField(cells[0], cfg), "no-such-strategy")


def test_reference_rk4_integrate_gpu_strategy(registered):
    op = cache.load_cache(os.path.join(OPERATORS, "mm_n4.bfct"))
    cfg = op.cfg
    c0 = basis.CoefficientField(inputs.bimodal(cfg.n_k, cfg.l_max, 1, seed=3)[0].copy(), cfg)
    tr_gpu = harness.rk4_integrate(op, c0, 0.01, 5, strategy="gpu")
    tr_cpu = harness.rk4_integrate(op, c0, 0.01, 5)
    assert tr_gpu.coeffs.shape == tr_cpu.coeffs.shape
    for s in range(tr_gpu.coeffs.shape[0]):
        assert _rel(tr_gpu.coeffs[s], tr_cpu.coeffs[s]) <= 1e-12, s
    assert tr_gpu.moment_drift() == 0.0
