"""The CPU oracle against the reference's golden vectors and known answers."""

import numpy as np
import pytest

from conftest import golden, golden_names, load_op
from oracle import q_oracle


@pytest.mark.parametrize("name", golden_names())
def test_oracle_matches_reference_golden(name):
    op = q_oracle.OracleOperator.from_operator(load_op(name))
    d = golden(name)
    for c, q in zip(d["cells"], d["q"]):
        assert q_oracle.rel_err(q_oracle.q_angular_first(op, c), q) < 1e-13
    assert q_oracle.rel_err(q_oracle.q_angular_first(op, d["c1"], d["c2"]), d["q12"]) < 1e-13
    # the reference's naive strategy agrees with its angular-first (test_contraction.py:57-65)
    assert q_oracle.rel_err(d["q_naive0"][0], d["q"][0]) < 1e-12


@pytest.mark.parametrize("name", ["hs_n2", "mm_n4", "hs_k4l6"])
def test_naive_and_angular_first_agree(name):
    op = q_oracle.OracleOperator.from_operator(load_op(name))
    c = golden(name)["cells"][0]
    assert q_oracle.rel_err(q_oracle.q_naive(op, c), q_oracle.q_angular_first(op, c)) < 1e-12


@pytest.mark.parametrize("name", ["hs_n2", "hs_n4"])
def test_known_answers(name):
    op = q_oracle.OracleOperator.from_operator(load_op(name))
    eq = np.zeros((op.n_k, op.n_q))
    eq[0, 0] = 1.0
    assert np.abs(q_oracle.q_angular_first(op, eq)).max() == 0.0
    assert np.abs(q_oracle.q_angular_first(op, np.zeros_like(eq))).max() == 0.0
    for c in golden(name)["cells"]:
        mass, mom, energy = q_oracle.moments(q_oracle.q_angular_first(op, c))
        assert mass == 0.0 and np.all(mom == 0.0) and energy == 0.0


def test_sort_guard():
    op = q_oracle.OracleOperator.from_operator(load_op("hs_n2"))
    perm = np.arange(op.q1.size)[::-1]
    bad = q_oracle.OracleOperator(op.n_k, op.n_q, op.q1[perm], op.q2[perm], op.q3[perm], op.tau[perm],
                                  op.g[perm], op.slice_starts, op.slice_tau, op.slice_q1, op.r)
    with pytest.raises(ValueError):
        q_oracle.q_angular_first(bad, np.zeros((op.n_k, op.n_q)))


@pytest.mark.parametrize("name", ["hs_n4", "mm_k4l6", "hs_n8"])
def test_oracle_bitwise_equals_live_reference(reference, name):
    """The restatement performs the reference's own operations in the same
    order (gather, CSR segment-sum matmul, einsum, bincount), so on the same
    numpy/scipy it is bit-identical to contraction.q_angular_first -- which is
    why bench.py may time it as the reference's CPU path on the GPU box
    (profiles/r01_cpu_ref_vs_port.txt: same speed per cell)."""
    import os

    from boltzfact import basis

    from conftest import OPERATORS

    ref_op = reference.cache.load_cache(os.path.join(OPERATORS, f"{name}.bfct"))
    op = q_oracle.OracleOperator.from_operator(load_op(name))
    ws = q_oracle.angular_workspace(op)
    for c in golden(name)["cells"]:
        ref = reference.contraction.q_angular_first(ref_op, basis.CoefficientField(c.copy(), ref_op.cfg)).values
        assert np.array_equal(q_oracle.q_angular_first(op, c, workspace=ws), ref)
