"""CPU oracle for the Q(f,f) hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module, and only as the checker / the timed reference
port.  The product path (``paper_2605_28475_b200``) never calls it.

It is a numpy restatement of the reference's contraction strategies
(``/root/reference/pkg/src/boltzfact/contraction.py``):

* :func:`q_angular_first` -- contraction.py:293-317.  Per (tau, q1) slice,
  Phi_S[a,b] = sum_{z in S} g_z f2[a,q2_z] f3[b,q3_z]  (:306-308),
  out_S[k1] = sum_{a,b} R[k1,a,b,tau_S] Phi_S[a,b]      (:309),
  Q[k1,q1_S] += out_S[k1]                               (:310-312).
* :func:`q_naive` -- contraction.py:236-260: full radial contraction per
  COO row, then weighted scatter into q1.  Independent summation order, used
  to cross-check the first.
* :func:`moments` -- basis.py:346-363.

Parity of this restatement is pinned by ``tests/test_oracle.py`` against the
golden fixtures in ``tests/golden/`` (produced by running the reference itself
in the build container, ``tests/golden/make_golden.py``) and against the
reference's own known answers (Q(eq) = 0, Q(0) = 0, bitwise-zero invariant
slots, bilinearity).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass
class OracleOperator:
    """Plain arrays of a factorized operator, 0-based indices."""

    n_k: int
    n_q: int
    q1: np.ndarray
    q2: np.ndarray
    q3: np.ndarray
    tau: np.ndarray
    g: np.ndarray
    slice_starts: np.ndarray
    slice_tau: np.ndarray
    slice_q1: np.ndarray
    r: np.ndarray  # (n_k, n_k, n_k, N_T)

    @classmethod
    def from_operator(cls, op) -> "OracleOperator":
        """From a reference or mirror FactorizedOperator (1-based COO columns)."""
        g = op.g
        z = lambda a: np.asarray(a, dtype=np.int64) - 1  # noqa: E731
        return cls(
            op.cfg.n_k,
            op.cfg.n_q,
            z(g.q1),
            z(g.q2),
            z(g.q3),
            z(g.tau),
            np.asarray(g.g, dtype=np.float64),
            np.asarray(g.slice_starts, dtype=np.int64),
            z(g.slice_tau),
            z(g.slice_q1),
            np.asarray(op.r.values, dtype=np.float64),
        )


def _sort_guard(op: OracleOperator) -> None:
    key = op.tau * op.n_q + op.q1
    if np.any(np.diff(key) < 0):  # contraction.py:297-301
        raise ValueError("COO rows must be sorted and grouped by (tau, q1)")


def q_angular_first(op: OracleOperator, f2: np.ndarray, f3: np.ndarray | None = None,
                    r_slices: np.ndarray | None = None) -> np.ndarray:
    """Q(f2, f3) of one cell, (n_k, n_q) -> (n_k, n_q)."""
    _sort_guard(op)
    f3 = f2 if f3 is None else f3
    n_k, n_q = op.n_k, op.n_q
    # operand columns of every row, the g weight folded into the slot-2 side
    left = f2[:, op.q2] * op.g  # (n_k, N_G)
    right = f3[:, op.q3]  # (n_k, N_G)
    outer = left[:, None, :] * right[None, :, :]  # (n_k, n_k, N_G)
    phi = np.add.reduceat(outer, op.slice_starts[:-1], axis=2)  # (n_k, n_k, N_S)
    if r_slices is None:
        r_slices = op.r[:, :, :, op.slice_tau]  # (n_k, n_k, n_k, N_S)
    out = np.einsum("kabs,abs->ks", r_slices, phi, optimize=True)
    q = np.zeros((n_k, n_q))
    for k1 in range(n_k):
        q[k1] = np.bincount(op.slice_q1, weights=out[k1], minlength=n_q)
    return q


def q_naive(op: OracleOperator, f2: np.ndarray, f3: np.ndarray | None = None) -> np.ndarray:
    """Row-by-row radial contraction (contraction.py:236-260 order)."""
    f3 = f2 if f3 is None else f3
    n_k, n_q = op.n_k, op.n_q
    q = np.zeros((n_k, n_q))
    bounds = np.concatenate(([0], np.flatnonzero(np.diff(op.tau)) + 1, [op.tau.size]))
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        t = op.tau[lo]
        psi = np.einsum("kab,az,bz->kz", op.r[:, :, :, t], f2[:, op.q2[lo:hi]], f3[:, op.q3[lo:hi]],
                        optimize=True) * op.g[lo:hi]
        for k1 in range(n_k):
            q[k1] += np.bincount(op.q1[lo:hi], weights=psi[k1], minlength=n_q)
    return q


def q_batch(op: OracleOperator, cells: np.ndarray, cells3: np.ndarray | None = None) -> np.ndarray:
    """Angular-first over a batch (B, n_k, n_q), one cell at a time."""
    rs = op.r[:, :, :, op.slice_tau]
    out = np.empty_like(cells)
    for i in range(cells.shape[0]):
        out[i] = q_angular_first(op, cells[i], None if cells3 is None else cells3[i], r_slices=rs)
    return out


_SQRT6 = math.sqrt(6.0)


def moments(values: np.ndarray):
    """(mass, momentum[3], energy) of one (n_k, n_q) field, basis.py:346-363."""
    mass = values[0, 0]
    mom = np.array([values[0, 3], values[0, 1], values[0, 2]]) if values.shape[1] > 1 else np.zeros(3)
    e2 = values[1, 0] if values.shape[0] > 1 else 0.0
    return float(mass), mom, float(0.5 * (3.0 * mass - _SQRT6 * e2))


def rel_err(got: np.ndarray, ref: np.ndarray) -> float:
    """max|got - ref| / max|ref| -- the reference's metric (test_contraction.py:63-65)."""
    scale = np.abs(ref).max()
    if scale == 0.0:
        return float(np.abs(got).max())
    return float(np.abs(got - ref).max() / scale)
