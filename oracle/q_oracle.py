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


def angular_workspace(op: OracleOperator):
    """The static pieces the reference caches per operator (contraction.py:110-130):
    the row -> slice segment-sum operator as a CSR 0/1 matrix (N_G x N_S) and
    the per-slice gather of R, contiguous as (n_k, n_k^2, N_S)."""
    import scipy.sparse as sp

    n_g = op.g.size
    n_s = op.slice_starts.size - 1
    ids = np.repeat(np.arange(n_s), np.diff(op.slice_starts))
    seg = sp.csr_matrix((np.ones(n_g), ids, np.arange(n_g + 1)), shape=(n_g, n_s))
    r_slices = np.ascontiguousarray(op.r[:, :, :, op.slice_tau].reshape(op.n_k, op.n_k * op.n_k, n_s))
    return seg, r_slices


def q_angular_first(op: OracleOperator, f2: np.ndarray, f3: np.ndarray | None = None,
                    r_slices: np.ndarray | None = None, workspace=None) -> np.ndarray:
    """Q(f2, f3) of one cell, (n_k, n_q) -> (n_k, n_q), contraction.py:293-317.

    Same operations as the reference (gather, CSR segment-sum matmul, einsum
    against the contiguous per-slice R, bincount scatter), so it is also the
    reference's CPU speed on the GPU box (tools/cpu_ref_vs_port.py).  Pass
    ``workspace=angular_workspace(op)`` to reuse the static pieces across
    cells, as the reference does; ``r_slices`` (n_k, n_k, n_k, N_S) is the
    older form of the R half of it."""
    _sort_guard(op)
    f3 = f2 if f3 is None else f3
    n_k, n_q = op.n_k, op.n_q
    if workspace is None:
        workspace = angular_workspace(op) if r_slices is None else (
            angular_workspace(op)[0], np.ascontiguousarray(r_slices.reshape(n_k, n_k * n_k, -1)))
    seg, rs = workspace
    # operand columns of every row, the g weight folded into the slot-2 side
    left = op.g * f2[:, op.q2]  # (n_k, N_G)
    outer = left[:, None, :] * f3[None, :, op.q3]  # (n_k, n_k, N_G)
    phi = np.asarray(outer.reshape(n_k * n_k, -1) @ seg)  # (n_k^2, N_S) segment sums
    out = np.einsum("kaS,aS->kS", rs, phi, optimize=True)
    q = np.empty((n_k, n_q))
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
    ws = angular_workspace(op)
    out = np.empty_like(cells)
    for i in range(cells.shape[0]):
        out[i] = q_angular_first(op, cells[i], None if cells3 is None else cells3[i], workspace=ws)
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
