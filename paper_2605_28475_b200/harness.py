"""GPU-resident RK4 relaxation (BASELINE config 5).

Mirrors ``boltzfact.harness.rk4_integrate`` (harness.py:79-120): classical
RK4 on dc/dt = Q(c, c), a divergence check after every step (harness.py:103-107,
``RuntimeError``), snapshots every ``record_every`` steps and at the end, and
an ``EvolutionTrace`` whose ``moment_drift()`` is the largest deviation of
mass/momentum/energy from the start (harness.py:55-76).

The batched form keeps the whole (B, n_k, n_q) state on the device; one step is
four Q launches plus the stage kernels (``bfq_rk4_step``).  Every step's
divergence check runs on the device into its own flag slot (one int32 per
step between records), and the flags are read back at record steps (and at the
end), so the step loop never synchronises; the ``RuntimeError`` then names the
exact first step whose state was not finite, with the reference's message
(harness.py:103-107).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .engine import plan_for
from .operator import CoefficientField, moments

__all__ = ["EvolutionTrace", "BatchTrace", "rk4_integrate", "rk4_integrate_batch"]


@dataclass
class EvolutionTrace:
    """Single-cell trajectory, same fields as the reference's (harness.py:55-76)."""

    times: np.ndarray
    coeffs: np.ndarray  # (n_records, n_k, n_q)
    mass: np.ndarray
    momentum: np.ndarray  # (n_records, 3)
    energy: np.ndarray
    cfg: object = field(repr=False)

    def mode(self, k: int, l: int, m: int) -> np.ndarray:
        return self.coeffs[:, k, l * l + l + m]

    def moment_drift(self) -> float:
        return float(max(np.abs(self.mass - self.mass[0]).max(),
                         np.abs(self.momentum - self.momentum[0]).max(),
                         np.abs(self.energy - self.energy[0]).max()))


@dataclass
class BatchTrace:
    """Batched trajectory: moments of every cell at every record step, plus
    full snapshots of the cells listed in ``watch``."""

    times: np.ndarray  # (n_records,)
    moments: np.ndarray  # (n_records, B, 5): mass, px, py, pz, energy
    watch: np.ndarray  # indices of the cells whose coefficients are kept
    snapshots: np.ndarray  # (n_records, len(watch), n_k, n_q)
    final: object  # torch tensor (B, n_k, n_q) on the device

    def moment_drift(self) -> float:
        """Largest |invariant(t) - invariant(0)| over all cells and records."""
        return float(np.abs(self.moments - self.moments[:1]).max())


def rk4_integrate_batch(op, c0, dt: float, n_steps: int, record_every: int = 1, watch=None,
                        device: int | None = None) -> BatchTrace:
    """Integrate every cell of ``c0`` (B, n_k, n_q) on the GPU."""
    import torch

    if dt <= 0 or n_steps < 1:
        raise ValueError("need positive dt and at least one step")
    plan = plan_for(op, device)
    dev = torch.device("cuda", plan.device)
    y = torch.as_tensor(np.ascontiguousarray(c0, dtype=np.float64) if isinstance(c0, np.ndarray) else c0,
                        dtype=torch.float64).to(dev).contiguous().clone()
    if y.dim() != 3 or tuple(y.shape[1:]) != (plan.n_k, plan.n_q):
        raise ValueError(f"state must have shape (B, {plan.n_k}, {plan.n_q})")
    b = y.shape[0]
    work = torch.empty((3,) + tuple(y.shape), dtype=torch.float64, device=dev)
    flags = torch.zeros(max(1, int(record_every)), dtype=torch.int32, device=dev)  # one slot per step
    mom = torch.empty((b, 5), dtype=torch.float64, device=dev)
    watch = np.arange(min(b, 4)) if watch is None else np.asarray(watch, dtype=np.int64)
    widx = torch.as_tensor(watch, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream

    times, moms, snaps = [], [], []

    def record(t):
        plan.moments_device(y.data_ptr(), mom.data_ptr(), b, stream)
        times.append(t)
        moms.append(mom.cpu().numpy().copy())
        snaps.append(y.index_select(0, widx).cpu().numpy())

    record(0.0)
    last = 0  # step of the previous record
    for step in range(1, n_steps + 1):
        slot = flags.data_ptr() + 4 * (step - last - 1)
        plan.rk4_step_device(y.data_ptr(), work.data_ptr(), b, dt, slot, stream)
        if step % record_every == 0 or step == n_steps:
            bad = torch.nonzero(flags[:step - last]).flatten()
            if bad.numel():
                first = last + 1 + int(bad[0])
                raise RuntimeError(f"integration diverged at step {first} (t={first * dt:.4g}); "
                                   "reduce dt below the stability bound")
            flags.zero_()
            last = step
            record(step * dt)
    return BatchTrace(np.array(times), np.stack(moms), watch, np.stack(snaps), y)


def rk4_integrate(op, c0, dt: float, n_steps: int, strategy: str = "gpu", record_every: int = 1) -> EvolutionTrace:
    """Single-cell drop-in for ``harness.rk4_integrate`` on the GPU."""
    if strategy != "gpu":
        raise ValueError(f"unknown strategy {strategy!r}")
    tr = rk4_integrate_batch(op, c0.values[None], dt, n_steps, record_every, watch=[0])
    coeffs = tr.snapshots[:, 0]
    ms, mom, en = [], [], []
    for snap in coeffs:
        m0, m1, m2 = moments(CoefficientField(snap, c0.cfg))
        ms.append(m0)
        mom.append(m1)
        en.append(m2)
    return EvolutionTrace(tr.times, coeffs, np.array(ms), np.array(mom), np.array(en), c0.cfg)
