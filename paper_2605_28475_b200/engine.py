"""Drop-in GPU strategy for the reference's operator API.

The reference dispatches ``evaluate(op, c, strategy)`` through the module
dictionary ``STRATEGIES`` (contraction.py:320-340); a strategy has the
signature ``fn(op, c, c2=None, stats=None) -> CoefficientField``
(contraction.py:236-238, :293-295).  This module provides

* :class:`GpuPlan`      -- the operator uploaded once to one device (C ABI plan),
                           cached on the operator object like ``_angular_cache``
                           (contraction.py:83-84, :114-132);
* :func:`q_gpu`         -- the single-cell strategy, same signature and
                           ``ContractionStats`` accounting as ``q_angular_first``;
* :func:`evaluate_batch`-- the throughput entry point: (B, n_k, n_q) float64
                           CUDA tensors, stream-ordered, no host sync;
* :func:`evaluate_host` -- host arrays in, host arrays out (pipelined copies);
* :func:`evaluate` / ``STRATEGIES`` -- the reference's dispatch, GPU only;
* :func:`register_with_reference` -- installs ``"gpu"`` into an imported
  ``boltzfact.contraction.STRATEGIES`` so the reference's own ``evaluate`` and
  ``harness.rk4_integrate(..., strategy="gpu")`` route here unchanged.
"""

from __future__ import annotations

import ctypes
import threading
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .operator import CoefficientField

__all__ = [
    "ContractionStats",
    "GpuPlan",
    "plan_for",
    "q_gpu",
    "evaluate_batch",
    "evaluate_host",
    "evaluate",
    "STRATEGIES",
    "register_with_reference",
    "linearize",
]


@dataclass
class ContractionStats:
    """Same fields as the reference's ContractionStats (contraction.py:51-73)."""

    strategy: str = ""
    flops: int = 0
    bytes_touched: int = 0
    wall_time: float = 0.0
    n_calls: int = 0

    def as_dict(self) -> dict:
        return {
            "strategy": self.strategy,
            "flops": self.flops,
            "bytes_touched": self.bytes_touched,
            "wall_time": self.wall_time,
            "n_calls": self.n_calls,
        }


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def make_desc(op):
    """``bfq_desc`` of a reference (or mirror) FactorizedOperator.

    Returns ``(desc, keepalive)``; the numpy arrays in ``keepalive`` back the
    descriptor's pointers and must outlive its use.  COO columns go from the
    reference's 1-based int32 (angular.py:260-269) to 0-based.
    """
    cfg, g, r = op.cfg, op.g, op.r
    zb = lambda a: np.ascontiguousarray(np.asarray(a, dtype=np.int64) - 1, dtype=np.int32)  # noqa: E731
    keep = dict(
        triplets=np.ascontiguousarray(np.asarray(g.channels.triplets, dtype=np.int32).reshape(-1)),
        q1=zb(g.q1), q2=zb(g.q2), q3=zb(g.q3), tau=zb(g.tau),
        g=np.ascontiguousarray(g.g, dtype=np.float64),
        slice_starts=np.ascontiguousarray(g.slice_starts, dtype=np.int64),
        slice_tau=zb(g.slice_tau), slice_q1=zb(g.slice_q1),
        r=np.ascontiguousarray(r.values, dtype=np.float64),
    )
    n_t = len(g.channels.triplets)
    if keep["r"].shape != (cfg.n_k, cfg.n_k, cfg.n_k, n_t):
        raise ValueError("physical tensor shape inconsistent with table")
    d = _lib.BfqDesc()
    d.k_max, d.l_max, d.gamma = cfg.k_max, cfg.l_max, float(cfg.gamma)
    d.n_t, d.n_g, d.n_s = n_t, keep["g"].size, keep["slice_tau"].size
    d.triplets = _ptr(keep["triplets"], ctypes.c_int32)
    for name in ("q1", "q2", "q3", "tau", "slice_tau", "slice_q1"):
        setattr(d, name, _ptr(keep[name], ctypes.c_int32))
    d.g = _ptr(keep["g"], ctypes.c_double)
    d.slice_starts = _ptr(keep["slice_starts"], ctypes.c_int64)
    d.r = _ptr(keep["r"], ctypes.c_double)
    d.conservation = int(bool(getattr(r, "conservation_applied", False)))
    d.detailed_balance = int(bool(getattr(r, "detailed_balance_applied", False)))
    return d, keep


def host_plan_info(op, smem_limit: int = 232448) -> dict:
    """CPU-only: validate ``op`` and report the plan the engine would build."""
    d, _keep = make_desc(op)
    info = _lib.BfqPlanInfo()
    _lib.check(_lib.lib().bfq_host_plan_info(ctypes.byref(d), int(smem_limit), ctypes.byref(info)))
    return {name: getattr(info, name) for name, _ in info._fields_}


class GpuPlan:
    """The factorized operator resident on one GPU (wraps ``bfq_plan*``)."""

    def __init__(self, handle: int, device: int, n_k: int, n_q: int, l_max: int, k_max: int, source: str):
        self._h = ctypes.c_void_p(handle)
        self.device = device
        self.n_k, self.n_q, self.l_max, self.k_max = n_k, n_q, l_max, k_max
        self.n_dof = n_k * n_q
        self.source = source
        info = _lib.BfqPlanInfo()
        _lib.check(_lib.lib().bfq_plan_get_info(self._h, ctypes.byref(info)))
        self.info = {name: getattr(info, name) for name, _ in info._fields_}
        fl, by = ctypes.c_double(), ctypes.c_double()
        _lib.check(_lib.lib().bfq_plan_work(self._h, ctypes.byref(fl), ctypes.byref(by)))
        self.flops_per_cell = fl.value
        self.bytes_per_cell = by.value

    # ---------------------------------------------------------------- builders
    @classmethod
    def from_operator(cls, op, device: int | None = None) -> "GpuPlan":
        """Upload a reference (or mirror) ``FactorizedOperator``."""
        device = _default_device() if device is None else int(device)
        d, _keep = make_desc(op)
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().bfq_plan_create(ctypes.byref(d), device, ctypes.byref(h)))
        cfg = op.cfg
        return cls(h.value, device, cfg.n_k, cfg.n_q, cfg.l_max, cfg.k_max, "operator")

    @classmethod
    def from_bfct(cls, path, device: int | None = None) -> "GpuPlan":
        """Native BFCT load + upload (no numpy detour), cache.py:92-166."""
        device = _default_device() if device is None else int(device)
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().bfq_plan_create_bfct(str(path).encode(), device, ctypes.byref(h)))
        info = _lib.BfqPlanInfo()
        _lib.check(_lib.lib().bfq_plan_get_info(h, ctypes.byref(info)))
        n_k, n_q = info.n_k, info.n_q
        l_max = int(round(n_q**0.5)) - 1
        return cls(h.value, device, n_k, n_q, l_max, n_k - 1, str(path))

    def close(self) -> None:
        if self._h is not None and self._h.value:
            _lib.lib().bfq_plan_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> ctypes.c_void_p:
        if self._h is None:
            raise RuntimeError("plan was closed")
        return self._h

    # ---------------------------------------------------------------- calls
    def eval_device(self, f2, f3, out, n_cells: int, stream: int) -> None:
        _lib.check(_lib.lib().bfq_eval(self.handle, f2, f3, out, int(n_cells), stream))

    def moments_device(self, c_ptr, out_ptr, n_cells: int, stream: int) -> None:
        _lib.check(_lib.lib().bfq_moments(self.handle, c_ptr, out_ptr, int(n_cells), stream))

    def rk4_step_device(self, y_ptr, work_ptr, n_cells: int, dt: float, flag_ptr, stream: int) -> None:
        _lib.check(_lib.lib().bfq_rk4_step(self.handle, y_ptr, work_ptr, int(n_cells), float(dt), flag_ptr, stream))


def _default_device() -> int:
    import torch

    if not torch.cuda.is_available():
        raise _lib.EngineUnavailable("no CUDA device visible: the Q(f,f) engine runs on the GPU only")
    return torch.cuda.current_device()


_plan_lock = threading.Lock()


def plan_for(op, device: int | None = None) -> GpuPlan:
    """The operator's plan on ``device``, built once and cached on ``op``."""
    if isinstance(op, GpuPlan):
        return op
    device = _default_device() if device is None else int(device)
    plans = getattr(op, "_gpu_plans", None)
    if plans is None or device not in plans:
        with _plan_lock:
            plans = getattr(op, "_gpu_plans", None)
            if plans is None:
                plans = {}
                object.__setattr__(op, "_gpu_plans", plans)
            if device not in plans:
                plans[device] = GpuPlan.from_operator(op, device)
    return plans[device]


def _check_batch(plan: GpuPlan, t, name: str):
    import torch

    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{name} must be a torch tensor")
    if t.dtype != torch.float64:
        raise ValueError(f"{name} must be float64, got {t.dtype}")
    if t.device.type != "cuda" or t.device.index != plan.device:
        raise ValueError(f"{name} must live on cuda:{plan.device}, got {t.device}")
    if t.dim() != 3 or tuple(t.shape[1:]) != (plan.n_k, plan.n_q):
        raise ValueError(f"{name} must have shape (B, {plan.n_k}, {plan.n_q}), got {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be C-contiguous")


def _overlaps(a, b) -> bool:
    """True when the byte ranges of two tensors intersect."""
    a0, b0 = a.data_ptr(), b.data_ptr()
    a1 = a0 + a.numel() * a.element_size()
    b1 = b0 + b.numel() * b.element_size()
    return a.numel() > 0 and b.numel() > 0 and a0 < b1 and b0 < a1


def evaluate_batch(op, f, f3=None, out=None, stream=None):
    """Q(f, f3) for every cell of ``f`` (B, n_k, n_q) on the GPU.

    ``f3=None`` (or ``f3 is f``) evaluates Q(f, f).  Stream-ordered on the
    current torch stream (or ``stream``); returns ``out``.
    """
    import torch

    plan = plan_for(op, f.device.index if hasattr(f, "device") and f.device.type == "cuda" else None)
    _check_batch(plan, f, "f")
    if f3 is not None and f3 is not f:
        _check_batch(plan, f3, "f3")
        if f3.shape != f.shape:
            raise ValueError("f and f3 must have the same shape")
    if out is None:
        out = torch.empty_like(f)
    else:
        _check_batch(plan, out, "out")
        if out.shape != f.shape:
            raise ValueError("out must have the shape of f")
        # CTAs of one tile read its cells while other CTAs already write Q:
        # an output that overlaps an input would be read back half-written
        for name, t in (("f", f), ("f3", f3)):
            if t is not None and _overlaps(out, t):
                raise ValueError(f"out must not overlap {name} (in-place evaluation is not supported)")
    st = (stream or torch.cuda.current_stream(plan.device)).cuda_stream
    p3 = None if f3 is None or f3 is f else f3.data_ptr()
    plan.eval_device(f.data_ptr(), p3, out.data_ptr(), f.shape[0], st)
    return out


def evaluate_host(op, values: np.ndarray, values3: np.ndarray | None = None) -> np.ndarray:
    """Host (B, n_k, n_q) float64 in, host Q out, through ``bfq_eval_host``."""
    plan = plan_for(op)
    v = np.ascontiguousarray(values, dtype=np.float64)
    if v.ndim != 3 or v.shape[1:] != (plan.n_k, plan.n_q):
        raise ValueError(f"values must have shape (B, {plan.n_k}, {plan.n_q})")
    v3 = None
    if values3 is not None:
        v3 = np.ascontiguousarray(values3, dtype=np.float64)
        if v3.shape != v.shape:
            raise ValueError("values3 must have the shape of values")
    out = np.empty_like(v)
    _lib.check(
        _lib.lib().bfq_eval_host(
            plan.handle, v.ctypes.data, None if v3 is None else v3.ctypes.data, out.ctypes.data, v.shape[0]
        )
    )
    return out


def _record(stats, op, dt: float) -> None:
    """angular_first accounting (contraction.py:314-316)."""
    if stats is None:
        return
    n_k = op.cfg.n_k
    n_g, n_s = op.g.n_g, op.g.n_s
    stats.strategy = "gpu"
    stats.flops += n_g * n_k**2 + n_s * n_k**3
    stats.bytes_touched += 8 * (n_g * (2 * n_k + 1 + n_k**2) + n_s * (n_k**2 + n_k**3))
    stats.wall_time += dt
    stats.n_calls += 1


def q_gpu(op, c, c2=None, stats=None):
    """Strategy ``"gpu"``: Q(c, c2) of one cell on the GPU.

    Signature and result type follow the reference strategies
    (contraction.py:293-317): returns ``type(c)(values, cfg)``.
    """
    cfg = op.cfg
    if c.values.shape != (cfg.n_k, cfg.n_q):
        raise ValueError("coefficient field does not match the operator")
    if c2 is not None and c2.values.shape != (cfg.n_k, cfg.n_q):
        raise ValueError("coefficient field does not match the operator")
    t0 = time.perf_counter()
    # one C-ABI call (bfq_eval_host: staged H2D, Q launch, D2H, sync) -- no torch
    # tensors on the per-cell path (profiles/r02_dropin_latency.json)
    q = evaluate_host(op, c.values[None], None if c2 is None else c2.values[None])[0]
    _record(stats, op, time.perf_counter() - t0)
    return type(c)(q, c.cfg)


def linearize(op, c_eq, device: int | None = None, chunk: int = 4096) -> np.ndarray:
    """Jacobian of Q at ``c_eq`` as a dense (n_dof, n_dof) matrix, on the GPU.

    Same result as the reference's ``linearize`` (contraction.py:343-369):
    column beta is dQ/dc_beta = Q(c_eq, e_beta) + Q(e_beta, c_eq) (slot-3 and
    slot-2 derivatives, the t3 / t2 terms of :360-368), evaluated as two
    batched bilinear launches with one basis vector e_beta per cell.
    """
    import torch

    plan = plan_for(op, device)
    dev = torch.device("cuda", plan.device)
    cfg = op.cfg
    n_dof = cfg.n_dof
    vals = np.ascontiguousarray(c_eq.values if hasattr(c_eq, "values") else c_eq, dtype=np.float64)
    if vals.shape != (cfg.n_k, cfg.n_q):
        raise ValueError("coefficient field does not match the operator")
    base = torch.from_numpy(vals).to(dev)
    jac_t = torch.empty((n_dof, n_dof), dtype=torch.float64, device=dev)  # row beta = column beta of J
    for b0 in range(0, n_dof, chunk):
        nb = min(chunk, n_dof - b0)
        e = torch.zeros((nb, n_dof), dtype=torch.float64, device=dev)
        e[torch.arange(nb, device=dev), torch.arange(b0, b0 + nb, device=dev)] = 1.0
        e = e.view(nb, cfg.n_k, cfg.n_q)
        c = base.expand(nb, cfg.n_k, cfg.n_q).contiguous()
        q3 = evaluate_batch(plan, c, e)  # Q(c_eq, e_beta): derivative through slot 3
        q2 = evaluate_batch(plan, e, c)  # Q(e_beta, c_eq): derivative through slot 2
        jac_t[b0:b0 + nb] = (q3 + q2).view(nb, n_dof)
    return jac_t.t().contiguous().cpu().numpy()


STRATEGIES = {"gpu": q_gpu}


def evaluate(op, c, strategy: str = "gpu", stats=None):
    """The reference's name dispatch (contraction.py:327-340), GPU strategies only."""
    try:
        fn = STRATEGIES[strategy]
    except KeyError:
        raise ValueError(f"unknown strategy {strategy!r}") from None
    return fn(op, c, stats=stats)


def register_with_reference(contraction_module=None) -> bool:
    """Install ``STRATEGIES["gpu"] = q_gpu`` into the reference's contraction
    module (imported as ``boltzfact.contraction`` unless given).  Returns False
    when the reference package is not importable."""
    if contraction_module is None:
        try:
            import boltzfact.contraction as contraction_module  # type: ignore
        except ImportError:
            return False
    contraction_module.STRATEGIES["gpu"] = q_gpu
    return True


def cell_field(values: np.ndarray, cfg) -> CoefficientField:
    return CoefficientField(values, cfg)
