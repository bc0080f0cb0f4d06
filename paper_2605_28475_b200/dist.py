"""Multi-GPU plumbing: one process per GPU, cells sharded, no data-path collective.

Spatial cells are independent: every rank owns a contiguous
block of the global batch and a replica of the operator.  The only collective
is a small all-reduce of conservation diagnostics (max |production| of mass,
momentum and energy, the cell count and a checksum), run once per batch or
per RK4 record step, outside the timed region.  Backend ``nccl`` on GPUs;
the same code runs on ``gloo`` for the CPU tests.
"""

from __future__ import annotations

import os

import numpy as np

__all__ = ["shard_range", "diagnostics_vector", "allreduce_diagnostics", "init_from_env", "max_over_ranks",
           "weak_scaling_rate"]

DIAG_FIELDS = ("max_mass", "max_px", "max_py", "max_pz", "max_energy", "cells", "checksum")


def shard_range(n_global: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block (start, count) of rank ``rank``; remainder to the first ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid world/rank")
    base, rem = divmod(n_global, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


def diagnostics_vector(moments, q):
    """Local diagnostics of one shard: ``moments`` (n, 5) of Q, ``q`` the shard's Q.

    Returns a float64 torch tensor [max|mass|, max|px|, max|py|, max|pz|,
    max|energy|, n_cells, sum(Q)] on the device of ``q``.
    """
    import torch

    dev = q.device
    n = q.shape[0]
    if n:
        m = moments.abs().amax(dim=0)
        chk = q.sum().reshape(1)
    else:
        m = torch.zeros(5, dtype=torch.float64, device=dev)
        chk = torch.zeros(1, dtype=torch.float64, device=dev)
    return torch.cat([m.to(torch.float64), torch.tensor([float(n)], dtype=torch.float64, device=dev),
                      chk.to(torch.float64)])


def allreduce_diagnostics(vec, group=None):
    """Combine shard diagnostics: MAX of the five maxima, SUM of count and checksum."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return vec
    mx = vec[:5].clone()
    sm = vec[5:].clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(sm, op=dist.ReduceOp.SUM, group=group)
    return torch.cat([mx, sm])


def max_over_ranks(value: float, device=None) -> float:
    """MAX of a per-rank scalar (a device-timed step time) over all ranks; the
    bench's step time is the slowest rank's (the job ends with it)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def weak_scaling_rate(cells_per_rank: int, evals_per_cell: int, local_ms: float, device=None) -> tuple[float, float]:
    """Whole-job cell-evaluations/s of a weak-scaling run: every rank evaluates
    ``cells_per_rank`` cells ``evals_per_cell`` times in ``local_ms`` of its own
    device time; the job's time is the max over ranks.  Returns (rate, max_ms)."""
    import torch.distributed as dist

    world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    ms = max_over_ranks(local_ms, device)
    return cells_per_rank * world * evals_per_cell / (ms / 1e3), ms


def init_from_env(backend: str = "nccl"):
    """(rank, world, local_rank) from torchrun's environment; initialises the
    process group when WORLD_SIZE > 1."""
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend)
    return rank, world, local


def as_dict(vec) -> dict:
    v = np.asarray(vec.cpu().numpy() if hasattr(vec, "cpu") else vec, dtype=np.float64)
    return dict(zip(DIAG_FIELDS, (float(x) for x in v)))
