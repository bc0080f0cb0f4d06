"""Multi-rank host logic on CPU (gloo, world size 2): sharding and the
diagnostics all-reduce that the GPU runs do over NCCL."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_28475_b200 import dist as bdist


def test_shard_range_covers_exactly():
    for n in (0, 1, 7, 8, 65536, 65537):
        for world in (1, 2, 3, 8):
            spans = [bdist.shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0
            for (s0, c0), (s1, _) in zip(spans, spans[1:]):
                assert s0 + c0 == s1
            assert sum(c for _, c in spans) == n
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q_all, m_all, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    start, count = bdist.shard_range(q_all.shape[0], world, rank)
    q = torch.from_numpy(q_all[start:start + count])
    m = torch.from_numpy(m_all[start:start + count])
    vec = bdist.allreduce_diagnostics(bdist.diagnostics_vector(m, q))
    out[rank] = vec.numpy()
    dist.barrier()
    dist.destroy_process_group()


def test_diagnostics_allreduce_gloo_world2():
    rng = np.random.default_rng(0)
    q_all = rng.normal(size=(13, 3, 9))
    m_all = rng.normal(size=(13, 5)) * 1e-17
    ref = bdist.diagnostics_vector(torch.from_numpy(m_all), torch.from_numpy(q_all)).numpy()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(2, _free_port(), q_all, m_all, out), nprocs=2, join=True)
        res = [out[0], out[1]]
    for r in res:
        assert np.array_equal(r[:6], ref[:6])
        assert abs(r[6] - ref[6]) <= 1e-12 * np.abs(q_all).sum()
    d = bdist.as_dict(res[0])
    assert d["cells"] == 13.0


def _timing_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    local_ms = [100.0, 125.0][rank]  # rank 1 is the slow one
    out[rank] = bdist.weak_scaling_rate(65536, 10, local_ms)
    dist.destroy_process_group()


def test_weak_scaling_rate_is_max_over_ranks_gloo_world2():
    """bench.py's aggregation: every rank reports the job rate over the slowest
    rank's time, cells counted over all ranks."""
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_timing_worker, args=(2, _free_port(), out), nprocs=2, join=True)
        res = [out[0], out[1]]
    for rate, ms in res:
        assert ms == 125.0
        assert rate == 65536 * 2 * 10 / 0.125
    assert bdist.weak_scaling_rate(100, 1, 50.0) == (2000.0, 50.0)  # no process group: one rank
