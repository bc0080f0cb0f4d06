"""Parity of the BENCHMARKED batches (SURVEY §8d pass criteria): the same
seeded generator, seed and batch size as bench.py, evaluated on the GPU in one
launch, checked against the CPU oracle on every cell of config 2 and on >= 256
stratified cells of configs 3, 4 and 5 (one Q evaluation), with the
reference's metric max|dQ| / max|Q_ref| <= 1e-12 per cell
(test_contraction.py:57-65, cli.py:371-386).  Also bfq_moments against the
oracle's basis.moments restatement."""

import os
import sys

import numpy as np
import pytest

from conftest import OPERATORS, ROOT
from oracle import q_oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2605_28475_b200 import engine  # noqa: E402

SEED = 20260520  # bench.py default


@pytest.mark.parametrize("config", ["hs8", "hs12", "mm10", "hs16"])
def test_benchmarked_batch_parity(config):
    opfile, n_global, _, _, sample = bench.CONFIGS[config]
    path = os.path.join(OPERATORS, opfile + ".bfct")
    if not os.path.exists(path):
        pytest.skip(f"{opfile} not shipped")
    op = bench.load_operator(opfile, 0)
    cfg = op.cfg
    host = bench.make_cells(config, cfg.n_k, cfg.l_max, n_global, seed=SEED, start=0, device=0)
    q = engine.evaluate_batch(op, torch.from_numpy(host).cuda())
    qh = q.cpu().numpy()
    # invariant slots bitwise zero on EVERY cell of the batch
    assert np.all(qh[:, 0, :4] == 0.0) and np.all(qh[:, 1, 0] == 0.0)
    idx = bench.stratified_indices(n_global, sample)
    assert idx.size == n_global if sample == 0 else idx.size >= 256
    ref, _ = bench.oracle_pool(path, host[idx])
    errs = np.array([q_oracle.rel_err(qh[j], ref[i]) for i, j in enumerate(idx)])
    assert errs.max() <= 1e-12, (config, int(idx[int(np.argmax(errs))]), float(errs.max()))


def test_moments_kernel_matches_oracle():
    op = bench.load_operator("hs_n8", 0)
    cfg = op.cfg
    host = bench.make_cells("hs8", cfg.n_k, cfg.l_max, 333, seed=SEED, start=0, device=0)
    host += np.random.default_rng(1).normal(scale=1e-3, size=host.shape)  # non-zero invariants
    f = torch.from_numpy(host).cuda()
    plan = engine.plan_for(op)
    out = torch.empty((host.shape[0], 5), dtype=torch.float64, device="cuda")
    plan.moments_device(f.data_ptr(), out.data_ptr(), host.shape[0], torch.cuda.current_stream().cuda_stream)
    got = out.cpu().numpy()
    for i in range(host.shape[0]):
        mass, mom, energy = q_oracle.moments(host[i])
        assert got[i, 0] == mass and np.array_equal(got[i, 1:4], mom) and got[i, 4] == energy, i
