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


def test_bench_two_ranks_functional():
    """The multi-rank bench path end to end on the GPU: ``bench.py --gpus 2``
    launches two ranks (gloo, sharing the device when only one exists), shards
    one fixed batch, checks rank 0's outputs against the oracle and reduces
    the per-rank times -- a functional check, not a scaling number."""
    import json
    import subprocess

    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--backend", "gloo",
                          "--config", "hs8", "--cells", "1000", "--steps", "2", "--warmup", "1", "--e2e-steps", "1",
                          "--parity-cells", "16"], capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_cells"] == 1000 and d["config"]["cells_per_rank"] == 500
    assert len(d["rank_ms"]) == 2 and d["ms_per_step"] > 0
    assert d["parity"]["pass"] and d["conservation"]["invariant_slots_exact"]
    assert d["conservation"]["cells"] == 1000.0
