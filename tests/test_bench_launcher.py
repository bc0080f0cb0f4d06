"""bench.py's multi-rank plumbing on CPU: ``--gpus 2`` re-launches itself under
torch.distributed.run, shards one fixed batch (strong) or gives every rank its
own batch (weak), and all-gathers / all-reduces over gloo -- the same code the
GPU runs drive over NCCL (no kernels in --dry-run)."""

import json
import os
import subprocess
import sys

import numpy as np

from conftest import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _run(*extra):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--backend", "gloo",
                          "--dry-run", "--config", "hs4", *extra], capture_output=True, text=True, timeout=600,
                         env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def test_strong_scaling_shards_one_batch_world2():
    d = _run("--cells", "65537")
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["global_cells"] == 65537
    assert d["shards"] == [[0, 32769], [32769, 32768]]
    assert d["diag_cells"] == 65537.0  # SUM all-reduce of the per-rank cell counts


def test_weak_scaling_world2():
    d = _run("--cells", "100", "--scaling", "weak")
    assert d["global_cells"] == 200 and d["shards"] == [[0, 100], [100, 100]]


def test_stratified_parity_sample():
    idx = bench.stratified_indices(65536, 256)
    assert idx[0] == 0 and idx[-1] == 65535 and 256 <= idx.size <= 259
    assert np.all(np.diff(idx) > 0)
    assert 65533 in idx and 65534 in idx  # the last tile
    gaps = np.diff(idx[:-3])
    assert gaps.max() - gaps.min() <= 1  # evenly spread over the batch
    assert np.array_equal(bench.stratified_indices(4096, 0), np.arange(4096))
    assert np.array_equal(bench.stratified_indices(5, 256), np.arange(5))
    assert bench.stratified_indices(0, 256).size == 0
