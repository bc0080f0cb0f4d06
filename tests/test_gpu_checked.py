"""Self-checking kernel build (stands in for compute-sanitizer, which is closed
on this pool): libbfq_checked.so bounds-checks every shared-memory, table and
output access of the Q kernels, times out mbarrier waits, asserts that the
conservation slots are computed exactly zero before the epilogue forces them,
and poisons released R-ring slots and consumed Phi rows with 1e300 under
randomized warp delays, so any race on those buffers fails the 1e-12 parity
against the oracle.  Runs tools/checked_run.py in a subprocess (the library
variant is chosen at import)."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)


def _run(env_extra, ops, cells):
    env = dict(os.environ, BFQ_LIB="checked", **env_extra)
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "checked_run.py"), "--ops", ops,
                          "--cells", str(cells)], capture_output=True, text=True, timeout=1500, env=env)
    lines = [json.loads(l) for l in res.stdout.splitlines() if l.startswith("{")]
    return res, lines


@pytest.mark.parametrize("env_extra,ops,cells", [
    ({}, "hs_n2,hs_n4,mm_k4l6,hs_n8,mm_n10,hs_n12,hs_n16", 11),
    ({"BFQ_KERNEL": "1"}, "hs_n4,hs_n8,hs_n12", 9),   # single-warp fallback kernel
    ({"BFQ_GENERIC": "1"}, "hs_n4,hs_n8,mm_n10", 9),  # run-time-size instantiations
    ({"BFQ_STAGES": "2"}, "hs_n8,hs_n12", 9),         # two-stage R ring
    ({"BFQ_CELLS": "1"}, "hs_n16", 5),                # one cell per tile, slices split over the warps
    ({"BFQ_HALF_DIAG": "0"}, "hs_n4,hs_n8,mm_n10,hs_n12", 9),  # packed-triangle self-symmetric channels (n_k = 11: shared tile)
    ({"BFQ_RK4_FUSED": "1"}, "mm_n4,hs_n8", 9),       # RK4 stages fused into the Q epilogue
    ({"BFQ_GENERIC": "1"}, "hs_n16", 3),              # run-time-size kernel with three tiles per axis
], ids=["default", "fallback", "generic", "stages2", "splitm", "packed_diag", "rk4_fused", "generic_mt3"])
def test_checked_kernels(env_extra, ops, cells):
    res, lines = _run(env_extra, ops, cells)
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-4000:]
    ran = [l for l in lines if "case" in l]
    assert ran and all(l["ok"] and l["violations"] == 0 for l in ran)
