"""Benchmark of the Q(f,f) hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config hs12|hs8|hs16|mm10|rk4|hs4|rbuild12|...] [--scaling strong|weak]

One step = one Q(f,f) evaluation of every cell of the rank's shard (one
``bfq_eval`` launch).  Default workload = BASELINE config 3: hard spheres,
N=L=12, a fixed 65,536-cell global batch sharded evenly over the GPUs
(strong scaling, as BASELINE config 3 states; ``--scaling weak`` gives every
GPU the full batch instead).  ``--gpus N`` without torchrun's environment
re-launches this script through ``torch.distributed.run`` with N ranks; under
torchrun the rank layout comes from RANK / WORLD_SIZE / LOCAL_RANK.  No
collective runs inside the timed region (cells are independent); the step
time is the max over ranks and NCCL is used only for the diagnostics
all-reduce after it.  After the timed region the run checks its OWN outputs:
a stratified sample of the timed batch (every cell for config 2) against the
CPU oracle, which is also the timed CPU baseline.  Rank 0 prints one JSON
line.  See DESIGN.md §4.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import platform
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (operator file, global cells, generator, description, parity sample (0 = every cell))
    "hs12": ("hs_n12", 65536, "pm", "config3: hard spheres N=L=12, perturbed Maxwellians", 256),
    "hs8": ("hs_n8", 4096, "pm", "config2: hard spheres N=L=8, perturbed Maxwellians", 0),
    "mm10": ("mm_n10", 32768, "bimodal", "config5 operator: Maxwell N=L=10, bimodal cells (single Q eval)", 256),
    "hs4": ("hs_n4", 65536, "pm", "hard spheres N=L=4 (small)", 256),
    "hs16": ("hs_n16", 16384, "pm", "config4: hard spheres N=L=16, perturbed Maxwellians", 256),
    "syn16": ("synth_n16", 16384, "pm", "config4 shape N=L=16 with a SYNTHETIC R (real Gaunt table, random "
                                        "slot-symmetric R with the reference's null-space zeroing): timing only", 64),
    "rk4": ("mm_n10", 32768, "bimodal", "config5: Maxwell N=L=10, bimodal cells, GPU-resident RK4 dt=0.01 "
                                         "(one step = one RK4 step = 4 Q(f,f) per cell)", 0),
}
# the operator build.  One step = one full R-tensor
# assembly (every channel's gain / loss integrals over both Duffy patches).
RBUILD = {
    "rbuild8": (8, 8, 1.0),
    "rbuild12": (12, 12, 1.0),
    "rbuild16": (16, 16, 1.0),
}
# the general projection basis.project(f, cfg, order) of
# sampled distributions.  One step = one projection of every cell's samples.
PROJ = {"proj12": (12, 12, 64, 4096), "proj8": (8, 8, 32, 16384)}
PROJ_METRIC = "projected cells/s (fp64 basis.project of sampled f, quadrature order as configured)"
METRIC = "Q(f,f) cell-evals/s (fp64, hard spheres L=N=12) and FP64/HBM roofline frac"
RBUILD_METRIC = "R-tensor assembly channel integrals/s (fp64, hard spheres, pad 16/16)"
FP64_PEAK_TFLOPS = 37.1  # DMMA.8x8x4 sustained, measured on this pool (profiles/fp64_peak.txt)
# SURVEY §8d "datasheet ~37 TF": 148 SMs x 128 FP64 tensor flop/clk/SM x 1.965 GHz max boost
FP64_NOMINAL_TFLOPS = 148 * 128 * 1.965e9 / 1e12
L2_BYTES = 132644864


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def make_cells(cfg_name, n_k, l_max, n, seed, start, device=None):
    """Seeded cells (host numpy); with ``device`` the Maxwellian projection runs
    on the GPU (bfq_project_maxwellians, same draws, equal to rounding)."""
    from paper_2605_28475_b200 import inputs

    gen = CONFIGS[cfg_name][2]
    if device is not None:
        if gen == "pm":
            return inputs.perturbed_maxwellians_device(n_k, l_max, n, seed=seed, start=start, device=device).cpu().numpy()
        return inputs.bimodal_device(n_k, l_max, n, seed=seed, start=start, device=device).cpu().numpy()
    if gen == "pm":
        return inputs.perturbed_maxwellians(n_k, l_max, n, seed=seed, start=start)
    return inputs.bimodal(n_k, l_max, n, seed=seed, start=start)


def stratified_indices(n, k):
    """``k`` cell indices spread evenly over [0, n): first and last cell, every
    stretch of the batch (hence every tile chunk of the grid), and the ragged
    last tile; ``k = 0`` or ``k >= n`` selects every cell."""
    import numpy as np

    if n == 0:
        return np.zeros(0, dtype=np.int64)
    if k <= 0 or k >= n:
        return np.arange(n, dtype=np.int64)
    idx = np.unique(np.round(np.linspace(0, n - 1, k)).astype(np.int64))
    tail = np.arange(max(0, n - 3), n, dtype=np.int64)  # the last (possibly partial) tile
    return np.unique(np.concatenate([idx, tail]))


# ------------------------------------------------------------------ CPU legs
REF_PKG = os.path.join(ROOT, "baseline", "_ref")  # the unmodified reference (pip --target), when shipped


def live_reference():
    """The reference's own package from baseline/_ref, or None."""
    if not os.path.isdir(os.path.join(REF_PKG, "boltzfact")):
        return None
    if REF_PKG not in sys.path:
        sys.path.insert(0, REF_PKG)
    try:
        from boltzfact import basis, cache, contraction  # noqa: F401
    except Exception:  # pragma: no cover - broken install
        return None
    return contraction


def _cpu_worker(args):
    """CPU Q of a block of cells in one process, one BLAS thread: the LIVE
    reference's evaluate(op, c) (angular_first, contraction.py:327-340) when
    baseline/_ref is shipped, else the oracle port of its operations
    (oracle/q_oracle.py).  Returns (Q, busy seconds, kind)."""
    path, cells = args[0], args[1]
    use_live = args[2] if len(args) > 2 else True
    import numpy as np

    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover
        threadpool_limits = None
    contraction = live_reference() if use_live else None
    out = np.empty_like(cells)
    if contraction is not None:
        from boltzfact import basis, cache

        op = cache.load_cache(path)
        contraction.evaluate(op, basis.CoefficientField(cells[0].copy(), op.cfg))  # builds the cached workspace
        ctx = threadpool_limits(limits=1) if threadpool_limits else None
        if ctx:
            ctx.__enter__()
        t0 = time.perf_counter()
        for i, c in enumerate(cells):
            out[i] = contraction.evaluate(op, basis.CoefficientField(np.array(c), op.cfg)).values
        dt = time.perf_counter() - t0
        if ctx:
            ctx.__exit__(None, None, None)
        return out, dt, "reference"
    from oracle import q_oracle
    from paper_2605_28475_b200.operator import load_cache

    op = q_oracle.OracleOperator.from_operator(load_cache(path))
    ws = q_oracle.angular_workspace(op)  # cached per operator, as the reference does
    ctx = threadpool_limits(limits=1) if threadpool_limits else None
    if ctx:
        ctx.__enter__()
    t0 = time.perf_counter()
    for i, c in enumerate(cells):
        out[i] = q_oracle.q_angular_first(op, c, workspace=ws)
    dt = time.perf_counter() - t0
    if ctx:
        ctx.__exit__(None, None, None)
    return out, dt, "port"


def oracle_pool(path, cells, cores=None, live=True):
    """Oracle Q of ``cells`` on ``cores`` host processes (one thread each),
    contiguous blocks, the pattern of cli.py:406-410.  Returns (q, info):
    cells/s over the slowest worker's busy time, plus the 1-core rate."""
    import multiprocessing as mp

    import numpy as np

    cores = max(1, min(cores or os.cpu_count() or 1, cells.shape[0]))
    _, t1, _ = _cpu_worker((path, cells[:2], live))  # 1-core rate (operator load + workspace excluded)
    bounds = np.linspace(0, cells.shape[0], cores + 1).round().astype(int)
    chunks = [(path, cells[bounds[i]:bounds[i + 1]], live) for i in range(cores) if bounds[i + 1] > bounds[i]]
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(len(chunks)) as pool:
        res = pool.map(_cpu_worker, chunks)
    wall = time.perf_counter() - t0
    q = np.concatenate([r[0] for r in res])
    busy = max(r[1] for r in res)
    return q, {"value": cells.shape[0] / busy, "cells": int(cells.shape[0]), "cores": len(chunks),
               "busy_s": busy, "wall_s": wall, "single_core_cells_per_s": 2.0 / t1, "kind": res[0][2]}


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rbuild_cpu_worker(args):
    k_max, l_max, gamma, grid, taus = args
    from oracle import r_oracle

    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover
        threadpool_limits = None
    ctx = threadpool_limits(limits=1) if threadpool_limits else None
    if ctx:
        ctx.__enter__()
    asm = r_oracle.Assembly(k_max, l_max, gamma, grid)
    trip = r_oracle.channels(l_max)
    t0 = time.perf_counter()
    for t in taus:
        asm.channel_half(*trip[t])
    dt = time.perf_counter() - t0
    if ctx:
        ctx.__exit__(None, None, None)
    return len(taus), dt


def rbuild_cpu_rate(config, per_core=1, cores=None):
    """Oracle port of kinematic.channel_half (the reference's per-channel work) on
    host cores, one thread per process: channel integrals/s (init excluded)."""
    import multiprocessing as mp

    from paper_2605_28475_b200 import rbuild

    k, l, gam = RBUILD[config]
    grid = rbuild.grid_sizes(k, l).as_tuple()[:7]
    n_t = rbuild.enumerate_channels(l).n_t
    cores = cores or os.cpu_count() or 1
    rng = __import__("random").Random(7)
    taus = rng.sample(range(n_t), min(n_t, per_core * cores))
    chunks = [(k, l, gam, grid, taus[i::cores]) for i in range(cores) if taus[i::cores]]
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(len(chunks)) as pool:
        res = pool.map(_rbuild_cpu_worker, chunks)
    wall = time.perf_counter() - t0
    done = sum(r[0] for r in res)
    busy = max(r[1] for r in res)
    return {"value": done / busy, "channels": done, "cores": len(chunks), "wall_s": wall, "busy_s": busy}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and throttle reasons during the timed region.  NVML in a
    background thread (2 ms period) plus explicit ``sample()`` calls placed
    while queued kernels are still running, so even a few-millisecond region
    is covered; falls back to ``nvidia-smi -lms`` without pynvml."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4))

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.nvml = None
        self.samples = []  # (sm MHz, max MHz, reason bits)

    def __enter__(self):
        import threading

        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM))
            self.stop = threading.Event()

            def loop():
                while not self.stop.is_set():
                    self.sample()
                    self.stop.wait(0.002)

            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
            return self
        except Exception:  # pragma: no cover - no NVML: nvidia-smi polling
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def sample(self):
        if self.nvml is None:
            return
        try:
            sm = float(self.nvml.nvmlDeviceGetClockInfo(self.handle, self.nvml.NVML_CLOCK_SM))
            bits = int(self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.handle))
            util = int(self.nvml.nvmlDeviceGetUtilizationRates(self.handle).gpu)
        except Exception:  # pragma: no cover
            return
        self.samples.append((sm, self.max_mhz, bits, util))

    def __exit__(self, *exc):
        self.lines = []
        if self.nvml is not None:
            self.stop.set()
            self.thread.join(timeout=5)
            return
        if self.proc is not None:
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        if self.nvml is not None:
            for s, m, bits, _ in self.samples:
                sm.append(s)
                mx = m
                reasons.update(name for name, bit in self.REASONS if bits & bit)
            if not sm:
                return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
            return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                    "samples": len(sm), "source": "nvml"}
        names = [n for n, _ in self.REASONS]
        for line in getattr(self, "lines", []):
            parts = [p.strip() for p in line.split(",")]
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except (ValueError, IndexError):
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ arms
def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path (oracle port of
    contraction.q_angular_first, the same operations and the same speed per
    cell, profiles/r01_cpu_ref_vs_port.txt) on all host cores, rank 0 only."""
    if rank != 0:
        return
    if args.config in RBUILD:
        rates, walls = [], []
        for _ in range(args.steps):
            r = rbuild_cpu_rate(args.config)
            rates.append(r["value"])
            walls.append(r["wall_s"])
        v = statistics.median(rates)
        k, l, gam = RBUILD[args.config]
        print(json.dumps({
            "impl": "reference", "metric": RBUILD_METRIC, "value": v, "unit": "channels/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(walls),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "none",
            "config": {"workload": f"R-tensor assembly N={k} L={l} gamma={gam}",
                       "step": "one channel per host core (random sample), oracle port of channel_half"},
            "cpu_baseline": {"value": v, "unit": "channels/s", "cores": r["cores"], "kind": "port",
                             "sample": f"{r['channels']} random channels, one per core", "cpu": cpu_model()},
            "e2e": {"value": v, "unit": "channels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }), flush=True)
        return
    if args.config in PROJ:  # the reference's basis.project einsums on sampled f, all host cores
        import multiprocessing as mp

        import numpy as np

        from paper_2605_28475_b200 import project as gproject
        from paper_2605_28475_b200.operator import SpectralConfig

        k, l, order, _ = PROJ[args.config]
        cfg = SpectralConfig(k, l, 1.0)
        pts = gproject.project_points(cfg, order)
        cores = os.cpu_count() or 1
        rng = np.random.default_rng(args.seed)
        u = rng.uniform(-0.3, 0.3, size=(cores, 3))
        t = rng.uniform(0.8, 1.2, size=cores)
        hs = np.stack([(2 * np.pi * t[i]) ** -1.5 * np.exp(-np.sum((pts - u[i]) ** 2, axis=1) / (2 * t[i]))
                       for i in range(cores)])
        rates, walls = [], []
        with mp.get_context("spawn").Pool(cores) as pool:
            for _ in range(args.steps):
                t0 = time.perf_counter()
                res = pool.map(_proj_worker, [(k, l, order, hs[i:i + 1]) for i in range(cores)])
                walls.append(time.perf_counter() - t0)
                rates.append(cores / max(r[1] for r in res))
        v = statistics.median(rates)
        print(json.dumps({
            "impl": "reference", "metric": PROJ_METRIC, "value": v, "unit": "cells/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(walls),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic drifting Maxwellians sampled on the host",
            "config": {"workload": f"basis.project of sampled f, N={k} L={l}, radial order {order}"},
            "cpu_baseline": {"value": v, "unit": "cells/s", "cores": cores, "kind": "port",
                             "sample": "one cell per core per step (oracle/project_oracle.py)", "cpu": cpu_model()},
            "e2e": {"value": v, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }), flush=True)
        return
    opfile, n_global, _, desc, _ = CONFIGS[args.config]
    from paper_2605_28475_b200.operator import load_cache

    path = os.path.join(ROOT, "operators", opfile + ".bfct")
    if not os.path.exists(path):
        print(json.dumps({"impl": "reference", "unavailable": f"operators/{opfile}.bfct (a multi-hour reference "
                          "CPU build) is not shipped with this snapshot"}), flush=True)
        return
    op = load_cache(path)
    cores = os.cpu_count() or 1
    # calibrate one cell, then size each step's sample to ~cpu_budget s per core
    probe = make_cells(args.config, op.cfg.n_k, op.cfg.l_max, 2, seed=args.seed, start=0)
    _, t2, _ = _cpu_worker((path, probe))
    per_core = max(1, int(args.cpu_budget / max(t2 / 2, 1e-6)))
    n_sample = min(n_global, per_core * cores)
    # the leading cells of the batch (per-cell CPU cost does not depend on the values;
    # generating the whole 65,536-cell batch on the host would take ~40 s)
    cells = make_cells(args.config, op.cfg.n_k, op.cfg.l_max, n_sample, seed=args.seed, start=0)
    for _ in range(args.warmup):
        oracle_pool(path, cells[:cores], cores)
    rates, walls = [], []
    for _ in range(args.steps):
        _, r = oracle_pool(path, cells, cores)
        rates.append(r["value"])
        walls.append(r["wall_s"])
        last = r
    v = statistics.median(rates)
    sample = (f"the first {n_sample} cells of the {n_global}-cell batch per step "
              f"({math.ceil(n_sample / last['cores'])} per core, ~{last['busy_s']:.1f} s of work per core); "
              "rate = sample / slowest worker's busy time")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "cells/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(walls),
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE.json distributions)",
        "config": {"workload": desc, "global_cells": n_global, "operator": opfile, "seed": args.seed,
                   "step": "one bounded sample of the workload on all host cores (multiprocessing pool)"},
        "cpu_baseline": {"value": v, "unit": "cells/s", "cores": last["cores"], "kind": last["kind"],
                         "sample": sample + ("; the live reference package (baseline/_ref): contraction.evaluate"
                                             if last["kind"] == "reference" else
                                             "; oracle/q_oracle.py (the reference's operations, bit-identical)"),
                         "cpu": cpu_model(), "single_core_cells_per_s": last["single_core_cells_per_s"]},
        "e2e": {"value": v, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def load_operator(opfile, device=0):
    """The reference-built cache; for config 4 (N=L=16, a multi-hour CPU build
    that is not always shipped) fall back to assembling it on the GPU (rbuild)."""
    from paper_2605_28475_b200.operator import SpectralConfig, load_cache

    path = os.path.join(ROOT, "operators", opfile + ".bfct")
    if os.path.exists(path) or opfile != "hs_n16":
        return load_cache(path)
    from paper_2605_28475_b200 import rbuild

    op = rbuild.build_operator(SpectralConfig(16, 16, 1.0), device=device)
    op._built_on_gpu = True
    return op


def run_rbuild(args, rank, world, local_rank):
    """R-tensor assembly on the GPU (include/bfr.h).  Replicas only: every rank
    assembles the full tensor (the build is one-time per operator)."""
    import torch

    from paper_2605_28475_b200 import rbuild
    from paper_2605_28475_b200.operator import SpectralConfig

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    k, l, gam = RBUILD[args.config]
    cfg = SpectralConfig(k, l, gam)
    grid = rbuild.grid_sizes(k, l)
    for _ in range(max(args.warmup, 0)):
        rbuild.assemble_r_tensor(cfg, grid, device=local_rank)
    stats, walls = [], []
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            t0 = time.perf_counter()
            r = rbuild.assemble_r_tensor(cfg, grid, device=local_rank)
            walls.append(time.perf_counter() - t0)
            stats.append(rbuild.last_stats())
    n_t = r.channels.n_t
    total_ms = sum(s["ms_total"] for s in stats)
    t = torch.tensor([total_ms, sum(walls)], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, wall_tot = float(t[0]), float(t[1])
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    st = stats[-1]
    contract_ms = statistics.mean(s["ms_contract"] for s in stats)
    achieved = 2.0 * st["alg_macs"] / (contract_ms / 1e3) / 1e12
    line = {
        "metric": RBUILD_METRIC, "value": n_t * world * args.steps / (total_ms / 1e3), "unit": "channels/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "none (deterministic quadrature grids)",
        "config": {"workload": f"R-tensor assembly N={k} L={l} gamma={gam} (kinematic.assemble_r_tensor)",
                   "grid": grid.as_tuple(), "channels": n_t,
                   "parallelism": f"replicas on {world} GPU(s)",
                   "l2": "working set (radial tables + integrand rows) larger than L2",
                   "points_per_patch": st["n_points"]},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": achieved / FP64_PEAK_TFLOPS, "traffic": None,
                     "kernel": "k_tri (channel contraction, DMMA m8n8k4)",
                     "alg_flops_per_step": 2.0 * st["alg_macs"],
                     "exec_flops_per_step": 2.0 * st["contract_macs"],
                     "contract_share_of_step": contract_ms / (total_ms / args.steps),
                     "peak_source": "measured FP64 DMMA.8x8x4 sustained (profiles/fp64_peak.txt)"},
        "e2e": {"value": n_t * world * args.steps / wall_tot, "unit": "channels/s",
                "h2d_bytes_per_step": None, "d2h_bytes_per_step": r.values.nbytes,
                "path": "rbuild.assemble_r_tensor (host tables -> bfr_assemble -> R on host)"},
        "gpu_launches": st["launches"] * args.steps,
        "clocks": clk.summary(),
        "build_s": {"device": total_ms / args.steps / 1e3, "wall": wall_tot / args.steps,
                    "reference_cpu_8proc_s": {"rbuild12": 1263.0}.get(args.config)},
    }
    if world == 1 and not args.no_cpu:
        cpu = rbuild_cpu_rate(args.config)
        line["cpu_baseline"] = {"value": cpu["value"], "unit": "channels/s", "cores": cpu["cores"], "kind": "port",
                                "sample": f"{cpu['channels']} random channels, one per core (oracle port of "
                                          "kinematic channel_half, 1 thread per process)"}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def _proj_worker(args):
    """Oracle restatement of basis.project on sampled f, one process (CPU baseline)."""
    k, l, order, samples = args
    from oracle.project_oracle import ProjectionOracle
    from paper_2605_28475_b200 import project as gproject

    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover
        threadpool_limits = None
    ctx = threadpool_limits(limits=1) if threadpool_limits else None
    if ctx:
        ctx.__enter__()
    orc = ProjectionOracle(k, l, gproject.projection_grid(l, order))
    t0 = time.perf_counter()
    out = [orc.project(s) for s in samples]
    dt = time.perf_counter() - t0
    if ctx:
        ctx.__exit__(None, None, None)
    return out, dt


def run_project(args, rank, world, local_rank):
    """General projection on the GPU (bfq_project_samples).  Replicas on N GPUs
    (each projects its own batch); samples are drifting Maxwellians evaluated
    on the device at the reference's quadrature points (generation outside
    the timed region), checked against the closed-form projection."""
    import numpy as np
    import torch

    from paper_2605_28475_b200 import inputs
    from paper_2605_28475_b200 import project as gproject
    from paper_2605_28475_b200.operator import SpectralConfig

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    k, l, order, n = PROJ[args.config]
    if args.cells:
        n = args.cells
    cfg = SpectralConfig(k, l, 1.0)
    pj = gproject.Projector(cfg, order, local_rank)
    pts = torch.from_numpy(gproject.project_points(cfg, order)).to(dev)
    rng = np.random.default_rng(args.seed + rank)
    u = rng.uniform(-0.3, 0.3, size=(n, 3))
    t = rng.uniform(0.8, 1.2, size=n)
    samples = torch.empty((n, pj.n_points), dtype=torch.float64, device=dev)
    ut, tt = torch.from_numpy(u).to(dev), torch.from_numpy(t).to(dev)
    for i in range(0, n, 64):
        d2 = ((pts[None, :, :] - ut[i:i + 64, None, :]) ** 2).sum(-1)
        samples[i:i + 64] = (2 * np.pi * tt[i:i + 64, None]) ** -1.5 * torch.exp(-d2 / (2 * tt[i:i + 64, None]))
    out = torch.empty((n, cfg.n_k, cfg.n_q), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(max(args.warmup, 0)):
        pj.project(samples, out)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local_rank) as clk:
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)
        for i in range(args.steps):
            starts[i].record(stream)
            pj.project(samples, out)
            ends[i].record(stream)
        clk.sample()
        torch.cuda.synchronize(dev)
    step_ms = [a.elapsed_time(b) for a, b in zip(starts, ends)]
    total_ms = starts[0].elapsed_time(ends[-1])
    tm = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    total_ms = float(tm[0])
    # parity: closed-form projection of the same drifting Maxwellians
    idx = stratified_indices(n, 64)
    got = out[torch.from_numpy(idx).to(dev)].cpu().numpy()
    ref = inputs.project_maxwellians(cfg.n_k, cfg.l_max, u[idx], t[idx])
    errs = [float(np.max(np.abs(got[j] - ref[j])) / np.max(np.abs(ref[j]))) for j in range(len(idx))]
    # end to end: samples from pinned host memory, projection, coefficients back
    e2e = None
    if args.e2e_steps != 0:
        nh = min(n, 512)
        hin = samples[:nh].cpu().pin_memory()
        hout = torch.empty((nh, cfg.n_k, cfg.n_q), dtype=torch.float64).pin_memory()
        dbuf = torch.empty_like(samples[:nh])
        dout = torch.empty_like(out[:nh])
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        ne = 3
        for _ in range(ne):
            dbuf.copy_(hin, non_blocking=True)
            pj.project(dbuf, dout)
            hout.copy_(dout, non_blocking=True)
        torch.cuda.synchronize(dev)
        el = time.perf_counter() - t0
        e2e = {"value": nh * ne * world / el, "unit": "cells/s", "h2d_bytes_per_step": hin.numel() * 8,
               "d2h_bytes_per_step": hout.numel() * 8, "steps": ne, "cells_per_step": nh,
               "path": "pinned host samples -> H2D -> bfq_project_samples -> D2H (PCIe-bound: "
                       f"{pj.n_points * 8 / 1e6:.1f} MB of samples per cell)"}
    if rank == 0:
        kern_s = statistics.mean(step_ms) / 1e3
        gbs = pj.bytes_per_cell * n / kern_s / 1e9
        tfs = pj.flops_per_cell * n / kern_s / 1e12
        hbm = measured_peaks().get("hbm_gbs", 6537.3)
        line = {
            "metric": PROJ_METRIC, "value": n * world * args.steps / (total_ms / 1e3), "unit": "cells/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: drifting Maxwellians (u ~ U(-0.3,0.3)^3, T ~ U(0.8,1.2)) sampled on the device",
            "config": {"workload": f"basis.project of sampled f, N={k} L={l}, radial order {order} "
                                   f"({pj.n_v}x{pj.n_t}x{pj.n_p} points per cell)", "cells_per_gpu": n,
                       "l2": f"inputs larger than L2 ({n * pj.n_points * 8 / 1e9:.1f} GB per GPU)"},
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                         "traffic": None, "kernel": "k_project_samples (DMMA azimuthal GEMM + polar/radial sums)",
                         "bytes_per_cell": pj.bytes_per_cell, "flops_per_cell": pj.flops_per_cell,
                         "fp64_tflops": tfs, "fp64_frac": tfs / FP64_PEAK_TFLOPS,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
            "e2e": e2e, "gpu_launches": args.steps, "clocks": clk.summary(),
            "parity": {"cells": int(len(idx)), "max_rel_err": max(errs), "bar": 1e-12,
                       "pass": bool(max(errs) <= 1e-12),
                       "against": "closed-form projection of the same Maxwellians (bfq_project_maxwellians path, "
                                  "itself pinned to the reference's project)"},
        }
        if world == 1 and not args.no_cpu:
            import multiprocessing as mp

            cores = os.cpu_count() or 1
            m = min(n, 2 * cores)
            hs = samples[:m].cpu().numpy()
            chunks = [(k, l, order, hs[i::cores]) for i in range(cores) if len(hs[i::cores])]
            with mp.get_context("spawn").Pool(len(chunks)) as pool:
                res = pool.map(_proj_worker, chunks)
            busy = max(r[1] for r in res)
            line["cpu_baseline"] = {"value": m / busy, "unit": "cells/s", "cores": len(chunks), "kind": "port",
                                    "sample": f"{m} cells' samples, 2 per process (oracle/project_oracle.py: "
                                              "basis.project's einsums on the sampled grid)", "cpu": cpu_model()}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    from paper_2605_28475_b200 import dist as bdist

    dry = args.dry_run
    dev = torch.device("cpu") if dry else torch.device("cuda", local_rank)
    if not dry:
        torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if args.backend == "nccl":
            # the communicator lines (nranks, NVLS/NVLink transport) go to stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    opfile, n_global, _, desc, psample = CONFIGS[args.config]
    if args.cells:
        n_global = args.cells
    strong = args.scaling == "strong"
    if strong:  # one fixed global batch, contiguous equal shards
        start, n_cells = bdist.shard_range(n_global, world, rank)
        total_cells = n_global
    else:  # every rank evaluates its own n_global cells
        start, n_cells = rank * n_global, n_global
        total_cells = n_global * world

    def gather(vals):
        """Per-rank float values -> list over ranks (all ranks)."""
        t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=dev)
        if dist is None:
            return [t.tolist()]
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return [o.tolist() for o in out]

    if dry:  # launcher / sharding / collective plumbing only (CPU test): no kernels, no timing
        shards = gather([start, n_cells])
        diag = bdist.allreduce_diagnostics(torch.tensor([0.0] * 5 + [float(n_cells), float(start)],
                                                        dtype=torch.float64))
        if rank == 0:
            print(json.dumps({"dry_run": True, "n_gpus": world, "scaling": args.scaling, "backend": args.backend,
                              "global_cells": total_cells, "shards": [[int(a), int(b)] for a, b in shards],
                              "diag_cells": float(diag[5])}), flush=True)
        if dist is not None:
            dist.destroy_process_group()
        return

    from paper_2605_28475_b200 import engine

    op = load_operator(opfile, local_rank)
    if getattr(op, "_built_on_gpu", False):
        desc += " [operator assembled on this GPU by bfr_assemble: reference build not present]"
    plan = engine.plan_for(op, local_rank)
    cfg = op.cfg
    host = make_cells(args.config, cfg.n_k, cfg.l_max, n_cells, seed=args.seed, start=start, device=local_rank)
    f = torch.from_numpy(host).to(dev)
    q = torch.empty_like(f)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    rk4 = args.config == "rk4"
    if rk4:
        y = f.clone()
        work = torch.empty((3,) + tuple(f.shape), dtype=torch.float64, device=dev)
        flag = torch.zeros(1, dtype=torch.int32, device=dev)

        def one_step():
            plan.rk4_step_device(y.data_ptr(), work.data_ptr(), n_cells, 0.01, flag.data_ptr(), stream.cuda_stream)
    else:
        def one_step():
            engine.evaluate_batch(plan, f, out=q)
    for _ in range(max(args.warmup, 0)):
        one_step()
    barrier()
    # Inputs (+ outputs) smaller than L2: flush L2 between timed steps by
    # writing a 256 MB buffer outside the per-step events; the step time is
    # then the sum of the per-step event intervals.
    flush = None
    if 2 * host.nbytes < 2 * L2_BYTES and not rk4:
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local_rank) as clk:
        barrier()
        t0 = time.perf_counter()
        for i in range(args.steps):
            if flush is not None:
                flush.fill_(i & 0xff)
            starts[i].record(stream)
            one_step()
            ends[i].record(stream)
        # (the sampler thread polls NVML every 2 ms while the queued steps run; a
        # synchronous NVML query between enqueues could starve the launch queue)
        clk.sample()
        barrier()
        wall = time.perf_counter() - t0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    local_ms = sum(step_ms) if flush is not None else starts[0].elapsed_time(ends[-1])
    q_per_step = 4 if rk4 else 1
    per_rank = gather([local_ms, n_cells, start])
    total_ms = max(r[0] for r in per_rank)  # the job ends with the slowest rank
    value = total_cells * args.steps * q_per_step / (total_ms / 1e3)
    ms_per_step = total_ms / args.steps

    # conservation diagnostics, all-reduced over NCCL after the timed region
    mom = torch.empty((n_cells, 5), dtype=torch.float64, device=dev)
    if rk4:
        mom0 = torch.empty_like(mom)
        plan.moments_device(f.data_ptr(), mom0.data_ptr(), n_cells, stream.cuda_stream)
        plan.moments_device(y.data_ptr(), mom.data_ptr(), n_cells, stream.cuda_stream)
        mom = mom - mom0  # drift of the invariants over the run
        if int(flag.item()):
            raise RuntimeError("RK4 diverged")
        out_t = y
    else:
        plan.moments_device(q.data_ptr(), mom.data_ptr(), n_cells, stream.cuda_stream)
        out_t = q
    diag = bdist.as_dict(bdist.allreduce_diagnostics(bdist.diagnostics_vector(mom, out_t)))
    slots_exact = bool((q[:, 0, : min(4, cfg.n_q)] == 0).all() and (cfg.n_k < 2 or (q[:, 1, 0] == 0).all())) \
        if not rk4 else None
    ok = torch.tensor([1.0 if (slots_exact is None or slots_exact) else 0.0], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)

    # end to end through the C ABI with host buffers, copies inside the timed region
    e2e = None
    if args.e2e_steps != 0 and not rk4:
        from paper_2605_28475_b200 import _lib

        lib = _lib.lib()
        e2e_steps = args.steps if args.e2e_steps < 0 else args.e2e_steps
        hin = torch.from_numpy(host).pin_memory()
        hout = torch.empty_like(hin).pin_memory()
        _lib.check(lib.bfq_eval_host(plan.handle, hin.data_ptr(), None, hout.data_ptr(), n_cells))  # warm
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            _lib.check(lib.bfq_eval_host(plan.handle, hin.data_ptr(), None, hout.data_ptr(), n_cells))
        el = time.perf_counter() - t0
        # pageable numpy buffers (staged through the plan's pinned chunks)
        pout = np.empty_like(host)
        n_pg = min(3, e2e_steps)
        t0 = time.perf_counter()
        for _ in range(n_pg):
            _lib.check(lib.bfq_eval_host(plan.handle, host.ctypes.data, None, pout.ctypes.data, n_cells))
        el_pg = time.perf_counter() - t0
        same_bits = bool(np.array_equal(pout, hout.numpy()))
        els = gather([el, el_pg])
        el, el_pg = max(r[0] for r in els), max(r[1] for r in els)
        bytes_ = n_cells * cfg.n_dof * 8
        e2e = {"value": total_cells * e2e_steps / el, "unit": "cells/s",
               "h2d_bytes_per_step": bytes_, "d2h_bytes_per_step": bytes_, "steps": e2e_steps,
               "path": "bfq_eval_host (C ABI, pinned host buffers, chunked H2D/Q/D2H pipeline over 3 streams)",
               "pageable": {"value": total_cells * n_pg / el_pg, "steps": n_pg, "bitwise_equal_to_pinned": same_bits,
                            "path": "bfq_eval_host on pageable numpy buffers (staged through pinned chunks)"}}

    # parity of the timed batch's own outputs against the CPU oracle (rank 0's shard)
    parity, cpu = None, None
    if rank == 0 and not args.no_parity and not rk4:
        from oracle import q_oracle
        from paper_2605_28475_b200.operator import save_cache

        oppath = os.path.join(ROOT, "operators", opfile + ".bfct")
        if getattr(op, "_built_on_gpu", False):  # the CPU port reads the same (GPU-built) operator
            import tempfile

            oppath = os.path.join(tempfile.mkdtemp(), opfile + ".bfct")
            save_cache(oppath, op)
        k = psample if args.parity_cells < 0 else args.parity_cells
        idx = stratified_indices(n_cells, k)
        qs = q[torch.from_numpy(idx).to(dev)].cpu().numpy()
        ref, cpu = oracle_pool(oppath, host[idx])
        errs = np.array([q_oracle.rel_err(qs[i], ref[i]) for i in range(len(idx))])
        worst = int(np.argmax(errs)) if len(idx) else 0
        parity = {"cells": int(len(idx)), "of": int(n_cells), "max_rel_err": float(errs.max()) if len(idx) else None,
                  "worst_cell": int(idx[worst]) if len(idx) else None, "bar": 1e-12,
                  "pass": bool(len(idx) and errs.max() <= 1e-12),
                  "selection": "every cell" if len(idx) == n_cells else
                  "stratified: evenly spread over the shard incl. first/last cell and the last tile",
                  "metric": "max|Q_gpu - Q_ref| / max|Q_ref| per cell (test_contraction.py:63-65)",
                  "against": ("the live reference's evaluate(op, c) (baseline/_ref)" if cpu["kind"] == "reference"
                              else "the CPU oracle (oracle/q_oracle.py)"),
                  "invariant_slots_exact": bool(ok.item() == 1.0)}
    elif rk4:
        parity = {"skipped": "RK4 trajectory parity is tests/test_gpu_rk4.py (reference golden, every 100th step)",
                  "moment_drift_max": max(diag[k] for k in ("max_mass", "max_px", "max_py", "max_pz", "max_energy"))}
    if dist is not None:
        dist.barrier()

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    flops_cell, bytes_cell = plan.flops_per_cell, plan.bytes_per_cell
    kern_s = statistics.mean(step_ms) / 1e3
    achieved = flops_cell * n_cells * q_per_step / kern_s / 1e12
    exec_tf = 2.0 * plan.info["exec_macs_per_cell"] * n_cells * q_per_step / kern_s / 1e12
    useful_tf = 2.0 * plan.info["useful_macs_per_cell"] * n_cells * q_per_step / kern_s / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tpath):
        try:  # ncu dram bytes per cell of the same kernel, scaled to this launch
            traffic = json.load(open(tpath))["dram_bytes_per_cell"] * n_cells
        except (OSError, ValueError, KeyError):
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": "cells/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json distributions)",
        "config": {"workload": desc, "operator": opfile, "global_cells": total_cells, "cells_per_rank": n_cells,
                   "parallelism": f"{'one fixed batch' if strong else 'one batch per GPU'} sharded over {world} "
                                  "GPU(s), contiguous blocks, no data-path collective",
                   "l2": ("L2 flushed between timed steps (256 MB write outside the step events; inputs "
                          "%.3f GB per GPU < 126 MB L2)" % (host.nbytes / 1e9)) if flush is not None else
                         ("inputs larger than L2 (%.2f GB per GPU vs 126 MB)" % (host.nbytes / 1e9)),
                   "seed": args.seed},
        "rank_ms": [r[0] for r in per_rank],
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                     "kernel": "bfq_q_kernel2 (fused stages 1-3, DMMA.8x8x4)",
                     "peak_source": "measured FP64 DMMA.8x8x4 sustained (profiles/fp64_peak.txt); "
                                    "MEASURED_PEAKS.json has no fp64 entry",
                     "nominal_peak": FP64_NOMINAL_TFLOPS, "nominal_frac": achieved / FP64_NOMINAL_TFLOPS,
                     "flops_per_cell": flops_cell,
                     "exec_dmma_macs_per_cell": plan.info["exec_macs_per_cell"],
                     "exec_tflops": exec_tf, "exec_frac": exec_tf / FP64_PEAK_TFLOPS,
                     "useful_macs_per_cell": plan.info["useful_macs_per_cell"],
                     "useful_tflops": useful_tf, "useful_frac": useful_tf / FP64_PEAK_TFLOPS,
                     "fracs_note": "frac: algorithmic FLOP (2(N_G n_k^2 + N_S n_k^3), SURVEY 8d) / peak; "
                                   "exec_frac: DMMA MACs issued incl. tile and row padding; useful_frac: MACs "
                                   "of the folded channels without padding (what the kernel must do)",
                     "hbm_frac": bytes_cell * n_cells / kern_s / 1e9 / measured_peaks().get("hbm_gbs", 6548.2)},
        "e2e": e2e,
        # RK4: 4 Q launches + 7 elementwise stage kernels (BFQ_RK4_FUSED=1: the 4 Q launches alone)
        "gpu_launches": args.steps * ((4 if os.environ.get("BFQ_RK4_FUSED", "0") not in ("", "0") else 11) if rk4 else 1),
        "clocks": clk.summary(),
        "parity": parity,
        "conservation": {"invariant_slots_exact": bool(ok.item() == 1.0), **diag},
        "wall_s": wall,
    }
    if rk4:
        line["rk4"] = {"dt": 0.01, "steps_per_s": args.steps / (total_ms / 1e3),
                       "full_run_estimate_s": 1000 * ms_per_step / 1e3}
    if world == 1 and cpu is not None:
        line["cpu_baseline"] = {
            "value": cpu["value"], "unit": "cells/s", "cores": cpu["cores"], "kind": cpu["kind"],
            "sample": f"the {cpu['cells']} parity cells of the timed batch, contiguous blocks over {cpu['cores']} "
                      f"processes (1 thread each), ~{cpu['busy_s']:.1f} s per process ("
                      + ("the live reference package from baseline/_ref: boltzfact.contraction.evaluate"
                         if cpu["kind"] == "reference" else
                         "oracle/q_oracle.py: the reference's q_angular_first operations, bit-identical to it and "
                         "the same speed per cell, profiles/r01_cpu_ref_vs_port.txt") + ")",
            "cpu": cpu_model(), "single_core_cells_per_s": cpu["single_core_cells_per_s"]}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def launch_ranks(args):
    """``--gpus N`` outside torchrun: re-run this script under
    torch.distributed.run with N local ranks; rank 0 prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1")))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="hs12", choices=sorted(CONFIGS) + sorted(RBUILD) + sorted(PROJ))
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: one fixed global batch sharded over the GPUs (BASELINE config 3); "
                         "weak: the batch per GPU")
    ap.add_argument("--cells", type=int, default=0, help="override the global batch (strong) / per-GPU batch (weak)")
    ap.add_argument("--seed", type=int, default=20260520)
    ap.add_argument("--e2e-steps", type=int, default=-1, help="-1: as many as --steps; 0: skip")
    ap.add_argument("--parity-cells", type=int, default=-1, help="-1: the config's default sample; 0: every cell")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=3.0, help="reference arm: seconds of work per core per step")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU oracle leg (parity and cpu_baseline)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--dry-run", action="store_true", help="launcher/sharding/collective plumbing only (no GPU)")
    args = ap.parse_args()
    if args.no_cpu:
        args.no_parity = True
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args))
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.backend == "gloo" and not args.dry_run:
        # functional multi-rank run on fewer GPUs than ranks (gloo only; NCCL
        # needs one GPU per rank): ranks share devices round-robin.  Not a
        # scaling measurement -- the ranks then contend for the same SMs.
        try:
            import torch

            n_dev = torch.cuda.device_count()
            if n_dev and local_rank >= n_dev:
                local_rank %= n_dev
        except Exception:  # pragma: no cover
            pass
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif args.config in RBUILD:
        run_rbuild(args, rank, world, local_rank)
    elif args.config in PROJ:
        run_project(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
