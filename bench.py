"""Benchmark of the Q(f,f) hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config hs12|hs8|mm10|hs4]

One step = one Q(f,f) evaluation of every cell of the rank's batch (one
``bfq_eval`` launch).  Default workload = BASELINE config 3 (hard spheres,
N=L=12, 65,536 cells per GPU; weak scaling: each rank evaluates its own
65,536-cell shard of a 65,536*N-cell global batch, no data-path collective).
Rank 0 prints one JSON line.  See DESIGN.md §Measurement.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (operator file, cells per GPU, generator, description)
    "hs12": ("hs_n12", 65536, "pm", "config3: hard spheres N=L=12, perturbed Maxwellians"),
    "hs8": ("hs_n8", 4096, "pm", "config2: hard spheres N=L=8, perturbed Maxwellians"),
    "mm10": ("mm_n10", 32768, "bimodal", "config5 operator: Maxwell N=L=10, bimodal cells (single Q eval)"),
    "hs4": ("hs_n4", 65536, "pm", "hard spheres N=L=4 (small)"),
    "hs16": ("hs_n16", 16384, "pm", "config4: hard spheres N=L=16, perturbed Maxwellians"),
    "syn16": ("synth_n16", 16384, "pm", "config4 shape N=L=16 with a SYNTHETIC R (real Gaunt table, random "
                                        "slot-symmetric R with the reference's null-space zeroing): timing only"),
    "rk4": ("mm_n10", 32768, "bimodal", "config5: Maxwell N=L=10, bimodal cells, GPU-resident RK4 dt=0.01 "
                                         "(one step = one RK4 step = 4 Q(f,f) per cell)"),
}
# the operator build.  One step = one full R-tensor
# assembly (every channel's gain / loss integrals over both Duffy patches).
RBUILD = {
    "rbuild8": (8, 8, 1.0),
    "rbuild12": (12, 12, 1.0),
    "rbuild16": (16, 16, 1.0),
}
METRIC = "Q(f,f) cell-evals/s (fp64, hard spheres L=N=12) and FP64/HBM roofline frac"
RBUILD_METRIC = "R-tensor assembly channel integrals/s (fp64, hard spheres, pad 16/16)"
FP64_PEAK_TFLOPS = 37.1  # DMMA.8x8x4 sustained, measured on this pool (profiles/fp64_peak.txt)


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


# ------------------------------------------------------------------ CPU legs
def _cpu_worker(args):
    path, cells = args
    from oracle import q_oracle
    from paper_2605_28475_b200.operator import load_cache

    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover
        threadpool_limits = None
    op = q_oracle.OracleOperator.from_operator(load_cache(path))
    ws = q_oracle.angular_workspace(op)  # cached per operator, as the reference does
    ctx = threadpool_limits(limits=1) if threadpool_limits else None
    if ctx:
        ctx.__enter__()
    t0 = time.perf_counter()
    for c in cells:
        q_oracle.q_angular_first(op, c, workspace=ws)
    dt = time.perf_counter() - t0
    if ctx:
        ctx.__exit__(None, None, None)
    return len(cells), dt


def cpu_port_rate(cfg_name, cells, budget_s=15.0, cores=None, path=None):
    """Oracle port (numpy restatement of q_angular_first) on host cores: cells/s."""
    import multiprocessing as mp

    path = path or os.path.join(ROOT, "operators", CONFIGS[cfg_name][0] + ".bfct")
    cores = cores or os.cpu_count() or 1
    # calibrate on one cell, then give every worker ~budget_s of work
    n1, dt1 = _cpu_worker((path, cells[:1]))
    per_worker = max(1, int(budget_s / max(dt1, 1e-6)))
    n = min(cells.shape[0], per_worker * cores)
    chunks = [(path, cells[i::cores][: per_worker]) for i in range(cores)]
    chunks = [c for c in chunks if len(c[1])]
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(len(chunks)) as pool:
        res = pool.map(_cpu_worker, chunks)
    wall = time.perf_counter() - t0
    done = sum(r[0] for r in res)
    busy = max(r[1] for r in res)
    return {"value": done / busy, "cells": done, "cores": len(chunks), "wall_s": wall, "busy_s": busy,
            "single_cell_s": dt1}


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
    contraction.q_angular_first) on all host cores, rank 0 only."""
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
                             "sample": f"{r['channels']} random channels, one per core"},
            "e2e": {"value": v, "unit": "channels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }), flush=True)
        return
    opfile, n_cells, _, desc = CONFIGS[args.config]
    from paper_2605_28475_b200.operator import load_cache

    path = os.path.join(ROOT, "operators", opfile + ".bfct")
    if not os.path.exists(path):
        print(json.dumps({"impl": "reference", "unavailable": f"operators/{opfile}.bfct (a multi-hour reference "
                          "CPU build) is not shipped with this snapshot"}), flush=True)
        return
    op = load_cache(path)
    cells = make_cells(args.config, op.cfg.n_k, op.cfg.l_max, 256, seed=args.seed, start=0)
    rates, walls = [], []
    for _ in range(args.warmup):
        cpu_port_rate(args.config, cells, budget_s=2.0)
    for _ in range(args.steps):
        r = cpu_port_rate(args.config, cells, budget_s=args.cpu_budget)
        rates.append(r["value"])
        walls.append(r["wall_s"])
        last = r
    v = statistics.median(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "cells/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(walls),
        "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json distributions)",
        "config": {"workload": desc, "cells_per_gpu": n_cells, "operator": opfile,
                   "step": "one bounded sample of the workload on all host cores (multiprocessing pool)"},
        "cpu_baseline": {"value": v, "unit": "cells/s", "cores": last["cores"], "kind": "port",
                         "sample": f"~{args.cpu_budget:.0f} s of per-core work per step, cells of {desc}"},
        "e2e": {"value": v, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def load_operator(opfile, device=0):
    """The reference-built cache; for config 4 (N=L=16, a multi-hour CPU build
    that is not shipped) fall back to assembling it on the GPU (rbuild)."""
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


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    from paper_2605_28475_b200 import dist as bdist
    from paper_2605_28475_b200 import engine

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    opfile, n_cells, _, desc = CONFIGS[args.config]
    if args.cells:
        n_cells = args.cells
    op = load_operator(opfile, local_rank)
    if getattr(op, "_built_on_gpu", False):
        desc += " [operator assembled on this GPU by bfr_assemble: reference build not present]"
    plan = engine.plan_for(op, local_rank)
    cfg = op.cfg
    host = make_cells(args.config, cfg.n_k, cfg.l_max, n_cells, seed=args.seed, start=rank * n_cells,
                      device=local_rank)
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
    l2_bytes = 132644864
    flush = None
    if 2 * host.nbytes < 2 * l2_bytes and not rk4:
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
            clk.sample()  # queued work is still running
        clk.sample()
        barrier()
        wall = time.perf_counter() - t0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms) if flush is not None else starts[0].elapsed_time(ends[-1])
    q_per_step = 4 if rk4 else 1
    # whole-job rate: cells of all ranks / the slowest rank's device time
    value, total_ms = bdist.weak_scaling_rate(n_cells, args.steps * q_per_step, total_ms, device=dev)
    ms_per_step = total_ms / args.steps

    # conservation diagnostics of the last step, all-reduced (max |production|,
    # or for RK4 the max drift of the invariants from the initial state)
    mom = torch.empty((n_cells, 5), dtype=torch.float64, device=dev)
    if rk4:
        mom0 = torch.empty_like(mom)
        plan.moments_device(f.data_ptr(), mom0.data_ptr(), n_cells, stream.cuda_stream)
        plan.moments_device(y.data_ptr(), mom.data_ptr(), n_cells, stream.cuda_stream)
        mom = mom - mom0
        if int(flag.item()):
            raise RuntimeError("RK4 diverged")
    else:
        plan.moments_device(q.data_ptr(), mom.data_ptr(), n_cells, stream.cuda_stream)
    diag = mom.abs().amax(dim=0)
    if dist is not None:
        dist.all_reduce(diag, op=dist.ReduceOp.MAX)
    conservation_max = float(diag.max().item())

    # end-to-end through the C ABI with host buffers (pinned), copies timed
    e2e = None
    if args.e2e_steps > 0 and not rk4:
        hin = torch.from_numpy(host).pin_memory()
        hout = torch.empty_like(hin).pin_memory()
        from paper_2605_28475_b200 import _lib

        lib = _lib.lib()
        lib.bfq_eval_host(plan.handle, hin.data_ptr(), None, hout.data_ptr(), n_cells)  # warm
        barrier()
        walls = []
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            _lib.check(lib.bfq_eval_host(plan.handle, hin.data_ptr(), None, hout.data_ptr(), n_cells))
            walls.append(time.perf_counter() - t0)
        # wall clock of the blocking host call (copies in the timed region), median step
        el = torch.tensor([statistics.median(walls) * args.e2e_steps], dtype=torch.float64, device=dev)
        if dist is not None:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        bytes_ = n_cells * cfg.n_dof * 8
        e2e = {"value": n_cells * world * args.e2e_steps / float(el.item()), "unit": "cells/s",
               "h2d_bytes_per_step": bytes_, "d2h_bytes_per_step": bytes_, "steps": args.e2e_steps,
               "path": "bfq_eval_host (C ABI, pinned host buffers, chunked H2D/Q/D2H pipeline)"}

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    flops_cell, bytes_cell = plan.flops_per_cell, plan.bytes_per_cell
    achieved = flops_cell * n_cells * q_per_step / (statistics.mean(step_ms) / 1e3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tpath):
        try:  # ncu dram bytes per cell of the same kernel, scaled to this launch
            traffic = json.load(open(tpath))["dram_bytes_per_cell"] * n_cells
        except (OSError, ValueError, KeyError):
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": "cells/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json distributions)",
        "config": {"workload": desc, "operator": opfile, "cells_per_gpu": n_cells, "global_cells": n_cells * world,
                   "parallelism": f"cells sharded over {world} GPU(s), no data-path collective",
                   "l2": ("L2 flushed between timed steps (256 MB write outside the step events; inputs "
                          "%.3f GB per GPU < 126 MB L2)" % (host.nbytes / 1e9)) if flush is not None else
                         ("inputs larger than L2 (%.2f GB per GPU vs 126 MB)" % (host.nbytes / 1e9)),
                   "seed": args.seed},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                     "peak_source": "measured FP64 DMMA.8x8x4 sustained (profiles/fp64_peak.txt); "
                                    "MEASURED_PEAKS.json has no fp64 entry",
                     "flops_per_cell": flops_cell, "exec_dmma_macs_per_cell": plan.info["exec_macs_per_cell"],
                     "hbm_frac": bytes_cell * n_cells / (statistics.mean(step_ms) / 1e3) / 1e9
                     / measured_peaks().get("hbm_gbs", 6456.5)},
        "e2e": e2e,
        "gpu_launches": args.steps * (7 if rk4 else 1),
        "clocks": clk.summary(),
        "conservation_max_abs": conservation_max,
        "wall_s": wall,
    }
    if rk4:
        line["rk4"] = {"dt": 0.01, "steps_per_s": args.steps / (total_ms / 1e3),
                       "full_run_estimate_s": 1000 * ms_per_step / 1e3,
                       "moment_drift_max": conservation_max}
    if world == 1 and not args.no_cpu:
        oppath = None
        if getattr(op, "_built_on_gpu", False):  # the CPU port reads the same (GPU-built) operator
            import tempfile

            from paper_2605_28475_b200.operator import save_cache

            oppath = os.path.join(tempfile.mkdtemp(), opfile + ".bfct")
            save_cache(oppath, op)
        cpu = cpu_port_rate(args.config, host[:256], budget_s=args.cpu_budget, path=oppath)
        line["cpu_baseline"] = {"value": cpu["value"], "unit": "cells/s", "cores": cpu["cores"], "kind": "port",
                                "sample": f"{cpu['cells']} cells of the same batch, ~{args.cpu_budget:.0f} s per core "
                                          "(oracle/q_oracle.py: the reference's q_angular_first operations, bit-identical to it and "
                                          "the same speed per cell, profiles/r01_cpu_ref_vs_port.txt; 1 thread per process)"}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="hs12", choices=sorted(CONFIGS) + sorted(RBUILD))
    ap.add_argument("--cells", type=int, default=0, help="override cells per GPU")
    ap.add_argument("--seed", type=int, default=20260520)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-budget", type=float, default=10.0, help="seconds of per-core CPU work per sample")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif args.config in RBUILD:
        run_rbuild(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
