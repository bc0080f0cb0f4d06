"""SASS evidence for the Q kernels (no GPU needed).

    python tools/sass_summary.py [--lib paper_2605_28475_b200/libbfq.so] > profiles/r02_sass_summary.txt

For every bfq_q_kernel2 / bfq_q_kernel instantiation in the built library:
registers, spill stores/loads and local-memory bytes (cuobjdump -res-usage),
static instruction counts of the FP64 tensor op (DMMA.8x8x4), the FP64 vector
ops (DFMA/DMUL/DADD), shared loads/stores, the bulk copy that fills the R ring
(UBLKCP = cp.async.bulk), the mbarrier ops (SYNCS.*) and any local-memory
instruction (LDL/STL = spills).  Static counts show what the compiler emitted;
the dynamic mix is in the ncu captures under profiles/.
"""

from __future__ import annotations

import argparse
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUOBJDUMP = "/usr/local/cuda/bin/cuobjdump"
CUFILT = "/usr/local/cuda/bin/cu++filt"

TRACK = ["DMMA", "DFMA", "DMUL", "DADD", "LDS", "STS", "LDG", "STG", "UBLKCP", "SYNCS", "BAR", "SHFL", "LDL", "STL"]


def demangle(name: str) -> str:
    try:
        return subprocess.run([CUFILT, name], capture_output=True, text=True).stdout.strip() or name
    except OSError:
        return name


def res_usage(lib: str) -> dict[str, str]:
    out = subprocess.run([CUOBJDUMP, "-res-usage", lib], capture_output=True, text=True).stdout
    usage, fn = {}, None
    for line in out.splitlines():
        m = re.match(r"\s*Function (\S+):", line)
        if m:
            fn = m.group(1)
            continue
        if fn and "REG:" in line:
            usage[fn] = line.strip()
            fn = None
    return usage


def sass_by_function(lib: str) -> dict[str, list[str]]:
    out = subprocess.run([CUOBJDUMP, "-sass", lib], capture_output=True, text=True).stdout
    funcs, cur = {}, None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        if cur is not None:
            m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
            if m:
                funcs[cur].append(m.group(1) + (m.group(2) or ""))
    return funcs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_2605_28475_b200", "libbfq.so"))
    ap.add_argument("--filter", default="bfq_q_kernel")
    a = ap.parse_args()
    usage = res_usage(a.lib)
    funcs = sass_by_function(a.lib)
    print(f"# SASS summary of {os.path.relpath(a.lib, ROOT)} (cuobjdump {a.lib.split('/')[-1]}, sm_100a)")
    print("# static instruction counts per kernel; DMMA = mma.sync.m8n8k4.f64 (FP64 tensor pipe),")
    print("# UBLKCP = cp.async.bulk global->shared (R ring), SYNCS = mbarrier ops, LDL/STL = local memory (spills)")
    for fn in sorted(funcs):
        if a.filter not in fn:
            continue
        ops = funcs[fn]
        cnt = collections.Counter(o.split(".")[0] for o in ops)
        variants = collections.Counter(o for o in ops if o.startswith(("DMMA", "UBLKCP", "SYNCS")))
        print()
        print(demangle(fn))
        print("  " + usage.get(fn, "(no res-usage line)"))
        print("  total " + str(len(ops)) + " | " + " ".join(f"{k}={cnt.get(k, 0)}" for k in TRACK))
        print("  forms: " + ", ".join(f"{k} x{v}" for k, v in sorted(variants.items())))
    return 0


if __name__ == "__main__":
    sys.exit(main())
