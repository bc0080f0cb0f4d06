"""Shared-memory wavefronts per SASS instruction class from an ncu source-page
CSV (``ncu -i rep --page source --csv --print-source sass``, optionally gzipped).

    python tools/ncu_smem_by_instr.py gpurun_out/prof/src_hs_n8.csv.gz [--top 25]

Groups the instructions by opcode (LDS / STS / LDG / ... ) and prints, per
group, executed instructions, shared wavefronts, the ideal count and the
excess (bank conflicts), then the individual instructions with the largest
wavefront counts -- where a kernel's shared-memory bandwidth goes.
"""
import argparse
import collections
import csv
import gzip
import io


def num(s):
    try:
        return float((s or "0").replace(",", ""))
    except ValueError:
        return 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    raw = gzip.open(a.path, "rt").read() if a.path.endswith(".gz") else open(a.path).read()
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1] if rows[0] and rows[0][0].startswith("Kernel") or len(rows[0]) < 5 else rows[0]
    start = rows.index(hdr) + 1
    ix = {k: hdr.index(k) for k in ("Address", "Source", "Instructions Executed", "L1 Wavefronts Shared",
                                    "L1 Wavefronts Shared Ideal", "Warp Stall Sampling (All Samples)")}
    groups = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0.0, 0])
    per = []
    tot_wf = tot_samples = 0.0
    for r in rows[start:]:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        key = op.split(".")[0] + ("." + op.split(".")[1] if op.startswith(("LDS", "STS", "LDG")) and "." in op else "")
        ex, wf, ide = num(r[ix["Instructions Executed"]]), num(r[ix["L1 Wavefronts Shared"]]), \
            num(r[ix["L1 Wavefronts Shared Ideal"]])
        smp = num(r[ix["Warp Stall Sampling (All Samples)"]])
        g = groups[key]
        g[0] += ex
        g[1] += wf
        g[2] += ide
        g[3] += smp
        g[4] += 1
        tot_wf += wf
        tot_samples += smp
        per.append((wf, ide, ex, smp, r[ix["Address"]], src))
    print(f"total shared wavefronts {tot_wf:.4g}, stall samples {tot_samples:.4g}")
    print(f"{'opcode':14s} {'static':>6s} {'executed':>12s} {'wavefronts':>12s} {'ideal':>12s} {'excess':>10s} "
          f"{'wf share':>8s} {'samples':>8s}")
    for k, (ex, wf, ide, smp, n) in sorted(groups.items(), key=lambda kv: -kv[1][1]):
        if wf == 0 and smp < 0.01 * tot_samples:
            continue
        print(f"{k:14s} {n:6d} {ex:12.4g} {wf:12.4g} {ide:12.4g} {wf - ide:10.3g} {wf / max(tot_wf, 1):8.1%} "
              f"{smp / max(tot_samples, 1):8.1%}")
    print("\ntop instructions by shared wavefronts:")
    for wf, ide, ex, smp, addr, src in sorted(per, reverse=True)[:a.top]:
        print(f"  {addr:>8s} wf {wf:10.4g} ideal {ide:10.4g} exec {ex:10.4g}  {src[:90]}")


if __name__ == "__main__":
    main()
