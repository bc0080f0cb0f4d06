"""Summarise an ncu report (raw page) into the numbers DESIGN.md cites."""
import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__warps_active.avg.per_cycle_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "sm__inst_executed.sum",
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(f"== {d.get('Kernel Name', '?')[:60]}")
        for k in KEYS:
            if k in d:
                print(f"  {k:85s} {d[k]:>16s} {units[hdr.index(k)]}")
        stalls = sorted(((float(d[k].replace(',', '') or 0), k) for k in hdr
                         if k.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in k), reverse=True)
        tot = sum(v for v, _ in stalls) or 1
        print("  stalls: " + ", ".join(f"{k.split('stalled_')[1]} {100 * v / tot:.0f}%" for v, k in stalls[:8]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
