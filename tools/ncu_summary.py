#!/usr/bin/env python
"""Summarise an ncu --set full report: duration, DRAM traffic, pipe
utilisation, occupancy, shared-memory conflicts and the top warp stall
reasons.   python tools/ncu_summary.py report.ncu-rep"""

import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe % active"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 inst % peak"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma pipe % active"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "occ limit (regs)"),
    ("launch__occupancy_limit_shared_mem", "occ limit (smem)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem st bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("smsp__inst_executed.sum", "instructions"),
    ("lts__t_sectors_op_red.sum", "L2 red sectors"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu pipe % peak"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"== {name[:110]}")
        for k, label in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {label:28s} {vals[i]:>16s} {units[i]}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(vals[i]), h.split("stalled_")[1].replace("_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        if stalls:
            stalls.sort(reverse=True)
            print("  top stalls (cycles/issued inst): " +
                  ", ".join(f"{n}={v:.2f}" for v, n in stalls[:7]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
