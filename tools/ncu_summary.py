#!/usr/bin/env python
"""Summarise ncu raw CSV exports (``ncu -i X.ncu-rep --page raw --csv``) into
the markdown table kept under profiles/.

    python tools/ncu_summary.py profiles/r01_ncu_full_decode_m6_raw.csv [...]
"""
import csv
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe (POPC) %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads/inst (32 = no divergence)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem st bank conflicts"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def load(path):
    with open(path) as f:
        rows = [r for r in csv.reader(f)]
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    head, units = rows[start], rows[start + 1]
    return [(head, units, r) for r in rows[start + 2:] if r]


def main(paths):
    for p in paths:
        for head, units, r in load(p):
            name = r[head.index("Kernel Name")] if "Kernel Name" in head else "?"
            print(f"### {p}\n\n`{name[:120]}`\n")
            print("| metric | value | unit |\n|---|---|---|")
            for key, label in METRICS:
                if key in head:
                    i = head.index(key)
                    print(f"| {label} (`{key}`) | {r[i]} | {units[i]} |")
            print()


if __name__ == "__main__":
    main(sys.argv[1:])
