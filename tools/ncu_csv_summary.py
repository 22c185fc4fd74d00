"""Summarise `ncu --page raw --csv` exports (no GPU needed) as a markdown table of the pipe counters the
P2P / M2L rooflines are argued from.

usage: python tools/ncu_csv_summary.py label=export.csv [label=export.csv ...]
Columns: duration, SM clock, FMA-pipe active %, XU (MUFU) instruction rate % of peak, issue-active %,
warps-active %, tensor-pipe % of elapsed, DRAM bytes, L2 / L1TEX throughput %, registers per thread.
"""
import csv
import sys

COLS = [
    ("duration", "gpu__time_duration.sum"),
    ("SM clock", "sm__cycles_elapsed.avg.per_second"),
    ("FMA pipe %", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("FP64 pipe %", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    ("XU (MUFU) inst %", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
    ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("tensor pipe %", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("DRAM read", "dram__bytes_read.sum"),
    ("L2 thru %", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("L1TEX thru %", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("regs", "launch__registers_per_thread"),
]


def rows_of(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, units = rows[hi], rows[hi + 1]
    for r in rows[hi + 2:]:
        if len(r) != len(hdr):
            continue
        d = {h: (v, u) for h, u, v in zip(hdr, units, r)}
        yield d


def fmt(d, key):
    if key not in d:
        return "-"
    v, u = d[key]
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    if u in ("%",):
        return f"{x:.1f}"
    if u in ("Ghz",):
        return f"{x:.2f} GHz"
    if u in ("usecond", "msecond", "nsecond", "us", "ms", "ns"):
        return f"{x:.1f} {u.replace('second', 's')}"
    if u in ("byte", "Kbyte", "Mbyte", "Gbyte"):
        return f"{x:.1f} {u.replace('byte', 'B')}"
    return f"{x:g}"


def main():
    print("| config | kernel | " + " | ".join(c for c, _ in COLS) + " |")
    print("|---|---|" + "---|" * len(COLS))
    for arg in sys.argv[1:]:
        label, path = arg.split("=", 1)
        for d in rows_of(path):
            name = d["Kernel Name"][0]
            short = name.split("(")[0].replace("void ", "").replace("kifmm::gpu::", "").replace("tc::", "")
            print(f"| {label} | `{short[:48]}` | " + " | ".join(fmt(d, k) for _, k in COLS) + " |")


if __name__ == "__main__":
    main()
