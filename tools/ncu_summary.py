"""Summarise ncu reports into profiles/ (run here, no GPU needed).

usage: python tools/ncu_summary.py name=report.ncu-rep[:i,j,...] [...] > profiles/<round>_ncu_summary.md
(name1,name2=report picks the report's kernels in order; default: the first kernel only)
Writes/updates profiles/ncu_summary.json with per-kernel figures used by bench.py.
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_tex.sum",
        "lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fma.sum", "sm__inst_executed_pipe_xu.sum", "sm__cycles_elapsed.avg.per_second",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for k, u, v in zip(hdr, units, r):
            m = re.search(r"[a-z0-9]+__[A-Za-z0-9_.]+$", k)
            k = m.group(0) if m else k
            if k in KEYS or k == "Kernel Name":
                d[k] = (v, u)
        res.append(d)
    return res


def to_bytes(v, u):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def main():
    js_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_summary.json")
    js = json.load(open(js_path)) if os.path.exists(js_path) else {}
    print("| kernel | name | duration | DRAM read+write / launch | tensor pipe % | SM thru % | L2 sectors % | regs |")
    print("|---|---|---|---|---|---|---|---|")
    for arg in sys.argv[1:]:
        names, path = arg.split("=", 1)
        names = names.split(",")
        for name, d in zip(names, raw(path)):
            dur = d.get("gpu__time_duration.sum", ("0", ""))
            rb = to_bytes(*d.get("dram__bytes_read.sum", ("0", "byte")))
            wb = to_bytes(*d.get("dram__bytes_write.sum", ("0", "byte")))
            g = lambda k: d.get(k, ("", ""))[0]  # noqa: E731
            print(f"| {name} | {d['Kernel Name'][0][:60]} | {dur[0]} {dur[1]} | {(rb + wb) / 1e6:.1f} MB | "
                  f"{g('sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed')} | "
                  f"{g('sm__throughput.avg.pct_of_peak_sustained_elapsed')} | "
                  f"{g('lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed')} | "
                  f"{g('launch__registers_per_thread')} |")
            js[name] = {"kernel": d["Kernel Name"][0], "duration": dur[0] + " " + dur[1],
                        "dram_bytes_per_launch": rb + wb, "source": os.path.basename(path),
                        **{k: g(k) for k in KEYS if g(k)}}
    json.dump(js, open(js_path, "w"), indent=1)


if __name__ == "__main__":
    main()
