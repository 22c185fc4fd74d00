"""Summarise an `ncu --page source --csv --print-source sass` export: per kernel, stall-reason totals and
the hottest SASS lines.  usage: python tools/ncu_src.py export.csv [top]"""
import csv
import sys
from collections import Counter

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
i = 0
while i < len(rows):
    r = rows[i]
    if r and r[0] == "Kernel Name":
        name = r[1]
        hdr = rows[i + 1]
        j = i + 2
        body = []
        while j < len(rows) and rows[j] and rows[j][0] != "Kernel Name":
            body.append(dict(zip(hdr, rows[j])))
            j += 1
        stalls = Counter()
        tot = 0
        for b in body:
            tot += int(b.get("Warp Stall Sampling (All Samples)", "0") or 0)
            for k, v in b.items():
                if k.startswith("stall_") and "(Not Issued)" not in k and v not in ("", "-"):
                    stalls[k] += int(v)
        print(f"== {name[:110]}\n   samples {tot}; stalls: " +
              ", ".join(f"{k[6:]} {100 * v / max(tot, 1):.1f}%" for k, v in stalls.most_common(8)))
        hot = sorted(body, key=lambda b: -int(b.get("Warp Stall Sampling (All Samples)", "0") or 0))[:top]
        for b in hot:
            s = int(b.get("Warp Stall Sampling (All Samples)", "0") or 0)
            top3 = sorted(((int(v), k[6:]) for k, v in b.items() if k.startswith("stall_") and "(Not" not in k
                           and v not in ("", "-") and int(v) > 0), reverse=True)[:3]
            print(f"   {100 * s / max(tot, 1):5.1f}%  {b['Address'][-5:]}  {b['Source'].strip()[:60]:60s} {top3}")
        i = j
    else:
        i += 1
