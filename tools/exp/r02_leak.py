"""Plan create / evaluate / destroy in a loop: device and host memory must not grow."""
import os, sys
sys.path.insert(0, ".")
import numpy as np, torch, psutil
from paper_2303_08394_b200 import fmm, generators
torch.zeros(1, device="cuda")
proc = psutil.Process(os.getpid())
ops = {}
rows = []
for i in range(40):
    prec = 32 if i % 2 == 0 else 64
    kind = ["uniform-cube", "sphere-surface", "two-cluster"][i % 3]
    pos, q = generators.sample(kind, 100000, seed=i, charges="signed", fp32=prec == 32)
    with fmm.Fmm(pos, fmm.FmmConfig(p=6, n_crit=60, precision=prec, gradient=i % 4 < 2)) as f:
        f.evaluate(q)
        f.evaluate(q, timed=True)
    torch.cuda.synchronize()
    free, total = torch.cuda.mem_get_info()
    rows.append((i, (total - free) / 1e6, proc.memory_info().rss / 1e6))
    if i % 5 == 4:
        print("iter %d: device used %.1f MB, host rss %.1f MB" % rows[-1], flush=True)
d0, d1 = rows[9][1], rows[-1][1]
h0, h1 = rows[9][2], rows[-1][2]
print("device growth after warm-up: %.1f MB; host rss growth: %.1f MB" % (d1 - d0, h1 - h0))
