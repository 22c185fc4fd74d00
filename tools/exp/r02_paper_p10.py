"""The paper's p = 10 setup (~1e6 points on a sphere surface, n_crit = 150, p = 10), fp64."""
import json, sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2303_08394_b200 import fmm, generators
pos, q = generators.sample("sphere-surface", 1000000, seed=0, charges="signed")
t0 = time.time()
with fmm.Fmm(pos, fmm.FmmConfig(p=10, n_crit=150, precision=64)) as f:
    t1 = time.time()
    pot, _, tm = f.evaluate(q, timed=True)
    pot, _, tm = f.evaluate(q, timed=True)
    idx = np.arange(0, len(q), 1000)
    d = fmm.direct(pos, q, targets=idx, precision=64)
    print(json.dumps({"setup": f.timings, "setup_total_s": round(t1 - t0, 2), "phases_ms": tm, "leaves": f.tree.n_leaves,
                      "err_vs_direct_1000": fmm.relative_error(pot[idx], d), "device_MB": f.info()["device_bytes"] / 1e6}))
