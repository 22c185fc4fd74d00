import os, sys, numpy as np
sys.path.insert(0, '.')
import oracle
from paper_2303_08394_b200 import fmm, generators
cases = [("uniform-cube", 100000, 100), ("two-cluster", 20000, 30)]
if len(sys.argv) > 1 and sys.argv[1] == "big":
    cases = [("uniform-cube", 1000000, 150)]
modes = [("tmem", "0", "64"), ("tmem", "1", "64"), ("smem", "0", "128"), ("smem", "1", "128")]
for kind, n, ncrit in cases:
    pos, q = generators.sample(kind, n, seed=2, charges="signed", fp32=True)
    ref = None
    for amode, pair, rowb in modes:
        os.environ["KIFMM_TC_AMODE"] = amode
        os.environ["KIFMM_TC_PAIR"] = pair
        os.environ["KIFMM_TC_ROWB"] = rowb
        f = fmm.Fmm(pos, fmm.FmmConfig(p=6, n_crit=ncrit, precision=32, m2l_backend=2))
        pot, _, tm = f.evaluate(q, timed=True)
        ms = [f.evaluate(q, timed=True)[2]["m2l_ms"] for _ in range(3)]
        if ref is None:
            r, _, _ = oracle.evaluate(f.tree, f.operators, q[f.tree.original_index])
            ii = np.empty_like(f.tree.original_index); ii[f.tree.original_index] = np.arange(f.tree.n)
            ref = r[ii]
        print(kind, n, amode, "pair", pair, "rowb", rowb, "err", fmm.relative_error(pot, ref), "m2l ms", min(ms), "total", tm["total_ms"], flush=True)
        f.close()
