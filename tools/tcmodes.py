import os, sys, numpy as np
sys.path.insert(0, '.')
import oracle
from paper_2303_08394_b200 import fmm, generators
cases = [("uniform-cube", 100000, 100), ("two-cluster", 20000, 30), ("sphere-surface", 100000, 60)]
if len(sys.argv) > 1 and sys.argv[1] == "big":
    cases = [("uniform-cube", 1000000, 150)]
modes = [("tf32", "0"), ("tf32", "1"), ("f16", "0"), ("f16", "1")]
for kind, n, ncrit in cases:
    pos, q = generators.sample(kind, n, seed=2, charges="signed", fp32=True)
    ref = None
    for k, pair in modes:
        os.environ["KIFMM_TC_KIND"] = k
        os.environ["KIFMM_TC_PAIR"] = pair
        f = fmm.Fmm(pos, fmm.FmmConfig(p=6, n_crit=ncrit, precision=32, gradient=True, m2l_backend=2))
        pot, g, tm = f.evaluate(q, timed=True)
        ms = [f.evaluate(q, timed=True)[2]["m2l_ms"] for _ in range(3)]
        if ref is None:
            r, rg, _ = oracle.evaluate(f.tree, f.operators, q[f.tree.original_index], gradient=True)
            ii = np.empty_like(f.tree.original_index); ii[f.tree.original_index] = np.arange(f.tree.n)
            ref, gref = r[ii], rg[ii]
        print(kind, n, k, "pair", pair, "err", fmm.relative_error(pot, ref), "gerr", fmm.relative_error(g, gref), "m2l ms", min(ms), "total", tm["total_ms"], flush=True)
        f.close()
