import os, sys, numpy as np
sys.path.insert(0, '.')
import oracle
from paper_2303_08394_b200 import fmm, generators
pos, q = generators.sample("uniform-cube", 100000, seed=2, charges="signed", fp32=True)
ref = None
for chunk in ["1", "4", "16", "64", "1000"]:
    os.environ["KIFMM_TC_CHUNK"] = chunk
    f = fmm.Fmm(pos, fmm.FmmConfig(p=6, n_crit=100, precision=32, gradient=False, m2l_backend=2))
    pot, _, tm = f.evaluate(q, timed=True)
    if ref is None:
        qr = q[f.tree.original_index]
        r, _, _ = oracle.evaluate(f.tree, f.operators, qr)
        ii = np.empty_like(f.tree.original_index); ii[f.tree.original_index] = np.arange(f.tree.n)
        ref = r[ii]
    print("chunk", chunk, "err", fmm.relative_error(pot, ref), "m2l ms", tm["m2l_ms"], flush=True)
    f.close()
