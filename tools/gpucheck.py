import sys, time, numpy as np
sys.path.insert(0, '.')
import oracle
from paper_2303_08394_b200 import fmm, generators
def inv(t):
    i = np.empty_like(t.original_index); i[t.original_index] = np.arange(t.n); return i
for kind, n, p, ncrit in [("uniform-cube", 5000, 6, 50), ("sphere-surface", 5000, 6, 50), ("two-cluster", 5000, 6, 30), ("uniform-cube", 3000, 4, 20)]:
    pos, q = generators.sample(kind, n, seed=1, charges="signed", fp32=True)
    for prec in (64, 32):
        cfg = fmm.FmmConfig(p=p, n_crit=ncrit, precision=prec, gradient=True, m2l_backend=1)
        f = fmm.Fmm(pos, cfg)
        pot, g, tm = f.evaluate(q, timed=True)
        qr = q[f.tree.original_index]
        ref, gref, _ = oracle.evaluate(f.tree, f.operators, qr, gradient=True)
        ii = inv(f.tree)
        d = oracle.direct(pos, q)
        print(kind, n, p, prec, "vs oracle", fmm.relative_error(pot, ref[ii]), "grad", fmm.relative_error(g, gref[ii]), "oracle vs direct", fmm.relative_error(ref[ii], d), flush=True)
        f.close()
