import sys, time, numpy as np
sys.path.insert(0, '.')
import oracle
from paper_2303_08394_b200 import fmm, generators
def inv(t):
    i = np.empty_like(t.original_index); i[t.original_index] = np.arange(t.n); return i
for kind, n, ncrit in [("uniform-cube", 5000, 50), ("two-cluster", 8000, 30), ("sphere-surface", 20000, 50), ("uniform-cube", 100000, 100)]:
    pos, q = generators.sample(kind, n, seed=2, charges="signed", fp32=True)
    res = {}
    for be in (1, 2):
        cfg = fmm.FmmConfig(p=6, n_crit=ncrit, precision=32, gradient=True, m2l_backend=be)
        f = fmm.Fmm(pos, cfg)
        pot, g, tm = f.evaluate(q, timed=True)
        res[be] = (pot, g, tm['m2l_ms'], f.info()['m2l_backend'])
        if be == 2:
            qr = q[f.tree.original_index]
            ref, gref, _ = oracle.evaluate(f.tree, f.operators, qr, gradient=True)
            ii = inv(f.tree)
        f.close()
    print(kind, n, "backend", res[2][3], "tc vs oracle", fmm.relative_error(res[2][0], ref[ii]), "grad", fmm.relative_error(res[2][1], gref[ii]),
          "simt vs oracle", fmm.relative_error(res[1][0], ref[ii]), "tc vs simt", fmm.relative_error(res[2][0], res[1][0]), "m2l ms simt/tc", res[1][2], res[2][2], flush=True)
