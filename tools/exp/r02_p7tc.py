"""fp32 p = 7: tcgen05 M2L (row width 224, 2-CTA pair) against the SIMT M2L -- parity and time."""
import json, sys
import numpy as np
sys.path.insert(0, ".")
from paper_2303_08394_b200 import fmm, generators
import oracle
def inv(t):
    i = np.empty_like(t.original_index); i[t.original_index] = np.arange(t.n); return i
for kind, n, ncrit in [("two-cluster", 4000, 8), ("uniform-cube", 20000, 60), ("sphere-surface", 200000, 100), ("uniform-cube", 1000000, 150)]:
    pos, q = generators.sample(kind, n, seed=7, charges="signed", fp32=True)
    for backend in (1, 0):
        with fmm.Fmm(pos, fmm.FmmConfig(p=7, n_crit=ncrit, precision=32, svd_cutoff=1e-8, gradient=True, m2l_backend=backend)) as f:
            pot, grad, tm = f.evaluate(q, timed=True)
            pot, grad, tm = f.evaluate(q, timed=True)
            rec = {"kind": kind, "n": n, "backend": f.info()["m2l_backend"], "total_ms": round(tm["total_ms"], 3), "m2l_ms": round(tm["m2l_ms"], 3)}
            if n <= 200000:
                qr = np.asarray(q, dtype=np.float64)[f.tree.original_index]
                phi, g, _ = oracle.evaluate(f.tree, f.operators, qr, gradient=True)
                ii = inv(f.tree)
                rec["pot_vs_oracle"] = fmm.relative_error(pot, phi[ii]); rec["grad_vs_oracle"] = fmm.relative_error(grad, g[ii])
            idx = np.arange(0, n, max(1, n // 1000))
            rec["pot_vs_direct"] = fmm.relative_error(pot[idx], fmm.direct(pos, q, targets=idx, precision=64))
            print(json.dumps(rec), flush=True)
