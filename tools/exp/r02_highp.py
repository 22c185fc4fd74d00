"""p = 8, 9, 10 on the any-width path: parity vs the oracle and accuracy vs direct summation."""
import json, sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2303_08394_b200 import fmm, generators
import oracle

def inv(t):
    i = np.empty_like(t.original_index); i[t.original_index] = np.arange(t.n); return i

cases = [("two-cluster", 3000, 30, 8, 64, 1e-12), ("uniform-cube", 4000, 60, 9, 64, 1e-12),
         ("sphere-surface", 4000, 60, 10, 64, 1e-12), ("uniform-cube", 4000, 60, 8, 32, 1e-8),
         ("two-cluster", 3000, 30, 10, 32, 1e-8)]
for kind, n, ncrit, p, prec, cut in cases:
    pos, q = generators.sample(kind, n, seed=5, charges="signed", fp32=prec == 32)
    t0 = time.time()
    with fmm.Fmm(pos, fmm.FmmConfig(p=p, n_crit=ncrit, precision=prec, svd_cutoff=cut, gradient=True)) as f:
        t1 = time.time()
        pot, grad, tm = f.evaluate(q, timed=True)
        pot2, grad2, _ = f.evaluate(q)
        qr = np.asarray(q, dtype=np.float64)[f.tree.original_index]
        phi, g, _ = oracle.evaluate(f.tree, f.operators, qr, gradient=True)
        ii = inv(f.tree)
        idx = np.arange(0, n, max(1, n // 500))
        d, dg = fmm.direct(pos, q, targets=idx, precision=64, gradient=True)
        print(json.dumps({"kind": kind, "n": n, "p": p, "precision": prec, "svd_cutoff": cut,
                          "backend": f.info()["m2l_backend"], "setup_s": round(t1 - t0, 2),
                          "eval_ms": round(tm["total_ms"], 3),
                          "pot_vs_oracle": fmm.relative_error(pot, phi[ii]),
                          "grad_vs_oracle": fmm.relative_error(grad, g[ii]),
                          "pot_vs_direct": fmm.relative_error(pot[idx], d),
                          "oracle_vs_direct": fmm.relative_error(phi[ii][idx], d),
                          "graph_equals_timed": bool(np.array_equal(pot, pot2) and np.array_equal(grad, grad2))}), flush=True)
