"""fp32 at p = 7: parity vs the oracle (same operators) and error vs direct summation as a function of the SVD cutoff."""
import json, sys
import numpy as np
sys.path.insert(0, ".")
from paper_2303_08394_b200 import fmm, generators
import oracle

def inv(t):
    i = np.empty_like(t.original_index); i[t.original_index] = np.arange(t.n); return i

for kind, n, ncrit in [("two-cluster", 4000, 8), ("uniform-cube", 20000, 60)]:
    pos, q = generators.sample(kind, n, seed=7, charges="signed", fp32=True)
    for p in (6, 7):
        for cut in (1e-12, 1e-10, 1e-8, 1e-7, 1e-6, 1e-5):
            with fmm.Fmm(pos, fmm.FmmConfig(p=p, n_crit=ncrit, precision=32, svd_cutoff=cut)) as f:
                pot, _, _ = f.evaluate(q)
                qr = np.asarray(q, dtype=np.float64)[f.tree.original_index]
                phi, _, _ = oracle.evaluate(f.tree, f.operators, qr, gradient=False)
                ref = phi[inv(f.tree)]
                idx = np.arange(0, n, max(1, n // 1000))
            d = fmm.direct(pos, q, targets=idx, precision=64)
            rec = {"kind": kind, "p": p, "cutoff": cut, "vs_oracle": fmm.relative_error(pot, ref)}
            if d is not None:
                rec["gpu_vs_direct"] = fmm.relative_error(pot[idx], d)
                rec["oracle_vs_direct"] = fmm.relative_error(ref[idx], d)
            print(json.dumps(rec), flush=True)
