"""fp32 accuracy vs tree depth: a uniform background plus a dense cluster of side `w` (depth grows as w shrinks)."""
import json, os, sys
import numpy as np
sys.path.insert(0, ".")
from paper_2303_08394_b200 import fmm
import oracle
rng = np.random.default_rng(3)
n = 20000
for w in (1e-1, 1e-2, 1e-3, 1e-4, 3e-5):
    a = rng.random((n // 2, 3))
    b = 0.3 + w * rng.random((n // 2, 3))
    pos = np.concatenate([a, b]).astype(np.float32).astype(np.float64)
    q = 2 * rng.random(n) - 1
    with fmm.Fmm(pos, fmm.FmmConfig(p=6, n_crit=30, precision=32, gradient=True)) as f:
        pot, g, _ = f.evaluate(q)
        qr = q[f.tree.original_index]
        phi, gr, _ = oracle.evaluate(f.tree, f.operators, qr, gradient=True)
        ii = np.empty_like(f.tree.original_index); ii[f.tree.original_index] = np.arange(f.tree.n)
        ref, gref = phi[ii], gr[ii]
        cl = slice(n // 2, n)
        print(json.dumps({"lib": os.environ.get("KIFMM_LIB", "default"), "cluster_side": w, "depth": int(f.tree.depth),
                          "pot_err": fmm.relative_error(pot, ref), "pot_err_cluster": fmm.relative_error(pot[cl], ref[cl]),
                          "pot_err_background": fmm.relative_error(pot[:n // 2], ref[:n // 2]),
                          "grad_err": fmm.relative_error(g, gref)}), flush=True)
