"""The concentrated blob of the mid-size randomised run (case 635): fp64 p = 6, int8 M2L vs DMMA M2L vs oracle."""
import json, sys
import numpy as np
sys.path.insert(0, ".")
from paper_2303_08394_b200 import fmm
import oracle
# replay the generator state of tools/exp/r02_fuzz_big.py is fragile; draw a similar blob instead
for seed in (1, 2, 3):
    rng = np.random.default_rng(seed)
    n = 100000
    pos = (0.5 + 0.1 * rng.standard_normal((n, 3)) * rng.random((n, 1)) ** 2) * 1e-3
    q = 2 * rng.random(n) - 1
    for backend in (4, 1):
        with fmm.Fmm(pos, fmm.FmmConfig(p=6, n_crit=300, precision=64, gradient=True, m2l_backend=backend)) as f:
            tree, ops = f.tree, f.operators
            qr = q[tree.original_index]
            pot, g, _ = f.evaluate(qr, input_order=False)
            M = oracle.upward_local(tree, ops, qr, 0, tree.n_leaves, 0)
            nl = tree.n_leaves; take = max(1, nl // 20)
            errs = []
            for lb in (0, (nl - take) // 2, nl - take):
                phi, gr = oracle.downward(tree, ops, qr, M, lb, lb + take, gradient=False)
                a, b = tree.leaf_ptr[lb], tree.leaf_ptr[lb + take]
                errs.append(fmm.relative_error(pot[a:b], phi[a:b]))
            # level-wise dynamic range of the multipole rows
            print(json.dumps({"seed": seed, "backend": backend, "depth": int(tree.depth), "leaves": int(nl), "errs": errs}), flush=True)
