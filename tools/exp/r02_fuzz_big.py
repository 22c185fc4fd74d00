"""Randomised mid-size check (50 k - 400 k points: 2-CTA pair kernels, queue-mode near field, chunked far works)
against the oracle on three leaf ranges (full upward pass, downward pass for the sampled leaves)."""
import json, sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2303_08394_b200 import fmm, generators
import oracle
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
t_end = time.time() + budget
ops_cache = {}
case = fails = 0
while time.time() < t_end:
    case += 1
    prec = int(rng.choice([32, 32, 64]))
    p = int(rng.choice([4, 5, 6, 7])) if prec == 32 else int(rng.choice([5, 6, 7, 8]))
    kind = str(rng.choice(["uniform-cube", "sphere-surface", "two-cluster", "blob"]))
    n = int(rng.integers(50000, 400000 if prec == 32 else 150000))
    ncrit = int(rng.choice([20, 40, 64, 150, 300]))
    grad = bool(rng.integers(0, 2))
    seed = int(rng.integers(0, 1000))
    if kind == "blob":
        pos = 0.5 + 0.1 * rng.standard_normal((n, 3)) * rng.random((n, 1)) ** 2
        q = 2 * rng.random(n) - 1
        if prec == 32:
            pos = pos.astype(np.float32).astype(np.float64)
    else:
        pos, q = generators.sample(kind, n, seed=seed, charges="signed", fp32=prec == 32)
    scale = float(rng.choice([1.0, 1.0, 1e-3, 50.0]))
    pos = pos * scale
    if prec == 32:
        pos = pos.astype(np.float32).astype(np.float64)
    cut = 1e-12 if prec == 64 or p < 7 else 1e-8
    rec = {"case": case, "kind": kind, "n": n, "n_crit": ncrit, "p": p, "precision": prec, "gradient": grad, "seed": seed, "scale": scale}
    try:
        with fmm.Fmm(pos, fmm.FmmConfig(p=p, n_crit=ncrit, precision=prec, gradient=grad, svd_cutoff=cut), operators=ops_cache) as f:
            tree, ops = f.tree, f.operators
            qr = q[tree.original_index]
            pot, g, _ = f.evaluate(qr.astype(f.dtype), input_order=False)
            pot_in, g_in, _ = f.evaluate(q.astype(f.dtype), input_order=True)
            rec.update(backend=f.info()["m2l_backend"], leaves=int(tree.n_leaves), depth=int(tree.depth))
        perm_ok = bool(np.array_equal(pot_in[tree.original_index], pot))
        M = oracle.upward_local(tree, ops, qr, 0, tree.n_leaves, 0)
        nl = tree.n_leaves
        take = max(1, int(nl * 0.01))
        rp, gp_, rg, gg_ = [], [], [], []
        for lb in (0, (nl - take) // 2, nl - take):
            phi, gr = oracle.downward(tree, ops, qr, M, lb, lb + take, gradient=grad)
            a, b = tree.leaf_ptr[lb], tree.leaf_ptr[lb + take]
            rp.append(phi[a:b]); gp_.append(pot[a:b])
            if grad:
                rg.append(gr[a:b]); gg_.append(g[a:b])
        ep = fmm.relative_error(np.concatenate(gp_), np.concatenate(rp))
        eg = fmm.relative_error(np.concatenate(gg_), np.concatenate(rg)) if grad else 0.0
        tp, tg = (1e-12, 1e-11) if prec == 64 else (1e-5, 5e-5)
        ok = perm_ok and ep <= tp and eg <= tg
        rec.update(pot_err=ep, grad_err=eg, perm_ok=perm_ok, ok=bool(ok))
    except Exception as e:  # noqa: BLE001
        rec.update(ok=False, error=repr(e)[:300])
    if not rec["ok"]:
        fails += 1
    print(json.dumps(rec), flush=True)
    if len(ops_cache) > 8:
        ops_cache.clear()
print(json.dumps({"cases": case, "failures": fails}), flush=True)
sys.exit(1 if fails else 0)
