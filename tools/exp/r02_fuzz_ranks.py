"""Randomised multi-rank check: the product's rank plans (one-GPU emulation, host exchange) against the single-rank
evaluate, for random clouds, orders, world sizes, cut levels, precision, gradient and output order."""
import json, sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2303_08394_b200 import fmm, generators

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2)
t_end = time.time() + budget
ops_cache = {}
case = fails = 0
while time.time() < t_end:
    case += 1
    prec = int(rng.choice([32, 64]))
    p = int(rng.choice([3, 4, 5, 6, 7])) if prec == 64 else int(rng.choice([3, 4, 5, 6]))
    kind = str(rng.choice(["uniform-cube", "sphere-surface", "two-cluster"]))
    n = int(rng.integers(2000, 40000))
    ncrit = int(rng.choice([10, 30, 64, 150]))
    world = int(rng.choice([2, 3, 4, 5, 8]))
    cut = int(rng.choice([0, 0, 2, 3]))
    grad = bool(rng.integers(0, 2))
    io = bool(rng.integers(0, 2))
    seed = int(rng.integers(0, 1000))
    pos, q = generators.sample(kind, n, seed=seed, charges="signed", fp32=prec == 32)
    rec = {"case": case, "kind": kind, "n": n, "n_crit": ncrit, "p": p, "precision": prec, "gradient": grad,
           "world": world, "cut_level": cut, "input_order": io, "seed": seed}
    try:
        kw = dict(p=p, n_crit=ncrit, precision=prec, gradient=grad)
        with fmm.Fmm(pos, fmm.FmmConfig(**kw), operators=ops_cache) as f:
            dt = f.dtype
            qq = (q if io else q[f.tree.original_index]).astype(dt)
            pot1, grad1, _ = f.evaluate(qq, input_order=io)
            tree, ops = f.tree, f.operators
        plans = [fmm.Fmm(pos, fmm.FmmConfig(**kw, rank=r, world_size=world, exchange=1, cut_level=cut), operators=ops,
                         tree=tree) for r in range(world)]
        try:
            info = [pl.info() for pl in plans]
            sends = [pl.evaluate_upward(qq, input_order=io) for pl in plans]
            hm = info[0]["halo_rows_max"]
            gathered = np.zeros((world, max(1, hm), info[0]["ne_pad"]), dtype=dt)
            for r, s in enumerate(sends):
                gathered[r, :s.shape[0]] = s
            outs = [pl.evaluate_downward(gathered) for pl in plans]
        finally:
            for pl in plans:
                pl.close()
        pot = np.sum([o[0] for o in outs], axis=0)
        same = 1e-13 if prec == 64 else 2e-6
        ep = fmm.relative_error(pot, pot1)
        eg = 0.0
        if grad:
            eg = fmm.relative_error(np.sum([o[1] for o in outs], axis=0), grad1)
        owned = sum(i["owned_particle_end"] - i["owned_particle_begin"] for i in info)
        ok = ep <= same and eg <= 10 * same and owned == n
        rec.update(pot_diff=ep, grad_diff=eg, halo_rows_max=int(hm), ok=bool(ok))
    except Exception as e:  # noqa: BLE001
        rec.update(ok=False, error=repr(e)[:300])
    if not rec["ok"]:
        fails += 1
    if not rec["ok"] or case % 10 == 0:
        print(json.dumps(rec), flush=True)
    if len(ops_cache) > 16:
        ops_cache.clear()
print(json.dumps({"cases": case, "failures": fails}), flush=True)
sys.exit(1 if fails else 0)
