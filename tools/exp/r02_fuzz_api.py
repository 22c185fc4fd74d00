"""Randomised API check: evaluate_many (K vectors), evaluate_device on random user streams (back to back on different
streams), input / reordered output order, graph on / off -- every route bit-identical to evaluate()."""
import json, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2303_08394_b200 import fmm, generators
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 4)
t_end = time.time() + budget
ops = {}
case = fails = 0
while time.time() < t_end:
    case += 1
    prec = int(rng.choice([32, 64]))
    p = int(rng.choice([4, 5, 6, 7]))
    kind = str(rng.choice(["uniform-cube", "sphere-surface", "two-cluster"]))
    n = int(rng.integers(500, 60000))
    ncrit = int(rng.choice([10, 40, 150]))
    grad = bool(rng.integers(0, 2)); io = bool(rng.integers(0, 2)); graph = bool(rng.integers(0, 2))
    K = int(rng.integers(1, 6))
    seed = int(rng.integers(0, 1000))
    pos, _ = generators.sample(kind, n, seed=seed, charges="signed", fp32=prec == 32)
    rec = dict(case=case, kind=kind, n=n, n_crit=ncrit, p=p, precision=prec, gradient=grad, input_order=io, graph=graph, K=K)
    try:
        cut = 1e-8 if (prec == 32 and p == 7) else 1e-12
        with fmm.Fmm(pos, fmm.FmmConfig(p=p, n_crit=ncrit, precision=prec, gradient=grad, use_graph=graph, svd_cutoff=cut), operators=ops) as f:
            dt = f.dtype
            tdt = torch.float32 if prec == 32 else torch.float64
            Q = (2 * rng.random((K, n)) - 1).astype(dt)
            single = [f.evaluate(Q[k], input_order=io)[:2] for k in range(K)]
            many = f.evaluate_many(Q, input_order=io)
            ok = all(np.array_equal(many[0][k], single[k][0]) for k in range(K))
            if grad:
                ok = ok and all(np.array_equal(many[1][k], single[k][1]) for k in range(K))
            # device route: K evaluates back to back on alternating user streams
            streams = [torch.cuda.Stream(), torch.cuda.Stream()]
            dq = [torch.from_numpy(Q[k]).cuda() for k in range(K)]
            dp = [torch.empty(n, dtype=tdt, device="cuda") for _ in range(K)]
            dg = [torch.empty((n, 3), dtype=tdt, device="cuda") if grad else None for _ in range(K)]
            torch.cuda.synchronize()
            for k in range(K):
                st = streams[k % 2]
                f.evaluate_device(dq[k].data_ptr(), dp[k].data_ptr(), dg[k].data_ptr() if grad else None,
                                  input_order=io, stream=st.cuda_stream)
            torch.cuda.synchronize()
            ok_dev = all(np.array_equal(dp[k].cpu().numpy(), single[k][0]) for k in range(K))
            if grad:
                ok_dev = ok_dev and all(np.array_equal(dg[k].cpu().numpy(), single[k][1]) for k in range(K))
        rec.update(many_ok=bool(ok), device_ok=bool(ok_dev), ok=bool(ok and ok_dev))
    except Exception as e:  # noqa: BLE001
        rec.update(ok=False, error=repr(e)[:300])
    if not rec["ok"]:
        fails += 1
    if not rec["ok"] or case % 10 == 0:
        print(json.dumps(rec), flush=True)
    if len(ops) > 12:
        ops.clear()
print(json.dumps({"cases": case, "failures": fails}), flush=True)
sys.exit(1 if fails else 0)
