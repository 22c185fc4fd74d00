"""Run every BASELINE config once on the GPU: plan time, evaluate time, error vs direct on 1000 targets."""
import os, sys, time, json, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_08394_b200 import fmm, generators
which = [int(x) for x in sys.argv[1:]] or [1, 2, 3, 4, 5]
for cid in which:
    c = generators.CONFIGS[cid]
    t0 = time.time()
    pos, q = generators.config_sample(cid)
    t1 = time.time()
    cfg = fmm.FmmConfig(p=c["p"], n_crit=c["n_crit"], precision=c["precision"], gradient=c["gradient"])
    f = fmm.Fmm(pos, cfg)
    t2 = time.time()
    dt = np.float32 if c["precision"] == 32 else np.float64
    qq = q.astype(dt)
    pot, g, tm = f.evaluate(qq, timed=True)
    tms = [f.evaluate(qq, timed=True)[2]["total_ms"] for _ in range(3)]
    tg = (generators.uniform(99, 0, 1000) * len(q)).astype(np.int64)
    d = fmm.direct(pos, q, targets=tg, precision=64)
    info = f.info()
    print(json.dumps({"config": cid, "n": len(q), "gen_s": round(t1 - t0, 2), "setup_s": {k: round(v, 2) for k, v in f.timings.items()},
                      "eval_ms": min(tms), "points_per_s": len(q) / (min(tms) * 1e-3),
                      "err_vs_direct_1000": fmm.relative_error(pot[tg], d), "leaves": f.tree.n_leaves, "depth": f.tree.depth,
                      "lists": f.tree.list_stats(), "phases": {k: round(v, 3) for k, v in tm.items()},
                      "m2l_backend": info["m2l_backend"], "device_MB": info["device_bytes"] / 1e6}), flush=True)
    f.close()
