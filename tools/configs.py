"""Run every BASELINE config once on the GPU: setup times, evaluate time (device-resident, CUDA
events, L2 flushed between steps; and the serialized per-phase run), error vs direct summation on
1000 sampled targets (potential and, where computed, gradient).  One JSON line per config.

usage: python tools/configs.py [config ids...]   (default 1 2 3 4 5)
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2303_08394_b200 import fmm, generators  # noqa: E402

which = [int(x) for x in sys.argv[1:]] or [1, 2, 3, 4, 5]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for cid in which:
    c = generators.CONFIGS[cid]
    t0 = time.time()
    pos, q = generators.config_sample(cid)
    t1 = time.time()
    cfg = fmm.FmmConfig(p=c["p"], n_crit=c["n_crit"], precision=c["precision"], gradient=c["gradient"])
    f = fmm.Fmm(pos, cfg)
    t2 = time.time()
    dt = np.float32 if c["precision"] == 32 else np.float64
    tdt = torch.float32 if c["precision"] == 32 else torch.float64
    qq = q.astype(dt)
    pot, g, tm = f.evaluate(qq, timed=True)
    # device-resident evaluate (the bench's `value` path) on an explicit stream
    n = len(q)
    dq = torch.from_numpy(qq).cuda()
    dpot = torch.empty(n, dtype=tdt, device="cuda")
    dgrad = torch.empty((n, 3), dtype=tdt, device="cuda") if c["gradient"] else None
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        def step():
            f.evaluate_device(dq.data_ptr(), dpot.data_ptr(), dgrad.data_ptr() if dgrad is not None else None,
                              input_order=True, stream=st.cuda_stream)
        for _ in range(3):
            step()
        ms = []
        for i in range(10):
            flush.fill_(float(i))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            step()
            b.record(st)
            b.synchronize()
            ms.append(a.elapsed_time(b))
    same = bool(np.array_equal(dpot.cpu().numpy(), pot))
    tg = (generators.uniform(99, 0, 1000) * n).astype(np.int64)
    d = fmm.direct(pos, q, targets=tg, precision=64, gradient=c["gradient"])
    dpot_ref, dgrad_ref = (d if c["gradient"] else (d, None))
    out = {"config": cid, "n": n, "precision": c["precision"], "p": c["p"], "n_crit": c["n_crit"],
           "gradient": c["gradient"], "gen_s": round(t1 - t0, 2), "plan_s": round(t2 - t1, 2),
           "setup_s": {k: round(v, 2) for k, v in f.timings.items()},
           "eval_ms_median": float(np.median(ms)), "eval_ms_min": float(np.min(ms)),
           "points_per_s": n / (float(np.median(ms)) * 1e-3),
           "device_path_equals_host_path": same,
           "err_vs_direct_1000": fmm.relative_error(pot[tg], dpot_ref),
           "leaves": f.tree.n_leaves, "depth": f.tree.depth, "lists": f.tree.list_stats(),
           "phases_serialized_ms": {k: round(v, 3) for k, v in tm.items()}}
    if c["gradient"]:
        out["grad_err_vs_direct_1000"] = fmm.relative_error(g[tg], dgrad_ref)
    info = f.info()
    out.update({"m2l_backend": info["m2l_backend"], "device_MB": info["device_bytes"] / 1e6})
    print(json.dumps(out), flush=True)
    f.close()
    del dq, dpot, dgrad
