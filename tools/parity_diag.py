"""Diagnostics of the fp32 GPU-vs-oracle error at a BASELINE config: the same oracle samples as
tests/test_gpu_configs.py, evaluated with each M2L / GEMM backend variant (env switches), plus the oracle's
own error vs fp64 direct summation on the sampled targets.

usage: python tools/parity_diag.py CONFIG [variant ...]   variants: default simt tcgemm0 tf32
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2303_08394_b200 import fmm, generators  # noqa: E402

cid = int(sys.argv[1])
variants = sys.argv[2:] or ["default", "simt", "tcgemm0", "tf32"]
FRACTION = {1: 0.2, 2: 0.01, 3: 0.01, 4: 0.004, 5: 0.001}
c = generators.CONFIGS[cid]
pos, q = generators.config_sample(cid)
ref = None
for v in variants:
    env = {"default": {}, "simt": {}, "tcgemm0": {"KIFMM_TC_GEMM": "0"}, "tf32": {"KIFMM_TC_KIND": "tf32"}}[v]
    for k in ("KIFMM_TC_GEMM", "KIFMM_TC_KIND"):
        os.environ.pop(k, None)
    os.environ.update(env)
    cfg = fmm.FmmConfig(p=c["p"], n_crit=c["n_crit"], precision=32, gradient=c["gradient"],
                        m2l_backend=1 if v == "simt" else 0)
    with fmm.Fmm(pos, cfg) as f:
        t, o = f.tree, f.operators
        qr = q[t.original_index]
        pot, grad, _ = f.evaluate(qr.astype(np.float32), input_order=False)
        backend = f.info()["m2l_backend"]
        if ref is None:
            M = oracle.upward_local(t, o, qr, 0, t.n_leaves, 0)
            take = max(1, int(t.n_leaves * FRACTION[cid]))
            rng = [(s, s + take) for s in (0, (t.n_leaves - take) // 2, t.n_leaves - take)]
            sel = np.concatenate([np.arange(t.leaf_ptr[a], t.leaf_ptr[b]) for a, b in rng])
            rp, rg = np.zeros(t.n), np.zeros((t.n, 3))
            for a, b in rng:
                phi, g = oracle.downward(t, o, qr, M, a, b, gradient=c["gradient"])
                rp[t.leaf_ptr[a]:t.leaf_ptr[b]] = phi[t.leaf_ptr[a]:t.leaf_ptr[b]]
                if c["gradient"]:
                    rg[t.leaf_ptr[a]:t.leaf_ptr[b]] = g[t.leaf_ptr[a]:t.leaf_ptr[b]]
            # oracle vs fp64 direct on 300 of the sampled targets
            sub = sel[:: max(1, sel.size // 300)]
            d = fmm.direct(t.positions, qr, targets=sub, precision=64, gradient=c["gradient"])
            dp, dg = d if c["gradient"] else (d, None)
            ref = dict(oracle_vs_direct=fmm.relative_error(rp[sub], dp),
                       oracle_grad_vs_direct=fmm.relative_error(rg[sub], dg) if c["gradient"] else None)
            print(json.dumps({"config": cid, **ref}), flush=True)
        # per-target relative error distribution
        e = np.abs(pot[sel] - rp[sel]) / np.abs(rp[sel]).max()
        rec = {"config": cid, "variant": v, "backend": backend,
               "pot_rel_l2": fmm.relative_error(pot[sel], rp[sel]),
               "pot_err_p50_p99_max_over_maxabs": [float(np.percentile(e, 50)), float(np.percentile(e, 99)), float(e.max())],
               "pot_vs_direct": fmm.relative_error(pot[sub], dp)}
        if c["gradient"]:
            rec["grad_rel_l2"] = fmm.relative_error(grad[sel], rg[sel])
        print(json.dumps(rec), flush=True)
