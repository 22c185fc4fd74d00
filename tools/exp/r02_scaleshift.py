"""Domains away from the unit cube: scaled and shifted clouds, fp32 and fp64, against the oracle."""
import json, sys
import numpy as np
sys.path.insert(0, ".")
from paper_2303_08394_b200 import fmm, generators
import oracle
for prec in (32, 64):
    for scale, shift in [(1.0, 0.0), (1e-4, 0.0), (1e4, 0.0), (1.0, 100.0), (1.0, -1000.0), (1e3, 5e4), (1e-3, 1.0)]:
        pos, q = generators.sample("two-cluster", 20000, seed=4, charges="signed")
        pos = pos * scale + shift
        if prec == 32:
            pos = pos.astype(np.float32).astype(np.float64)
        try:
            with fmm.Fmm(pos, fmm.FmmConfig(p=6, n_crit=40, precision=prec, gradient=True)) as f:
                pot, g, _ = f.evaluate(q)
                qr = q[f.tree.original_index]
                phi, gr, _ = oracle.evaluate(f.tree, f.operators, qr, gradient=True)
                ii = np.empty_like(f.tree.original_index); ii[f.tree.original_index] = np.arange(f.tree.n)
                print(json.dumps({"precision": prec, "scale": scale, "shift": shift, "depth": int(f.tree.depth),
                                  "pot_err": fmm.relative_error(pot, phi[ii]), "grad_err": fmm.relative_error(g, gr[ii])}), flush=True)
        except Exception as e:
            print(json.dumps({"precision": prec, "scale": scale, "shift": shift, "error": repr(e)[:200]}), flush=True)
