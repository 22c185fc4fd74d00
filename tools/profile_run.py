"""Minimal driver for ncu: build the config-2 plan and run a few evaluates."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2303_08394_b200 import fmm, generators  # noqa: E402

cfg_id = int(os.environ.get("KIFMM_CFG", "2"))
backend = int(os.environ.get("KIFMM_M2L", "0"))
c = generators.CONFIGS[cfg_id]
pos, q = generators.config_sample(cfg_id)
f = fmm.Fmm(pos, fmm.FmmConfig(p=c["p"], n_crit=c["n_crit"], precision=c["precision"], gradient=c["gradient"],
                               m2l_backend=backend))
qq = q.astype(np.float32 if c["precision"] == 32 else np.float64)
for _ in range(int(os.environ.get("KIFMM_ITERS", "2"))):
    pot, g, tm = f.evaluate(qq, timed=True)
print(tm)
print(f.info())
