import os, sys, numpy as np
sys.path.insert(0, '.')
from paper_2303_08394_b200 import fmm, generators
pos, q = generators.config_sample(2)
for pair in ("0", "1"):
    for chunk in ["24", "48", "98", "200", "400"]:
        os.environ["KIFMM_TC_CHUNK"] = chunk; os.environ["KIFMM_TC_PAIR"] = pair
        f = fmm.Fmm(pos, fmm.FmmConfig(p=6, n_crit=150, precision=32, gradient=True, m2l_backend=2))
        ms = [f.evaluate(q, timed=True)[2]["m2l_ms"] for _ in range(4)]
        print("pair", pair, "chunk", chunk, "m2l ms", min(ms), flush=True)
        f.close()
