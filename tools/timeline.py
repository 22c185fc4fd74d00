"""Experiments: per-kernel-class timeline of one captured evaluate (build with -DKIFMM_TIMELINE_PROBES,
e.g. tools/build_variant.sh tl -DKIFMM_TIMELINE_PROBES; run with KIFMM_LIB=variants/tl.so KIFMM_TIMELINE=1
KIFMM_NEAR_DEBUG=1).  The library prints the timeline to stderr after each evaluate."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2303_08394_b200 import fmm, generators  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = generators.CONFIGS[cfg_id]
pos, q = generators.config_sample(cfg_id)
f = fmm.Fmm(pos, fmm.FmmConfig(p=c["p"], n_crit=c["n_crit"], precision=c["precision"], gradient=c["gradient"]))
qq = q.astype(np.float32 if c["precision"] == 32 else np.float64)
for i in range(4):
    print(f"--- evaluate {i}", file=sys.stderr, flush=True)
    f.evaluate(qq)
