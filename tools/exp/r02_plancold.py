"""Cold vs warm plan creation in one process (KIFMM_PLAN_TIMING prints the phases)."""
import os, sys, time
os.environ["KIFMM_PLAN_TIMING"] = "1"
sys.path.insert(0, ".")
import torch
torch.zeros(1, device="cuda")
from paper_2303_08394_b200 import fmm, generators
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = generators.CONFIGS[cid]
pos, q = generators.config_sample(cid)
cfg = fmm.FmmConfig(p=c["p"], n_crit=c["n_crit"], precision=c["precision"], gradient=c["gradient"])
for i in range(3):
    t0 = time.perf_counter()
    f = fmm.Fmm(pos, cfg)
    t1 = time.perf_counter()
    f.evaluate(q.astype("float32" if c["precision"] == 32 else "float64"))
    t2 = time.perf_counter()
    print(f"== creation {i}: Fmm() {t1 - t0:.3f} s {f.timings}  first evaluate {t2 - t1:.3f} s", flush=True)
    f.close()
