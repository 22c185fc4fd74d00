"""Experiments: time one config's evaluate (device-resident, L2 flushed, CUDA events) and its phases.

usage: KIFMM_LIB=variants/x.so python tools/near_time.py [cfg] [steps]  -> one JSON line
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2303_08394_b200 import fmm, generators  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
c = generators.CONFIGS[cfg_id]
pos, q = generators.config_sample(cfg_id)
ndt = np.float32 if c["precision"] == 32 else np.float64
tdt = torch.float32 if c["precision"] == 32 else torch.float64
f = fmm.Fmm(pos, fmm.FmmConfig(p=c["p"], n_crit=c["n_crit"], precision=c["precision"], gradient=c["gradient"],
                               m2l_backend=int(os.environ.get("KIFMM_M2L_BACKEND", "0"))))
n = len(q)
dq = torch.from_numpy(q.astype(ndt)).cuda()
dpot = torch.empty(n, dtype=tdt, device="cuda")
dgrad = torch.empty((n, 3), dtype=tdt, device="cuda") if c["gradient"] else None
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)


def step():
    f.evaluate_device(dq.data_ptr(), dpot.data_ptr(), dgrad.data_ptr() if dgrad is not None else None,
                      input_order=True, stream=stream.cuda_stream)


for _ in range(5):
    step()
ms = []
for i in range(steps):
    flush.fill_(float(i))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    step()
    b.record(stream)
    b.synchronize()
    ms.append(a.elapsed_time(b))
ph = []
for _ in range(10):
    ph.append(f.evaluate(q.astype(ndt), timed=True)[2])
out = {"lib": os.environ.get("KIFMM_LIB", "default"), "cfg": cfg_id, "ms_median": float(np.median(ms)),
       "ms_min": float(np.min(ms))}
out.update({k: round(float(np.median([p[k] for p in ph])), 4) for k in ph[0] if k.endswith("_ms")})
print(json.dumps(out))
