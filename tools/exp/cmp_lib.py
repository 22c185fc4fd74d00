"""Experiments: evaluate a config with the library in KIFMM_LIB and compare with a saved reference output.
usage: KIFMM_LIB=variants/x.so python tools/exp/cmp_lib.py cfg save|check /tmp/ref.npz"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

from paper_2303_08394_b200 import fmm, generators  # noqa: E402

cfg_id, mode, path = int(sys.argv[1]), sys.argv[2], sys.argv[3]
c = generators.CONFIGS[cfg_id]
pos, q = generators.config_sample(cfg_id)
with fmm.Fmm(pos, fmm.FmmConfig(p=c["p"], n_crit=c["n_crit"], precision=c["precision"], gradient=c["gradient"])) as f:
    qq = q.astype(f.dtype)
    f.evaluate(qq)
    pot, grad, _ = f.evaluate(qq)
if mode == "save":
    np.savez(path, pot=pot, grad=grad if grad is not None else np.zeros(1))
else:
    z = np.load(path)
    e = float(np.linalg.norm(pot - z["pot"]) / np.linalg.norm(z["pot"]))
    eg = float(np.linalg.norm(grad - z["grad"]) / np.linalg.norm(z["grad"])) if grad is not None else 0.0
    print(f"cmp {os.environ.get('KIFMM_LIB')} cfg {cfg_id}: rel pot {e:.3e} grad {eg:.3e} bitexact {np.array_equal(pot, z['pot'])}")
