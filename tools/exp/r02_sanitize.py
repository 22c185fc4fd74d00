"""Small evaluates for compute-sanitizer (memcheck / initcheck / synccheck): every kernel family once."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2303_08394_b200 import fmm, generators
cases = [("two-cluster", 3000, 20, 5, 32, True), ("uniform-cube", 4000, 40, 6, 32, True),
         ("sphere-surface", 3000, 30, 4, 32, False), ("two-cluster", 2000, 20, 6, 64, True),
         ("uniform-cube", 2000, 30, 7, 64, False), ("uniform-cube", 1500, 30, 3, 32, True)]
for kind, n, nc, p, prec, grad in cases:
    pos, q = generators.sample(kind, n, seed=3, charges="signed", fp32=prec == 32)
    with fmm.Fmm(pos, fmm.FmmConfig(p=p, n_crit=nc, precision=prec, gradient=grad)) as f:
        pot, g, _ = f.evaluate(q)
        pot2, _, _ = f.evaluate(q, timed=True)
        idx = np.arange(0, n, 7)
        d = fmm.direct(pos, q, targets=idx, precision=64)
        print(kind, n, p, prec, "backend", f.info()["m2l_backend"], "err vs direct %.2e" % fmm.relative_error(pot[idx], d),
              "timed == graph:", bool(np.array_equal(pot, pot2)), flush=True)
