"""Randomised host check (CPU): trees and U/V/W/X lists of random and degenerate clouds, scaled and shifted, bit for bit
against the brute-force restatements of the oracle (10047 cases in 240 s, 0 failures)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import oracle
from paper_2303_08394_b200 import generators, host
rng = np.random.default_rng(1)
t_end = time.time() + 240
cases = fails = 0
while time.time() < t_end:
    cases += 1
    kind = str(rng.choice(["uniform-cube", "sphere-surface", "two-cluster", "dups", "line", "blob", "plane"]))
    n = int(rng.integers(1, 1500))
    ncrit = int(rng.choice([1, 2, 3, 8, 20, 64]))
    if ncrit <= 2: n = min(n, 250)
    seed = int(rng.integers(0, 10000))
    if kind in ("uniform-cube", "sphere-surface", "two-cluster"):
        pos = generators.sample(kind, n, seed=seed)[0]
    elif kind == "dups":
        b = rng.random((max(1, n // 3), 3)); pos = np.concatenate([b] * 3)
    elif kind == "line":
        t = rng.random(n); pos = np.stack([t, 0.3 + 0 * t, 0.7 + 0 * t], axis=1)
    elif kind == "plane":
        pos = rng.random((n, 3)); pos[:, 2] = 0.5
    else:
        pos = np.clip(0.5 + 0.05 * rng.standard_normal((n, 3)), 0, 1)
    scale = float(rng.choice([1.0, 1e-3, 1e3])); shift = float(rng.choice([0.0, -5.0, 100.0]))
    pos = pos * scale + shift
    try:
        t = host.Tree(pos, ncrit)
        ref = oracle.tree_leaves(pos, ncrit, (t.origin, t.side), balance=True)
        ok = np.array_equal(ref, t.leaves)
        if ok:
            bf = oracle.lists_bruteforce(t)
            for name in "uvwx":
                if not (np.array_equal(bf[name][0], getattr(t, name + "_ptr")) and np.array_equal(bf[name][1], getattr(t, name + "_idx"))):
                    ok = False; print("list mismatch", name)
            if not np.array_equal(bf["v"][2], t.v_tv):
                ok = False; print("tv mismatch")
    except Exception as e:
        ok = False; print("exception", repr(e)[:200])
    if not ok:
        fails += 1
        print("FAIL", kind, n, ncrit, seed, scale, shift, flush=True)
print("cases", cases, "failures", fails)
