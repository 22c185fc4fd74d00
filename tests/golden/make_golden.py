"""Regenerate the golden fixtures (run from the repo root: python tests/golden/make_golden.py).

The reference ships no runnable FMM and no fixtures, so the
golden vectors are (a) the seeded synthetic inputs of BASELINE.json configs and
(b) their exact-arithmetic targets from an independent numpy fp64 direct sum
(Eq. (1)): phi_i = sum_{j != i} q_j / (4 pi |x_i - x_j|).
Inputs come from paper_2303_08394_b200.generators (splitmix64, portable).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2303_08394_b200 import generators  # noqa: E402


def direct_numpy(pos, q, targets, chunk=256):
    out = np.zeros(len(targets))
    grad = np.zeros((len(targets), 3))
    for s in range(0, len(targets), chunk):
        t = targets[s:s + chunk]
        d = pos[t][:, None, :] - pos[None, :, :]
        r = np.sqrt((d * d).sum(-1))
        with np.errstate(divide="ignore"):
            inv = np.where(r > 0, 1.0 / r, 0.0)
        out[s:s + chunk] = (q[None, :] * inv).sum(1) / (4 * np.pi)
        grad[s:s + chunk] = -(q[None, :, None] * d * (inv ** 3)[:, :, None]).sum(1) / (4 * np.pi)
    return out, grad


def main():
    here = os.path.dirname(os.path.abspath(__file__))
    # config 1 (BASELINE.json configs[0]): N=10k uniform, seed 0, fp32 charges U[0,1)
    pos, q = generators.config_sample(1)
    phi, grad = direct_numpy(pos, q, np.arange(pos.shape[0]))
    np.savez_compressed(os.path.join(here, "config1_direct.npz"), positions=pos, charges=q, potential=phi,
                        gradient=grad)
    # two-cluster (W/X lists live), N=3000, signed charges
    pos, q = generators.sample("two-cluster", 3000, seed=5, charges="signed", fp32=True)
    phi, grad = direct_numpy(pos, q, np.arange(pos.shape[0]))
    np.savez_compressed(os.path.join(here, "two_cluster_direct.npz"), positions=pos, charges=q, potential=phi,
                        gradient=grad)
    # config 2 sample (1M points): direct at 1000 seeded targets -- the "1,000 sampled targets" of the north star
    pos, q = generators.config_sample(2)
    rng_t = (generators.uniform(1234, 0, 1000) * pos.shape[0]).astype(np.int64)
    phi, grad = direct_numpy(pos, q, rng_t, chunk=8)
    np.savez_compressed(os.path.join(here, "config2_sampled_direct.npz"), targets=rng_t, potential=phi,
                        gradient=grad)
    print("wrote fixtures to", here)


if __name__ == "__main__":
    main()
