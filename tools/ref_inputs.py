"""Build the oracle's inputs for a BASELINE config in THIS (child) process and save them as .npz, so the
timed reference process (bench.py --impl reference) never maps the product library: tree, lists and
operator cache come from the product's host C++ (bit-exact with the oracle's brute-force restatements,
tests/test_tree_lists.py, tests/test_lists_baseline.py), charges from the seeded generator.

usage: python tools/ref_inputs.py CONFIG OUT.npz
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import views  # noqa: E402
from paper_2303_08394_b200 import generators, host  # noqa: E402


def main():
    cid, out = int(sys.argv[1]), sys.argv[2]
    c = generators.CONFIGS[cid]
    pos, q = generators.config_sample(cid)
    tree = host.Tree(pos, c["n_crit"])
    ops = host.Operators(c["p"], domain_side=tree.side)
    tmp = out + ".tmp.npz"
    views.save(tmp, tree, ops, reference_level=ops.view.reference_level)
    with np.load(tmp) as z:
        d = dict(z)
    d["charges_reordered"] = np.ascontiguousarray(q[tree.original_index])
    np.savez(out, **d)
    os.remove(tmp)


if __name__ == "__main__":
    main()
