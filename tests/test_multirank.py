"""Multi-rank evaluate on CPU (gloo, world_size 2): the Morton-range partition
of the product host library + the partitioned evaluate restated in the oracle
(upward on owned subtrees -> all-gather of multipoles -> redundant top levels
-> downward on owned leaves) must reproduce the single-rank result exactly.
This is the host-side logic of the NCCL path."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2303_08394_b200 import generators, host


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kind, n, n_crit, p, cut, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pos, q = generators.sample(kind, n, seed=11, charges="signed")
    t = host.Tree(pos, n_crit)
    o = host.Operators(p, domain_side=t.side)
    qr = q[t.original_index]
    lb = t.partition(world, o.n_e, cut_level=cut)
    M = oracle.upward_local(t, o, qr, lb[rank], lb[rank + 1], cut, threads=2)
    Mt = torch.from_numpy(M)
    dist.all_reduce(Mt, op=dist.ReduceOp.SUM)  # owned slices are disjoint: a sum is an all-gather
    M = oracle.upward_top(t, o, Mt.numpy(), cut, threads=2)
    phi, g = oracle.downward(t, o, qr, M, lb[rank], lb[rank + 1], gradient=True, threads=2)
    a, b = t.leaf_ptr[lb[rank]], t.leaf_ptr[lb[rank + 1]]
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), a=a, b=b, phi=phi[a:b], g=g[a:b])
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,n,n_crit,p,cut", [("uniform-cube", 4000, 20, 4, 2),
                                                 ("two-cluster", 4000, 10, 5, 2),
                                                 ("sphere-surface", 3000, 15, 4, 3)])
def test_two_rank_matches_single_rank(tmp_path, kind, n, n_crit, p, cut):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), kind, n, n_crit, p, cut, str(tmp_path)), nprocs=world, join=True)
    pos, q = generators.sample(kind, n, seed=11, charges="signed")
    t = host.Tree(pos, n_crit)
    o = host.Operators(p, domain_side=t.side)
    ref, gref, _ = oracle.evaluate(t, o, q[t.original_index], gradient=True)
    got, gg = np.zeros(t.n), np.zeros((t.n, 3))
    covered = np.zeros(t.n, bool)
    for r in range(world):
        d = np.load(tmp_path / f"rank{r}.npz")
        got[d["a"]:d["b"]] = d["phi"]
        gg[d["a"]:d["b"]] = d["g"]
        covered[d["a"]:d["b"]] = True
    assert covered.all()
    assert np.array_equal(got, ref)
    assert np.array_equal(gg, gref)
