"""Multi-rank evaluate on CPU (gloo, world_size 2 and 3): the product's partition and halo-exchange
tables (kifmm_halo_plan) drive the partitioned algorithm restated in the oracle --
upward on each rank's owned subtrees -> all-gather of ONLY the export rows (one slot of max_export rows
per rank, as the GPU plan's ncclAllGather) -> every rank recomputes the nodes spanning ranks -> downward
on owned leaves -- and must reproduce the single-rank result bit for bit.  A row missing from the
export tables would reach the receiving rank as zeros and break the equality.  This is the host-side
logic of the NCCL path; tests/test_multirank_gpu.py runs the product's device path."""
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
    h = t.halo(world, o.n_e, cut_level=cut)
    lb = h.leaf_begin
    qr = q[t.original_index]
    # upward over the owned subtrees: nodes whose leaves all lie in [lb[rank], lb[rank+1]) (cut 0 = every level)
    M = oracle.upward_local(t, o, qr, lb[rank], lb[rank + 1], 0, threads=2)
    own = np.flatnonzero(h.up_owner == rank)
    assert not np.any(M[np.flatnonzero(h.up_owner != rank)]), "upward wrote rows it does not own"
    del own
    send = np.zeros((max(1, h.max_export), o.n_e))
    send[:len(h.exports[rank])] = M[h.exports[rank]]
    slots = [torch.zeros_like(torch.from_numpy(send)) for _ in range(world)]
    dist.all_gather(slots, torch.from_numpy(send))
    for r in range(world):
        if r != rank:
            M[h.exports[r]] = slots[r].numpy()[:len(h.exports[r])]
    # nodes spanning ranks, children first (levels descending)
    span = np.flatnonzero(h.up_owner < 0)
    span = span[np.argsort(-t.node_level()[span], kind="stable")]
    oracle.m2m_nodes(t, o, span, M)
    phi, g = oracle.downward(t, o, qr, M, lb[rank], lb[rank + 1], gradient=True, threads=2)
    a, b = t.leaf_ptr[lb[rank]], t.leaf_ptr[lb[rank + 1]]
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), a=a, b=b, phi=phi[a:b], g=g[a:b],
             shipped=sum(len(e) for e in h.exports), owned=int(np.count_nonzero(h.up_owner >= 0)))
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,n,n_crit,p,cut,world", [("uniform-cube", 4000, 20, 4, 2, 2),
                                                       ("two-cluster", 4000, 10, 5, 0, 2),
                                                       ("sphere-surface", 3000, 15, 4, 3, 2),
                                                       ("two-cluster", 5000, 8, 4, 0, 3)])
def test_ranks_match_single_rank(tmp_path, kind, n, n_crit, p, cut, world):
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
        assert d["shipped"] < d["owned"]  # a halo, not every owned multipole
    assert covered.all()
    assert np.array_equal(got, ref)
    assert np.array_equal(gg, gref)
