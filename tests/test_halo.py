"""The product's multi-GPU partition and halo-exchange tables (kifmm_halo_plan), checked on
the CPU against the direct definition of what each rank's downward pass reads:

  reads(r) = V(b) for every node b at level >= 2 with an owned leaf below it     (M2L)
           + W(a) for every owned leaf a                                          (M2P)
           + the children of every node recomputed by all ranks (up_owner -1)     (M2M above the cut)

Every row rank r reads must be computed by r itself (owned, or recomputed from rows it has) or be
shipped by its owner in the all-gather; and every shipped row must be read by some other rank.
"""
import numpy as np
import pytest

from paper_2303_08394_b200 import generators, host


def _trees():
    yield "uniform", host.Tree(generators.sample("uniform-cube", 30000, seed=1)[0], 30)
    yield "sphere", host.Tree(generators.sample("sphere-surface", 30000, seed=2)[0], 30)
    yield "two-cluster", host.Tree(generators.sample("two-cluster", 30000, seed=3)[0], 20)


TREES = list(_trees())


def _leaf_range(t):
    lo = np.full(t.n_nodes, np.iinfo(np.int64).max)
    hi = np.full(t.n_nodes, -1)
    for leaf in range(t.n_leaves):
        n = t.leaf_node[leaf]
        while n >= 0:
            lo[n] = min(lo[n], leaf)
            hi[n] = max(hi[n], leaf + 1)
            n = t.node_parent[n]
    return lo, hi


@pytest.mark.parametrize("name,t", TREES, ids=[n for n, _ in TREES])
@pytest.mark.parametrize("world,cut", [(2, 0), (3, 0), (4, 2), (4, 0), (8, 0), (8, 3)])
def test_halo_tables_cover_every_read(name, t, world, cut):
    h = t.halo(world, n_e=98, cut_level=cut)
    lb = h.leaf_begin
    assert lb[0] == 0 and lb[-1] == t.n_leaves and np.all(np.diff(lb) >= 0)
    lo, hi = _leaf_range(t)
    lvl = t.node_level()
    owner_of = np.searchsorted(lb, np.arange(t.n_leaves), side="right") - 1
    # owner = the rank holding every leaf below the node; -1 only for non-leaf nodes spanning ranks
    for n in range(t.n_nodes):
        r = owner_of[lo[n]]
        if hi[n] <= lb[r + 1]:
            assert h.up_owner[n] == r
        else:
            assert h.up_owner[n] == -1 and t.node_leaf[n] < 0
    shipped = [set(e.tolist()) for e in h.exports]
    for s in range(world):
        assert all(h.up_owner[n] == s for n in shipped[s])
        assert len(shipped[s]) <= h.max_export
    redundant = [n for n in range(t.n_nodes) if h.up_owner[n] < 0]
    read_by_other = [set() for _ in range(world)]
    for r in range(world):
        owned_leaves = range(lb[r], lb[r + 1])
        active = set()
        for leaf in owned_leaves:
            n = t.leaf_node[leaf]
            while n >= 0 and n not in active:
                active.add(n)
                n = t.node_parent[n]
        reads = set()
        for b in active:
            if lvl[b] >= 2:
                reads.update(t.v_idx[t.v_ptr[b]:t.v_ptr[b + 1]].tolist())
        for leaf in owned_leaves:
            reads.update(t.w_idx[t.w_ptr[leaf]:t.w_ptr[leaf + 1]].tolist())
        for n in redundant:
            if lvl[n] >= 2:
                reads.update(c for c in t.node_children[n].tolist() if c >= 0)
        for n in reads:
            o = h.up_owner[n]
            if o == r or o == -1:
                continue
            assert n in shipped[o], (name, world, r, n, o)
            read_by_other[o].add(n)
    for s in range(world):  # nothing is shipped that no other rank reads
        assert shipped[s] == read_by_other[s], (name, world, s)


def test_auto_cut_balances_clustered_cloud():
    """Cut level 0 (auto) picks a finer alignment when the level-2 boxes cannot balance the ranks (a dense
    cluster inside one level-2 box): no rank is left without leaves."""
    t = dict(TREES)["two-cluster"]
    fixed = t.partition(8, 98, cut_level=2)
    auto = t.partition(8, 98, cut_level=0)
    assert np.any(np.diff(fixed) == 0)
    assert np.all(np.diff(auto) > 0)


def test_single_rank_owns_everything():
    t = dict(TREES)["sphere"]
    h = t.halo(1, n_e=98)
    assert np.all(h.up_owner == 0) and h.max_export == 0 and len(h.exports[0]) == 0
