"""tree and interaction_lists.

Lists must be bit-exact with a brute-force restatement of the definitions
(oracle/oracle.cpp `oracle_lists_bruteforce`), trees with a brute-force
recursive split + pairwise balance (`oracle_tree_leaves`).
"""
import itertools

import numpy as np
import pytest

import oracle
from paper_2303_08394_b200 import InvalidArgument, generators, host


def _clouds():
    yield "uniform", generators.sample("uniform-cube", 3000, seed=1)[0], 10
    yield "sphere", generators.sample("sphere-surface", 3000, seed=2)[0], 10
    yield "two-cluster", generators.sample("two-cluster", 3000, seed=3)[0], 8
    yield "two-cluster-fine", generators.sample("two-cluster", 1500, seed=4)[0], 1
    rng = np.random.default_rng(5)
    yield "gauss-blob", np.clip(0.5 + 0.08 * rng.standard_normal((2500, 3)), 0, 1), 4


def test_single_leaf():
    pos = generators.sample("uniform-cube", 10, seed=0)[0]
    t = host.Tree(pos, 10)
    assert t.n_leaves == 1 and t.depth == 0 and t.n_nodes == 1
    assert list(t.u_idx) == [0]


def test_two_per_octant():
    pts = []
    for o in itertools.product((0.25, 0.75), repeat=3):
        pts.append(np.array(o) - 0.05)
        pts.append(np.array(o) + 0.05)
    t = host.Tree(np.array(pts), 2, domain=((0, 0, 0), 1.0))
    assert t.n_leaves == 8 and t.depth == 1
    assert all(host.level(int(k)) == 1 for k in t.leaves)


def test_point_outside_domain():
    with pytest.raises(InvalidArgument):
        host.Tree(np.array([[0.5, 0.5, 0.5], [1.5, 0.5, 0.5]]), 1, domain=((0, 0, 0), 1.0))


@pytest.mark.parametrize("name,pos,n_crit", list(_clouds()), ids=lambda x: x if isinstance(x, str) else "")
def test_tree_matches_bruteforce(name, pos, n_crit):
    t = host.Tree(pos, n_crit)
    ref = oracle.tree_leaves(pos, n_crit, (t.origin, t.side), balance=True)
    assert np.array_equal(ref, t.leaves)
    unb = host.Tree(pos, n_crit, balance=False)
    ref_u = oracle.tree_leaves(pos, n_crit, (t.origin, t.side), balance=False)
    assert np.array_equal(ref_u, unb.leaves)


@pytest.mark.parametrize("name,pos,n_crit", list(_clouds()), ids=lambda x: x if isinstance(x, str) else "")
def test_tree_invariants(name, pos, n_crit):
    t = host.Tree(pos, n_crit)
    lv = t.leaves
    # leaf ranges cover [0, N) disjointly and in order
    assert t.leaf_ptr[0] == 0 and t.leaf_ptr[-1] == t.n and np.all(np.diff(t.leaf_ptr) > 0)
    # n_crit or MAX_LEVEL
    cnt = np.diff(t.leaf_ptr)
    lvls = lv & np.uint64(0xF)
    assert np.all((cnt <= n_crit) | (lvls == 15))
    # permutation integrity
    assert np.array_equal(np.sort(t.original_index), np.arange(t.n))
    assert np.array_equal(t.positions, pos[t.original_index])
    # each reordered particle lies in its leaf's cube
    for li in range(0, t.n_leaves, max(1, t.n_leaves // 50)):
        c, h = host.node_bounds(int(lv[li]), t.origin, t.side)
        p = t.positions[t.leaf_ptr[li]:t.leaf_ptr[li + 1]]
        assert np.all(np.abs(p - np.array(c)) <= h * (1 + 1e-12))
    # 2:1 balance over adjacent leaf pairs, brute force
    keys = [int(k) for k in lv]
    for a in keys:
        for b in keys:
            if host.is_adjacent(a, b):
                assert abs(host.level(a) - host.level(b)) <= 1
    # every non-root node's parent exists
    for n in range(1, t.n_nodes):
        assert t.node_parent[n] >= 0 and t.node_key[t.node_parent[n]] == host.parent(int(t.node_key[n]))


def test_balance_idempotent():
    pos = generators.sample("two-cluster", 2000, seed=9)[0]
    t = host.Tree(pos, 3)
    t2 = host.Tree(t.positions, 3, domain=(t.origin, t.side))
    assert np.array_equal(t.leaves, t2.leaves)


@pytest.mark.parametrize("name,pos,n_crit", list(_clouds()), ids=lambda x: x if isinstance(x, str) else "")
def test_lists_bit_exact(name, pos, n_crit):
    t = host.Tree(pos, n_crit)
    bf = oracle.lists_bruteforce(t)
    assert np.array_equal(bf["u"][0], t.u_ptr) and np.array_equal(bf["u"][1], t.u_idx)
    assert np.array_equal(bf["v"][0], t.v_ptr) and np.array_equal(bf["v"][1], t.v_idx)
    assert np.array_equal(bf["v"][2], t.v_tv)
    assert np.array_equal(bf["w"][0], t.w_ptr) and np.array_equal(bf["w"][1], t.w_idx)
    assert np.array_equal(bf["x"][0], t.x_ptr) and np.array_equal(bf["x"][1], t.x_idx)


@pytest.mark.parametrize("name,pos,n_crit", list(_clouds()), ids=lambda x: x if isinstance(x, str) else "")
def test_list_properties(name, pos, n_crit):
    t = host.Tree(pos, n_crit)
    nl, nn = t.n_leaves, t.n_nodes
    lvl = t.node_level()
    u = {a: set(t.u_idx[t.u_ptr[a]:t.u_ptr[a + 1]]) for a in range(nl)}
    for a in range(nl):
        assert a in u[a]
        for b in u[a]:
            assert a in u[b]  # U symmetric
    v = {b: set(t.v_idx[t.v_ptr[b]:t.v_ptr[b + 1]]) for b in range(nn)}
    for b in range(nn):
        for s in v[b]:
            assert b in v[s]  # V symmetric
            assert lvl[s] == lvl[b] >= 2
    # W / X duality (X on all nodes)
    for a in range(nl):
        for s in t.w_idx[t.w_ptr[a]:t.w_ptr[a + 1]]:
            assert a in set(t.x_idx[t.x_ptr[s]:t.x_ptr[s + 1]])
    assert np.diff(t.u_ptr).max() <= 60
    assert np.diff(t.v_ptr).max() <= 189
    assert np.diff(t.x_ptr).max() <= 19
    # transfer vectors consistent with geometry
    tv = host.transfer_vectors()
    for b in range(0, nn, max(1, nn // 30)):
        ab = np.array(host.decode(int(t.node_key[b]))[0])
        for e in range(t.v_ptr[b], t.v_ptr[b + 1]):
            asrc = np.array(host.decode(int(t.node_key[t.v_idx[e]]))[0])
            assert np.array_equal(tv[t.v_tv[e]], asrc - ab)


def test_uniform_tree_has_empty_w_x():
    pos = generators.sample("uniform-cube", 20000, seed=0)[0]
    t = host.Tree(pos, 64)
    s = t.list_stats()
    assert s["W"][2] == 0 and s["X"][2] == 0
    assert len(set((t.leaves & np.uint64(0xF)).tolist())) == 1


def test_transfer_vectors():
    tv = host.transfer_vectors()
    assert tv.shape == (316, 3)
    assert np.all(np.max(np.abs(tv), axis=1) >= 2) and np.all(np.abs(tv) <= 3)
    assert len({tuple(x) for x in tv}) == 316
    assert [tuple(x) for x in tv] == sorted(tuple(x) for x in tv)


def test_interior_v_list_is_189():
    pos = generators.sample("uniform-cube", 40000, seed=0)[0]
    t = host.Tree(pos, 100)  # uniform depth 3 (512 leaves)
    lvl = t.node_level()
    interior = [b for b in range(t.n_nodes) if lvl[b] == 3 and
                all(2 <= x <= 5 for x in host.decode(int(t.node_key[b]))[0])]
    assert interior and all(t.v_ptr[b + 1] - t.v_ptr[b] == 189 for b in interior)


def test_sphere_stats_scaled():  # SPEC.md:183 (scaled-down sphere, n_crit=150)
    pos = generators.sample("sphere-surface", 10000, seed=0)[0]
    t = host.Tree(pos, 150)
    s = t.list_stats()
    assert t.n_leaves > 8 and s["U"][1] > 5


def test_partition_contiguous_and_aligned():
    pos = generators.sample("uniform-cube", 50000, seed=0)[0]
    t = host.Tree(pos, 64)
    for w in (1, 2, 3, 4, 8):
        lb = t.partition(w, n_e=98, cut_level=2)
        assert lb[0] == 0 and lb[-1] == t.n_leaves and np.all(np.diff(lb) >= 0)
        for b in lb[1:-1]:
            if 0 < b < t.n_leaves:  # boundaries never split a level-2 box
                ka, kb = int(t.leaves[b - 1]), int(t.leaves[b])
                anc = lambda k: host.decode(k)[0] if host.level(k) <= 2 else tuple(  # noqa: E731
                    x >> (host.level(k) - 2) for x in host.decode(k)[0])
                assert anc(ka) != anc(kb)
