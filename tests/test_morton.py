"""morton module KATs and properties."""
import itertools

import numpy as np
import pytest

from paper_2303_08394_b200 import InvalidArgument, host


def test_encode_root_is_zero():
    assert host.encode((0, 0, 0), 0) == 0


def test_round_trip_examples():
    k = host.encode((1, 0, 0), 1)
    assert host.decode(k) == ((1, 0, 0), 1)
    rng = np.random.default_rng(0)
    for _ in range(2000):
        lvl = int(rng.integers(0, 16))
        a = tuple(int(x) for x in rng.integers(0, 2 ** lvl, 3))
        assert host.decode(host.encode(a, lvl)) == (a, lvl)


def test_level1_raw_order_is_z_order():
    keys = [host.encode((x, y, z), 1) for z in (0, 1) for y in (0, 1) for x in (0, 1)]
    assert len(set(keys)) == 8
    assert keys == sorted(keys)  # octant order x + 2y + 4z == ascending raw


def test_parent_examples():
    root = host.encode((0, 0, 0), 0)
    for c in host.children(root):
        assert host.parent(c) == root
    assert host.parent(host.encode((3, 2, 1), 2)) == host.encode((1, 1, 0), 1)
    rng = np.random.default_rng(1)
    for _ in range(1000):
        lvl = int(rng.integers(0, 15))
        k = host.encode(tuple(int(x) for x in rng.integers(0, 2 ** lvl, 3)), lvl)
        assert all(host.parent(c) == k for c in host.children(k))


def test_children_examples():
    ch = host.children(0)
    assert ch == sorted(ch)
    anchors = sorted(host.decode(c)[0] for c in ch)
    assert anchors == sorted(itertools.product((0, 1), repeat=3))
    # children tile the parent cube
    pc, ph = host.node_bounds(0)
    for c in ch:
        cc, chh = host.node_bounds(c)
        assert chh == ph / 2
        assert all(abs(cc[d] - pc[d]) == pytest.approx(ph / 2) for d in range(3))


def test_errors():
    with pytest.raises(InvalidArgument):
        host.encode((2, 0, 0), 1)
    with pytest.raises(InvalidArgument):
        host.encode((0, 0, 0), 16)
    with pytest.raises(InvalidArgument):
        host.parent(0)
    with pytest.raises(InvalidArgument):
        host.children(host.encode((0, 0, 0), 15))


def test_neighbors_examples():
    assert host.neighbors(0) == []
    assert len(host.neighbors(host.encode((0, 0, 0), 1))) == 7
    n = host.neighbors(host.encode((1, 1, 1), 2))
    assert len(n) == 26 and n == sorted(n)


def test_neighbors_symmetric():
    for lvl in (1, 2, 3):
        keys = [host.encode(a, lvl) for a in itertools.product(range(2 ** lvl), repeat=3)]
        for k in keys[:: max(1, len(keys) // 40)]:
            for nb in host.neighbors(k):
                assert k in host.neighbors(nb)


def test_is_adjacent_examples():
    a, b = host.children(0)[:2]
    assert host.is_adjacent(a, b)
    for c in host.children(a):
        assert not host.is_adjacent(0, c)
    l1 = host.encode((0, 0, 0), 1)
    assert host.is_adjacent(l1, host.encode((2, 0, 0), 2))
    assert not host.is_adjacent(l1, host.encode((3, 0, 0), 2))


def _brute_adjacent(ka, kb):
    (aa, la), (ab, lb) = host.decode(ka), host.decode(kb)
    lo_a = [x / 2 ** la for x in aa]
    hi_a = [(x + 1) / 2 ** la for x in aa]
    lo_b = [x / 2 ** lb for x in ab]
    hi_b = [(x + 1) / 2 ** lb for x in ab]
    touch = all(lo_a[d] <= hi_b[d] and lo_b[d] <= hi_a[d] for d in range(3))
    a_in_b = all(lo_a[d] >= lo_b[d] and hi_a[d] <= hi_b[d] for d in range(3))
    b_in_a = all(lo_b[d] >= lo_a[d] and hi_b[d] <= hi_a[d] for d in range(3))
    return touch and not (a_in_b or b_in_a)


def test_is_adjacent_matches_cube_overlap_oracle():
    keys = [host.encode(a, l) for l in range(0, 4) for a in itertools.product(range(2 ** l), repeat=3)]
    rng = np.random.default_rng(3)
    for _ in range(20000):
        i, j = rng.integers(0, len(keys), 2)
        ka, kb = keys[i], keys[j]
        assert host.is_adjacent(ka, kb) == _brute_adjacent(ka, kb)
        assert host.is_adjacent(ka, kb) == host.is_adjacent(kb, ka)


def test_node_bounds_examples():
    c, h = host.node_bounds(0, (0, 0, 0), 1.0)
    assert c == (0.5, 0.5, 0.5) and h == 0.5
    c, h = host.node_bounds(host.encode((1, 0, 0), 1), (0, 0, 0), 1.0)
    assert c == (0.75, 0.25, 0.25) and h == 0.25


def test_cross_level_raw_order_is_spatial():
    # ancestors sort before descendants and Z-order is preserved across levels
    k2 = host.encode((3, 1, 0), 2)
    par = host.parent(k2)
    assert par < k2
    assert host.children(k2)[0] > k2
