"""Host-side modules of the evaluate path, mirroring the reference's module API.

morton, kernel, surface,
tree + interaction_lists and operators/precompute
 -- all implemented in C++ inside libkifmm_b200.so; this file
only marshals arrays.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check, lib

MAX_LEVEL = 15


# ------------------------------------------------------------------ morton
def encode(anchor, level: int) -> int:
    """key of (anchor, level)."""
    a = (C.c_uint32 * 3)(*[int(x) for x in anchor])
    out = C.c_uint64()
    check(lib.kifmm_morton_encode(a, int(level), C.byref(out)), "encode")
    return out.value


def decode(key: int):
    a = (C.c_uint32 * 3)()
    lvl = C.c_int32()
    check(lib.kifmm_morton_decode(int(key), a, C.byref(lvl)), "decode")
    return (a[0], a[1], a[2]), lvl.value


def level(key: int) -> int:
    return int(key) & 0xF


def parent(key: int) -> int:
    out = C.c_uint64()
    check(lib.kifmm_morton_parent(int(key), C.byref(out)), "parent")
    return out.value


def children(key: int):
    out = (C.c_uint64 * 8)()
    check(lib.kifmm_morton_children(int(key), out), "children")
    return list(out)


def neighbors(key: int):
    out = (C.c_uint64 * 26)()
    n = lib.kifmm_morton_neighbors(int(key), out)
    return list(out[:n])


def is_adjacent(a: int, b: int) -> bool:
    return bool(lib.kifmm_morton_is_adjacent(int(a), int(b)))


def node_bounds(key: int, origin=(0.0, 0.0, 0.0), side: float = 1.0):
    o = (C.c_double * 3)(*origin)
    c = (C.c_double * 3)()
    h = C.c_double()
    lib.kifmm_morton_node_bounds(int(key), o, float(side), c, C.byref(h))
    return (c[0], c[1], c[2]), h.value


# ------------------------------------------------------------------ kernel
def laplace(x, y) -> float:
    """1/(4 pi |x-y|), 0 at x == y."""
    return lib.kifmm_laplace((C.c_double * 3)(*x), (C.c_double * 3)(*y))


def kernel_matrix(sources, targets) -> np.ndarray:
    """K[j, i] = laplace(sources_i, targets_j)."""
    s = np.ascontiguousarray(sources, dtype=np.float64).reshape(-1, 3)
    t = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1, 3)
    out = np.empty((t.shape[0], s.shape[0]), dtype=np.float64)
    lib.kifmm_kernel_matrix(s.ctypes.data, s.shape[0], t.ctypes.data, t.shape[0], out.ctypes.data)
    return out


# ----------------------------------------------------------------- surface
def surface_count(p: int) -> int:
    return lib.kifmm_surface_count(int(p))


def surface_grid(p: int) -> np.ndarray:
    """boundary points of the p^3 grid on [-1,1]^3, lexicographic."""
    n = surface_count(p)
    if n < 0:
        from .errors import InvalidArgument
        raise InvalidArgument("surface_grid: p must be >= 2")
    out = np.empty((n, 3), dtype=np.float64)
    check(lib.kifmm_surface_grid(int(p), out.ctypes.data), "surface_grid")
    return out


def scaled_surface(grid, center, half_side: float, alpha: float) -> np.ndarray:
    """center + alpha * half_side * grid."""
    return np.asarray(center, dtype=np.float64)[None, :] + alpha * half_side * np.asarray(grid)


def transfer_vectors() -> np.ndarray:
    out = np.empty((316, 3), dtype=np.int32)
    n = lib.kifmm_transfer_vectors(out.ctypes.data)
    return out[:n]


# -------------------------------------------------------------------- tree
def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(int(n),)).view(dtype)


class Tree:
    """LinearTree + InteractionLists built in C++.

    Arrays are zero-copy views into C++-owned memory, valid while this object
    lives.  Lists are CSR with members in ascending raw key order.
    """

    def __init__(self, positions, n_crit: int, domain=None, balance: bool = True, threads: int = 0):
        pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
        dom = None
        if domain is not None:
            origin, side = domain
            dom = np.array(list(origin) + [side], dtype=np.float64)
        h = C.c_void_p()
        check(lib.kifmm_tree_build(pos.ctypes.data, pos.shape[0], int(n_crit),
                                   dom.ctypes.data if dom is not None else None,
                                   1 if balance else 0, int(threads), C.byref(h)), "build_tree")
        self._h = h
        self.view = _lib.TreeView()
        check(lib.kifmm_tree_get_view(h, C.byref(self.view)), "tree_view")
        v = self.view
        self.n = v.n_particles
        self.depth = v.depth
        self.n_overfull = v.n_overfull
        self.n_leaves = v.n_leaves
        self.n_nodes = v.n_nodes
        self.origin = tuple(v.origin)
        self.side = v.side
        nl, nn = v.n_leaves, v.n_nodes
        self.positions = _arr(v.positions, 3 * self.n, np.float64).reshape(-1, 3)
        self.original_index = _arr(v.original_index, self.n, np.int64)
        self.node_key = _arr(v.node_key, nn, np.uint64)
        self.level_ptr = _arr(v.level_ptr, self.depth + 2, np.int64)
        self.node_parent = _arr(v.node_parent, nn, np.int64)
        self.node_children = _arr(v.node_children, 8 * nn, np.int64).reshape(-1, 8)
        self.node_leaf = _arr(v.node_leaf, nn, np.int64)
        self.leaf_node = _arr(v.leaf_node, nl, np.int64)
        self.leaf_ptr = _arr(v.leaf_ptr, nl + 1, np.int64)
        self.u_ptr = _arr(v.u_ptr, nl + 1, np.int64)
        self.u_idx = _arr(v.u_idx, self.u_ptr[-1], np.int64)
        self.v_ptr = _arr(v.v_ptr, nn + 1, np.int64)
        self.v_idx = _arr(v.v_idx, self.v_ptr[-1], np.int64)
        self.v_tv = _arr(v.v_tv, self.v_ptr[-1], np.int32)
        self.w_ptr = _arr(v.w_ptr, nl + 1, np.int64)
        self.w_idx = _arr(v.w_idx, self.w_ptr[-1], np.int64)
        self.x_ptr = _arr(v.x_ptr, nn + 1, np.int64)
        self.x_idx = _arr(v.x_idx, self.x_ptr[-1], np.int64)

    @property
    def leaves(self) -> np.ndarray:
        return self.node_key[self.leaf_node]

    def node_level(self) -> np.ndarray:
        return (self.node_key & np.uint64(0xF)).astype(np.int64)

    def list_stats(self) -> dict:
        """min/mean/max of |U|,|V|,|W|,|X| (SPEC.md:273 `stats`)."""
        out = {}
        lvl = self.node_level()
        for name, ptr, mask in (("U", self.u_ptr, None), ("V", self.v_ptr, lvl >= 2),
                                ("W", self.w_ptr, None), ("X", self.x_ptr, self.node_leaf >= 0)):
            sz = np.diff(ptr)
            if mask is not None:
                sz = sz[mask]
            out[name] = (int(sz.min()) if sz.size else 0, float(sz.mean()) if sz.size else 0.0,
                         int(sz.max()) if sz.size else 0)
        return out

    def partition(self, world_size: int, n_e: int, gradient: bool = False, cut_level: int = 0) -> np.ndarray:
        out = np.zeros(world_size + 1, dtype=np.int64)
        check(lib.kifmm_partition_leaves(C.byref(self.view), int(n_e), int(gradient), int(world_size),
                                         int(cut_level), out.ctypes.data), "partition")
        return out

    def halo(self, world_size: int, n_e: int, gradient: bool = False, cut_level: int = 0) -> "Halo":
        """Multi-GPU partition + halo-exchange tables (kifmm_halo_plan)."""
        return Halo(self, world_size, n_e, gradient, cut_level)

    def close(self):
        if getattr(self, "_h", None):
            lib.kifmm_tree_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Halo:
    """Partition and halo-exchange tables of a world_size-rank evaluate (include/kifmm.h kifmm_halo_view):
    leaf_begin (world + 1), up_owner (n_nodes; -1 = recomputed by every rank), exports[r] (node rows rank
    r contributes to the all-gather), max_export (rows per all-gather slot)."""

    def __init__(self, tree: Tree, world_size: int, n_e: int, gradient: bool = False, cut_level: int = 0):
        h = C.c_void_p()
        check(lib.kifmm_halo_plan(C.byref(tree.view), int(n_e), int(gradient), int(world_size), int(cut_level),
                                  C.byref(h)), "halo_plan")
        try:
            v = _lib.HaloView()
            check(lib.kifmm_halo_get_view(h, C.byref(v)), "halo_view")
            w = v.world_size
            self.world_size, self.cut_level, self.max_export = w, v.cut_level, int(v.max_export)
            self.leaf_begin = _arr(v.leaf_begin, w + 1, np.int64).copy()
            self.up_owner = _arr(v.up_owner, v.n_nodes, np.int32).copy()
            ptr = _arr(v.export_ptr, w + 1, np.int64).copy()
            idx = _arr(v.export_idx, ptr[-1], np.int64).copy()
            self.exports = [idx[ptr[r]:ptr[r + 1]] for r in range(w)]
        finally:
            lib.kifmm_halo_destroy(h)


# --------------------------------------------------------------- operators
class Operators:
    """OperatorCache: factored pinvs, M2M/L2L composites, M2L K_t."""

    def __init__(self, p: int = 6, alpha_inner: float = 1.05, alpha_outer: float = 2.95,
                 svd_cutoff: float = 1e-12, domain_side: float = 1.0, threads: int = 0, _handle=None):
        if _handle is None:
            h = C.c_void_p()
            check(lib.kifmm_precompute(int(p), float(alpha_inner), float(alpha_outer), float(svd_cutoff),
                                       float(domain_side), int(threads), C.byref(h)), "precompute")
        else:
            h = _handle
        self._h = h
        self.view = _lib.OperatorView()
        check(lib.kifmm_operators_get_view(h, C.byref(self.view)), "operators_view")
        v = self.view
        ne, nc = v.n_e, v.n_c
        self.p, self.n_e, self.n_c = v.p, ne, nc
        self.alpha_inner, self.alpha_outer, self.svd_cutoff = v.alpha_inner, v.alpha_outer, v.svd_cutoff
        self.domain_side, self.ref_half_side = v.domain_side, v.ref_half_side
        self.fingerprint = v.fingerprint
        self.surface = _arr(v.surface, 3 * ne, np.float64).reshape(ne, 3)
        ku, kd = v.uc2e_rank, v.dc2e_rank
        self.uc2e = (_arr(v.uc2e_u, nc * ku, np.float64).reshape(nc, ku), _arr(v.uc2e_s, ku, np.float64),
                     _arr(v.uc2e_v, ne * ku, np.float64).reshape(ne, ku))
        self.dc2e = (_arr(v.dc2e_u, nc * kd, np.float64).reshape(nc, kd), _arr(v.dc2e_s, kd, np.float64),
                     _arr(v.dc2e_v, ne * kd, np.float64).reshape(ne, kd))
        self.m2m = _arr(v.m2m, 8 * ne * ne, np.float64).reshape(8, ne, ne)
        self.l2l = _arr(v.l2l, 8 * ne * ne, np.float64).reshape(8, ne, ne)
        self.m2l = _arr(v.m2l, v.n_m2l * nc * ne, np.float64).reshape(v.n_m2l, nc, ne)

    def save(self, path: str) -> None:
        check(lib.kifmm_operators_save(self._h, str(path).encode()), "save_cache")

    @classmethod
    def load(cls, path: str, expected_fingerprint: int = 0) -> "Operators":
        h = C.c_void_p()
        check(lib.kifmm_operators_load(str(path).encode(), int(expected_fingerprint), C.byref(h)), "load_cache")
        return cls(_handle=h)

    def close(self):
        if getattr(self, "_h", None):
            lib.kifmm_operators_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def svd(a) -> tuple:
    """The in-repo one-sided Jacobi SVD used by precompute."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    m, n = a.shape
    u = np.empty((m, n)), np.empty(n), np.empty((n, n))
    check(lib.kifmm_svd(a.ctypes.data, m, n, u[0].ctypes.data, u[1].ctypes.data, u[2].ctypes.data), "svd")
    return u
