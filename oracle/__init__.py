"""TEST INFRASTRUCTURE ONLY: ctypes wrapper of oracle/_build/liboracle.so.

The fp64 CPU restatement of the reference evaluate (see oracle/oracle.h).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arm may import this package; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} missing: run `make oracle`")

_lib = C.CDLL(LIB_PATH)
P, i32, i64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double


class Timings(C.Structure):
    _fields_ = [(n, f64) for n in ("p2m_ms", "m2m_ms", "m2l_ms", "p2l_ms", "l2l_ms", "near_ms", "l2p_ms",
                                   "m2p_ms", "total_ms")] + \
        [(n, i64) for n in ("m2m_levels", "m2l_levels", "l2l_levels", "p2m_calls", "near_calls", "l2p_calls",
                            "m2p_calls", "p2l_calls")]

    def as_dict(self):
        return {n: (int if t is i64 else float)(getattr(self, n)) for n, t in self._fields_}


_lib.oracle_evaluate.argtypes = [P, P, P, P, P, i32, i64, i64, C.POINTER(Timings)]
_lib.oracle_upward_local.argtypes = [P, P, P, i64, i64, i32, P, i32]
_lib.oracle_upward_top.argtypes = [P, P, i32, P, i32]
_lib.oracle_downward.argtypes = [P, P, P, P, i64, i64, P, P, i32, C.POINTER(Timings)]
_lib.oracle_direct.argtypes = [P, P, i64, P, i64, P, P, i32]
_lib.oracle_direct.restype = None
_lib.oracle_tree_leaves.argtypes = [P, i64, i32, P, i32, P, i64]
_lib.oracle_tree_leaves.restype = i64
_lib.oracle_max_threads.argtypes = []
_lib.oracle_max_threads.restype = i32
_lib.oracle_relative_error.argtypes = [P, P, i64]
_lib.oracle_relative_error.restype = f64


def _ptr(a):
    return None if a is None else a.ctypes.data


def evaluate(tree, ops, charges_reordered, gradient=False, threads=0, leaf_range=None):
    """Full fp64 evaluate; returns (potential, gradient|None, timings) in REORDERED order."""
    q = np.ascontiguousarray(charges_reordered, dtype=np.float64)
    n = tree.n
    phi = np.zeros(n)
    g = np.zeros((n, 3)) if gradient else None
    lb, le = leaf_range if leaf_range is not None else (0, tree.n_leaves)
    tm = Timings()
    _lib.oracle_evaluate(C.addressof(tree.view), C.addressof(ops.view), q.ctypes.data, phi.ctypes.data, _ptr(g),
                         int(threads), int(lb), int(le), C.byref(tm))
    return phi, g, tm.as_dict()


def upward_local(tree, ops, charges_reordered, leaf_begin, leaf_end, cut_level, threads=0):
    q = np.ascontiguousarray(charges_reordered, dtype=np.float64)
    M = np.zeros((tree.n_nodes, ops.n_e))
    _lib.oracle_upward_local(C.addressof(tree.view), C.addressof(ops.view), q.ctypes.data, int(leaf_begin),
                             int(leaf_end), int(cut_level), M.ctypes.data, int(threads))
    return M


def upward_top(tree, ops, M, cut_level, threads=0):
    M = np.ascontiguousarray(M, dtype=np.float64)
    _lib.oracle_upward_top(C.addressof(tree.view), C.addressof(ops.view), int(cut_level), M.ctypes.data,
                           int(threads))
    return M


_lib.oracle_m2m_nodes.argtypes = [P, P, i64, P, P]


def m2m_nodes(tree, ops, nodes, M):
    """M2M of `nodes` (children before parents) into M (n_nodes x n_e, updated in place and returned)."""
    nd = np.ascontiguousarray(nodes, dtype=np.int64)
    assert M.flags.c_contiguous and M.dtype == np.float64
    _lib.oracle_m2m_nodes(C.addressof(tree.view), C.addressof(ops.view), nd.size, nd.ctypes.data, M.ctypes.data)
    return M


def downward(tree, ops, charges_reordered, M, leaf_begin, leaf_end, gradient=False, threads=0):
    q = np.ascontiguousarray(charges_reordered, dtype=np.float64)
    M = np.ascontiguousarray(M, dtype=np.float64)
    phi = np.zeros(tree.n)
    g = np.zeros((tree.n, 3)) if gradient else None
    tm = Timings()
    _lib.oracle_downward(C.addressof(tree.view), C.addressof(ops.view), q.ctypes.data, M.ctypes.data,
                         int(leaf_begin), int(leaf_end), phi.ctypes.data, _ptr(g), int(threads), C.byref(tm))
    return phi, g


def direct(positions, charges, targets=None, gradient=False, threads=0):
    """O(N*M) fp64 direct sum at `targets` (indices) or all points."""
    pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
    q = np.ascontiguousarray(charges, dtype=np.float64)
    tg = None if targets is None else np.ascontiguousarray(targets, dtype=np.int64)
    m = pos.shape[0] if tg is None else tg.shape[0]
    phi = np.zeros(m)
    g = np.zeros((m, 3)) if gradient else None
    _lib.oracle_direct(pos.ctypes.data, q.ctypes.data, pos.shape[0], _ptr(tg), m, phi.ctypes.data, _ptr(g),
                       int(threads))
    return (phi, g) if gradient else phi


class Csr(C.Structure):
    _fields_ = [("u_ptr", C.POINTER(i64)), ("u_idx", C.POINTER(i64)), ("v_ptr", C.POINTER(i64)),
                ("v_idx", C.POINTER(i64)), ("v_tv", C.POINTER(i32)), ("w_ptr", C.POINTER(i64)),
                ("w_idx", C.POINTER(i64)), ("x_ptr", C.POINTER(i64)), ("x_idx", C.POINTER(i64)),
                ("n_u", i64), ("n_v", i64), ("n_w", i64), ("n_x", i64)]


_lib.oracle_lists_subset.argtypes = [P, i64, P, i64, P, i32, C.POINTER(Csr)]
_lib.oracle_csr_free.argtypes = [C.POINTER(Csr)]
_lib.oracle_csr_free.restype = None


def lists_for(tree, leaf_targets=None, node_targets=None, threads=0):
    """Brute-force U/W (per target leaf) and V/X (per target node) lists from the SPEC definitions,
    as CSR rows in the order of the given targets (all leaves / all nodes when None)."""
    lt = np.arange(tree.n_leaves, dtype=np.int64) if leaf_targets is None else np.ascontiguousarray(
        leaf_targets, dtype=np.int64)
    nt = np.arange(tree.n_nodes, dtype=np.int64) if node_targets is None else np.ascontiguousarray(
        node_targets, dtype=np.int64)
    c = Csr()
    rc = _lib.oracle_lists_subset(C.addressof(tree.view), lt.size, lt.ctypes.data, nt.size, nt.ctypes.data,
                                  int(threads), C.byref(c))
    if rc != 0:
        raise RuntimeError(f"oracle_lists_subset failed ({rc})")

    def arr(p, n, dt):
        return np.ctypeslib.as_array(p, shape=(int(n),)).astype(dt, copy=True) if n else np.zeros(0, dt)
    try:
        out = {"u": (arr(c.u_ptr, lt.size + 1, np.int64), arr(c.u_idx, c.n_u, np.int64)),
               "v": (arr(c.v_ptr, nt.size + 1, np.int64), arr(c.v_idx, c.n_v, np.int64),
                     arr(c.v_tv, c.n_v, np.int32)),
               "w": (arr(c.w_ptr, lt.size + 1, np.int64), arr(c.w_idx, c.n_w, np.int64)),
               "x": (arr(c.x_ptr, nt.size + 1, np.int64), arr(c.x_idx, c.n_x, np.int64))}
    finally:
        _lib.oracle_csr_free(C.byref(c))
    return out


def lists_bruteforce(tree, threads=0):
    """Brute-force U/V/W/X CSR of the whole tree (every leaf / node a target)."""
    return lists_for(tree, None, None, threads)


def tree_leaves(positions, n_crit, domain, balance=True):
    """Brute-force recursive split + pairwise balance; sorted leaf keys."""
    pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
    origin, side = domain
    dom = np.array(list(origin) + [side], dtype=np.float64)
    out = np.zeros(max(64, 8 * pos.shape[0]), dtype=np.uint64)
    n = _lib.oracle_tree_leaves(pos.ctypes.data, pos.shape[0], int(n_crit), dom.ctypes.data, 1 if balance else 0,
                                out.ctypes.data, out.size)
    if n < 0:
        raise RuntimeError("oracle_tree_leaves failed")
    return out[:n]


def max_threads():
    """OpenMP threads the oracle uses with threads = 0 (omp_get_max_threads())."""
    return int(_lib.oracle_max_threads())


def relative_error(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64).ravel()
    b = np.ascontiguousarray(b, dtype=np.float64).ravel()
    return float(_lib.oracle_relative_error(a.ctypes.data, b.ctypes.data, a.size))
