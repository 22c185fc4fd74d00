"""TEST INFRASTRUCTURE ONLY: the oracle's inputs (LinearTree + InteractionLists + OperatorCache)
as plain numpy arrays, so a process can run the oracle without loading the product library.

`save(path, tree, ops)` writes the arrays of any objects with the attributes of
paper_2303_08394_b200.host.Tree / Operators (duck-typed: this module imports nothing from the
product); `load(path)` returns (TreeData, OperatorData) whose `.view` are ctypes structures with the
layout of kifmm_tree_view / kifmm_operator_view (include/kifmm.h), which is all oracle_* reads.
bench.py's reference arm builds the inputs in a child process (tools/ref_inputs.py) and loads them
here, so only oracle/_build/liboracle.so is mapped into the timed reference process.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double


class TreeView(C.Structure):  # kifmm_tree_view
    _fields_ = [
        ("n_particles", i64), ("depth", i32), ("n_overfull", i32), ("n_leaves", i64), ("n_nodes", i64),
        ("origin", f64 * 3), ("side", f64),
        ("positions", C.POINTER(f64)), ("original_index", C.POINTER(i64)), ("node_key", C.POINTER(u64)),
        ("level_ptr", C.POINTER(i64)), ("node_parent", C.POINTER(i64)), ("node_children", C.POINTER(i64)),
        ("node_leaf", C.POINTER(i64)), ("leaf_node", C.POINTER(i64)), ("leaf_ptr", C.POINTER(i64)),
        ("u_ptr", C.POINTER(i64)), ("u_idx", C.POINTER(i64)), ("v_ptr", C.POINTER(i64)),
        ("v_idx", C.POINTER(i64)), ("v_tv", C.POINTER(i32)), ("w_ptr", C.POINTER(i64)),
        ("w_idx", C.POINTER(i64)), ("x_ptr", C.POINTER(i64)), ("x_idx", C.POINTER(i64)),
    ]


class OperatorView(C.Structure):  # kifmm_operator_view
    _fields_ = [
        ("p", i32), ("n_e", i32), ("n_c", i32), ("reference_level", i32),
        ("alpha_inner", f64), ("alpha_outer", f64), ("svd_cutoff", f64), ("domain_side", f64),
        ("ref_half_side", f64), ("surface", C.POINTER(f64)),
        ("uc2e_rank", i32), ("uc2e_u", C.POINTER(f64)), ("uc2e_s", C.POINTER(f64)), ("uc2e_v", C.POINTER(f64)),
        ("dc2e_rank", i32), ("dc2e_u", C.POINTER(f64)), ("dc2e_s", C.POINTER(f64)), ("dc2e_v", C.POINTER(f64)),
        ("m2m", C.POINTER(f64)), ("l2l", C.POINTER(f64)), ("n_m2l", i32), ("m2l", C.POINTER(f64)),
        ("fingerprint", u64),
    ]


TREE_ARRAYS = {"positions": np.float64, "original_index": np.int64, "node_key": np.uint64, "level_ptr": np.int64,
               "node_parent": np.int64, "node_children": np.int64, "node_leaf": np.int64, "leaf_node": np.int64,
               "leaf_ptr": np.int64, "u_ptr": np.int64, "u_idx": np.int64, "v_ptr": np.int64, "v_idx": np.int64,
               "v_tv": np.int32, "w_ptr": np.int64, "w_idx": np.int64, "x_ptr": np.int64, "x_idx": np.int64}
TREE_SCALARS = ("n", "depth", "n_overfull", "n_leaves", "n_nodes", "side")
OPS_SCALARS = ("p", "n_e", "n_c", "alpha_inner", "alpha_outer", "svd_cutoff", "domain_side", "ref_half_side",
               "fingerprint")


def save(path, tree, ops, reference_level=2):
    d = {f"t_{k}": np.ascontiguousarray(getattr(tree, k), dtype=v) for k, v in TREE_ARRAYS.items()}
    d.update({f"t_{k}": np.array(getattr(tree, k)) for k in TREE_SCALARS})
    d["t_origin"] = np.array(tree.origin, dtype=np.float64)
    d.update({f"o_{k}": np.array(getattr(ops, k)) for k in OPS_SCALARS})
    d["o_reference_level"] = np.array(reference_level)
    d["o_surface"] = np.ascontiguousarray(ops.surface)
    for name in ("uc2e", "dc2e"):
        u, s, v = getattr(ops, name)
        d[f"o_{name}_u"], d[f"o_{name}_s"], d[f"o_{name}_v"] = (np.ascontiguousarray(x) for x in (u, s, v))
    for name in ("m2m", "l2l", "m2l"):
        d[f"o_{name}"] = np.ascontiguousarray(getattr(ops, name))
    np.savez(path, **d)


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class TreeData:
    """Host.Tree-shaped holder of the arrays (the attributes the oracle wrappers use)."""

    def __init__(self, z):
        for k, v in TREE_ARRAYS.items():
            setattr(self, k, np.ascontiguousarray(z[f"t_{k}"], dtype=v))
        self.n, self.depth, self.n_overfull = int(z["t_n"]), int(z["t_depth"]), int(z["t_n_overfull"])
        self.n_leaves, self.n_nodes, self.side = int(z["t_n_leaves"]), int(z["t_n_nodes"]), float(z["t_side"])
        self.origin = tuple(float(x) for x in z["t_origin"])
        v = self.view = TreeView()
        v.n_particles, v.depth, v.n_overfull = self.n, self.depth, self.n_overfull
        v.n_leaves, v.n_nodes, v.side = self.n_leaves, self.n_nodes, self.side
        v.origin = (f64 * 3)(*self.origin)
        for k, dt in TREE_ARRAYS.items():
            ct = {np.float64: f64, np.int64: i64, np.uint64: u64, np.int32: i32}[dt]
            setattr(v, k, _p(getattr(self, k), ct))


class OperatorData:
    def __init__(self, z):
        self.p, self.n_e, self.n_c = int(z["o_p"]), int(z["o_n_e"]), int(z["o_n_c"])
        self.surface = np.ascontiguousarray(z["o_surface"])
        self.uc2e = tuple(np.ascontiguousarray(z[f"o_uc2e_{x}"]) for x in "usv")
        self.dc2e = tuple(np.ascontiguousarray(z[f"o_dc2e_{x}"]) for x in "usv")
        self.m2m, self.l2l, self.m2l = (np.ascontiguousarray(z[f"o_{x}"]) for x in ("m2m", "l2l", "m2l"))
        v = self.view = OperatorView()
        v.p, v.n_e, v.n_c, v.reference_level = self.p, self.n_e, self.n_c, int(z["o_reference_level"])
        for k in ("alpha_inner", "alpha_outer", "svd_cutoff", "domain_side", "ref_half_side"):
            setattr(v, k, float(z[f"o_{k}"]))
        v.fingerprint = int(z["o_fingerprint"])
        v.surface = _p(self.surface, f64)
        v.uc2e_rank, v.dc2e_rank = self.uc2e[1].size, self.dc2e[1].size
        v.uc2e_u, v.uc2e_s, v.uc2e_v = (_p(a, f64) for a in self.uc2e)
        v.dc2e_u, v.dc2e_s, v.dc2e_v = (_p(a, f64) for a in self.dc2e)
        v.m2m, v.l2l, v.m2l = _p(self.m2m, f64), _p(self.l2l, f64), _p(self.m2l, f64)
        v.n_m2l = self.m2l.shape[0]


def load(path):
    with np.load(path) as z:
        return TreeData(z), OperatorData(z)
