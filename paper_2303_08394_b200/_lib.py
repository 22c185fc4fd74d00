"""ctypes binding of libkifmm_b200.so (include/kifmm.h).

The library is built in-tree (`make lib`, or __graft_entry__.build()).  There
is no fallback: if the shared object is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

from .errors import STATUS_TO_ERROR, KifmmError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KIFMM_LIB") or os.path.join(_HERE, "lib", "libkifmm_b200.so")  # override: experiments

i32, i64, u64, f32, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double
P = C.c_void_p


class TreeView(C.Structure):
    _fields_ = [
        ("n_particles", i64), ("depth", i32), ("n_overfull", i32),
        ("n_leaves", i64), ("n_nodes", i64),
        ("origin", f64 * 3), ("side", f64),
        ("positions", C.POINTER(f64)), ("original_index", C.POINTER(i64)),
        ("node_key", C.POINTER(u64)), ("level_ptr", C.POINTER(i64)),
        ("node_parent", C.POINTER(i64)), ("node_children", C.POINTER(i64)),
        ("node_leaf", C.POINTER(i64)), ("leaf_node", C.POINTER(i64)),
        ("leaf_ptr", C.POINTER(i64)),
        ("u_ptr", C.POINTER(i64)), ("u_idx", C.POINTER(i64)),
        ("v_ptr", C.POINTER(i64)), ("v_idx", C.POINTER(i64)), ("v_tv", C.POINTER(i32)),
        ("w_ptr", C.POINTER(i64)), ("w_idx", C.POINTER(i64)),
        ("x_ptr", C.POINTER(i64)), ("x_idx", C.POINTER(i64)),
    ]


class OperatorView(C.Structure):
    _fields_ = [
        ("p", i32), ("n_e", i32), ("n_c", i32), ("reference_level", i32),
        ("alpha_inner", f64), ("alpha_outer", f64), ("svd_cutoff", f64),
        ("domain_side", f64), ("ref_half_side", f64),
        ("surface", C.POINTER(f64)),
        ("uc2e_rank", i32), ("uc2e_u", C.POINTER(f64)), ("uc2e_s", C.POINTER(f64)), ("uc2e_v", C.POINTER(f64)),
        ("dc2e_rank", i32), ("dc2e_u", C.POINTER(f64)), ("dc2e_s", C.POINTER(f64)), ("dc2e_v", C.POINTER(f64)),
        ("m2m", C.POINTER(f64)), ("l2l", C.POINTER(f64)),
        ("n_m2l", i32), ("m2l", C.POINTER(f64)),
        ("fingerprint", u64),
    ]


class HaloView(C.Structure):
    _fields_ = [
        ("world_size", i32), ("cut_level", i32), ("n_nodes", i64),
        ("leaf_begin", C.POINTER(i64)), ("up_owner", C.POINTER(i32)),
        ("export_ptr", C.POINTER(i64)), ("export_idx", C.POINTER(i64)), ("max_export", i64),
    ]


class GpuOptions(C.Structure):
    _fields_ = [
        ("precision", i32), ("gradient", i32), ("device", i32), ("rank", i32),
        ("world_size", i32), ("cut_level", i32), ("nccl_unique_id", P),
        ("m2l_backend", i32), ("use_graph", i32), ("exchange", i32),
    ]


class GpuTimings(C.Structure):
    _fields_ = [(n, f32) for n in (
        "total_ms", "upload_ms", "p2m_ms", "m2m_ms", "exchange_ms", "p2l_ms", "m2l_ms",
        "down_solve_ms", "l2l_ms", "leaf_ms", "download_ms", "upward_ms", "downward_ms")]

    def as_dict(self):
        return {n: float(getattr(self, n)) for n, _ in self._fields_}


class GpuPlanInfo(C.Structure):
    _fields_ = [
        ("n_particles", i64), ("n_leaves", i64), ("n_nodes", i64),
        ("owned_leaf_begin", i64), ("owned_leaf_end", i64),
        ("owned_particle_begin", i64), ("owned_particle_end", i64),
        ("near_pairs", i64), ("l2p_pairs", i64), ("m2p_pairs", i64), ("p2m_pairs", i64), ("p2l_pairs", i64),
        ("m2l_pairs", i64), ("m2l_padded_pairs", i64),
        ("n_e", i32), ("n_c", i32), ("ne_pad", i32), ("m2l_backend", i32),
        ("device_bytes", i64), ("kernel_launches", i32), ("halo_rows_max", i64), ("halo_rows_mine", i64),
        ("m2m_levels", i32), ("m2l_levels", i32), ("l2l_levels", i32), ("m2l_launch_levels", i32),
        ("p2m_leaves", i64), ("near_leaves", i64), ("l2p_leaves", i64), ("m2p_leaves", i64), ("p2l_nodes", i64),
    ]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -j lib` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    return C.CDLL(LIB_PATH)


lib = _load()

_SIGS = {
    "kifmm_last_error": (C.c_char_p, []),
    "kifmm_version": (C.c_char_p, []),
    "kifmm_morton_encode": (i32, [C.POINTER(C.c_uint32), i32, C.POINTER(u64)]),
    "kifmm_morton_decode": (i32, [u64, C.POINTER(C.c_uint32), C.POINTER(i32)]),
    "kifmm_morton_parent": (i32, [u64, C.POINTER(u64)]),
    "kifmm_morton_children": (i32, [u64, C.POINTER(u64)]),
    "kifmm_morton_neighbors": (i32, [u64, C.POINTER(u64)]),
    "kifmm_morton_is_adjacent": (i32, [u64, u64]),
    "kifmm_morton_node_bounds": (None, [u64, C.POINTER(f64), f64, C.POINTER(f64), C.POINTER(f64)]),
    "kifmm_laplace": (f64, [C.POINTER(f64), C.POINTER(f64)]),
    "kifmm_kernel_matrix": (None, [P, i64, P, i64, P]),
    "kifmm_surface_count": (i32, [i32]),
    "kifmm_surface_grid": (i32, [i32, P]),
    "kifmm_tree_build": (i32, [P, i64, i32, P, i32, i32, C.POINTER(P)]),
    "kifmm_tree_get_view": (i32, [P, C.POINTER(TreeView)]),
    "kifmm_tree_destroy": (None, [P]),
    "kifmm_transfer_vectors": (i32, [P]),
    "kifmm_partition_leaves": (i32, [C.POINTER(TreeView), i32, i32, i32, i32, P]),
    "kifmm_halo_plan": (i32, [C.POINTER(TreeView), i32, i32, i32, i32, C.POINTER(P)]),
    "kifmm_halo_get_view": (i32, [P, C.POINTER(HaloView)]),
    "kifmm_halo_destroy": (None, [P]),
    "kifmm_precompute": (i32, [i32, f64, f64, f64, f64, i32, C.POINTER(P)]),
    "kifmm_operators_get_view": (i32, [P, C.POINTER(OperatorView)]),
    "kifmm_operators_destroy": (None, [P]),
    "kifmm_operators_save": (i32, [P, C.c_char_p]),
    "kifmm_operators_load": (i32, [C.c_char_p, u64, C.POINTER(P)]),
    "kifmm_svd": (i32, [P, i32, i32, P, P, P]),
    "kifmm_gpu_plan_create": (i32, [C.POINTER(GpuOptions), C.POINTER(TreeView), C.POINTER(OperatorView),
                                    C.POINTER(P)]),
    "kifmm_gpu_evaluate": (i32, [P, P, P, P, i32, C.POINTER(GpuTimings)]),
    "kifmm_gpu_evaluate_device": (i32, [P, P, P, P, i32, P]),
    "kifmm_gpu_evaluate_many": (i32, [P, i32, C.POINTER(P), C.POINTER(P), C.POINTER(P), i32]),
    "kifmm_gpu_evaluate_upward": (i32, [P, P, i32, P]),
    "kifmm_gpu_evaluate_downward": (i32, [P, P, P, P]),
    "kifmm_gpu_plan_get_info": (i32, [P, C.POINTER(GpuPlanInfo)]),
    "kifmm_gpu_last_timings": (i32, [P, C.POINTER(GpuTimings)]),
    "kifmm_gpu_plan_destroy": (None, [P]),
    "kifmm_gpu_nccl_unique_id": (i32, [P]),
    "kifmm_gpu_direct": (i32, [i32, i32, P, P, i64, P, i64, P, P]),
    "kifmm_gpu_fma_peak": (i32, [i32, i32, C.POINTER(f64)]),
}

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED = tuple(_SIGS)


def last_error() -> str:
    msg = lib.kifmm_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "") -> None:
    """Raise the reference-taxonomy exception for a non-zero status."""
    if status == 0:
        return
    cls = STATUS_TO_ERROR.get(int(status), KifmmError)
    msg = last_error()
    raise cls(f"{what}: {msg}" if what else msg)
