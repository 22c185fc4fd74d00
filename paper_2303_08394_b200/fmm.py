"""The orchestrator: `Fmm` plan object and `run`.

Mirrors the reference's single API object (Fig. 2):
host C++ builds tree, lists and the operator cache; the evaluate section of
`run` ("zero state -> upward -> downward -> permute back") is the
GPU plan behind the kifmm_gpu_* C ABI.  There is no CPU evaluate in this
package: without a CUDA device `Fmm` raises DeviceError.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import time

import numpy as np

from . import _lib, host
from ._lib import check, lib
from .errors import CacheMismatch, CorruptArchive, InvalidArgument


@dataclasses.dataclass
class FmmConfig:
    """FmmConfig plus the GPU knobs of SURVEY 5 ("precision, gradient, n_gpus")."""
    p: int = 6
    n_crit: int = 150
    alpha_inner: float = 1.05
    alpha_outer: float = 2.95
    svd_cutoff: float = 1e-12        # SPEC default (an fp64 setting); fp32 plans at p = 7 need ~1e-8 (tests/test_gpu.py)
    threads: int = 0                 # host threads for tree/lists/precompute (0 = all)
    precision: int = 32              # 32 or 64
    gradient: bool = False
    device: int = 0
    m2l_backend: int = 0             # 0 auto, 1 SIMT / fp64 DMMA, 2 tcgen05 (fp32, p = 4..7: fp16 3-term split; tf32 via KIFMM_TC_KIND),
    #                                  4 tcgen05 int8 Ozaki scheme (fp64, p = 6, 7; the fp64 default there)
    use_graph: bool = True
    rank: int = 0
    world_size: int = 1
    cut_level: int = 0                # multi-GPU partition alignment level (0 = auto)
    nccl_unique_id: bytes | None = None
    exchange: int = 0                # world_size > 1: 0 NCCL all-gather, 1 host (evaluate_upward / _downward)
    cache: str | None = None         # operator cache archive path

    def validate(self):
        if self.p < 2:
            raise InvalidArgument("p must be >= 2")
        if self.n_crit < 1:
            raise InvalidArgument("n_crit must be >= 1")
        if not (0 < self.alpha_inner < self.alpha_outer):
            raise InvalidArgument("need 0 < alpha_inner < alpha_outer")
        if not (0 < self.svd_cutoff < 1):
            raise InvalidArgument("svd_cutoff must be in (0, 1)")
        if self.precision not in (32, 64):
            raise InvalidArgument("precision must be 32 or 64")


def operator_fingerprint(p: int, alpha_inner: float, alpha_outer: float, svd_cutoff: float, side: float) -> int:
    """FNV-1a over (kernel id, p, alphas, cutoff, side); equals operator_fingerprint() in operators.cpp."""
    import struct
    data = b"laplace3d-1/(4pi r)-v1\x00" + struct.pack("<i", int(p)) + struct.pack(
        "<dddd", alpha_inner, alpha_outer, svd_cutoff, side)
    h = 1469598103934665603
    for b in data:
        h ^= b
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def load_or_precompute(cfg: FmmConfig, domain_side: float) -> host.Operators:
    """Cache policy of SPEC.md:544/571: load on fingerprint match, else rebuild (warn) and save."""
    if cfg.cache and os.path.exists(cfg.cache):
        fp = operator_fingerprint(cfg.p, cfg.alpha_inner, cfg.alpha_outer, cfg.svd_cutoff, domain_side)
        try:
            return host.Operators.load(cfg.cache, fp)
        except (CacheMismatch, CorruptArchive) as e:
            import warnings
            warnings.warn(f"operator cache {cfg.cache} rejected ({e}); rebuilding")
    ops = host.Operators(cfg.p, cfg.alpha_inner, cfg.alpha_outer, cfg.svd_cutoff, domain_side, cfg.threads)
    if cfg.cache:
        ops.save(cfg.cache)
    return ops


class Fmm:
    """Plan: tree + lists + operators on the host, evaluate on the GPU."""

    def __init__(self, positions, config: FmmConfig | None = None,
                 operators: host.Operators | dict | None = None, tree: host.Tree | None = None):
        """`operators`: a precomputed operator set (its domain side must equal the tree's), or a dict used as
        an in-memory operator cache keyed by fingerprint (load on fingerprint match, else
        precompute and insert) -- point clouds whose bounding cubes differ get their own entries."""
        cfg = config or FmmConfig()
        cfg.validate()
        self.config = cfg
        self.timings = {}
        t0 = time.perf_counter()
        self.tree = tree if tree is not None else host.Tree(positions, cfg.n_crit, threads=cfg.threads)
        t1 = time.perf_counter()
        if isinstance(operators, dict):
            fp = operator_fingerprint(cfg.p, cfg.alpha_inner, cfg.alpha_outer, cfg.svd_cutoff, self.tree.side)
            if fp not in operators:
                operators[fp] = load_or_precompute(cfg, self.tree.side)
            self.operators = operators[fp]
        else:
            self.operators = operators if operators is not None else load_or_precompute(cfg, self.tree.side)
        t2 = time.perf_counter()
        self.timings.update(tree_s=t1 - t0, precompute_s=t2 - t1)
        self.dtype = np.float32 if cfg.precision == 32 else np.float64
        self._uid = None
        opts = _lib.GpuOptions()
        opts.precision = cfg.precision
        opts.gradient = 1 if cfg.gradient else 0
        opts.device = cfg.device
        opts.rank = cfg.rank
        opts.world_size = cfg.world_size
        opts.cut_level = cfg.cut_level
        if cfg.nccl_unique_id is not None:
            self._uid = C.create_string_buffer(bytes(cfg.nccl_unique_id), 128)
            opts.nccl_unique_id = C.cast(self._uid, C.c_void_p)
        opts.m2l_backend = cfg.m2l_backend
        opts.use_graph = 1 if cfg.use_graph else 0
        opts.exchange = int(cfg.exchange)
        h = C.c_void_p()
        check(lib.kifmm_gpu_plan_create(C.byref(opts), C.byref(self.tree.view), C.byref(self.operators.view),
                                        C.byref(h)), "gpu_plan_create")
        self._h = h
        self.timings["plan_s"] = time.perf_counter() - t2
        self.n = self.tree.n

    # -------------------------------------------------------------- evaluate
    def evaluate(self, charges, input_order: bool = True, timed: bool = False):
        """Potentials (and gradients) for `charges` (input order by default).

        Returns (potential, gradient | None, timings | None).
        """
        q = np.ascontiguousarray(charges, dtype=self.dtype)
        if q.shape != (self.n,):
            raise InvalidArgument(f"charges must have shape ({self.n},)")
        pot = np.empty(self.n, dtype=self.dtype)
        grad = np.empty((self.n, 3), dtype=self.dtype) if self.config.gradient else None
        tm = _lib.GpuTimings() if timed else None
        check(lib.kifmm_gpu_evaluate(self._h, q.ctypes.data, pot.ctypes.data,
                                     grad.ctypes.data if grad is not None else None, 1 if input_order else 0,
                                     C.byref(tm) if tm is not None else None), "gpu_evaluate")
        return pot, grad, (tm.as_dict() if tm is not None else None)

    def evaluate_ptr(self, q_ptr: int, pot_ptr: int, grad_ptr: int | None, input_order: bool = True,
                     timed: bool = False):
        """Raw-pointer variant (host or pinned buffers, e.g. torch pinned tensors)."""
        tm = _lib.GpuTimings() if timed else None
        check(lib.kifmm_gpu_evaluate(self._h, C.c_void_p(q_ptr), C.c_void_p(pot_ptr),
                                     C.c_void_p(grad_ptr) if grad_ptr else None, 1 if input_order else 0,
                                     C.byref(tm) if tm is not None else None), "gpu_evaluate")
        return tm.as_dict() if tm is not None else None

    def evaluate_many(self, charges, input_order: bool = True):
        """Potentials (and gradients) for K independent charge vectors (array K x N), pipelined:
        the copies of one vector overlap the evaluate of its neighbours (kifmm_gpu_evaluate_many).

        Returns (potential K x N, gradient K x N x 3 | None).
        """
        q = np.ascontiguousarray(charges, dtype=self.dtype)
        if q.ndim != 2 or q.shape[1] != self.n:
            raise InvalidArgument(f"charges must have shape (K, {self.n})")
        k = q.shape[0]
        pot = np.empty((k, self.n), dtype=self.dtype)
        grad = np.empty((k, self.n, 3), dtype=self.dtype) if self.config.gradient else None
        self.evaluate_many_ptr([q[i].ctypes.data for i in range(k)], [pot[i].ctypes.data for i in range(k)],
                               [grad[i].ctypes.data for i in range(k)] if grad is not None else None, input_order)
        return pot, grad

    def evaluate_many_ptr(self, q_ptrs, pot_ptrs, grad_ptrs=None, input_order: bool = True):
        """Raw-pointer variant of evaluate_many (lists of host buffer addresses; pinned buffers overlap)."""
        k = len(q_ptrs)
        if len(pot_ptrs) != k or (grad_ptrs is not None and len(grad_ptrs) != k):
            raise InvalidArgument("evaluate_many: pointer lists differ in length")
        arr = C.c_void_p * max(k, 1)
        qa, pa = arr(*q_ptrs), arr(*pot_ptrs)
        ga = arr(*grad_ptrs) if grad_ptrs is not None else None
        check(lib.kifmm_gpu_evaluate_many(self._h, k, C.cast(qa, C.POINTER(C.c_void_p)),
                                          C.cast(pa, C.POINTER(C.c_void_p)),
                                          C.cast(ga, C.POINTER(C.c_void_p)) if ga is not None else None,
                                          1 if input_order else 0), "gpu_evaluate_many")

    def evaluate_device(self, d_charges: int, d_potential: int, d_gradient: int | None = None,
                        input_order: bool = True, stream: int | None = None):
        """Device-pointer variant; asynchronous on `stream` (cudaStream_t as int) or the plan stream."""
        check(lib.kifmm_gpu_evaluate_device(self._h, C.c_void_p(d_charges), C.c_void_p(d_potential),
                                            C.c_void_p(d_gradient) if d_gradient else None,
                                            1 if input_order else 0, C.c_void_p(stream) if stream else None),
              "gpu_evaluate_device")

    # ------------------------------------------- host-exchange multi-rank halves (exchange = 1)
    def evaluate_upward(self, charges, input_order: bool = True) -> np.ndarray:
        """Upward pass of this rank; returns its export rows (halo_rows_max x ne_pad, plan precision) for
        the caller's all-gather (kifmm_gpu_evaluate_upward)."""
        q = np.ascontiguousarray(charges, dtype=self.dtype)
        if q.shape != (self.n,):
            raise InvalidArgument(f"charges must have shape ({self.n},)")
        inf = self.info()
        rows = np.zeros((max(1, inf["halo_rows_max"]), inf["ne_pad"]), dtype=self.dtype)
        check(lib.kifmm_gpu_evaluate_upward(self._h, q.ctypes.data, 1 if input_order else 0, rows.ctypes.data),
              "gpu_evaluate_upward")
        return rows[:inf["halo_rows_max"]]

    def evaluate_downward(self, gathered):
        """Downward pass of this rank from the all-gathered rows (world_size x halo_rows_max x ne_pad);
        returns (potential, gradient | None) like evaluate() (kifmm_gpu_evaluate_downward)."""
        g = np.ascontiguousarray(gathered, dtype=self.dtype)
        pot = np.zeros(self.n, dtype=self.dtype)
        grad = np.zeros((self.n, 3), dtype=self.dtype) if self.config.gradient else None
        check(lib.kifmm_gpu_evaluate_downward(self._h, g.ctypes.data if g.size else None, pot.ctypes.data,
                                              grad.ctypes.data if grad is not None else None),
              "gpu_evaluate_downward")
        return pot, grad

    def last_timings(self) -> dict:
        """Device times of the last timed evaluate and of the last upward / downward halves
        (kifmm_gpu_last_timings)."""
        tm = _lib.GpuTimings()
        check(lib.kifmm_gpu_last_timings(self._h, C.byref(tm)), "gpu_last_timings")
        return tm.as_dict()

    def info(self) -> dict:
        inf = _lib.GpuPlanInfo()
        check(lib.kifmm_gpu_plan_get_info(self._h, C.byref(inf)), "plan_info")
        return inf.as_dict()

    def close(self):
        if getattr(self, "_h", None):
            lib.kifmm_gpu_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def run(positions, charges, config: FmmConfig | None = None):
    """SPEC.md:540 `run`: potentials in input order (+ gradient) and per-phase timings."""
    f = Fmm(positions, config)
    try:
        pot, grad, tm = f.evaluate(charges, input_order=True, timed=True)
        tm = dict(tm)
        tm.update(f.timings)
        return pot, grad, tm
    finally:
        f.close()


def direct(positions, charges, targets=None, precision: int = 64, gradient: bool = False, device: int = 0):
    """Direct summation on the GPU (verification kernel K10)."""
    dt = np.float32 if precision == 32 else np.float64
    pos = np.ascontiguousarray(positions, dtype=dt).reshape(-1, 3)
    q = np.ascontiguousarray(charges, dtype=dt)
    n = pos.shape[0]
    tg = np.arange(n, dtype=np.int64) if targets is None else np.ascontiguousarray(targets, dtype=np.int64)
    pot = np.empty(tg.shape[0], dtype=dt)
    grad = np.empty((tg.shape[0], 3), dtype=dt) if gradient else None
    check(lib.kifmm_gpu_direct(precision, device, pos.ctypes.data, q.ctypes.data, n, tg.ctypes.data, tg.shape[0],
                               pot.ctypes.data, grad.ctypes.data if grad is not None else None), "gpu_direct")
    return (pot, grad) if gradient else pot


def relative_error(a, b) -> float:
    """||a - b||_2 / ||b||_2; zero-norm reference is an error."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    if a.shape != b.shape:
        raise InvalidArgument("relative_error: length mismatch")
    nb = np.linalg.norm(b)
    if nb == 0:
        raise InvalidArgument("relative_error: zero-norm reference")
    return float(np.linalg.norm(a - b) / nb)


def fma_peak(precision: int = 32, device: int = 0) -> float:
    out = C.c_double()
    check(lib.kifmm_gpu_fma_peak(device, precision, C.byref(out)), "fma_peak")
    return out.value
