"""The product's multi-rank device path on the GPU.

One-GPU emulation (always runs): world_size plans -- one per rank, all on device 0, built with
exchange = 1 -- run their upward halves (P2M, M2M of the owned subtrees, export rows gathered by
gather_rows_kernel), the test all-gathers the export rows on the host exactly as ncclAllGather lays them
out (slot r = rank r's rows), and each plan runs its downward half (scatter of the other ranks' rows +
their fp16 split, recomputed spanning nodes, M2L / P2L / L2L, leaves).  Everything but the NCCL call
itself is the product path; the ranks never wait on one another (the host exchange sits between two
synchronous calls).  Their combined output must equal the single-rank evaluate to fp64 rounding (fp64)
or fp32 accumulation-order differences (fp32), and the oracle within the parity gates.

Two GPUs (skipped on a one-GPU box): the same through NCCL, one process per GPU.
"""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2303_08394_b200 import fmm, generators

pytestmark = pytest.mark.gpu


def _emulated(pos, q, cfg_kw, world, input_order=True):
    plans = [fmm.Fmm(pos, fmm.FmmConfig(**cfg_kw, rank=r, world_size=world, exchange=1)) for r in range(world)]
    try:
        info = [p.info() for p in plans]
        dt = plans[0].dtype
        qq = q if input_order else q[plans[0].tree.original_index]
        sends = [p.evaluate_upward(qq.astype(dt), input_order=input_order) for p in plans]
        hm = info[0]["halo_rows_max"]
        gathered = np.zeros((world, max(1, hm), info[0]["ne_pad"]), dtype=dt)
        for r, s in enumerate(sends):
            gathered[r, :s.shape[0]] = s
        outs = [p.evaluate_downward(gathered) for p in plans]
        for p in plans:  # device spans of the two halves (kifmm_gpu_last_timings; tools/scale_projection.py)
            tm = p.last_timings()
            assert tm["upward_ms"] > 0 and tm["downward_ms"] > 0
        return outs, info, plans[0].tree
    finally:
        for p in plans:
            p.close()


CASES = [("uniform-cube", 60000, 40, 6, 32, 2), ("two-cluster", 50000, 20, 6, 32, 3),
         ("sphere-surface", 60000, 40, 6, 32, 4), ("two-cluster", 30000, 20, 5, 64, 2),
         ("uniform-cube", 40000, 30, 7, 64, 3)]


@pytest.mark.parametrize("kind,n,n_crit,p,precision,world", CASES)
def test_host_exchange_ranks_match_single_rank(require_gpu, kind, n, n_crit, p, precision, world):
    pos, q = generators.sample(kind, n, seed=17, charges="signed", fp32=precision == 32)
    kw = dict(p=p, n_crit=n_crit, precision=precision, gradient=True)
    with fmm.Fmm(pos, fmm.FmmConfig(**kw)) as f:
        pot1, grad1, _ = f.evaluate(q)
        qr = q[f.tree.original_index]
        ref, gref, _ = oracle.evaluate(f.tree, f.operators, qr, gradient=True)
        inv = np.empty_like(f.tree.original_index)
        inv[f.tree.original_index] = np.arange(f.tree.n)
        ref, gref = ref[inv], gref[inv]
    outs, info, tree = _emulated(pos, q, kw, world)
    # input order: every rank writes its own particles and zeros elsewhere
    pot = np.sum([o[0] for o in outs], axis=0)
    grad = np.sum([o[1] for o in outs], axis=0)
    owned = np.zeros(tree.n, int)
    for i in info:
        owned[tree.original_index[i["owned_particle_begin"]:i["owned_particle_end"]]] += 1
    assert np.all(owned == 1)
    assert all(i["halo_rows_mine"] <= i["halo_rows_max"] for i in info)
    same = 1e-13 if precision == 64 else 2e-6
    assert fmm.relative_error(pot, pot1) <= same and fmm.relative_error(grad, grad1) <= 10 * same
    gate_p, gate_g = (1e-12, 1e-11) if precision == 64 else (1e-5, 5e-5)
    assert fmm.relative_error(pot, ref) <= gate_p and fmm.relative_error(grad, gref) <= gate_g


def test_host_exchange_reordered_output(require_gpu):
    """input_order = 0: each rank writes only its contiguous reordered particle range."""
    pos, q = generators.sample("two-cluster", 40000, seed=19, charges="signed")
    kw = dict(p=5, n_crit=20, precision=64, gradient=False)
    with fmm.Fmm(pos, fmm.FmmConfig(**kw)) as f:
        ref, _, _ = f.evaluate(q[f.tree.original_index], input_order=False)
    outs, info, tree = _emulated(pos, q, kw, 3, input_order=False)
    got = np.zeros(tree.n)
    for (pot, _), i in zip(outs, info):
        a, b = i["owned_particle_begin"], i["owned_particle_end"]
        assert not np.any(np.delete(pot, np.arange(a, b)))
        got[a:b] = pot[a:b]
    assert fmm.relative_error(got, ref) <= 1e-13


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _nccl_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    from paper_2303_08394_b200._lib import lib
    import ctypes
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    buf = ctypes.create_string_buffer(128)
    if rank == 0:
        lib.kifmm_gpu_nccl_unique_id(buf)
    obj = [bytes(buf.raw)]
    dist.broadcast_object_list(obj, src=0)
    pos, q = generators.sample("uniform-cube", 200000, seed=23, charges="signed", fp32=True)
    cfg = fmm.FmmConfig(p=6, n_crit=60, precision=32, gradient=True, device=rank, rank=rank, world_size=world,
                        nccl_unique_id=obj[0])
    with fmm.Fmm(pos, cfg) as f:
        pot, grad, _ = f.evaluate(q)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), pot=pot, grad=grad)
    dist.destroy_process_group()


def test_nccl_two_gpus_match_single_rank(require_gpu, tmp_path):
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (this pool leases one; the one-GPU emulation above covers the device path)")
    mp.spawn(_nccl_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    pos, q = generators.sample("uniform-cube", 200000, seed=23, charges="signed", fp32=True)
    with fmm.Fmm(pos, fmm.FmmConfig(p=6, n_crit=60, precision=32, gradient=True)) as f:
        pot1, grad1, _ = f.evaluate(q)
    r = [np.load(tmp_path / f"r{k}.npz") for k in range(2)]
    assert fmm.relative_error(r[0]["pot"] + r[1]["pot"], pot1) <= 2e-6
    assert fmm.relative_error(r[0]["grad"] + r[1]["grad"], grad1) <= 2e-5
