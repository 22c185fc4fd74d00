"""Benchmark of the B200 KIFMM evaluate (BASELINE.json metric).

Workload (N=1 GPU): BASELINE config 2 -- 1,000,000 points uniform in [0,1]^3,
fp32 charges U[0,1), p=6 (n_e=152), n_crit=150 (uniform depth 5), potential +
gradient, fp32.  Synthetic seeded data (splitmix64, generators.py).

  value : points/s of the evaluate with charges already resident in HBM
          (device pointers, CUDA events on the launch stream, L2 flushed with a
          256 MiB write between timed steps), max over ranks.
  e2e   : points/s through the public API with pinned host buffers, every step
          copying its charges in and its potential & gradient out: K steps as one
          Fmm.evaluate_many_ptr call over K charge vectors (H2D / evaluate / D2H
          pipelined on three streams), wall clock.  e2e.single_call: one synchronous
          Fmm.evaluate_ptr per step (no overlap).
  roofline: the dominant kernel (M2L) -- useful flops 2*n_e*n_c per V pair over
          its measured launch time, against the measured peak of the unit it uses.
  cpu_baseline: the fp64 C++ oracle (restatement of SPEC.md) on all host cores,
          full evaluates (mean of 3).

`--impl reference` times that CPU restatement alone -- full evaluates, inputs built
in a child process so only liboracle.so is mapped (the reference ships no runnable
FMM) -- and prints the same JSON schema with "impl": "reference".
For N > 1 (torchrun, or `--gpus N` alone: bench.py then starts N ranks itself) the
leaves are Morton-partitioned across ranks (strong scaling of the same 1M-point
problem) with an NCCL all-gather of halo multipoles.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = 2
# BASELINE.json configs (mirrors paper_2303_08394_b200.generators.CONFIGS, which the reference arm must not
# import: importing the package maps the product library)
CONFIGS_META = {
    1: dict(kind="uniform-cube", p=5, n_crit=64, gradient=False),
    2: dict(kind="uniform-cube", p=6, n_crit=150, gradient=True),
    3: dict(kind="sphere-surface", p=6, n_crit=150, gradient=False),
    4: dict(kind="uniform-cube", p=7, n_crit=150, gradient=False),
    5: dict(kind="uniform-cube", p=6, n_crit=128, gradient=False),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=CONFIG)
    ap.add_argument("--m2l-backend", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def metric_name(config):
    """BASELINE.json's metric for the configuration it is quoted on (config 2); other configs say which."""
    if config == CONFIG:
        return "FMM evaluate points/sec at N=1M p=6"
    return f"FMM evaluate points/sec (BASELINE config {config})"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Clocks:
    """nvidia-smi sampler around the timed region (B200_PROFILING.md clocks line).

    Samples carry nvidia-smi's own timestamp; summary() keeps only those taken
    between the wall-clock bounds of the timed loop."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.out = ""
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        import datetime
        sm, mx, reasons, n_all = [], None, set(), 0
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 10:
                continue
            n_all += 1
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                clk, cmax = float(f[2]), float(f[3])
            except ValueError:
                continue
            mx = cmax
            if self.t0 is not None and not (self.t0 - 0.05 <= ts <= (self.t1 or ts) + 0.05):
                continue
            sm.append(clk)
            for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"),
                                 f[6:10]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "samples_total": n_all}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def ncu_traffic(name):
    """Per-launch DRAM bytes of a kernel from the committed ncu summary, or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f).get(name, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def cpu_info():
    """Host CPU of the baseline run (nproc, model, OpenMP threads)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def oracle_full_evaluate(tree, ops, q_reordered, gradient, steps):
    """The fp64 C++ oracle (restatement of SPEC.md's evaluate) -- the WHOLE evaluate (P2M, M2M, M2L,
    P2L, L2L, L2P, M2P, near field over every leaf), all host threads; returns per-step seconds."""
    import oracle  # CPU baseline / reference leg only
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        oracle.evaluate(tree, ops, q_reordered, gradient=gradient, threads=0)
        times.append(time.perf_counter() - t0)
    return times


def run_reference(args):
    """Reference arm: the reference's CPU evaluate, i.e. the oracle (the reference ships no runnable FMM,
    SURVEY 0 / 8c), timed over full evaluates.  Its inputs (tree, lists, operators, charges) are built in
    a child process (tools/ref_inputs.py) and loaded from .npz, so this process maps liboracle.so only."""
    import tempfile

    rank, world, _ = dist_env()
    if rank != 0:
        return
    c = CONFIGS_META[args.config]
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, f"config{args.config}.npz")
        t0 = time.perf_counter()
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ref_inputs.py"), str(args.config), path],
                       check=True)
        setup_s = time.perf_counter() - t0
        import oracle
        from oracle import views
        tree, ops = views.load(path)
        with np.load(path) as z:
            qr = np.ascontiguousarray(z["charges_reordered"])
    steps, warm = max(1, min(args.steps, 10)), min(args.warmup, 1)
    oracle_full_evaluate(tree, ops, qr, c["gradient"], warm)
    times = oracle_full_evaluate(tree, ops, qr, c["gradient"], steps)
    t = float(np.mean(times))
    value = tree.n / t
    threads = oracle.max_threads()
    desc = (f"fp64 C++ oracle (restatement of SPEC.md's evaluate), the full evaluate of all {tree.n} points "
            f"({tree.n_leaves} leaves) per step, {threads} OpenMP threads; mean of {steps} steps after {warm} "
            f"warm-up (std {float(np.std(times)) * 1e3:.1f} ms); tree/lists/operators built in a child process")
    line = {
        "impl": "reference", "metric": metric_name(args.config), "value": value, "unit": "points/s",
        "n_gpus": world, "steps": steps, "warmup": warm, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"BASELINE config {args.config}: N={tree.n} {c['kind']}, p={c['p']}, "
                               f"n_crit={c['n_crit']}, gradient={c['gradient']}", "parallelism": "cpu-openmp",
                   "steps_requested": args.steps, "warmup_requested": args.warmup},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": threads, "kind": "port", "sample": desc,
                         **cpu_info(), "omp_max_threads": threads},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup_s": round(setup_s, 2),
    }
    print(json.dumps(line), flush=True)


def _free_port():
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def _rank_entry(rank, argv, world, port):
    os.environ.update({"RANK": str(rank), "LOCAL_RANK": str(rank), "WORLD_SIZE": str(world),
                       "LOCAL_WORLD_SIZE": str(world), "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    sys.argv = argv
    main()


def main():
    args = parse()
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is not None and int(env_world) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}; refusing to time a different "
                 "number of GPUs than requested")
    if args.impl == "reference":
        return run_reference(args)  # rank 0 only; CPU
    if env_world is None and args.gpus > 1:
        # not launched by torchrun: start one process per GPU ourselves (rendezvous on 127.0.0.1)
        import torch
        import torch.multiprocessing as mp
        if torch.cuda.device_count() < args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but only {torch.cuda.device_count()} CUDA devices visible")
        mp.spawn(_rank_entry, args=(list(sys.argv), args.gpus, _free_port()), nprocs=args.gpus, join=True)
        return

    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2303_08394_b200 import fmm, generators

    c = generators.CONFIGS[args.config]
    pos, q = generators.config_sample(args.config)
    n = pos.shape[0]
    prec = c["precision"]
    tdt = torch.float32 if prec == 32 else torch.float64
    ndt = np.float32 if prec == 32 else np.float64

    uid = None
    if world > 1:
        from paper_2303_08394_b200._lib import lib
        import ctypes
        buf = ctypes.create_string_buffer(128)
        if rank == 0:
            lib.kifmm_gpu_nccl_unique_id(buf)
        obj = [bytes(buf.raw)]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]

    cfg = fmm.FmmConfig(p=c["p"], n_crit=c["n_crit"], precision=prec, gradient=c["gradient"], device=local,
                        m2l_backend=args.m2l_backend, rank=rank, world_size=world, nccl_unique_id=uid)
    f = fmm.Fmm(pos, cfg)
    info = f.info()
    setup = {k: round(v, 3) for k, v in f.timings.items()}  # host tree + lists, operator precompute, plan

    # ---- device-resident run (value)
    dq = torch.from_numpy(q.astype(ndt)).to("cuda")
    dpot = torch.empty(n, dtype=tdt, device="cuda")
    dgrad = torch.empty((n, 3), dtype=tdt, device="cuda") if c["gradient"] else None
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.Stream()  # explicit non-default stream: plan kernels and timing events share it
    torch.cuda.set_stream(stream)
    sp = stream.cuda_stream

    def step():
        f.evaluate_device(dq.data_ptr(), dpot.data_ptr(), dgrad.data_ptr() if dgrad is not None else None,
                          input_order=True, stream=sp)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with Clocks(local) as clk:
        time.sleep(0.5)  # let the sampler start before the timed region
        clk.mark_start()
        for i in range(args.steps):
            flush.fill_(float(i))  # L2 flush between timed steps (256 MiB > 126 MB L2)
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize()
        clk.mark_end()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = float(sum(step_ms))
    if dist:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    ms_per_step = total_ms / args.steps
    value = n / (ms_per_step * 1e-3)

    # ---- per-phase device times (same kernels, events between phases, not graph-captured)
    phases = []
    qh = q.astype(ndt)
    for _ in range(10):
        _, _, tm = f.evaluate(qh, timed=True)
        phases.append(tm)
    ph = {k: float(np.mean([p[k] for p in phases])) for k in phases[0]}

    # ---- end-to-end through the public API with pinned host buffers (e2e)
    hq = torch.from_numpy(qh).pin_memory()
    hpot = torch.empty(n, dtype=tdt).pin_memory()
    hgrad = torch.empty((n, 3), dtype=tdt).pin_memory() if c["gradient"] else None
    for _ in range(args.warmup):
        f.evaluate_ptr(hq.data_ptr(), hpot.data_ptr(), hgrad.data_ptr() if hgrad is not None else None)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        f.evaluate_ptr(hq.data_ptr(), hpot.data_ptr(), hgrad.data_ptr() if hgrad is not None else None)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_single = n * args.steps / e2e_s
    # pipelined: the same K steps as ONE evaluate_many call over K right-hand sides (a ring of 4 pinned
    # host input / output buffer sets); every step still copies its charges in and its results out
    ring = 4
    rq = [torch.from_numpy(qh).pin_memory() for _ in range(ring)]
    rpot = [torch.empty(n, dtype=tdt).pin_memory() for _ in range(ring)]
    rgrad = [torch.empty((n, 3), dtype=tdt).pin_memory() for _ in range(ring)] if c["gradient"] else None

    def many(k):
        f.evaluate_many_ptr([rq[i % ring].data_ptr() for i in range(k)], [rpot[i % ring].data_ptr() for i in range(k)],
                            [rgrad[i % ring].data_ptr() for i in range(k)] if rgrad is not None else None)

    many(max(args.warmup, 2))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    many(args.steps)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = n * args.steps / e2e_s
    if not np.array_equal(rpot[(args.steps - 1) % ring].numpy(), hpot.numpy()):
        raise RuntimeError("evaluate_many result differs from evaluate")
    esz = 4 if prec == 32 else 8
    h2d = n * esz
    d2h = n * esz * (4 if c["gradient"] else 1)

    if rank != 0:
        f.close()
        if dist:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (M2L)
    peaks = measured_peaks()
    n_e = info["n_e"]
    m2l_flops = 2.0 * n_e * info["n_c"] * info["m2l_pairs"]
    m2l_s = ph["m2l_ms"] * 1e-3
    achieved = m2l_flops / m2l_s / 1e12 if m2l_s > 0 else 0.0
    if info["m2l_backend"] == 2:
        bf16 = peaks.get("bf16_tflops", 1590.0)
        peak, bound, src = bf16 / 3.0, "tensor", ("measured dense bf16 (= fp16 kind::f16 rate) / 3: the 3-term "
                                                  "fp16 split issues 3 MMAs per useful MAC; " +
                                                  ("of measured" if peaks else "of fallback"))
    elif info["m2l_backend"] == 3:
        tf32 = peaks.get("bf16_tflops", 1590.0) / 2.0
        peak, bound, src = tf32 / 3.0, "tensor", ("measured bf16/2 (TF32) / 3 (3xTF32 issues 3 MMAs per "
                                                  "useful MAC), " + ("of measured" if peaks else "of fallback"))
    elif info["m2l_backend"] == 4:
        # int8 Ozaki scheme: 36 digit-slice products per useful fp64 MAC at 2x the bf16 MMA rate
        i8 = 2.0 * peaks.get("bf16_tflops", 1590.0)
        peak, bound, src = i8 / 36.0, "tensor", ("measured dense bf16 x 2 (kind::i8 rate) / 36: the 8-slice Ozaki "
                                                 "scheme issues 36 int8 MMAs per useful fp64 MAC; " +
                                                 ("of measured" if peaks else "of fallback"))
    else:
        fp32 = fmm.fma_peak(32, local) / 1e12
        peak, bound, src = fp32, "tensor", ("FP32 SIMT kernel: peak = FFMA throughput measured in this run "
                                            "(MEASURED_PEAKS.json has no FP32 entry); 'tensor' here means the "
                                            "compute roof, not tensor cores")
    roof = {"bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak if peak else None, "traffic": ncu_traffic("m2l"),
            "kernel": {1: "M2L (gather_gemm_kernel / gather_dmma_kernel)", 4: "M2L (m2l_oz_kernel)"}.get(
                info["m2l_backend"], "M2L (m2l_tc_kernel)"),
            "peak_source": src,
            "work": f"2*n_e*n_c flop per V pair x {info['m2l_pairs']} V pairs per launch",
            "m2l_ms": ph["m2l_ms"]}
    p2p_pairs = info["near_pairs"] + info["l2p_pairs"] + info["m2p_pairs"]
    pair_flops = 19.0 if c["gradient"] else 11.0
    fp32_peak = fmm.fma_peak(32, local) / 1e12 if prec == 32 else fmm.fma_peak(64, local) / 1e12
    p2p = {"achieved_tflops": p2p_pairs * pair_flops / (ph["leaf_ms"] * 1e-3) / 1e12 if ph["leaf_ms"] else None,
           "peak_tflops": fp32_peak, "pairs": p2p_pairs, "flop_per_pair": pair_flops, "leaf_ms": ph["leaf_ms"]}
    p2p["frac"] = p2p["achieved_tflops"] / fp32_peak if p2p["achieved_tflops"] else None
    # nominal: SMs x 128 FP32 lanes (64 FP64) x 2 flop x max SM clock; the FFMA probe above
    # runs at whatever clock the power cap allows at that moment
    nominal = torch.cuda.get_device_properties(local).multi_processor_count * (128 if prec == 32 else 64) * 2 * \
        (clk.summary().get("sm_max_mhz") or 1965.0) * 1e6 / 1e12
    p2p["peak_nominal_tflops"] = nominal
    p2p["frac_nominal"] = p2p["achieved_tflops"] / nominal if p2p["achieved_tflops"] else None
    p2p["span"] = "near field (self + U list) and far field (L2P + M2P) kernels of the serialized timed run"

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        import oracle
        qr = q[f.tree.original_index]
        ts = oracle_full_evaluate(f.tree, f.operators, qr, c["gradient"], 3)
        th = oracle.max_threads()
        cpu = {"value": n / float(np.mean(ts)), "unit": "points/s", "cores": th, "kind": "port",
               "sample": f"fp64 C++ oracle, the full evaluate of all {n} points per step, {th} OpenMP threads, "
                         f"mean of 3 (std {float(np.std(ts)) * 1e3:.1f} ms)", **cpu_info(), "omp_max_threads": th}

    line = {
        "metric": metric_name(args.config), "value": value, "unit": "points/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32" if prec == 32 else "f64", "data": "synthetic",
        "config": {"workload": f"BASELINE config {args.config}: N={n} {c['kind']} (seed 0), p={c['p']}, "
                               f"n_crit={c['n_crit']}, gradient={c['gradient']}, depth {f.tree.depth}, "
                               f"{f.tree.n_leaves} leaves",
                   "parallelism": f"morton-range x{world}" if world > 1 else "single-gpu",
                   "l2": "flushed (256 MiB write) between timed steps",
                   "m2l_backend": {1: "simt/dmma", 2: "tcgen05-f16x3", 3: "tcgen05-3xtf32",
                                   4: "tcgen05-i8-ozaki"}.get(info["m2l_backend"])},
        "e2e": {"value": e2e, "unit": "points/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "Fmm.evaluate_many_ptr (kifmm_gpu_evaluate_many): K steps = K charge vectors from pinned "
                       "host buffers, H2D / evaluate / D2H pipelined on three streams; wall clock",
                "single_call": {"value": e2e_single, "unit": "points/s",
                                "api": "Fmm.evaluate_ptr (kifmm_gpu_evaluate) once per step, synchronous"}},
        "gpu_launches": int(info["kernel_launches"]) * args.steps,
        "setup_s": dict(setup, note="tree_s: host C++ tree + U/V/W/X lists; precompute_s: operator cache (SVDs, "
                                    "K_t); plan_s: GPU plan creation (upload, work lists, warm-up); all outside "
                                    "the timed evaluate window (SURVEY 8d)"),
        "roofline": roof, "p2p": p2p, "phases_ms": ph, "clocks": clk.summary(), "cpu_baseline": cpu,
        "plan": {k: info[k] for k in ("n_leaves", "n_nodes", "near_pairs", "m2l_pairs", "m2l_padded_pairs",
                                      "device_bytes", "kernel_launches")},
    }
    print(json.dumps(line), flush=True)
    f.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
