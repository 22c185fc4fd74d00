"""Projected 2/4/8-GPU evaluate time from per-rank work measured on ONE B200 (not a multi-GPU measurement).

This pool gives one GPU, so the N-GPU path cannot be timed on NVLink hardware.  What can be measured is each
rank's share of the work: for every rank r of an N-rank partition this script builds the product's rank-r plan
(`world_size = N, exchange = 1`: the halves of the evaluate with the halo exchange done by the caller), runs
the upward half of all ranks, all-gathers their export rows on the host exactly as ncclAllGather lays them out,
and times every rank's upward and downward halves on the device (CUDA events inside
kifmm_gpu_evaluate_upward / _downward, host copies excluded).  The ranks run one after another -- they never
wait on one another.  The combined output is checked against the single-rank evaluate.

  projected_ms(N) = max_r upward_ms(r) + allgather_ms + max_r downward_ms(r)
  allgather_ms    = bytes received per GPU (N - 1 slots of halo_rows_max rows) / NVLINK_GBS

NVLINK_GBS defaults to 700 GB/s (an assumed effective all-gather rate under NVLink 5's 900 GB/s per
direction); the exchange is < 1 % of the step either way.  One JSON line per (config, N).

usage: python tools/scale_projection.py [config ids...]   (default 4 5)
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2303_08394_b200 import fmm, generators, host  # noqa: E402

NVLINK_GBS = float(os.environ.get("NVLINK_GBS", "700"))
REPS = 3
which = [int(x) for x in sys.argv[1:]] or [4, 5]
worlds = [int(x) for x in os.environ.get("WORLDS", "2,4,8").split(",")]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

for cid in which:
    c = generators.CONFIGS[cid]
    pos, q = generators.config_sample(cid)
    n = len(q)
    dt = np.float32 if c["precision"] == 32 else np.float64
    tdt = torch.float32 if c["precision"] == 32 else torch.float64
    qq = q.astype(dt)
    kw = dict(p=c["p"], n_crit=c["n_crit"], precision=c["precision"], gradient=c["gradient"])
    tree = host.Tree(pos, c["n_crit"])
    ops = fmm.load_or_precompute(fmm.FmmConfig(**kw), tree.side)
    # ---- one GPU: the device-resident evaluate (CUDA graph), L2 flushed between steps
    with fmm.Fmm(pos, fmm.FmmConfig(**kw), operators=ops, tree=tree) as f:
        pot1, grad1, _ = f.evaluate(qq)
        dq = torch.from_numpy(qq).cuda()
        dpot = torch.empty(n, dtype=tdt, device="cuda")
        dgrad = torch.empty((n, 3), dtype=tdt, device="cuda") if c["gradient"] else None
        st = torch.cuda.Stream()
        ms = []
        with torch.cuda.stream(st):
            for i in range(3 + REPS):
                flush.fill_(float(i))
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                f.evaluate_device(dq.data_ptr(), dpot.data_ptr(), dgrad.data_ptr() if dgrad is not None else None,
                                  input_order=True, stream=st.cuda_stream)
                b.record(st)
                b.synchronize()
                if i >= 3:
                    ms.append(a.elapsed_time(b))
        one_ms = float(np.median(ms))
        one_info = f.info()
        del dq, dpot, dgrad
    print(json.dumps({"config": cid, "n_gpus": 1, "measured_ms": one_ms, "points_per_s": n / (one_ms * 1e-3),
                      "kind": "measured (single GPU, CUDA graph)", "device_MB": one_info["device_bytes"] / 1e6}),
          flush=True)
    for world in worlds:
        def plan(r):
            return fmm.Fmm(pos, fmm.FmmConfig(**kw, rank=r, world_size=world, exchange=1), operators=ops, tree=tree)
        # pass 1: every rank's export rows
        sends, infos = [], []
        for r in range(world):
            with plan(r) as f:
                infos.append(f.info())
                sends.append(f.evaluate_upward(qq))
        hm = infos[0]["halo_rows_max"]
        gathered = np.zeros((world, max(1, hm), infos[0]["ne_pad"]), dtype=dt)
        for r, s in enumerate(sends):
            gathered[r, :s.shape[0]] = s
        del sends
        # pass 2: time both halves of every rank; assemble the output
        pot = np.zeros(n, dtype=dt)
        grad = np.zeros((n, 3), dtype=dt) if c["gradient"] else None
        up, dn, ranks = [], [], []
        for r in range(world):
            with plan(r) as f:
                u, d = [], []
                for rep in range(1 + REPS):
                    flush.fill_(float(rep))
                    f.evaluate_upward(qq)
                    tu = f.last_timings()["upward_ms"]
                    flush.fill_(float(rep))
                    o = f.evaluate_downward(gathered)
                    td = f.last_timings()["downward_ms"]
                    if rep:
                        u.append(tu)
                        d.append(td)
                pot += o[0]
                if grad is not None:
                    grad += o[1]
                i = infos[r]
                up.append(float(np.median(u)))
                dn.append(float(np.median(d)))
                ranks.append({"rank": r, "upward_ms": up[-1], "downward_ms": dn[-1],
                              "leaves": i["owned_leaf_end"] - i["owned_leaf_begin"],
                              "particles": i["owned_particle_end"] - i["owned_particle_begin"],
                              "near_pairs": i["near_pairs"], "m2l_pairs": i["m2l_pairs"],
                              "halo_rows_exported": i["halo_rows_mine"], "device_MB": i["device_bytes"] / 1e6})
        es = 4 if c["precision"] == 32 else 8
        recv_bytes = (world - 1) * hm * infos[0]["ne_pad"] * es
        ag_ms = recv_bytes / (NVLINK_GBS * 1e9) * 1e3
        proj = max(up) + ag_ms + max(dn)
        work = [a + b for a, b in zip(up, dn)]
        rec = {"config": cid, "n_gpus": world, "kind": "PROJECTED from per-rank halves timed on one B200",
               "projected_ms": proj, "points_per_s": n / (proj * 1e-3), "speedup_vs_1": one_ms / proj,
               "efficiency": one_ms / proj / world, "max_upward_ms": max(up), "max_downward_ms": max(dn),
               "allgather_ms": ag_ms, "allgather_recv_MB_per_gpu": recv_bytes / 1e6, "nvlink_GBs_assumed": NVLINK_GBS,
               "rank_work_imbalance": max(work) / (sum(work) / world), "sum_rank_work_over_one_gpu": sum(work) / one_ms,
               "rel_err_vs_single_rank": fmm.relative_error(pot, pot1), "ranks": ranks}
        if grad is not None:
            rec["grad_rel_err_vs_single_rank"] = fmm.relative_error(grad, grad1)
        print(json.dumps(rec), flush=True)
