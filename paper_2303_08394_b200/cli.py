"""Command-line harness (SPEC.md:633-692 `cli`): generate | precompute | run | bench | stats | verify.

    python -m paper_2303_08394_b200 generate --dist sphere-surface --n 100000 --seed 1 --out pts.bin
    python -m paper_2303_08394_b200 stats --input pts.bin --n-crit 150
    python -m paper_2303_08394_b200 precompute --input pts.bin --p 6 --cache ops.kifmm
    python -m paper_2303_08394_b200 run --input pts.bin --p 6 --n-crit 150 --cache ops.kifmm --verify
    python -m paper_2303_08394_b200 bench --dist sphere-surface --sizes 25000,50000,100000 --repeats 5
    python -m paper_2303_08394_b200 verify --input pts.bin --p 6 --tolerance 1e-5

Particle file: 8-byte little-endian count N, then N x 3 float64 positions (row-major), then
N float64 charges.  Reports are one JSON document on stdout (or --out).  Exit codes:
0 success, 1 usage, 2 data error, 3 numerical failure.  Threads: --threads > FMM_NUM_THREADS > all cores.
`generate`, `precompute` and `stats` are host-only; `run`, `bench` and `verify` evaluate on the GPU (there
is no CPU evaluate in this package) and verify against the GPU's fp64 direct-sum kernel.
"""
from __future__ import annotations

import argparse
import json
import os
import struct
import sys
import time

import numpy as np

EXIT_OK, EXIT_USAGE, EXIT_DATA, EXIT_NUMERICAL = 0, 1, 2, 3


class UsageError(Exception):
    pass


# ------------------------------------------------------------------ particle file
def write_particles(path: str, positions, charges) -> None:
    pos = np.ascontiguousarray(positions, dtype="<f8").reshape(-1, 3)
    q = np.ascontiguousarray(charges, dtype="<f8").reshape(-1)
    if pos.shape[0] != q.shape[0]:
        raise ValueError("positions and charges differ in length")
    with open(path, "wb") as f:
        f.write(struct.pack("<Q", pos.shape[0]))
        f.write(pos.tobytes())
        f.write(q.tobytes())


def read_particles(path: str):
    from .errors import CorruptArchive
    with open(path, "rb") as f:
        head = f.read(8)
        if len(head) != 8:
            raise CorruptArchive(f"{path}: truncated header")
        (n,) = struct.unpack("<Q", head)
        body = f.read()
    if len(body) != 32 * n:
        raise CorruptArchive(f"{path}: expected {32 * n} payload bytes for N={n}, found {len(body)}")
    arr = np.frombuffer(body, dtype="<f8")
    return arr[:3 * n].reshape(n, 3).astype(np.float64), arr[3 * n:].astype(np.float64)


# ------------------------------------------------------------------ helpers
def _threads(args) -> int:
    if getattr(args, "threads", None) is not None:
        return int(args.threads)
    env = os.environ.get("FMM_NUM_THREADS")
    return int(env) if env else 0


def _config(args, **extra):
    from . import fmm
    return fmm.FmmConfig(p=args.p, n_crit=args.n_crit, alpha_inner=args.alpha_inner, alpha_outer=args.alpha_outer,
                         svd_cutoff=args.svd_cutoff, threads=_threads(args), precision=args.precision,
                         gradient=args.gradient, device=args.device, cache=args.cache, **extra)


def _emit(doc: dict, out: str | None) -> None:
    text = json.dumps(doc, indent=1)
    if out:
        with open(out, "w") as f:
            f.write(text + "\n")
    else:
        print(text)


def _list_stats(tree) -> dict:
    return {k: {"min": v[0], "mean": v[1], "max": v[2]} for k, v in tree.list_stats().items()}


def _verify(fmm_mod, pos, q, pot, targets: int, seed: int):
    n = pos.shape[0]
    if n <= targets:
        tg = np.arange(n, dtype=np.int64)
    else:
        rng = np.random.default_rng(seed)
        tg = np.sort(rng.choice(n, targets, replace=False)).astype(np.int64)
    ref = fmm_mod.direct(pos, q, targets=tg, precision=64)
    return fmm_mod.relative_error(pot[tg], ref), int(tg.size)


# ------------------------------------------------------------------ subcommands
def cmd_generate(args) -> int:
    from . import generators
    if args.n < 1:
        raise UsageError("--n must be >= 1")
    pos, q = generators.sample(args.dist, args.n, seed=args.seed, charges=args.charges)
    if args.dist == "sphere-surface" and not args.unit_sphere:
        pos = 0.5 + 0.5 * pos  # radius 0.5 side about the unit cube's centre
    write_particles(args.out, pos, q)
    _emit({"generated": args.out, "n": int(args.n), "distribution": args.dist, "seed": args.seed,
           "charges": args.charges}, None)
    return EXIT_OK


def cmd_stats(args) -> int:
    from . import host
    pos, _ = read_particles(args.input)
    t0 = time.perf_counter()
    t = host.Tree(pos, args.n_crit, threads=_threads(args))
    _emit({"n": int(t.n), "n_crit": args.n_crit, "depth": int(t.depth), "leaves": int(t.n_leaves),
           "nodes": int(t.n_nodes), "overfull_leaves": int(t.n_overfull), "lists": _list_stats(t),
           "tree_and_lists_s": time.perf_counter() - t0}, args.out)
    return EXIT_OK


def cmd_precompute(args) -> int:
    from . import host
    if args.side is not None:
        side = float(args.side)
    elif args.input:
        pos, _ = read_particles(args.input)
        side = host.Tree(pos, max(1, pos.shape[0]), threads=_threads(args)).side  # one leaf: just the domain
    else:
        raise UsageError("precompute needs --input or --side (the operators depend on the domain side)")
    if not args.cache:
        raise UsageError("precompute needs --cache PATH")
    t0 = time.perf_counter()
    ops = host.Operators(args.p, args.alpha_inner, args.alpha_outer, args.svd_cutoff, side, _threads(args))
    ops.save(args.cache)
    _emit({"cache": args.cache, "p": args.p, "n_e": ops.n_e, "domain_side": side, "fingerprint": ops.fingerprint,
           "precompute_s": time.perf_counter() - t0}, args.out)
    return EXIT_OK


def _run_once(args, pos, q):
    from . import fmm
    f = fmm.Fmm(pos, _config(args))
    try:
        dt = f.dtype
        pot, grad, tm = f.evaluate(q.astype(dt), timed=True)
        rep = {"config": {k: getattr(f.config, k) for k in ("p", "n_crit", "alpha_inner", "alpha_outer",
                                                             "svd_cutoff", "precision", "gradient", "threads")},
               "n": int(f.n), "depth": int(f.tree.depth), "leaves": int(f.tree.n_leaves),
               "operator_ms": {k: v for k, v in tm.items() if k.endswith("_ms")},
               "setup_s": dict(f.timings), "lists": _list_stats(f.tree), "m2l_backend": f.info()["m2l_backend"]}
        return pot, grad, rep
    finally:
        f.close()


def cmd_run(args) -> int:
    from . import fmm
    pos, q = read_particles(args.input)
    pot, _, rep = _run_once(args, pos, q)
    rep["total_ms"] = rep["operator_ms"].get("total_ms")
    if args.verify:
        err, m = _verify(fmm, pos, q, pot, args.verify_targets, args.seed)
        rep["relative_error_vs_direct"] = err
        rep["verify_targets"] = m
    if args.potentials:
        np.save(args.potentials, pot)
    _emit(rep, args.out)
    return EXIT_OK


def cmd_verify(args) -> int:
    from . import fmm
    pos, q = read_particles(args.input)
    pot, _, rep = _run_once(args, pos, q)
    err, m = _verify(fmm, pos, q, pot, args.verify_targets, args.seed)
    ok = err <= args.tolerance
    rep.update({"relative_error_vs_direct": err, "verify_targets": m, "tolerance": args.tolerance, "pass": ok})
    _emit(rep, args.out)
    return EXIT_OK if ok else EXIT_NUMERICAL


def cmd_bench(args) -> int:
    """per size, `repeats` runs; mean +- sample std of the total (tree + lists + plan +
    evaluate, operators cached) and of each evaluate phase; plus the direct sum at the same sizes (GPU
    fp64 kernel, skipped above --direct-max)."""
    from . import fmm, generators
    sizes = [int(float(s)) for s in args.sizes.split(",")]
    if sizes != sorted(sizes):
        raise UsageError("--sizes must be ascending")
    rows, ops = [], {}  # in-memory operator cache keyed by fingerprint (the domain side differs per cloud)
    for n in sizes:
        pos, q = generators.sample(args.dist, n, seed=args.seed, charges=args.charges)
        tot, phases = [], []
        fmm.Fmm(pos, _config(args), operators=ops).close()  # operators cached before the timed repeats
        for _ in range(args.repeats):
            t0 = time.perf_counter()
            f = fmm.Fmm(pos, _config(args), operators=ops)
            _, _, tm = f.evaluate(q.astype(f.dtype), timed=True)
            tot.append(time.perf_counter() - t0)
            phases.append(tm)
            f.close()
        row = {"n": n, "total_s_mean": float(np.mean(tot)),
               "total_s_std": float(np.std(tot, ddof=1)) if len(tot) > 1 else 0.0,
               "evaluate_ms": {k: [float(np.mean([p[k] for p in phases])),
                                   float(np.std([p[k] for p in phases], ddof=1)) if len(phases) > 1 else 0.0]
                               for k in phases[0]}}
        if n <= args.direct_max:
            t0 = time.perf_counter()
            fmm.direct(pos, q, precision=64)
            row["direct_s"] = time.perf_counter() - t0
        rows.append(row)
    if len(sizes) > 1:
        slope = float(np.polyfit(np.log(sizes), np.log([r["total_s_mean"] for r in rows]), 1)[0])
    else:
        slope = None
    _emit({"distribution": args.dist, "repeats": args.repeats, "rows": rows, "loglog_slope_total": slope}, args.out)
    return EXIT_OK


# ------------------------------------------------------------------ parser
def _common(ap, fmm_flags=True):
    ap.add_argument("--threads", type=int, default=None)
    ap.add_argument("--out", default=None)
    ap.add_argument("--seed", type=int, default=0)
    if fmm_flags:
        ap.add_argument("--p", type=int, default=6)
        ap.add_argument("--n-crit", type=int, default=150)
        ap.add_argument("--alpha-inner", type=float, default=1.05)
        ap.add_argument("--alpha-outer", type=float, default=2.95)
        ap.add_argument("--svd-cutoff", type=float, default=1e-12)
        ap.add_argument("--cache", default=None)
        ap.add_argument("--precision", type=int, choices=(32, 64), default=64)
        ap.add_argument("--gradient", action="store_true")
        ap.add_argument("--device", type=int, default=0)
        ap.add_argument("--l2p-cache-local", action="store_true",
                        help="accepted for SPEC compatibility (SPEC.md:506): the GPU layout is leaf-contiguous")


def build_parser():
    ap = argparse.ArgumentParser(prog="kifmm", description=__doc__.split("\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("generate")
    g.add_argument("--dist", choices=("sphere-surface", "uniform-cube", "two-cluster"), default="sphere-surface")
    g.add_argument("--n", type=int, required=True)
    g.add_argument("--charges", choices=("unit", "uniform", "signed"), default="unit")
    g.add_argument("--unit-sphere", action="store_true", help="unit sphere at the origin (BASELINE config 3)")
    _common(g, fmm_flags=False)
    g.set_defaults(fn=cmd_generate)
    s = sub.add_parser("stats")
    s.add_argument("--input", required=True)
    s.add_argument("--n-crit", type=int, default=150)
    _common(s, fmm_flags=False)
    s.set_defaults(fn=cmd_stats)
    pc = sub.add_parser("precompute")
    pc.add_argument("--input", default=None)
    pc.add_argument("--side", type=float, default=None)
    _common(pc)
    pc.set_defaults(fn=cmd_precompute)
    r = sub.add_parser("run")
    r.add_argument("--input", required=True)
    r.add_argument("--verify", action="store_true")
    r.add_argument("--verify-targets", type=int, default=1000)
    r.add_argument("--potentials", default=None, help="save the potentials (.npy, input order)")
    _common(r)
    r.set_defaults(fn=cmd_run)
    v = sub.add_parser("verify")
    v.add_argument("--input", required=True)
    v.add_argument("--tolerance", type=float, default=1e-5)
    v.add_argument("--verify-targets", type=int, default=1000)
    _common(v)
    v.set_defaults(fn=cmd_verify)
    b = sub.add_parser("bench")
    b.add_argument("--dist", choices=("sphere-surface", "uniform-cube", "two-cluster"), default="sphere-surface")
    b.add_argument("--sizes", default="25000,50000,100000,200000")
    b.add_argument("--repeats", type=int, default=5)
    b.add_argument("--charges", choices=("unit", "uniform", "signed"), default="unit")
    b.add_argument("--direct-max", type=int, default=200000)
    _common(b)
    b.set_defaults(fn=cmd_bench)
    return ap


def main(argv=None) -> int:
    from .errors import CacheMismatch, CorruptArchive, DeviceError, InvalidArgument, IoError, KifmmError, \
        NumericalError
    ap = build_parser()
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return EXIT_OK if e.code == 0 else EXIT_USAGE
    try:
        return args.fn(args)
    except UsageError as e:
        print(f"kifmm {args.cmd}: {e}", file=sys.stderr)
        return EXIT_USAGE
    except NumericalError as e:
        print(f"kifmm {args.cmd}: numerical failure: {e}", file=sys.stderr)
        return EXIT_NUMERICAL
    except (InvalidArgument, IoError, CacheMismatch, CorruptArchive, DeviceError, KifmmError, OSError,
            ValueError) as e:
        print(f"kifmm {args.cmd}: {type(e).__name__}: {e}", file=sys.stderr)
        return EXIT_DATA


if __name__ == "__main__":
    sys.exit(main())
