"""GPU parity tests (run on a B200 with -m gpu): the CUDA evaluate through the
C ABI against the fp64 oracle on identical inputs.

Tolerances (north star, BASELINE.json): relative L2 <= 1e-12 for fp64 and
<= 1e-5 for fp32 (potentials); gradients (an extension) use
1e-11 (fp64) and 5e-5 (fp32).  Both oracle and GPU consume the same fp64
operator matrices and factored pseudo-inverses (SURVEY 8c parity protocol).
"""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2303_08394_b200 import InvalidArgument, fmm, generators, host

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL = {64: (1e-12, 1e-11), 32: (1e-5, 5e-5)}


def _inv(t):
    i = np.empty_like(t.original_index)
    i[t.original_index] = np.arange(t.n)
    return i


def _ref(f, q, gradient):
    qr = np.asarray(q, dtype=np.float64)[f.tree.original_index]
    phi, g, _ = oracle.evaluate(f.tree, f.operators, qr, gradient=gradient)
    ii = _inv(f.tree)
    return phi[ii], (g[ii] if g is not None else None)


CASES = [("uniform-cube", 6000, 40, 4), ("uniform-cube", 5000, 50, 6), ("sphere-surface", 8000, 40, 6),
         ("two-cluster", 6000, 20, 5), ("two-cluster", 4000, 8, 7), ("uniform-cube", 3000, 30, 2)]


@pytest.mark.parametrize("kind,n,n_crit,p", CASES)
@pytest.mark.parametrize("precision,backend", [(64, 0), (32, 1), (32, 0)],
                         ids=["fp64", "fp32-simt", "fp32-auto"])
def test_parity_vs_oracle(require_gpu, kind, n, n_crit, p, precision, backend):
    """backend 0 = the production choice (tcgen05 M2L and GEMMs for fp32 p = 4, 5, 6; int8 tcgen05 or DMMA for fp64),
    1 = the SIMT M2L / GEMM kernels."""
    if precision == 32 and p >= 7:
        pytest.skip("fp32 at p=7: kept spectrum cond ~1e11, see test_fp32_p7_accuracy_bound")
    pos, q = generators.sample(kind, n, seed=7, charges="signed", fp32=precision == 32)
    cfg = fmm.FmmConfig(p=p, n_crit=n_crit, precision=precision, gradient=True, m2l_backend=backend)
    with fmm.Fmm(pos, cfg) as f:
        pot, grad, _ = f.evaluate(q)
        ref, gref = _ref(f, q, True)
    tp, tg = TOL[precision]
    assert fmm.relative_error(pot, ref) <= tp
    assert fmm.relative_error(grad, gref) <= tg


def test_fp32_p7_accuracy_bound(require_gpu):
    """fp32 at p=7 is outside every BASELINE config (p=7 is the fp64 config 4) and
    its check->equivalent solve is ill-conditioned; the
    documented bound is 5e-4 relative L2."""
    pos, q = generators.sample("two-cluster", 4000, seed=7, charges="signed", fp32=True)
    with fmm.Fmm(pos, fmm.FmmConfig(p=7, n_crit=8, precision=32)) as f:
        pot, _, _ = f.evaluate(q)
        ref, _ = _ref(f, q, False)
    assert fmm.relative_error(pot, ref) <= 5e-4


def test_randomised_clouds_short(require_gpu):
    """A short run of the randomised GPU-vs-oracle tool (random size, leaf capacity, order 2-8, distribution,
    degenerate clouds, scale / shift, charge range, precision, gradient): every case inside the parity gates."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "randomised_gpu.py"), "20", "5"], cwd=root,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("precision", [32, 64])
@pytest.mark.parametrize("scale,shift", [(1e-4, 0.0), (1e4, 0.0), (1.0, -1000.0), (1e3, 5e4), (1e-3, 1.0)])
def test_scaled_and_shifted_domains(require_gpu, scale, shift, precision):
    """Clouds away from the unit cube.  K_t scales with 1 / side: the fp16 split of the tcgen05 M2L takes its
    power-of-two scale from the largest operator entry (a fixed 2^8 gave NaN for a domain of side 1e-4 and 1.1e-5
    at side 1e4, tools/exp/r02_scaleshift.py)."""
    pos, q = generators.sample("two-cluster", 20000, seed=4, charges="signed")
    pos = pos * scale + shift
    if precision == 32:
        pos = pos.astype(np.float32).astype(np.float64)
    with fmm.Fmm(pos, fmm.FmmConfig(p=6, n_crit=40, precision=precision, gradient=True)) as f:
        pot, grad, _ = f.evaluate(q)
        ref, gref = _ref(f, q, True)
    tp, tg = (1e-12, 1e-11) if precision == 64 else (2e-6, 2e-6)
    assert fmm.relative_error(pot, ref) <= tp
    assert fmm.relative_error(grad, gref) <= tg


@pytest.mark.parametrize("kind,n,n_crit,p,precision", [
    ("uniform-cube", 60000, 60, 6, 32), ("two-cluster", 40000, 30, 6, 32), ("sphere-surface", 30000, 40, 5, 32),
    ("two-cluster", 20000, 30, 7, 64), ("uniform-cube", 20000, 60, 5, 64), ("two-cluster", 6000, 30, 8, 64)])
def test_no_state_carries_between_evaluates(require_gpu, kind, n, n_crit, p, precision):
    """A plan keeps no state from one evaluate to the next: charges A, then B (sparse and 1e6 times larger), then
    zeros, then A again reproduce A bit for bit; B equals a fresh plan's B; zeros give zeros.  Covers the fp32
    tcgen05 path (split buffers, partial rows, near-field queue), the fp64 int8 path (per-level exponents
    recomputed every evaluate) and the column-blocked GEMMs of p = 8, through the graph and the eager launch."""
    pos, qa = generators.sample(kind, n, seed=41, charges="signed", fp32=precision == 32)
    rng = np.random.default_rng(5)
    qb = np.where(rng.random(n) < 0.01, 1e6 * (2 * rng.random(n) - 1), 0.0)
    cfg = fmm.FmmConfig(p=p, n_crit=n_crit, precision=precision, gradient=True)
    with fmm.Fmm(pos, cfg) as f:
        a1 = f.evaluate(qa)[:2]
        b1 = f.evaluate(qb)[:2]
        z = f.evaluate(np.zeros(n))[:2]
        a2 = f.evaluate(qa)[:2]
        a3 = f.evaluate(qa, timed=True)[:2]
        tree, ops = f.tree, f.operators
    with fmm.Fmm(pos, cfg, operators=ops, tree=tree) as g:
        b2 = g.evaluate(qb)[:2]
    for x, y in ((a1, a2), (a1, a3), (b1, b2)):
        assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1])
    assert not np.any(z[0]) and not np.any(z[1])


@pytest.mark.parametrize("side,depth_min", [(1e-2, 9), (1e-3, 12), (1e-4, 15)])
def test_fp32_deep_cluster(require_gpu, side, depth_min):
    """fp32 on a clustered cloud (a dense cube of the given side in a uniform background, tree depth 10-15): the
    surface geometry of the fp32 kernels is node-local with the centre as a float pair, so the parity gate holds
    at any depth -- absolute fp32 coordinates gave 9e-6 / 1.1e-4 / 2.6e-4 here (tools/exp/r02_deep.py)."""
    rng = np.random.default_rng(3)
    n = 20000
    pos = np.concatenate([rng.random((n // 2, 3)), 0.3 + side * rng.random((n // 2, 3))])
    pos = pos.astype(np.float32).astype(np.float64)
    q = 2 * rng.random(n) - 1
    with fmm.Fmm(pos, fmm.FmmConfig(p=6, n_crit=30, precision=32, gradient=True)) as f:
        assert f.tree.depth >= depth_min
        pot, grad, _ = f.evaluate(q)
        ref, gref = _ref(f, q, True)
    assert fmm.relative_error(pot, ref) <= 3e-6
    assert fmm.relative_error(grad, gref) <= 5e-6


@pytest.mark.parametrize("precision", [32, 64])
@pytest.mark.parametrize("kind,n_crit", [("dups", 1), ("dups", 2), ("line", 1)])
def test_degenerate_clouds_max_depth(require_gpu, kind, n_crit, precision):
    """Clouds that drive the tree to its maximum depth (15): every point three times with n_crit < 3, and points
    on a line with n_crit = 1 (cases found by the randomised GPU-vs-oracle runs, tests/randomised_gpu.py)."""
    rng = np.random.default_rng(11)
    if kind == "dups":
        base = rng.random((100, 3))
        pos, q = np.concatenate([base] * 3), np.tile(2 * rng.random(100) - 1, 3)
    else:
        t = np.sort(rng.random(300))
        pos, q = np.stack([t, 0.5 + 0 * t, 0.25 + 0 * t], axis=1), 2 * rng.random(300) - 1
    if precision == 32:
        pos = pos.astype(np.float32).astype(np.float64)
    with fmm.Fmm(pos, fmm.FmmConfig(p=5, n_crit=n_crit, precision=precision)) as f:
        assert f.tree.depth == 15
        pot, _, _ = f.evaluate(q)
        ref, _ = _ref(f, q, False)
    assert np.all(np.isfinite(pot))
    assert fmm.relative_error(pot, ref) <= TOL[precision][0]


@pytest.mark.parametrize("kind,n,n_crit,p,precision,cutoff", [
    ("two-cluster", 3000, 30, 8, 64, 1e-12), ("sphere-surface", 4000, 60, 10, 64, 1e-12),
    ("uniform-cube", 4000, 60, 9, 32, 1e-8)])
def test_high_orders(require_gpu, kind, n, n_crit, p, precision, cutoff):
    """p = 8, 9, 10 (row widths 320, 448, 512; the paper's L2P experiment uses p = 10) on the any-width
    kernels: parity gates against the oracle, and the graph launch equals the eager timed run."""
    pos, q = generators.sample(kind, n, seed=5, charges="signed", fp32=precision == 32)
    cfg = fmm.FmmConfig(p=p, n_crit=n_crit, precision=precision, svd_cutoff=cutoff, gradient=True)
    with fmm.Fmm(pos, cfg) as f:
        assert f.info()["m2l_backend"] == 1
        pot, grad, _ = f.evaluate(q)
        pot2, grad2, _ = f.evaluate(q, timed=True)
        ref, gref = _ref(f, q, True)
    assert np.array_equal(pot, pot2) and np.array_equal(grad, grad2)
    tp, tg = TOL[precision]
    assert fmm.relative_error(pot, ref) <= tp
    assert fmm.relative_error(grad, gref) <= tg


@pytest.mark.parametrize("kind,n,n_crit", [("two-cluster", 4000, 8), ("uniform-cube", 20000, 60)])
def test_fp32_p7_with_fp32_cutoff(require_gpu, kind, n, n_crit):
    """fp32 at p = 7 meets the fp32 gate once the pseudo-inverse cutoff suits fp32: the SPEC default
    (svd_cutoff 1e-12, an fp64 setting) keeps singular values down to 1e-11 of the largest, and the
    fp32 rounding of the resulting densities costs 1e-4; with svd_cutoff = 1e-8 the same plan agrees
    with the oracle (same operators) to < 1e-6 and is closer to direct summation than p = 6
    (tools/exp/r02_p7cut.py: 3.7e-7 / 6.6e-7 against 1.3e-6 / 2.9e-6 with the SIMT M2L; 1.1e-6 / 7.6e-7
    with the tcgen05 M2L, tools/exp/r02_p7tc.py)."""
    pos, q = generators.sample(kind, n, seed=7, charges="signed", fp32=True)
    with fmm.Fmm(pos, fmm.FmmConfig(p=7, n_crit=n_crit, precision=32, svd_cutoff=1e-8, gradient=True)) as f:
        assert f.info()["m2l_backend"] == 2  # tcgen05 M2L, row width 224 (2-CTA pair kernel); SIMT solves / M2M / L2L
        pot, grad, _ = f.evaluate(q)
        ref, gref = _ref(f, q, True)
    assert fmm.relative_error(pot, ref) <= 2e-6
    assert fmm.relative_error(grad, gref) <= 1e-5
    idx = np.arange(0, n, max(1, n // 1000))
    assert fmm.relative_error(pot[idx], fmm.direct(pos, q, targets=idx, precision=64)) <= 2e-6


@pytest.mark.parametrize("variant", [("f16", "0", 2), ("f16", "1", 2), ("tf32", "0", 3), ("tf32", "1", 3)],
                         ids=["f16x3", "f16x3-2cta", "tf32x3", "tf32x3-2cta"])
@pytest.mark.parametrize("kind,n,n_crit", [("uniform-cube", 20000, 60), ("sphere-surface", 30000, 50),
                                           ("two-cluster", 20000, 30)])
def test_tcgen05_m2l_parity(require_gpu, monkeypatch, kind, n, n_crit, variant):
    """Every tensor-core M2L variant (kind::f16 3-term split / kind::tf32 3xTF32, 1-CTA / 2-CTA pair)."""
    monkeypatch.setenv("KIFMM_TC_KIND", variant[0])
    monkeypatch.setenv("KIFMM_TC_PAIR", variant[1])
    pos, q = generators.sample(kind, n, seed=8, charges="signed", fp32=True)
    cfg = fmm.FmmConfig(p=6, n_crit=n_crit, precision=32, gradient=True, m2l_backend=2)
    with fmm.Fmm(pos, cfg) as f:
        assert f.info()["m2l_backend"] == variant[2]
        pot, grad, _ = f.evaluate(q)
        ref, gref = _ref(f, q, True)
    assert fmm.relative_error(pot, ref) <= 1e-5
    assert fmm.relative_error(grad, gref) <= 5e-5


def test_single_leaf_equals_direct(require_gpu):
    pos, q = generators.sample("uniform-cube", 200, seed=1, charges="uniform")
    with fmm.Fmm(pos, fmm.FmmConfig(p=6, n_crit=500, precision=64)) as f:
        assert f.tree.n_leaves == 1
        pot, _, _ = f.evaluate(q)
    assert fmm.relative_error(pot, oracle.direct(pos, q)) <= 1e-13


def test_golden_config1(require_gpu):  # BASELINE config 1 (p=5, n_crit=64), fp32
    g = np.load(os.path.join(GOLD, "config1_direct.npz"))
    pos, q = g["positions"], g["charges"]
    with fmm.Fmm(pos, fmm.FmmConfig(p=5, n_crit=64, precision=32, gradient=True)) as f:
        pot, grad, _ = f.evaluate(q)
        ref, gref = _ref(f, q, True)
    assert fmm.relative_error(pot, ref) <= 1e-5
    assert fmm.relative_error(pot, g["potential"]) <= 1e-4


def test_config2_full_size(require_gpu):
    """BASELINE config 2 at full size (1M points, p=6, fp32, gradient): GPU vs the
    fp64 oracle on all points, and vs direct summation on the 1,000 committed
    sampled targets (north star)."""
    pos, q = generators.config_sample(2)
    with fmm.Fmm(pos, fmm.FmmConfig(p=6, n_crit=150, precision=32, gradient=True)) as f:
        pot, grad, _ = f.evaluate(q.astype(np.float32))
        pot2, grad2, _ = f.evaluate(q.astype(np.float32))
        ref, gref = _ref(f, q, True)
        backend = f.info()["m2l_backend"]
    assert np.array_equal(pot, pot2) and np.array_equal(grad, grad2)  # deterministic
    assert fmm.relative_error(pot, ref) <= 1e-5, backend
    assert fmm.relative_error(grad, gref) <= 5e-5
    gold = np.load(os.path.join(GOLD, "config2_sampled_direct.npz"))
    tg = gold["targets"]
    assert fmm.relative_error(pot[tg], gold["potential"]) <= 1e-5
    assert fmm.relative_error(grad[tg], gold["gradient"]) <= 1e-4
    # the GPU direct-sum kernel (K10) agrees with the fp64 numpy fixture
    d = fmm.direct(pos, q, targets=tg, precision=64)
    assert fmm.relative_error(d, gold["potential"]) <= 1e-12


def test_size_independent_properties(require_gpu):
    pos, q = generators.sample("sphere-surface", 200000, seed=9, charges="signed", fp32=True)
    with fmm.Fmm(pos, fmm.FmmConfig(p=6, n_crit=150, precision=32)) as f:
        a, _, _ = f.evaluate(q.astype(np.float32))
        b, _, _ = f.evaluate((2.0 * q).astype(np.float32))  # scaling by 2 is exact
        z, _, _ = f.evaluate(np.zeros(f.n, np.float32))
        # reordered-order interface agrees with input order
        r, _, _ = f.evaluate(q[f.tree.original_index].astype(np.float32), input_order=False)
    assert np.array_equal(b, 2.0 * a)
    assert not np.any(z)
    assert np.array_equal(r, a[f.tree.original_index])


def test_direct_kernel(require_gpu):
    pos, q = generators.sample("two-cluster", 3000, seed=10, charges="signed")
    tg = np.arange(0, 3000, 7)
    d64, g64 = fmm.direct(pos, q, targets=tg, precision=64, gradient=True)
    r, gr = oracle.direct(pos, q, targets=tg, gradient=True)
    assert fmm.relative_error(d64, r) <= 1e-13 and fmm.relative_error(g64, gr) <= 1e-12
    d32 = fmm.direct(pos, q, targets=tg, precision=32)
    assert fmm.relative_error(d32, r) <= 1e-5


def test_evaluate_device_and_graph(require_gpu):
    import torch
    pos, q = generators.sample("uniform-cube", 50000, seed=12, charges="uniform", fp32=True)
    with fmm.Fmm(pos, fmm.FmmConfig(p=5, n_crit=64, precision=32, gradient=True, use_graph=True)) as f:
        host_pot, host_grad, _ = f.evaluate(q)
        dq = torch.from_numpy(q.astype(np.float32)).cuda()
        dp = torch.empty(f.n, device="cuda")
        dg = torch.empty((f.n, 3), device="cuda")
        s = torch.cuda.Stream()
        f.evaluate_device(dq.data_ptr(), dp.data_ptr(), dg.data_ptr(), stream=s.cuda_stream)
        s.synchronize()
    assert np.array_equal(dp.cpu().numpy(), host_pot)
    assert np.array_equal(dg.cpu().numpy(), host_grad)


def test_invalid_arguments(require_gpu):
    pos, q = generators.sample("uniform-cube", 1000, seed=0)
    with fmm.Fmm(pos, fmm.FmmConfig(p=3, n_crit=20)) as f:
        with pytest.raises(InvalidArgument):
            f.evaluate(q[:10])
    with pytest.raises(InvalidArgument):
        fmm.Fmm(pos, fmm.FmmConfig(p=11, n_crit=20))  # n_e > 512 (p > 10) unsupported on the GPU
    with pytest.raises(InvalidArgument):
        fmm.Fmm(pos, fmm.FmmConfig(precision=16))


def test_run_api(require_gpu):  # run(particles, config) -> potentials (input order) + timings
    pos, q = generators.sample("sphere-surface", 20000, seed=13, charges="unit")
    pot, grad, tm = fmm.run(pos, q, fmm.FmmConfig(p=6, n_crit=50, precision=64))
    assert grad is None and tm["total_ms"] > 0 and "tree_s" in tm
    assert fmm.relative_error(pot[:500], oracle.direct(pos, q, targets=np.arange(500))) <= 1e-5


def test_near_queue_mode_bit_identical(require_gpu, monkeypatch):
    """Queue mode (near field taken by side-stream blocks from a counter, drained after L2L) computes
    every leaf work in exactly one block: results equal the standalone launch bit for bit
    (KIFMM_NEAR_WS=0 one leaf_eval_f2 block per work, 1 the warp-specialised kernel in queue mode, 2 also
    standalone; KIFMM_NEAR_BPS = side blocks per SM, 0 = no queue)."""
    pos, q = generators.sample("two-cluster", 60000, seed=21, charges="signed", fp32=True)
    cfg = fmm.FmmConfig(p=6, n_crit=40, precision=32, gradient=True)
    out = {}
    for ws in ("0", "1", "2"):
        for bps in ("0", "1", "2"):
            monkeypatch.setenv("KIFMM_NEAR_WS", ws)
            monkeypatch.setenv("KIFMM_NEAR_BPS", bps)
            with fmm.Fmm(pos, cfg) as f:
                out[ws, bps] = f.evaluate(q)[:2]
                if bps == "0":
                    out[ws, "timed"] = f.evaluate(q, timed=True)[:2]
    ref = out["0", "0"]
    for k, v in out.items():
        assert np.array_equal(v[0], ref[0]) and np.array_equal(v[1], ref[1]), k


@pytest.mark.parametrize("pair", ["0", "1"], ids=["1cta", "2cta"])
@pytest.mark.parametrize("p,kind,n,n_crit", [(4, "uniform-cube", 40000, 40), (5, "uniform-cube", 40000, 64),
                                             (5, "sphere-surface", 30000, 50), (4, "two-cluster", 20000, 30)])
def test_tcgen05_path_other_orders(require_gpu, monkeypatch, p, kind, n, n_crit, pair):
    """The tcgen05 M2L and GEMM chain are instantiated per row width (n_e padded to 32): 64 (p = 4),
    128 (p = 5) and 160 (p = 6).  fp32 plans at p = 4, 5 take that path by default (m2l_backend 2), in the
    single-CTA and the 2-CTA pair kernels, and meet the fp32 parity gates against the oracle."""
    monkeypatch.setenv("KIFMM_TC_PAIR", pair)
    pos, q = generators.sample(kind, n, seed=31, charges="signed", fp32=True)
    with fmm.Fmm(pos, fmm.FmmConfig(p=p, n_crit=n_crit, precision=32, gradient=True)) as f:
        assert f.info()["m2l_backend"] == 2
        pot, grad, _ = f.evaluate(q)
        ref, gref = _ref(f, q, True)
    assert fmm.relative_error(pot, ref) <= 1e-5
    assert fmm.relative_error(grad, gref) <= 5e-5


def test_simt_gemms_with_tcgen05_m2l(require_gpu, monkeypatch):
    """fp32 solves / M2M / L2L on the SIMT GEMM (KIFMM_TC_GEMM=0) next to the tcgen05 M2L."""
    monkeypatch.setenv("KIFMM_TC_GEMM", "0")
    pos, q = generators.sample("sphere-surface", 30000, seed=22, charges="signed", fp32=True)
    with fmm.Fmm(pos, fmm.FmmConfig(p=6, n_crit=50, precision=32, gradient=True)) as f:
        assert f.info()["m2l_backend"] == 2
        pot, grad, _ = f.evaluate(q)
        ref, gref = _ref(f, q, True)
    assert fmm.relative_error(pot, ref) <= 1e-5
    assert fmm.relative_error(grad, gref) <= 5e-5


@pytest.mark.parametrize("n_crit", [1, 4, 20])
@pytest.mark.parametrize("precision", [64, 32])
def test_small_trees_spec_invariant(require_gpu, n_crit, precision):
    """N <= 200, n_crit in {1, 4, 20}, p = 6 agrees with direct summation to 1e-5 (deep,
    ragged trees: a leaf per particle at n_crit = 1); and with the fp64 oracle to the parity bar."""
    pos, q = generators.sample("uniform-cube", 200, seed=31 + n_crit, charges="signed", fp32=precision == 32)
    with fmm.Fmm(pos, fmm.FmmConfig(p=6, n_crit=n_crit, precision=precision, gradient=True)) as f:
        pot, grad, _ = f.evaluate(q)
        ref, gref = _ref(f, q, True)
    assert fmm.relative_error(pot, oracle.direct(pos, q)) <= 1e-5
    tp, tg = TOL[precision]
    assert fmm.relative_error(pot, ref) <= tp
    assert fmm.relative_error(grad, gref) <= tg


@pytest.mark.parametrize("n", [1, 2, 3, 77])
def test_tiny_inputs(require_gpu, n):
    pos, q = generators.sample("uniform-cube", n, seed=40 + n, charges="signed")
    with fmm.Fmm(pos, fmm.FmmConfig(p=4, n_crit=2, precision=64, gradient=True)) as f:
        pot, grad, _ = f.evaluate(q)
        ref, gref = _ref(f, q, True)
    assert np.all(np.isfinite(pot)) and np.all(np.isfinite(grad))
    if n == 1:  # a lone particle sees nothing (r = 0 -> 0)
        assert not np.any(pot) and not np.any(grad) and not np.any(ref)
    else:
        assert fmm.relative_error(pot, ref) <= 1e-12 and fmm.relative_error(grad, gref) <= 1e-11


def test_coincident_particles(require_gpu):
    """Duplicated positions: the r = 0 convention masks self and coincident pairs on the
    GPU exactly as in the oracle; a leaf that cannot be split below MAX_LEVEL stays over-full."""
    base, _ = generators.sample("two-cluster", 400, seed=50, charges="signed")
    pos = np.repeat(base, 3, axis=0)
    q = generators.sample("uniform-cube", len(pos), seed=51, charges="signed")[1]
    for precision in (64, 32):
        p_ = pos.astype(np.float32).astype(np.float64) if precision == 32 else pos
        q_ = q.astype(np.float32).astype(np.float64) if precision == 32 else q
        with fmm.Fmm(p_, fmm.FmmConfig(p=6, n_crit=2, precision=precision, gradient=True)) as f:
            pot, grad, _ = f.evaluate(q_)
            ref, gref = _ref(f, q_, True)
        assert np.all(np.isfinite(pot)) and np.all(np.isfinite(grad))
        ep, eg = fmm.relative_error(pot, ref), fmm.relative_error(grad, gref)
        # fp32 cannot resolve level-15 geometry (box half side 2^-16 of the domain against a 2^-24
        # relative coordinate rounding), so duplicates driving the tree to MAX_LEVEL cost fp32 accuracy;
        # fp64 stays at the parity bar
        tp, tg = TOL[precision] if precision == 64 else (2e-3, 1e-2)
        assert ep <= tp and eg <= tg, (precision, f.tree.depth, ep, eg)


@pytest.mark.parametrize("gradient,input_order", [(True, True), (False, True), (True, False)])
def test_evaluate_many_equals_evaluate(require_gpu, gradient, input_order):
    """kifmm_gpu_evaluate_many (copies pipelined against the evaluates on three streams, double-buffered
    staging) returns, for every right-hand side, exactly what one evaluate call returns."""
    pos, _ = generators.sample("uniform-cube", 40000, seed=5, fp32=True)
    cfg = fmm.FmmConfig(p=6, n_crit=40, precision=32, gradient=gradient)
    qs = np.stack([generators.sample("uniform-cube", 40000, seed=100 + k, charges="signed", fp32=True)[1]
                   for k in range(5)]).astype(np.float32)
    with fmm.Fmm(pos, cfg) as f:
        pots, grads = f.evaluate_many(qs, input_order=input_order)
        for k in range(len(qs)):
            p1, g1, _ = f.evaluate(qs[k], input_order=input_order)
            assert np.array_equal(pots[k], p1)
            if gradient:
                assert np.array_equal(grads[k], g1)
            else:
                assert grads is None
        empty = f.evaluate_many(np.zeros((0, 40000), np.float32))
        assert empty[0].shape == (0, 40000)


@pytest.mark.parametrize("p", [5, 6, 7])
def test_fp64_dmma_gemm_matches_simt(require_gpu, monkeypatch, p):
    """fp64 GEMMs (solves, M2M, M2L, L2L) on the DMMA tensor op agree with the SIMT DFMA kernel
    (KIFMM_DMMA=0) to fp64 rounding, and both with the oracle within the fp64 gate."""
    pos, q = generators.sample("two-cluster", 6000, seed=41, charges="signed")
    out = {}
    for dm in ("0", "1"):
        monkeypatch.setenv("KIFMM_DMMA", dm)
        with fmm.Fmm(pos, fmm.FmmConfig(p=p, n_crit=30, precision=64, gradient=True)) as f:
            out[dm] = f.evaluate(q)[:2]
            ref, gref = _ref(f, q, True)
    assert fmm.relative_error(out["1"][0], out["0"][0]) <= 1e-13
    assert fmm.relative_error(out["1"][0], ref) <= 1e-12
    assert fmm.relative_error(out["1"][1], gref) <= 1e-11


def test_schedule_switches_bit_identical(require_gpu, monkeypatch):
    """Scheduling-only switches change no arithmetic: the split downward chain (KIFMM_DN_SPLIT) and
    programmatic dependent launch (KIFMM_PDL) give bit-identical results; the tap-set face split of the
    M2L tiles (KIFMM_TC_FACE) regroups rows into tiles and stays within fp32 rounding."""
    pos, q = generators.sample("uniform-cube", 200000, seed=13, charges="signed", fp32=True)
    cfg = fmm.FmmConfig(p=6, n_crit=40, precision=32, gradient=True)
    out = {}
    for name, env in [("ref", {}), ("nosplit", {"KIFMM_DN_SPLIT": "0"}), ("nopdl", {"KIFMM_PDL": "0"}),
                      ("noface", {"KIFMM_TC_FACE": "0"})]:
        for k in ("KIFMM_DN_SPLIT", "KIFMM_PDL", "KIFMM_TC_FACE"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        with fmm.Fmm(pos, cfg) as f:
            out[name] = f.evaluate(q)[:2]
    for name in ("nosplit", "nopdl"):
        assert np.array_equal(out[name][0], out["ref"][0]) and np.array_equal(out[name][1], out["ref"][1]), name
    assert fmm.relative_error(out["noface"][0], out["ref"][0]) <= 1e-6


@pytest.mark.parametrize("dist,n,ncrit,p", [("uniform-cube", 20000, 40, 7), ("sphere-surface", 20000, 30, 6),
                                            ("two-cluster", 12000, 20, 7)])
def test_fp64_int8_ozaki_m2l(require_gpu, dist, n, ncrit, p):
    """fp64 M2L on the int8 tensor cores (m2l_backend 4, the fp64 default for p = 6, 7) against the DMMA
    kernel (backend 1) and the fp64 oracle: the digit-sliced products are exact in int32, so the two
    backends agree to fp64 rounding and both meet the 1e-12 parity gate."""
    pos, q = generators.sample(dist, n, seed=17, charges="signed")
    out = {}
    for b in (4, 1):
        with fmm.Fmm(pos, fmm.FmmConfig(p=p, n_crit=ncrit, precision=64, gradient=True, m2l_backend=b)) as f:
            assert f.info()["m2l_backend"] == b
            out[b] = f.evaluate(q)[:2]
            if b == 4:
                ref, gref = _ref(f, q, True)
    e41 = fmm.relative_error(out[4][0], out[1][0])
    e4 = fmm.relative_error(out[4][0], ref)
    eg4 = fmm.relative_error(out[4][1], gref)
    print(f"ozaki {dist} p={p}: vs DMMA {e41:.2e}, vs oracle {e4:.2e} (gradient {eg4:.2e})")
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.path.join("gpurun_out", "ozaki_r02.jsonl"), "a") as fh:
        fh.write(json.dumps({"dist": dist, "n": n, "n_crit": ncrit, "p": p, "charges": "signed",
                             "rel_l2_vs_dmma": e41, "rel_l2_vs_oracle": e4, "rel_l2_gradient_vs_oracle": eg4,
                             "lib": os.environ.get("KIFMM_LIB", "default")}) + "\n")
    assert e41 <= 1e-12 and e4 <= 1e-12 and eg4 <= 1e-11


def test_fp64_int8_ozaki_dynamic_range(require_gpu):
    """The int8 digits are relative to each LEVEL's largest multipole, so rows far below it keep fewer
    bits.  Charges spanning six decades (log-uniform, random signs) on a clustered cloud still meet the
    fp64 gate against the DMMA kernel and the oracle."""
    pos, _ = generators.sample("two-cluster", 12000, seed=41)
    rng = np.random.default_rng(41)
    q = rng.choice([-1.0, 1.0], size=len(pos)) * 10.0 ** rng.uniform(-6, 0, size=len(pos))
    out = {}
    for b in (4, 1):
        with fmm.Fmm(pos, fmm.FmmConfig(p=7, n_crit=20, precision=64, m2l_backend=b)) as f:
            out[b] = f.evaluate(q)[0]
            if b == 4:
                ref, _ = _ref(f, q, False)
    assert fmm.relative_error(out[4], out[1]) <= 1e-12
    assert fmm.relative_error(out[4], ref) <= 1e-12


def test_int8_m2l_is_fp64_only(require_gpu):
    pos, q = generators.sample("uniform-cube", 3000, seed=1, charges="signed", fp32=True)
    with pytest.raises(InvalidArgument):
        fmm.Fmm(pos, fmm.FmmConfig(p=6, n_crit=40, precision=32, m2l_backend=4))


def test_fp64_near_serial_bit_identical(require_gpu, monkeypatch):
    """fp64 runs the near field on the plan stream after L2L (KIFMM_NEAR_SERIAL, the fp64 default) or on
    the side stream next to the tree passes: the same kernels and accumulation order, bit-identical."""
    pos, q = generators.sample("uniform-cube", 20000, seed=31, charges="signed")
    out = {}
    for v in ("1", "0"):
        monkeypatch.setenv("KIFMM_NEAR_SERIAL", v)
        with fmm.Fmm(pos, fmm.FmmConfig(p=6, n_crit=40, precision=64, gradient=True)) as f:
            out[v] = f.evaluate(q)[:2]
    assert np.array_equal(out["1"][0], out["0"][0]) and np.array_equal(out["1"][1], out["0"][1])


@pytest.mark.parametrize("gradient,input_order", [(False, True), (True, True), (True, False)])
def test_far_surface_chunks(require_gpu, monkeypatch, gradient, input_order):
    """Far works with many (M2P) surfaces are cut into chunks whose partial sums far_combine_kernel adds in
    chunk order: the result equals the unchunked far kernel (KIFMM_FAR_CHUNK=0) to fp32 summation order,
    in input order and in reordered order, with and without gradient, and meets the oracle gate."""
    pos, q = generators.sample("sphere-surface", 60000, seed=29, charges="signed", fp32=True)
    cfg = fmm.FmmConfig(p=6, n_crit=40, precision=32, gradient=gradient)
    out = {}
    for ch in ("0", "3"):
        monkeypatch.setenv("KIFMM_FAR_CHUNK", ch)
        with fmm.Fmm(pos, cfg) as f:
            qq = q if input_order else q[f.tree.original_index]
            out[ch] = f.evaluate(qq, input_order=input_order)[:2]
            if ch == "3":
                ref, gref = _ref(f, q, gradient)
                if not input_order:
                    ref = ref[f.tree.original_index]
                    gref = gref[f.tree.original_index] if gradient else None
    assert fmm.relative_error(out["3"][0], out["0"][0]) <= 1e-6
    assert fmm.relative_error(out["3"][0], ref) <= 1e-5
    if gradient:
        assert fmm.relative_error(out["3"][1], out["0"][1]) <= 1e-6
        assert fmm.relative_error(out["3"][1], gref) <= 5e-5
