"""operators/precompute and persistence.

Eigen3 (the reference's SVD, CMakeLists.txt:16) is un-vendored and absent, so
the in-repo Jacobi SVD is cross-checked against numpy.linalg.svd (LAPACK).
"""
import os

import numpy as np
import pytest

from paper_2303_08394_b200 import CacheMismatch, CorruptArchive, InvalidArgument, fmm, host


@pytest.fixture(scope="module")
def ops6():
    return host.Operators(p=6, domain_side=1.0)


def test_jacobi_svd_matches_lapack():
    rng = np.random.default_rng(0)
    # (300, 280) and the odd (270, 257) take the parallel round-robin order (n >= 256; a bye column when odd)
    for shape in ((40, 40), (60, 30), (300, 280), (270, 257)):
        a = rng.standard_normal(shape)
        u, s, v = host.svd(a)
        s_np = np.linalg.svd(a, compute_uv=False)
        assert np.allclose(s, s_np, rtol=1e-13, atol=1e-13 * s_np[0])
        assert np.allclose(u @ np.diag(s) @ v.T, a, atol=1e-12)
        assert np.allclose(v.T @ v, np.eye(shape[1]), atol=1e-12)


def test_precompute_independent_of_thread_count():
    """Operators do not depend on the host thread count: p = 6 (serial cyclic SVDs next to the M2L
    matrices) and p = 8 (parallel round-robin Jacobi batch)."""
    for p in (6, 8):
        a = host.Operators(p=p, domain_side=1.0, threads=1)
        b = host.Operators(p=p, domain_side=1.0, threads=3)
        for x, y in zip(a.uc2e + a.dc2e + (a.m2m, a.l2l, a.m2l), b.uc2e + b.dc2e + (b.m2m, b.l2l, b.m2l)):
            assert np.array_equal(x, y), p


def test_svd_of_check_matrix(ops6):
    # singular values of K(up-check <- up-equivalent) agree with LAPACK to 1e-13 sigma_max
    g = host.surface_grid(6)
    h2 = 1.0 / 8
    K = host.kernel_matrix(1.05 * h2 * g, 2.95 * h2 * g)
    s_np = np.linalg.svd(K, compute_uv=False)
    U, S, V = ops6.uc2e
    assert np.max(np.abs(S - s_np[:len(S)])) <= 1e-13 * s_np[0]
    # factored pinv residual on the numerical row space
    rng = np.random.default_rng(1)
    for _ in range(5):
        v = V @ rng.standard_normal(V.shape[1])  # a vector in the kept row space
        rec = V @ ((U.T @ (K @ v)) / S)
        assert np.linalg.norm(rec - v) / np.linalg.norm(v) <= 1e-6


def test_shapes_and_counts():
    o = host.Operators(p=2, domain_side=1.0)
    assert o.n_e == o.n_c == 8
    assert o.m2m.shape == (8, 8, 8) and o.l2l.shape == (8, 8, 8)
    assert o.m2l.shape == (316, 8, 8)
    assert np.all(np.isfinite(o.m2l))


def test_m2l_matrices_are_kernel_matrices(ops6):
    # K_t = kernel_matrix(source up-equivalent at offset t, target down-check) at level 2
    tv = host.transfer_vectors()
    g = host.surface_grid(6)
    h2 = 1.0 / 8
    for t in (0, 100, 315):
        src = np.array(tv[t]) * 2 * h2 + 1.05 * h2 * g
        tgt = 1.05 * h2 * g
        assert np.array_equal(ops6.m2l[t], host.kernel_matrix(src, tgt))


def test_m2m_composite(ops6):
    # M2M_o = uc2e_inv(2) K(child ue(3) -> parent uc(2)), factored in fp64
    g = host.surface_grid(6)
    h2, h3 = 1.0 / 8, 1.0 / 16
    U, S, V = ops6.uc2e
    for o in (0, 5, 7):
        c = np.array([(1 if o & 1 else -1), (1 if o & 2 else -1), (1 if o & 4 else -1)]) * h3
        K = host.kernel_matrix(c + 1.05 * h3 * g, 2.95 * h2 * g)
        ref = V @ ((U.T @ K) / S[:, None])
        assert np.allclose(ops6.m2m[o], ref, rtol=1e-9, atol=1e-9 * np.abs(ref).max())


def test_m2m_far_field(ops6):  # parent expansion reproduces the far field
    g = host.surface_grid(6)
    h2, h3 = 1.0 / 8, 1.0 / 16
    U, S, V = ops6.uc2e
    rng = np.random.default_rng(2)
    o = 3
    c = np.array([(1 if o & 1 else -1), (1 if o & 2 else -1), (1 if o & 4 else -1)]) * h3
    pts = c + (rng.random((20, 3)) - 0.5) * 2 * h3
    q = rng.random(20)
    # child multipole (level 3 => scale 2^(2-3))
    chk = host.kernel_matrix(pts, c + 2.95 * h3 * g) @ q
    m_child = 0.5 * (V @ ((U.T @ chk) / S))
    m_par = ops6.m2m[o] @ m_child
    far = np.array([[1.3, 0.2, -0.7], [-0.9, 1.1, 0.4]])
    direct = host.kernel_matrix(pts, far) @ q
    via = host.kernel_matrix(1.05 * h2 * g, far) @ m_par
    assert np.max(np.abs(via - direct) / np.abs(direct)) <= 1e-5


def test_p2m_far_field(ops6):  # unit charge at the leaf centre, 10 widths away
    g = host.surface_grid(6)
    h2 = 1.0 / 8
    U, S, V = ops6.uc2e
    chk = host.kernel_matrix(np.zeros((1, 3)), 2.95 * h2 * g) @ np.ones(1)
    m = V @ ((U.T @ chk) / S)
    tgt = np.array([[10 * 2 * h2, 0.0, 0.0]])
    est = host.kernel_matrix(1.05 * h2 * g, tgt) @ m
    exact = host.laplace((0, 0, 0), tgt[0])
    assert abs(est[0] - exact) / exact <= 1e-5


def test_invalid_config():
    with pytest.raises(InvalidArgument):
        host.Operators(p=1)
    with pytest.raises(InvalidArgument):
        host.Operators(p=4, alpha_inner=3.0, alpha_outer=2.0)
    with pytest.raises(InvalidArgument):
        host.Operators(p=4, svd_cutoff=0.0)


def test_cache_round_trip(tmp_path, ops6):
    path = str(tmp_path / "ops.cache")
    ops6.save(path)
    back = host.Operators.load(path, ops6.fingerprint)
    for a, b in ((ops6.m2l, back.m2l), (ops6.m2m, back.m2m), (ops6.l2l, back.l2l), (ops6.uc2e[0], back.uc2e[0]),
                 (ops6.uc2e[1], back.uc2e[1]), (ops6.dc2e[2], back.dc2e[2]), (ops6.surface, back.surface)):
        assert a.tobytes() == b.tobytes()
    assert back.fingerprint == ops6.fingerprint
    assert fmm.operator_fingerprint(6, 1.05, 2.95, 1e-12, 1.0) == ops6.fingerprint
    # 64-byte aligned segments
    raw = open(path, "rb").read()
    header = int(raw[:15])
    assert header % 64 == 0


def test_cache_failures(tmp_path, ops6):
    path = str(tmp_path / "ops.cache")
    ops6.save(path)
    with pytest.raises(CacheMismatch):
        host.Operators.load(path, ops6.fingerprint ^ 1)
    raw = open(path, "rb").read()
    trunc = str(tmp_path / "trunc.cache")
    open(trunc, "wb").write(raw[: len(raw) // 2])
    with pytest.raises(CorruptArchive):
        host.Operators.load(trunc, ops6.fingerprint)
    foreign = str(tmp_path / "foreign.cache")
    open(foreign, "wb").write(raw.replace(b"KIFMM-OPERATOR-CACHE 1", b"KIFMM-OPERATOR-CACHE 9", 1))
    with pytest.raises(CacheMismatch):
        host.Operators.load(foreign, 0)
    with pytest.raises(Exception):
        host.Operators.load(str(tmp_path / "missing.cache"), 0)


def test_load_or_precompute(tmp_path):
    cfg = fmm.FmmConfig(p=3, cache=str(tmp_path / "c.cache"))
    a = fmm.load_or_precompute(cfg, 2.0)
    assert os.path.exists(cfg.cache)
    b = fmm.load_or_precompute(cfg, 2.0)
    assert a.m2l.tobytes() == b.m2l.tobytes()
    with pytest.warns(UserWarning):
        c = fmm.load_or_precompute(cfg, 3.0)  # different domain -> fingerprint mismatch -> rebuild
    assert c.domain_side == 3.0
