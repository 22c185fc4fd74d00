"""kernel and surface KATs."""
import itertools
import math

import numpy as np
import pytest

from paper_2303_08394_b200 import InvalidArgument, host


def test_laplace_examples():
    assert host.laplace((0, 0, 0), (1, 0, 0)) == pytest.approx(1 / (4 * math.pi), rel=1e-15)
    assert abs(host.laplace((0, 0, 0), (1, 0, 0)) - 0.0795774715) < 1e-10
    assert host.laplace((0.3, 0.2, 0.1), (0.3, 0.2, 0.1)) == 0.0
    assert host.laplace((0, 0, 0), (0, 2, 0)) == pytest.approx(0.5 * host.laplace((0, 0, 0), (1, 0, 0)))


def test_laplace_symmetry_homogeneity():
    rng = np.random.default_rng(0)
    for _ in range(100):
        x, y = rng.random(3), rng.random(3)
        assert host.laplace(x, y) == host.laplace(y, x)
        t = 3.7
        assert host.laplace(t * x, t * y) == pytest.approx(host.laplace(x, y) / t, rel=1e-14)


def test_kernel_matrix_examples():
    assert host.kernel_matrix([[0, 0, 0]], [[1, 0, 0]])[0, 0] == pytest.approx(1 / (4 * math.pi))
    assert host.kernel_matrix([[1, 2, 3]], [[1, 2, 3]])[0, 0] == 0.0
    rng = np.random.default_rng(1)
    s, t, q = rng.random((7, 3)), rng.random((5, 3)), rng.random(7)
    K = host.kernel_matrix(s, t)
    loop = np.array([sum(q[i] * host.laplace(s[i], t[j]) for i in range(7)) for j in range(5)])
    assert np.allclose(K @ q, loop, rtol=1e-14, atol=0)


def test_p2p_double_loop():  # SPEC.md:310-312 (through kernel_matrix, K q == p2p)
    rng = np.random.default_rng(2)
    s, q = rng.random((100, 3)), rng.random(100)
    K = host.kernel_matrix(s, s)
    d = s[:, None, :] - s[None, :, :]
    r = np.sqrt((d * d).sum(-1))
    with np.errstate(divide="ignore"):
        ref = (np.where(r > 0, 1 / r, 0) * q[None, :]).sum(1) / (4 * np.pi)
    assert np.max(np.abs(K @ q - ref) / np.abs(ref)) < 1e-13
    assert np.all(host.kernel_matrix(s, s) @ np.zeros(100) == 0)


@pytest.mark.parametrize("p", range(2, 17))
def test_surface_count(p):
    g = host.surface_grid(p)
    assert g.shape == (6 * (p - 1) ** 2 + 2, 3) == (host.surface_count(p), 3)
    assert np.all(np.max(np.abs(g), axis=1) == 1.0)
    assert len({tuple(x) for x in g}) == len(g)


def test_surface_examples():
    assert host.surface_grid(2).shape[0] == 8
    assert host.surface_grid(6).shape[0] == 152
    with pytest.raises(InvalidArgument):
        host.surface_grid(1)


def test_surface_cube_symmetries():
    g = host.surface_grid(5)
    pts = {tuple(np.round(x, 12)) for x in g}
    for perm in itertools.permutations(range(3)):
        for signs in itertools.product((-1, 1), repeat=3):
            h = g[:, perm] * np.array(signs)
            assert {tuple(np.round(x, 12)) for x in h} == pts


def test_scaled_surface():
    g = host.surface_grid(4)
    s = host.scaled_surface(g, (0.5, 0.5, 0.5), 0.5, 1.0)
    assert np.allclose(np.max(np.abs(s - 0.5), axis=1), 0.5)
    s = host.scaled_surface(g, (0.5, 0.5, 0.5), 0.5, 2.95)
    assert np.allclose(np.max(np.abs(s - 0.5), axis=1), 1.475)
