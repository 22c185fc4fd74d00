"""CPU checks of the numerical argument behind the fp64 M2L on the int8 tensor cores (m2l_oz.cuh, DESIGN
9.2): the digit split, its bounds, the int32 headroom of the tap chunking, and the accuracy of the
triangular truncation -- restated in numpy (the device code cannot run here)."""
import numpy as np

S = 8  # digit slices per operand (KIFMM_OZ_SLICES)


def level_exp(m):
    """E with max|x| 2^-E < 1/2 (oz::level_exp)."""
    return int(np.frexp(m)[1]) + 1 if m > 0 else 0


def digits(x, e):
    """x 2^-e = sum_i d_i 2^-7i, d_i = rint(128 y) of the running remainder (oz_slice_kernel)."""
    y = np.ldexp(x, -e)
    out = []
    for _ in range(S):
        y = y * 128.0
        d = np.rint(y)
        y = y - d
        out.append(d.astype(np.int64))
    return np.stack(out), y


def test_level_exponent_matches_device_formula():
    # device: ilogb(m) + 2; numpy frexp returns the exponent of m = f 2^k, f in [0.5, 1): k = ilogb + 1
    for m in (1e-300, 0.3, 0.5, 1.0, 1.5, 7.99, 8.0, 1e300):
        e = level_exp(m)
        assert m * 2.0 ** -e < 0.5 and m * 2.0 ** -e >= 0.125


def test_digits_are_signed_7_bit_and_exact():
    rng = np.random.default_rng(0)
    x = rng.standard_normal(20000) * 10.0 ** rng.uniform(-6, 3, 20000)
    e = level_exp(np.abs(x).max())
    d, rest = digits(x, e)
    assert np.abs(d).max() <= 64  # int8 with headroom: |y| < 1/2 before every step
    # every step is exact in fp64 (scaling by 128, subtracting an integer): the digits and the remainder
    # reproduce x exactly, and the remainder is below 2^-7S of the level scale
    recon = sum(np.ldexp(d[i].astype(np.float64), e - 7 * (i + 1)) for i in range(S))
    assert np.allclose(recon + np.ldexp(rest, e - 7 * S), x, rtol=0, atol=0)
    assert np.abs(rest).max() <= 0.5


def test_int32_headroom_of_tap_chunks():
    # tap_max<NP>() = 2^31 / (S NP 64 64): the largest digit-sum group holds S products
    for np_, expect in ((224, 292), (160, 409)):
        tap_max = (2 ** 31 - 1) // (S * np_ * 64 * 64)
        assert tap_max == expect
        assert S * np_ * 64 * 64 * tap_max < 2 ** 31


def test_triangular_truncation_accuracy():
    """sum_{i + j <= S + 1} D_i E_j^T 2^-7(i+j) against the fp64 product, for a tap-like block."""
    rng = np.random.default_rng(1)
    n, k = 64, 218
    a = rng.standard_normal((n, k)) * 10.0 ** rng.uniform(-3, 0, (n, 1))  # rows of different magnitudes
    b = rng.standard_normal((k, k))
    ea, eb = level_exp(np.abs(a).max()), level_exp(np.abs(b).max())
    da, _ = digits(a, ea)
    db, _ = digits(b, eb)
    acc = np.zeros((n, k))
    for i in range(1, S + 1):
        for j in range(1, S + 1):
            if i + j <= S + 1:
                prod = da[i - 1] @ db[j - 1].T  # exact integer product (int64 here, int32 on the device)
                assert np.abs(prod).max() < 2 ** 31
                acc += np.ldexp(prod.astype(np.float64), -7 * (i + j))
    approx = np.ldexp(acc, ea + eb)
    exact = a @ b.T
    rel = np.linalg.norm(approx - exact) / np.linalg.norm(exact)
    assert rel < 1e-13, rel
