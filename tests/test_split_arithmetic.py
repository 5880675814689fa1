"""Arithmetic behind DESIGN.md reading R14 (FP16 operands of the tensor-core translations),
checked on the CPU with numpy emulations of the two operand formats: a three-product split
A_h B_h + A_h B_r + A_r B_h with 11-bit heads and remainders loses the same accuracy whether the
heads / remainders are TF32 numbers or power-of-two row-scaled fp16 numbers, and the scaling is
what makes that true (unscaled fp16 flushes small rows).  Products are summed in fp64 here, so
only the operand representation is compared (the translations are matrix
products; the paper fixes no precision)."""
import numpy as np


def _tf32(x):
    """round-to-nearest (ties away, as cvt.rna) to TF32: 10 explicit mantissa bits"""
    b = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x1000) & 0xFFFFE000
    return b.astype(np.uint32).view(np.float32)


def _split_tf32(x):
    h = _tf32(x)
    return h.astype(np.float64), _tf32((x - h.astype(np.float64)).astype(np.float32)).astype(np.float64)


def _pow2_scale(amax):
    """2^(12 - floor(log2 amax)) per row (1 for zero rows), as split_rows_h_kernel"""
    e = np.floor(np.log2(np.where(amax > 0, amax, 1.0)))
    return np.where(amax > 0, np.exp2(12 - e), 1.0)


def _split_fp16(x, scaled=True):
    s = _pow2_scale(np.abs(x).max(axis=1, keepdims=True)) if scaled else np.ones((x.shape[0], 1))
    a = (x * s).astype(np.float32)
    h = a.astype(np.float16)
    r = (a - h.astype(np.float32)).astype(np.float16)
    return h.astype(np.float64) / s, r.astype(np.float64) / s


def _three_products(split_a, split_b, A, B):
    ah, ar = split_a(A)
    bh, br = split_b(B)
    return ah @ bh.T + ah @ br.T + ar @ bh.T


def _rel(x, ref):
    return np.linalg.norm(x - ref) / np.linalg.norm(ref)


def test_scaled_fp16_split_matches_the_tf32_split():
    rng = np.random.default_rng(0)
    for spread in (0, 4, 8):          # decades of magnitude spread inside each row
        A = rng.standard_normal((96, 456)) * 10.0 ** (-spread * rng.random((96, 456)))
        B = rng.standard_normal((64, 456)) * 10.0 ** (-spread * rng.random((64, 456)))
        B *= 10.0 ** rng.uniform(-12, 12, (64, 1))          # state rows of any magnitude
        ref = A @ B.T
        e_tf32 = _rel(_three_products(_split_tf32, _split_tf32, A, B), ref)
        e_fp16 = _rel(_three_products(_split_fp16, _split_fp16, A, B), ref)
        assert e_tf32 < 4e-7 and e_fp16 < 4e-7, (spread, e_tf32, e_fp16)
        assert e_fp16 < 2.0 * e_tf32 + 1e-9, (spread, e_tf32, e_fp16)
        # one product alone (11 bits) is three orders worse: the split is what gives fp32 accuracy
        ah, _ = _split_fp16(A)
        bh, _ = _split_fp16(B)
        assert _rel(ah @ bh.T, ref) > 100 * e_fp16


def test_fp16_needs_the_row_scale():
    rng = np.random.default_rng(1)
    A = rng.standard_normal((32, 200))
    B = rng.standard_normal((16, 200)) * 1e-9               # below the fp16 subnormal range
    ref = A @ B.T
    unscaled = _three_products(lambda x: _split_fp16(x, False), lambda x: _split_fp16(x, False), A, B)
    assert np.abs(unscaled).max() == 0.0                    # flushed to zero
    assert _rel(_three_products(_split_fp16, _split_fp16, A, B), ref) < 4e-7


def test_scale_is_an_exact_power_of_two_and_bounds_the_row():
    rng = np.random.default_rng(2)
    x = rng.standard_normal((50, 64)) * 10.0 ** rng.uniform(-30, 30, (50, 1))
    s = _pow2_scale(np.abs(x).max(axis=1, keepdims=True))
    m, _ = np.frexp(s)
    assert np.all(m == 0.5)                                 # exact powers of two
    top = np.abs(x * s).max(axis=1)
    assert np.all(top >= 2.0 ** 12) and np.all(top < 2.0 ** 13)   # below the fp16 maximum 65504
    assert _pow2_scale(np.zeros((1, 1)))[0, 0] == 1.0
