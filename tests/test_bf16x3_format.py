"""CPU check of the bf16x3 leaf format's error budget (no GPU).

cfg5's leaves multiply fp32 operands as x = hi + lo, hi = bf16_rn(x),
lo = bf16_rn(x - hi), computing hi_a.hi_b + hi_a.lo_b + lo_a.hi_b (csrc/
elementwise.cu lincomb_split_kernel, csrc/tc_gemm.cu tc_pair_kernel<..., B3>).
Here the split is emulated bit-exactly in NumPy (round-to-nearest-even to the
top 16 bits of the fp32 pattern, as __float2bfloat16_rn) and the three products
accumulated in float64, isolating the format's own error from the tensor core's
fp32 accumulation: per product <= 2^-15 relative Frobenius, and a 2-level
Strassen with these leaves stays far inside cfg5's 1e-4."""

import numpy as np
import pytest


def bf16_rn(x: np.ndarray) -> np.ndarray:
    """float32 -> nearest bf16 (ties to even), returned as float32."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return r.astype(np.uint32).view(np.float32)


def split(x: np.ndarray):
    hi = bf16_rn(x)
    lo = bf16_rn((x - hi).astype(np.float32))
    return hi, lo


def mm3(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    ah, al = (v.astype(np.float64) for v in split(a))
    bh, bl = (v.astype(np.float64) for v in split(b))
    return ah @ bh + ah @ bl + al @ bh


def test_bf16_rounding_matches_definition():
    x = np.array([1.0, 1.00390625, 1.005859375, -3.14159265, 2.0 ** -20, 65504.0], dtype=np.float32)
    h = bf16_rn(x)
    assert np.all(h.view(np.uint32) & 0xFFFF == 0)
    # nearest: |x - h| <= half an ulp of bf16 (8 significant bits)
    assert np.all(np.abs(x - h) <= np.abs(x) * 2.0 ** -8)
    assert h[1] == 1.0            # 1 + 2^-8 is a tie: even mantissa (1.0)
    assert h[2] == 1.0078125      # above the tie: rounds up


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_split_reconstruction(seed):
    x = np.random.default_rng(seed).uniform(-4, 4, 100000).astype(np.float32)
    hi, lo = split(x)
    rec = hi.astype(np.float64) + lo.astype(np.float64)
    assert np.max(np.abs(rec - x) / np.abs(x)) <= 2.0 ** -16


@pytest.mark.parametrize("n,k", [(64, 512), (128, 4096)])
def test_product_error(n, k):
    rng = np.random.default_rng(n + k)
    a = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    b = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    ref = a.astype(np.float64) @ b.astype(np.float64)
    err = np.linalg.norm(mm3(a, b) - ref) / np.linalg.norm(ref)
    assert err <= 2.0 ** -15, err


def _strassen(a, b, base, leaf):
    n = a.shape[0]
    if n <= base:
        return leaf(a, b)
    h = n // 2
    A = {q: a[i * h:(i + 1) * h, j * h:(j + 1) * h] for q, (i, j) in
         {"00": (0, 0), "01": (0, 1), "10": (1, 0), "11": (1, 1)}.items()}
    B = {q: b[i * h:(i + 1) * h, j * h:(j + 1) * h] for q, (i, j) in
         {"00": (0, 0), "01": (0, 1), "10": (1, 0), "11": (1, 1)}.items()}
    f = np.float32
    M1 = _strassen((A["00"] + A["11"]).astype(f), (B["00"] + B["11"]).astype(f), base, leaf)
    M2 = _strassen((A["10"] + A["11"]).astype(f), B["00"], base, leaf)
    M3 = _strassen(A["00"], (B["01"] - B["11"]).astype(f), base, leaf)
    M4 = _strassen(A["11"], (B["10"] - B["00"]).astype(f), base, leaf)
    M5 = _strassen((A["00"] + A["01"]).astype(f), B["11"], base, leaf)
    M6 = _strassen((A["10"] - A["00"]).astype(f), (B["00"] + B["01"]).astype(f), base, leaf)
    M7 = _strassen((A["01"] - A["11"]).astype(f), (B["10"] + B["11"]).astype(f), base, leaf)
    return np.block([[M1 + M4 - M5 + M7, M3 + M5], [M2 + M4, M1 - M2 + M3 + M6]])


def test_two_level_strassen_with_bf16x3_leaves():
    """fp32 S/T sums (as the GPU forms them), bf16x3 leaves: the relative
    Frobenius error vs the f64 product stays well under cfg5's 1e-4.  Measured
    here 1.7e-5 (f64 leaves: 1.5e-7; one classic bf16x3 product: 3.8e-6 -- the
    two Strassen levels amplify the leaf error ~4.6x through the S/T sums and
    the C combination); the GPU's fp32 accumulation adds a little (2.3e-5 at
    n = 16384, tests/test_gpu_strassen.py)."""
    n = 256
    rng = np.random.default_rng(1005)
    a = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    b = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    ref = a.astype(np.float64) @ b.astype(np.float64)
    c = _strassen(a, b, n // 4, mm3)
    err = np.linalg.norm(c - ref) / np.linalg.norm(ref)
    assert err <= 3e-5, err
