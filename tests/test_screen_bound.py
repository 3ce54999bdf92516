"""The fp32 screening bound of the selection kernel (csrc/select.cuh), checked on
the CPU with a restatement of its arithmetic: every score the kernel computes in
fp32 -- 8 lanes x (two interleaved FFMA2 partial sums over 4-element float4
steps), lane sums, a 3-level shuffle tree -- lies within
gamma_(d+4) |x|_2 |q|_2 + 2^-100 of the exact dot product, on random rows and on
rows built for heavy cancellation.  (Test infrastructure: numpy only.)"""

import math

import numpy as np
import pytest


def screen_gamma(d: int) -> float:
    """csrc/select.cuh screen_gamma, as the host computes it."""
    n, u = float(d + 4), 2.0 ** -24
    g = n * u / (1.0 - n * u)
    return float(np.float32(g * (1.0 + 2.0 ** -20) * (1.0 + 1.2e-7)))


def fma32(a, b, c):
    """fp32 fused multiply-add: the product is exact in fp64, one rounding."""
    return np.float32(np.float64(a) * np.float64(b) + np.float64(c))


def kernel_dot32(x: np.ndarray, q: np.ndarray) -> np.float32:
    """group_dots (screened): lane l8 owns float4 m of column 4*(l8 + 8m); per
    float4 two FFMA2 on (x.x, x.y) and (x.z, x.w) into a float2 accumulator;
    lane value = acc.x + acc.y; tree: l += shfl_down(4), (2), (1)."""
    d = x.shape[0]
    lanes = []
    for l8 in range(8):
        ax = ay = np.float32(0)
        for m in range(d // 32):
            c = 4 * (l8 + 8 * m)
            ax = fma32(x[c], q[c], ax)
            ay = fma32(x[c + 1], q[c + 1], ay)
            ax = fma32(x[c + 2], q[c + 2], ax)
            ay = fma32(x[c + 3], q[c + 3], ay)
        lanes.append(np.float32(ax + ay))
    for off in (4, 2, 1):
        lanes = [np.float32(lanes[i] + lanes[i + off]) if i + off < 8 else lanes[i]
                 for i in range(8)]
    return lanes[0]


def kernel_bound(x: np.ndarray, q: np.ndarray) -> float:
    """|x|_2 |q|_2 gamma + 2^-100, every step rounded upward (an upper bound
    of what the kernel computes with __ffma2_ru / __fadd_ru / __fsqrt_ru /
    __fmul_ru)."""
    up = lambda v: np.nextafter(np.float32(v), np.float32(np.inf))
    nx = up(np.sqrt(up(np.sum(np.float64(x) ** 2))))
    nq = up(np.sqrt(up(np.sum(np.float64(q) ** 2))))
    return float(up(up(np.float64(nx) * nq) * screen_gamma(x.shape[0]))) + 2.0 ** -100


@pytest.mark.parametrize("d", [64, 128])
def test_screen_bound_random_and_cancelling(d):
    rng = np.random.default_rng(d)
    worst = 0.0
    for trial in range(300):
        q = rng.standard_normal(d).astype(np.float32) * np.float32(0.125)
        if trial % 3 == 0:
            x = rng.standard_normal(d).astype(np.float32) * np.float32(0.125)
        elif trial % 3 == 1:
            # heavy cancellation: pairs of large opposite contributions
            x = (rng.choice([-1.0, 1.0], d) * (2.0 ** rng.integers(-6, 12, d))).astype(np.float32)
            x[1::2] = -x[0::2] * q[0::2] / np.where(q[1::2] == 0, 1, q[1::2])
        else:
            # magnitudes over 30 orders
            x = (rng.standard_normal(d) * 10.0 ** rng.integers(-15, 15, d)).astype(np.float32)
        exact = math.fsum(float(a) * float(b) for a, b in zip(x, q))
        s32 = float(kernel_dot32(x, q))
        b = kernel_bound(x, q)
        assert abs(s32 - exact) <= b, (trial, s32, exact, b)
        if b > 0:
            worst = max(worst, abs(s32 - exact) / b)
    assert worst < 1.0


def test_gamma_matches_the_bound_formula():
    # gamma_(d+4) = (d+4) u / (1 - (d+4) u), u = 2^-24, with 2^-20 headroom
    for d in (64, 128, 256):
        n = d + 4
        g = n * 2.0 ** -24 / (1 - n * 2.0 ** -24)
        assert g * (1 + 2.0 ** -20) <= screen_gamma(d) <= g * (1 + 2.0 ** -18)
