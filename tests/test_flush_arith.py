"""The two float64 shortcuts of the K1 flush kernels (ott_flush.cu), checked against exact
rational arithmetic on the CPU:

* line_params, 2-bit: RN(range / 3) as Markstein's FMA correction of RN(range * RN(1/3))
  (quant.py:64 divides in float64);
* threshold_tie: floor(fl((v - x_min) / step)) >= k decided without the division as
  fma(-k, step, v - x_min) >= -delta_k step, delta_k the distance from k to the rounding
  midpoint below it (2^(e-53), or 2^(e-54) for k = 2^e), exact when v - x_min is close to k step.

The GPU parity suite checks the kernels bit-exactly against the oracle. These tests pin the
arithmetic claims themselves, including significands near 1, 4/3 and 2."""
import math
from fractions import Fraction

import numpy as np

C3 = 1.0 / 3.0


def fma(a, b, c):  # correctly rounded a * b + c
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def div3(x):
    q0 = x * C3
    return fma(fma(-q0, 3.0, x), C3, q0)


def test_markstein_division_by_three_is_correctly_rounded():
    rng = np.random.default_rng(5)
    xs = []
    for e in range(-40, 41, 3):
        for m in range(64):
            xs += [float.fromhex("0x1.%013xp%d" % (((1 << 52) - 1 - m), e)),  # significand near 2
                   float.fromhex("0x1.%013xp%d" % (m, e)),  # near 1
                   float.fromhex("0x1.%013xp%d" % ((0x5555555555555 + m - 32) & ((1 << 52) - 1), e))]  # near 4/3
    xs += [float(v) for v in (rng.random(4000) + 1.0) * 2.0 ** rng.integers(-30, 30, 4000)]
    # ranges of fp16 lines (differences of two fp16 values, exact in float64)
    h = rng.standard_normal((4000, 2)) * 2.0 ** rng.integers(-14, 14, (4000, 1))
    h = h.astype(np.float16).astype(np.float64)
    xs += [abs(a - b) for a, b in h if np.isfinite(a) and np.isfinite(b) and a != b]
    for x in xs:
        assert div3(x) == x / 3.0, x.hex()


def tie_delta(k):  # ott_flush.cu tie_delta
    e = k.bit_length() - 1
    return 2.0 ** (e - 53 - (1 if k & (k - 1) == 0 else 0))


def test_threshold_tie_without_division():
    rng = np.random.default_rng(6)
    seen = {}
    for it in range(40000):
        step = float(rng.random() * 2.0 ** int(rng.integers(-24, 12)))
        if step == 0.0:
            continue
        k = int(rng.integers(1, 3)) if it % 2 else int(rng.integers(1, 255))  # levels up to 255 (8-bit)
        d = k * step  # RN(k step)
        j = int(rng.integers(-5, 6))
        for _ in range(abs(j)):
            d = float(np.nextafter(d, math.inf if j > 0 else -math.inf))
        ref = math.floor(d / step) >= k
        assert (fma(-k, step, d) >= -step * tie_delta(k)) == ref, (step, k, j)
        seen[ref] = seen.get(ref, 0) + 1
    assert min(seen.get(True, 0), seen.get(False, 0)) > 1000
