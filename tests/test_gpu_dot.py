"""C5 on the device, pinned to exact arithmetic (reading C5).

minife_exact_round is the rounding step every CG dot ends with (warp-parallel carry
normalisation + round-to-nearest-even, exact.cuh).  Its expected values come from Python's
exact integer arithmetic: int / int true division is correctly rounded (ties to even), so
RN(sum w_i 2^(32 i - 1074)) = (sum w_i 2^(32 i)) / 2^1074 needs no float arithmetic at all.
minife_dot (the full device dot) is compared with the oracle's exact dot (itself pinned to
math.fsum in test_oracle_dot_spmv.py).
"""
import math
import struct

import numpy as np
import pytest

import oracle as O

M = pytest.importorskip("paper_1505_08023_b200")

pytestmark = pytest.mark.gpu

DIGITS = 68


def exact_rn(words):
    """RN of the accumulator value by exact integer arithmetic (Python int true division)."""
    if len(words) > DIGITS and words[DIGITS] != 0:
        return math.nan
    v = sum(int(w) << (32 * i) for i, w in enumerate(words[:DIGITS]))
    if v == 0:
        return 0.0
    try:
        return v / (1 << 1074)
    except OverflowError:
        return math.inf if v > 0 else -math.inf


def bits(x):
    return struct.unpack("<q", struct.pack("<d", x))[0]


def same(a, b):
    if math.isnan(a) or math.isnan(b):
        return math.isnan(a) and math.isnan(b)
    return bits(a) == bits(b)


def check(words):
    words = [int(w) for w in words]
    got = M.exact_round(np.array(words, dtype=np.int64))
    want = exact_rn(words)
    assert same(got, want), (words, got, want)


def words_for(x: float):
    """Accumulator words holding exactly the double x (one 32-bit chunk per word)."""
    from fractions import Fraction
    v = Fraction(x) * (1 << 1074)            # every double is an integer multiple of 2^-1074
    assert v.denominator == 1
    v = int(v)
    w = [0] * DIGITS
    neg = v < 0
    v = abs(v)
    i = 0
    while v:
        w[i] = (v & 0xffffffff) * (-1 if neg else 1)
        v >>= 32
        i += 1
    return w


def test_exact_round_special_values():
    check([0] * DIGITS)                                      # exact zero -> +0.0
    assert bits(M.exact_round([0] * DIGITS)) == 0
    check([1 << 32, -1] + [0] * 66)                          # cancels to zero -> +0.0
    assert bits(M.exact_round([1 << 32, -1])) == 0
    check([1])                                               # smallest subnormal
    check([-1])
    check([0, 0, 0] + [0] * 64 + [1])                        # 2^(32*67-1074): huge but finite
    check([0] * 67 + [1 << 40])                              # overflows -> inf
    check([0] * 67 + [-(1 << 40)])                           # -> -inf
    w = [0] * 72
    w[68] = 1                                                # non-finite flag -> NaN
    assert math.isnan(M.exact_round(w))
    for x in (1.0, -1.0, 0.1, -3.75, 5e-324, 2.2250738585072014e-308, 1.7976931348623157e308,
              math.pi * 1e-300, -math.e * 1e200):
        got = M.exact_round(words_for(x))
        assert same(got, x), (x, got)


def test_exact_round_ties_and_carries():
    # one = 2^0: word holding 2^1074 -> digit 33, bit 18
    one = [0] * DIGITS
    one[33] = 1 << 18
    check(one)
    # 1 + 2^-53 (exact tie, even -> 1), 1 + 3 2^-53 (tie, rounds up), 1 + 2^-53 + tiny, ...
    base = (1 << 1074)
    for num in (base + (base >> 53), base + 3 * (base >> 53), base + (base >> 53) + 1,
                base - (base >> 54), base - (base >> 54) - 1, -(base + (base >> 53))):
        w = []
        v = num
        neg = v < 0
        v = abs(v)
        for i in range(DIGITS):
            w.append(((v >> (32 * i)) & 0xffffffff) * (-1 if neg else 1))
        check(w)
    # long carry chains: digits that are all ones, borrowed from above, mixed signs
    check([0xffffffff] * 40 + [0] * 28)
    check([-1] + [0] * 39 + [1])
    check([1] + [0] * 50 + [-1])                             # negative, just above -2^(32*51)
    check([(1 << 63) - 1] * DIGITS)                          # max words: carries everywhere
    check([-(1 << 63)] * DIGITS)
    check([(1 << 63) - 1, -(1 << 63)] * 34)


def test_exact_round_random_words():
    rng = np.random.default_rng(1505)
    for trial in range(300):
        kind = trial % 5
        w = np.zeros(DIGITS, dtype=np.int64)
        if kind == 0:                                        # dense, full int64 range
            w[:] = rng.integers(-(1 << 63), (1 << 63) - 1, DIGITS, dtype=np.int64)
        elif kind == 1:                                      # sparse, small magnitudes
            idx = rng.integers(0, DIGITS, 5)
            w[idx] = rng.integers(-(1 << 33), 1 << 33, 5)
        elif kind == 2:                                      # near-cancelling top digits
            t = int(rng.integers(3, DIGITS))
            w[t] = 1
            w[t - 1] = -(1 << 32) + int(rng.integers(0, 3))
            w[:t - 1] = rng.integers(-(1 << 20), 1 << 20, t - 1)
        elif kind == 3:                                      # typical CG accumulator: a band
            lo = int(rng.integers(0, 50))
            w[lo:lo + 6] = rng.integers(-(1 << 50), 1 << 50, 6)
        else:                                                # subnormal range
            w[:3] = rng.integers(-(1 << 40), 1 << 40, 3)
        check(w.tolist())


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_dot_matches_oracle(seed):
    rng = np.random.default_rng(seed)
    n = 200_003
    u = rng.uniform(-1, 1, n)
    v = rng.uniform(-1, 1, n)
    assert same(M.dot(u, v), O.dot(u, v))
    # huge dynamic range and cancellation: sum of (a, -a) pairs plus small terms
    a = rng.standard_normal(n) * np.exp2(rng.integers(-600, 600, n))
    b = rng.standard_normal(n) * np.exp2(rng.integers(-400, 400, n))
    u2 = np.concatenate([a, a, [1e-300, 3.0]])
    v2 = np.concatenate([b, -b, [1e-10, 1.0]])
    got = M.dot(u2, v2)
    assert same(got, O.dot(u2, v2))
    assert same(got, math.fsum([1e-300 * 1e-10, 3.0]))
    perm = rng.permutation(u2.size)                          # order independence
    assert same(M.dot(u2[perm], v2[perm]), got)


def test_dot_edge_cases():
    e = np.zeros(0)
    assert bits(M.dot(e, e)) == 0                            # empty -> +0.0
    z = np.array([-0.0, 0.0, -0.0])
    assert bits(M.dot(z, np.ones(3))) == 0                   # exact zero -> +0.0
    assert math.isnan(M.dot(np.array([1.0, np.inf]), np.array([1.0, 1.0])))
    assert math.isnan(M.dot(np.array([np.nan]), np.array([0.0])))
    t = np.array([1.0, 2.0 ** -53])                          # tie: 1 + 2^-53 -> 1
    assert M.dot(t, np.ones(2)) == 1.0
    t = np.array([1.0, 2.0 ** -53, 2.0 ** -200])             # above the tie -> next up
    assert M.dot(t, np.ones(3)) == np.nextafter(1.0, 2.0)
    # exact result above the binade of the largest term, still finite
    t = np.array([2.0 ** 1000, 2.0 ** 1000, 2.0 ** 1000])
    assert M.dot(t, np.ones(3)) == 3 * 2.0 ** 1000
