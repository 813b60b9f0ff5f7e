"""Pins for the oracle's SpMV (C4; Fig 3.1) and exactly-rounded dot (C5).

The dot is pinned to Python's math.fsum, which is documented to return the correctly
rounded sum of its float inputs: fed the rounded products fl(u_i v_i) it is exactly C5's
definition, computed by an unrelated algorithm (Shewchuk partials).  SpMV is pinned to
SPEC's hand examples, a dense numpy product, and the signed-zero rule of C4.
"""
import math

import numpy as np
import pytest

import oracle as O


def fsum_dot(u, v):
    return math.fsum((np.asarray(u) * np.asarray(v)).tolist())


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_dot_random_vs_fsum(seed):
    rng = np.random.default_rng(seed)
    n = 5000
    u = rng.standard_normal(n) * np.exp(rng.uniform(-30, 30, n))
    v = rng.standard_normal(n)
    assert O.dot(u, v) == fsum_dot(u, v)


def test_dot_cancellation():
    u = np.array([1e16, 1.0, -1e16, 3.0, 1e-30])
    v = np.ones_like(u)
    assert O.dot(u, v) == fsum_dot(u, v) == 4.0 + 1e-30
    # catastrophic: huge terms cancel exactly, tiny survive
    u = np.array([1e300, 1e-300, -1e300])
    assert O.dot(u, np.ones(3)) == 1e-300


def test_dot_ties_to_even():
    one = 1.0
    e = 2.0 ** -53
    # 1 + 2^-53 is a tie -> rounds to even (1.0)
    assert O.dot([one, e], [1.0, 1.0]) == 1.0
    # any sticky bit below breaks the tie upwards
    assert O.dot([one, e, 2.0 ** -200], [1.0, 1.0, 1.0]) == 1.0 + 2.0 ** -52
    # (1 + 2^-52) + 2^-53 is a tie with odd last bit -> rounds up to 1 + 2^-51
    assert O.dot([one + 2.0 ** -52, e], [1.0, 1.0]) == 1.0 + 2.0 ** -51
    # negative mirror
    assert O.dot([-one, -e], [1.0, 1.0]) == -1.0


def test_dot_subnormals_and_range():
    tiny = 5e-324
    u = np.array([tiny, tiny, 3 * tiny, -tiny, 2.0 ** -1022, 1e-310])
    v = np.ones_like(u)
    assert O.dot(u, v) == fsum_dot(u, v)
    # products that underflow are rounded first (fl(u*v)), then summed exactly
    u = np.array([1e-200, 1e-200, 3e-170])
    v = np.array([1e-200, 3e-150, 1e-160])
    assert O.dot(u, v) == fsum_dot(u, v)
    rng = np.random.default_rng(7)
    u = rng.standard_normal(3000) * np.exp(rng.uniform(-700, 700, 3000))
    v = rng.standard_normal(3000)
    assert O.dot(u, v) == fsum_dot(u, v)


def test_dot_zero_overflow_nonfinite():
    assert O.dot([0.0, -0.0], [1.0, 1.0]) == 0.0
    assert math.copysign(1.0, O.dot([1.0, -1.0], [1.0, 1.0])) == 1.0    # exact zero -> +0.0
    big = np.finfo(np.float64).max
    assert O.dot([big, big], [1.0, 1.0]) == math.inf
    assert O.dot([big, big, -big], [1.0, 1.0, 1.0]) == big     # exact, no spurious overflow
    assert math.isnan(O.dot([1.0, math.inf], [1.0, 1.0]))
    assert math.isnan(O.dot([1.0, math.nan], [1.0, 1.0]))
    assert O.dot([], []) == 0.0


def test_dot_order_independent():
    rng = np.random.default_rng(11)
    u = rng.standard_normal(2000) * 1e5
    v = rng.standard_normal(2000)
    perm = rng.permutation(2000)
    assert O.dot(u, v) == O.dot(u[perm], v[perm])


def test_spmv_spec_examples():
    # S:214 identity -> y = x
    n = 6
    rp = np.arange(n + 1, dtype=np.int64)
    x = np.linspace(-1, 1, n)
    assert np.array_equal(O.spmv(rp, np.arange(n), np.ones(n), x), x)
    # rows {0: [(0,1),(1,2)], 1: [(1,3)]}, x = (1,1) -> (3,3)
    y = O.spmv(np.array([0, 2, 3]), np.array([0, 1, 1]), np.array([1.0, 2.0, 3.0]),
               np.array([1.0, 1.0]))
    assert np.array_equal(y, [3.0, 3.0])


def test_spmv_random_vs_dense():
    # random 20x20, 30% density -> dense oracle to <= 1e-13 relative
    rng = np.random.default_rng(5)
    D = rng.standard_normal((20, 20)) * (rng.uniform(size=(20, 20)) < 0.3)
    rp = [0]
    cols, vals = [], []
    for i in range(20):
        nz = np.nonzero(D[i])[0]
        cols += nz.tolist()
        vals += D[i, nz].tolist()
        rp.append(len(cols))
    x = rng.standard_normal(20)
    y = O.spmv(np.array(rp), np.array(cols), np.array(vals), x)
    ref = D @ x
    assert np.abs(y - ref).max() <= 1e-13 * np.abs(D).sum(axis=1).max()


def test_spmv_left_fold_and_signed_zero():
    # C4: s = +0.0; s = fl(s + fl(a x)) in stored order; an all-(-0) row gives +0.0
    y = O.spmv(np.array([0, 2]), np.array([0, 1]), np.array([-1.0, -2.0]),
               np.array([0.0, 0.0]))
    assert y[0] == 0.0 and math.copysign(1.0, y[0]) == 1.0
    # order matters in fp: (1e16 + 1) - 1e16 = 0 in a left fold, 1 in the other order
    y = O.spmv(np.array([0, 3]), np.array([0, 1, 2]), np.array([1e16, 1.0, -1e16]),
               np.ones(3))
    assert y[0] == 0.0
    y = O.spmv(np.array([0, 3]), np.array([0, 1, 2]), np.array([1e16, -1e16, 1.0]),
               np.ones(3))
    assert y[0] == 1.0
