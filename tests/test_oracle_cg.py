"""Pins for the oracle's CG (C6) on systems with known solutions.

Independent references: CG's finite-termination property on tiny SPD systems,
exact rational solves of the assembled FE system written here with fractions.Fraction
(closed-form element entries h/3, 0, -h/12, -h/12 from SPEC S:134, dense assembly, symmetric
elimination, Gaussian elimination), numpy.linalg.solve at 10^3, and CG's monotone A-norm
error.
"""
import itertools
from fractions import Fraction

import numpy as np
import pytest

import oracle as O


def csr_from_dense(D):
    rp, cols, vals = [0], [], []
    for i in range(D.shape[0]):
        nz = np.nonzero(D[i])[0]
        cols += nz.tolist()
        vals += D[i, nz].tolist()
        rp.append(len(cols))
    return (np.array(rp, dtype=np.int64), np.array(cols, dtype=np.int64),
            np.array(vals, dtype=np.float64))


def test_identity_one_iteration():
    n = 7
    b = np.linspace(-3, 5, n)
    rp, c, v = csr_from_dense(np.eye(n))
    r = O.cg(rp, c, v, b, 50, 1e-12)
    assert r.status == O.OR_OK and r.converged == 1 and r.iters == 1
    assert np.array_equal(r.x, b)


def test_2x2_spec_example():
    rp, c, v = csr_from_dense(np.array([[4.0, 1.0], [1.0, 3.0]]))
    r = O.cg(rp, c, v, np.array([1.0, 2.0]), 10, 1e-14)
    assert r.status == O.OR_OK and r.converged and r.iters <= 2
    np.testing.assert_allclose(r.x, [1 / 11, 7 / 11], atol=1e-15)


def test_status_codes():
    # pAp < 0 -> not SPD
    rp, c, v = csr_from_dense(np.array([[-1.0]]))
    r = O.cg(rp, c, v, np.array([1.0]), 5, 0.0)
    assert r.status == O.OR_ENOTSPD and r.iters == 0
    # b = 0: rr = 0 and pAp = 0 -> converged with zero iterations
    rp, c, v = csr_from_dense(np.eye(3))
    r = O.cg(rp, c, v, np.zeros(3), 5, 0.0)
    assert r.status == O.OR_OK and r.converged and r.iters == 0 and r.hist[0] == 0.0
    # NaN in the matrix -> diverged
    r = O.cg(np.array([0, 1]), np.array([0]), np.array([np.nan]), np.array([1.0]), 5, 0.0)
    assert r.status == O.OR_EDIVERGED
    # invalid arguments
    r = O.cg(rp, c, v, np.ones(3), 0, 0.0)
    assert r.status == O.OR_EINVAL


def exact_fe_solution(n):
    """Exact rational solution of the Dirichlet-eliminated FE system on an n^3 cube."""
    h = Fraction(1, n)
    Kd = {0: h / 3, 1: Fraction(0), 2: -h / 12, 3: -h / 12}
    N = n + 1
    rows = N ** 3
    A = [[Fraction(0)] * rows for _ in range(rows)]
    for ez, ey, ex in itertools.product(range(n), repeat=3):
        nodes = [(ex + (a & 1)) + N * ((ey + ((a >> 1) & 1)) + N * (ez + ((a >> 2) & 1)))
                 for a in range(8)]
        for a in range(8):
            for b in range(8):
                A[nodes[a]][nodes[b]] += Kd[bin(a ^ b).count("1")]

    def xyz(g):
        return g % N, (g // N) % N, g // (N * N)

    bc = [any(c in (0, n) for c in xyz(g)) for g in range(rows)]
    val = [Fraction(1) if xyz(g)[0] == n else Fraction(0) for g in range(rows)]
    free = [g for g in range(rows) if not bc[g]]
    M = [[A[i][j] for j in free] + [-sum(A[i][k] * val[k] for k in range(rows) if bc[k])]
         for i in free]
    m = len(free)
    for col in range(m):       # Gauss-Jordan, exact
        piv = next(r for r in range(col, m) if M[r][col] != 0)
        M[col], M[piv] = M[piv], M[col]
        pv = M[col][col]
        M[col] = [e / pv for e in M[col]]
        for r in range(m):
            if r != col and M[r][col] != 0:
                f = M[r][col]
                M[r] = [a - f * b for a, b in zip(M[r], M[col])]
    x = list(val)
    for k, g in enumerate(free):
        x[g] = M[k][m]
    return x


def test_exact_rationals_small_meshes():
    # values quoted in SURVEY §8(c) P6 must agree with the exact computation here
    x2 = exact_fe_solution(2)
    assert x2[13] == Fraction(3, 8)
    x3 = exact_fe_solution(3)
    assert x3[1 + 4 * (1 + 4 * 1)] == Fraction(12, 175)
    assert x3[2 + 4 * (1 + 4 * 1)] == Fraction(72, 175)
    x4 = exact_fe_solution(4)
    assert x4[2 + 5 * (2 + 5 * 2)] == Fraction(234, 1127)


@pytest.mark.parametrize("n", [2, 3, 4])
def test_oracle_cg_matches_exact_solution(n):
    xe = np.array([float(v) for v in exact_fe_solution(n)])
    s = O.assemble(n, n, n)
    r = O.cg(s.row_ptr, s.col, s.val, s.b, 200, 1e-14)
    assert r.status == O.OR_OK and r.converged
    assert np.abs(r.x - xe).max() <= 1e-14


def test_10cubed_against_direct_solve():
    s = O.assemble(10, 10, 10)
    A = np.zeros((s.rows, s.rows))
    for i in range(s.rows):
        A[i, s.col[s.row_ptr[i]:s.row_ptr[i + 1]]] = s.val[s.row_ptr[i]:s.row_ptr[i + 1]]
    xd = np.linalg.solve(A, s.b)
    r = O.cg(s.row_ptr, s.col, s.val, s.b, 200, 1e-14)
    assert r.status == O.OR_OK and r.converged and r.iters < 60
    assert np.abs(r.x - xd).max() <= 1e-13
    # recurrence residual vs explicit b - A x
    true_res = np.linalg.norm(s.b - A @ r.x)
    assert abs(true_res - r.hist[-1]) <= 1e-10 * r.hist[0]
    # tol = 0 runs exactly max_iters (benchmark mode)
    r0 = O.cg(s.row_ptr, s.col, s.val, s.b, 200, 0.0)
    assert r0.iters == 200 and r0.converged == 0 and r0.hist.size == 201
    assert np.all(np.isfinite(r0.hist))


def test_energy_norm_monotone():
    # ||x_k - x*||_A strictly decreases
    s = O.assemble(4, 4, 4)
    A = np.zeros((s.rows, s.rows))
    for i in range(s.rows):
        A[i, s.col[s.row_ptr[i]:s.row_ptr[i + 1]]] = s.val[s.row_ptr[i]:s.row_ptr[i + 1]]
    xs = np.linalg.solve(A, s.b)
    prev = np.inf
    for k in range(1, 12):
        r = O.cg(s.row_ptr, s.col, s.val, s.b, k, 0.0)
        if r.iters < k:
            break
        e = r.x - xs
        en = float(e @ A @ e)
        if en < 1e-28:          # at rounding level (7 distinct eigen-components here)
            break
        assert en < prev
        prev = en


def test_history_prefix_property():
    # running K iterations and K' > K iterations share the first K+1 history entries
    s = O.assemble(6, 5, 4)
    a = O.cg(s.row_ptr, s.col, s.val, s.b, 10, 0.0)
    b = O.cg(s.row_ptr, s.col, s.val, s.b, 25, 0.0)
    assert np.array_equal(a.hist, b.hist[:11])
