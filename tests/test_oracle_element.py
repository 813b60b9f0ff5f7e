"""Pins for the oracle's element operator (C1).

Independent of the oracle: 2x2x2 Gauss-Legendre quadrature of grad(phi_a).grad(phi_b) for
trilinear phi (exact for these integrands on boxes), written here with numpy's
leggauss nodes, and the textbook unit-cube values x12 (h/3, 0, -h/12, -h/12).
"""
import numpy as np
import pytest

import oracle as O


def gauss_element_matrix(hx, hy, hz):
    g, w = np.polynomial.legendre.leggauss(2)
    pts = (g + 1.0) / 2.0     # map to [0, 1]
    wts = w / 2.0
    h = np.array([hx, hy, hz])
    K = np.zeros((8, 8))
    for i, xi in enumerate(pts):
        for j, eta in enumerate(pts):
            for k, zeta in enumerate(pts):
                wq = wts[i] * wts[j] * wts[k] * hx * hy * hz
                grads = []
                for a in range(8):
                    bits = [(a >> d) & 1 for d in range(3)]
                    t = [xi, eta, zeta]
                    val1 = [t[d] if bits[d] else 1.0 - t[d] for d in range(3)]
                    dval = [(1.0 if bits[d] else -1.0) / h[d] for d in range(3)]
                    grads.append(np.array([
                        dval[0] * val1[1] * val1[2],
                        val1[0] * dval[1] * val1[2],
                        val1[0] * val1[1] * dval[2]]))
                for a in range(8):
                    for b in range(8):
                        K[a, b] += wq * grads[a] @ grads[b]
    return K


@pytest.mark.parametrize("h", [(1.0, 1.0, 1.0), (0.1, 0.1, 0.1), (1 / 300, 1 / 300, 1 / 300),
                               (1 / 600, 1 / 300, 1 / 300), (0.5, 0.25, 0.125)])
def test_matches_gauss_quadrature(h):
    K = O.element_matrix(*h)
    G = gauss_element_matrix(*h)
    scale = np.abs(G).max()
    assert np.abs(K - G).max() <= 1e-15 * scale * 4


def test_unit_cube_times_12():
    # diagonal h/3, edge-adjacent 0, face-diagonal -h/12, body-diagonal -h/12
    K = O.element_matrix(1.0, 1.0, 1.0) * 12.0
    np.testing.assert_allclose(K[0], [4, 0, 0, -1, 0, -1, -1, -1], atol=1e-14)
    h = 0.1
    K = O.element_matrix(h, h, h)
    np.testing.assert_allclose(np.diag(K), np.full(8, h / 3), rtol=1e-15)


@pytest.mark.parametrize("h", [(0.1, 0.1, 0.1), (1 / 600, 1 / 300, 1 / 300), (0.3, 0.7, 0.2)])
def test_symmetric_and_zero_row_sums(h):
    K = O.element_matrix(*h)
    assert np.array_equal(K, K.T)          # exact symmetry
    assert np.abs(K.sum(axis=1)).max() <= 1e-15 * np.abs(K).max() * 8


def test_depends_only_on_difference_pattern():
    K = O.element_matrix(0.2, 0.3, 0.4)
    for a in range(8):
        for b in range(8):
            d = a ^ b
            assert K[a, b] == K[0, d]


# SURVEY §8(c)-C1 test vectors: the canonical rounding sequence of C1,
# K(d) = fl(fl(T_x + T_y) + T_z), T_a = fl(fl(S_a M_b) M_c), evaluated for the configs'
# element sizes (h_a = fl(1/n_a)).  Index of d = (dx, dy, dz) in row 0: dx + 2 dy + 4 dz.
# These values were derived outside this repo and are stored as the shortest
# round-trip decimal strings, so each comparison below is bit-exact.  A reordered product
# (e.g. fl(S fl(M_b M_c))) or a re-associated sum moves at least one of them by an ulp.
C1_VECTORS = [
    ((10, 10, 10), {0: "0.033333333333333326", 1: "0.0", 3: "-0.008333333333333331",
                    7: "-0.008333333333333331"}),
    ((300, 300, 300), {0: "0.0011111111111111111", 3: "-0.0002777777777777778",
                       7: "-0.0002777777777777778"}),
    ((600, 300, 300), {0: "0.0011111111111111111", 1: "-0.0005555555555555556",
                       2: "0.0002777777777777778", 3: "-0.00041666666666666664",
                       6: "0.0", 7: "-0.0002777777777777778"}),
]


@pytest.mark.parametrize("n,vec", C1_VECTORS)
def test_c1_canonical_vectors(n, vec):
    K = O.element_matrix(1.0 / n[0], 1.0 / n[1], 1.0 / n[2])
    for d, s in vec.items():
        assert K[0, d] == float(s), (n, d, K[0, d].hex(), float(s).hex())
    # n = 10: the canonical K(000) is one ulp below fl(h/3) -- the rounding sequence matters
    if n == (10, 10, 10):
        assert K[0, 0] != 0.1 / 3.0


@pytest.mark.parametrize("n", [(10, 10, 10), (300, 300, 300), (600, 300, 300), (7, 3, 5)])
def test_c1_within_few_ulp_of_exact_rationals(n):
    """Exact K(d) of the trilinear brick (tensor product of the 1-D stiffness [1,-1]/h and
    mass [1/3, 1/6] h factors) evaluated in rationals at the rounded h_a = fl(1/n_a): the
    canonical floating-point sequence (four roundings per term, two additions) stays within a
    few ulp of the sum of the terms' magnitudes (the sum cancels: zero row sums)."""
    from fractions import Fraction as F
    h = [F(1.0 / m) for m in n]
    for d in range(8):
        dd = [(d >> k) & 1 for k in range(3)]
        exact = F(0)
        scale = F(0)
        for a in range(3):
            S = (-1 if dd[a] else 1) / h[a]
            M = F(1)
            for b in range(3):
                if b != a:
                    M *= h[b] / (6 if dd[b] else 3)
            exact += S * M
            scale += abs(S * M)
        K = O.element_matrix(*[float(x) for x in h])[0, d]
        if exact == 0:
            assert K == 0.0
        else:
            ulp = np.spacing(float(scale))
            assert abs(F(K) - exact) <= 4 * F(ulp), (n, d)
