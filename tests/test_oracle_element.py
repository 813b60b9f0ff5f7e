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
