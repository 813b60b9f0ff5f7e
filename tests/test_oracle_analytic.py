"""Pins for the analytical solution (C8) and FE verification.

Independent references: boundary values (the series must vanish on five faces), the
six-face superposition identity (the six rotated problems sum to the constant 1 inside the
cube, so u(1/2,1/2,1/2) = 1/6 exactly), and second-order FE convergence.
"""
import numpy as np
import pytest

import oracle as O


def test_centre_is_one_sixth():
    assert abs(O.analytic(0.5, 0.5, 0.5, 300) - 1.0 / 6.0) <= 1e-13


@pytest.mark.parametrize("pt", [(0.3, 0.6, 0.2), (0.1, 0.45, 0.8), (0.77, 0.21, 0.5)])
def test_six_face_superposition(pt):
    x, y, z = pt
    u = lambda a, b, c: O.analytic(a, b, c, 300)   # noqa: E731  (u = 1 on the face a = 1)
    total = (u(x, y, z) + u(1 - x, y, z) + u(y, x, z) + u(1 - y, x, z) + u(z, x, y) +
             u(1 - z, x, y))
    assert abs(total - 1.0) <= 1e-10


def test_homogeneous_faces():
    for (x, y, z) in [(0.0, 0.3, 0.4), (0.5, 0.0, 0.5), (0.5, 1.0, 0.5), (0.7, 0.2, 0.0),
                      (0.2, 0.6, 1.0)]:
        assert abs(O.analytic(x, y, z, 300)) <= 1e-12


def test_series_converged_in_terms():
    # doubling the term cap changes interior values by <= 1e-10
    for pt in [(0.5, 0.5, 0.5), (0.2, 0.5, 0.5), (0.9, 0.3, 0.7)]:
        assert abs(O.analytic(*pt, 300) - O.analytic(*pt, 150)) <= 1e-10


def fe_solution(n):
    s = O.assemble(n, n, n)
    r = O.cg(s.row_ptr, s.col, s.val, s.b, 2000, 1e-12)
    assert r.status == O.OR_OK and r.converged
    return r.x


def at(x, n, p):
    N = n + 1
    ix, iy, iz = (int(round(c * n)) for c in p)
    return x[ix + N * (iy + N * iz)]


PROBES = [(0.5, 0.5, 0.5), (0.2, 0.5, 0.5), (0.8, 0.5, 0.5), (0.5, 0.2, 0.5), (0.6, 0.3, 0.7)]


def test_fe_error_second_order():
    errs = {}
    for n in (10, 20):
        x = fe_solution(n)
        h = 1.0 / n
        for p in PROBES:
            e = at(x, n, p) - O.analytic(*p, 300)
            assert abs(e) <= 2.0 * h * h, (n, p, e)
            errs[(n, p)] = abs(e)
    for p in PROBES:
        assert errs[(20, p)] < errs[(10, p)]     # refinement monotonicity
        # O(h^2): halving h divides the error by ~4
        assert 2.5 < errs[(10, p)] / errs[(20, p)] < 6.0
