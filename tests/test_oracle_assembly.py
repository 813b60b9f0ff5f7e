"""Pins for the oracle's FE assembly and Dirichlet elimination (C2, C3; P:36, P:48, P:52,
P:251-266).

Independent references: a dense numpy assembly from the Gauss-quadrature element matrix of
test_oracle_element (no oracle arithmetic), the textbook interior-row stencil x12/h
{32, 0 x6, -2 x12, -1 x8} with zero row sum, and the definition of symmetric elimination.
"""
import itertools

import numpy as np
import pytest

import oracle as O
from tests.test_oracle_element import gauss_element_matrix


def dense_assembly(nx, ny, nz):
    NX, NY, NZ = nx + 1, ny + 1, nz + 1
    rows = NX * NY * NZ
    A = np.zeros((rows, rows))
    Ke = gauss_element_matrix(1.0 / nx, 1.0 / ny, 1.0 / nz)
    for ez, ey, ex in itertools.product(range(nz), range(ny), range(nx)):
        nodes = [(ex + (a & 1)) + NX * ((ey + ((a >> 1) & 1)) + NY * (ez + ((a >> 2) & 1)))
                 for a in range(8)]
        for a in range(8):
            for b in range(8):
                A[nodes[a], nodes[b]] += Ke[a, b]
    return A


def to_dense(s, val):
    A = np.zeros((s.rows, s.rows))
    for i in range(s.rows):
        for k in range(s.row_ptr[i], s.row_ptr[i + 1]):
            A[i, s.col[k]] = val[k]
    return A


def coords(n, gid):
    nx, ny, nz = n
    return gid % (nx + 1), (gid // (nx + 1)) % (ny + 1), gid // ((nx + 1) * (ny + 1))


def is_bc(n, gid):
    ix, iy, iz = coords(n, gid)
    return ix in (0, n[0]) or iy in (0, n[1]) or iz in (0, n[2])


@pytest.mark.parametrize("n", [(2, 2, 2), (3, 2, 4), (4, 4, 4), (5, 3, 2)])
def test_assembly_matches_dense_quadrature(n):
    s = O.assemble(*n, keep_pre_bc=True)
    A = to_dense(s, s.val_pre_bc)
    D = dense_assembly(*n)
    assert np.abs(A - D).max() <= 1e-15 * np.abs(D).max() * 16
    assert np.array_equal(A, A.T)                       # exact symmetry
    assert np.abs(A.sum(axis=1)).max() <= 1e-15 * np.abs(D).max() * 64   # row sums 0
    assert np.all(s.b_pre_bc == 0.0)                    # zero source (G6)


def test_interior_row_stencil():
    n = 6
    h = 1.0 / n
    s = O.assemble(n, n, n, keep_pre_bc=True)
    gid = 3 + 7 * (3 + 7 * 3)
    cols = s.col[s.row_ptr[gid]:s.row_ptr[gid + 1]]
    vals = s.val_pre_bc[s.row_ptr[gid]:s.row_ptr[gid + 1]] * 12.0 / h
    assert cols.size == 27
    expect = []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                k = abs(dx) + abs(dy) + abs(dz)
                expect.append({0: 32.0, 1: 0.0, 2: -2.0, 3: -1.0}[k])
    np.testing.assert_allclose(vals, expect, atol=1e-12)
    assert abs(vals.sum()) < 1e-12


@pytest.mark.parametrize("n", [(2, 2, 2), (3, 3, 3), (4, 3, 5)])
def test_dirichlet_definition(n):
    s = O.assemble(*n, keep_pre_bc=True)
    A0 = to_dense(s, s.val_pre_bc)
    A = to_dense(s, s.val)
    rows = s.rows
    v = np.array([1.0 if coords(n, g)[0] == n[0] else 0.0 for g in range(rows)])
    bc = np.array([is_bc(n, g) for g in range(rows)])
    # constrained rows: identity rows, b = v
    for i in np.where(bc)[0]:
        e = np.zeros(rows)
        e[i] = 1.0
        assert np.array_equal(A[i], e)
        assert s.b[i] == v[i]
    # free rows: constrained columns eliminated, b = -sum_i A_ji v_i
    for j in np.where(~bc)[0]:
        assert np.all(A[j, bc] == 0.0)
        assert np.array_equal(A[j, ~bc], A0[j, ~bc])
        assert abs(s.b[j] - (-(A0[j, bc] * v[bc]).sum())) <= 1e-15
    assert np.array_equal(A, A.T)
    # pattern unchanged (G5): structural zeros are still stored
    assert s.val.size == s.val_pre_bc.size
    # count of 1.0 rhs entries = (ny+1)(nz+1)
    assert int((s.b == 1.0).sum()) == (n[1] + 1) * (n[2] + 1)


def test_rhs_next_to_hot_face_equals_h():
    # free rows adjacent to x=1 away from other faces: b = -(-8 - 4) h/12 = h
    n = 6
    s = O.assemble(n, n, n)
    gid = (n - 1) + (n + 1) * (3 + (n + 1) * 3)
    assert abs(s.b[gid] - 1.0 / n) <= 1e-15
    gid = 1 + (n + 1) * (3 + (n + 1) * 3)        # next to x = 0: b = 0
    assert s.b[gid] == 0.0


@pytest.mark.parametrize("n", [2, 3, 4])
def test_spd_after_bc(n):
    s = O.assemble(n, n, n)
    A = to_dense(s, s.val)
    ev = np.linalg.eigvalsh(A)
    assert ev.min() > 0.0


@pytest.mark.parametrize("n", [(4, 3, 5), (6, 6, 6)])
def test_single_row_routine_matches_full_assembly(n):
    s = O.assemble(*n)
    for gid in range(s.rows):
        cols, vals, b = O.row(*n, gid)
        assert np.array_equal(cols, s.col[s.row_ptr[gid]:s.row_ptr[gid + 1]])
        assert np.array_equal(vals, s.val[s.row_ptr[gid]:s.row_ptr[gid + 1]])
        assert b == s.b[gid]
