"""Pins for the oracle's mesh indexing and matrix structure (Fig 3.6).

Each check is fixed by something other than the oracle: SPEC's worked examples, the closed
form nnz = prod(3N_a - 2) (BASELINE.json's nnz figures), and a brute-force "two nodes share
an element" enumeration, which is the definition of the FE sparsity pattern.
"""
import itertools

import numpy as np
import pytest

import oracle as O


def test_node_id_spec_examples():
    # S:58-60
    assert O.node_id((3, 3, 3), 0, 0, 0) == 0
    assert O.node_id((3, 3, 3), 1, 1, 1) == 13
    assert O.node_id((3, 3, 3), -1, 0, 0) < 0
    # G3: per-axis check -- ix = 3 on a 3-wide line must not wrap to the next line
    assert O.node_id((3, 3, 3), 3, 0, 0) < 0
    assert O.node_id((3, 3, 3), 0, 3, 0) < 0


def test_node_id_bijection():
    nodes = (4, 3, 5)
    ids = [O.node_id(nodes, ix, iy, iz)
           for iz in range(5) for iy in range(3) for ix in range(4)]
    assert ids == list(range(60))   # x-fastest enumeration = ascending ids


@pytest.mark.parametrize("n,rows,nnz", [((1, 1, 1), 8, 64), ((2, 2, 2), 27, 343),
                                        ((3, 3, 3), 64, 1000)])
def test_structure_small_counts(n, rows, nnz):
    # S:205-207 and the closed form
    row_ptr, col = O.structure(*n)
    assert row_ptr.size - 1 == rows
    assert row_ptr[-1] == nnz


@pytest.mark.parametrize("n", [(1, 1, 1), (4, 4, 4), (5, 3, 2), (10, 10, 10), (7, 1, 3)])
def test_nnz_closed_form(n):
    N = [a + 1 for a in n]
    expect = (3 * N[0] - 2) * (3 * N[1] - 2) * (3 * N[2] - 2)
    assert O.lib().or_structure_nnz(*n) == expect


def test_nnz_100_matches_baseline():
    # BASELINE.json configs[1]: "1.03M rows, ~27.3M nnz"; 27,270,901
    assert O.lib().or_structure_nnz(100, 100, 100) == 27270901 == (3 * 101 - 2) ** 3


@pytest.mark.parametrize("n", [(2, 2, 2), (3, 2, 4), (1, 3, 2)])
def test_pattern_equals_shared_element_relation(n):
    """Brute force: (i, j) is stored iff nodes i and j belong to a common element."""
    nx, ny, nz = n
    NX, NY = nx + 1, ny + 1
    rows = (nx + 1) * (ny + 1) * (nz + 1)
    pairs = set()
    for ez, ey, ex in itertools.product(range(nz), range(ny), range(nx)):
        nodes = [(ex + (a & 1)) + NX * ((ey + ((a >> 1) & 1)) + NY * (ez + ((a >> 2) & 1)))
                 for a in range(8)]
        for i in nodes:
            for j in nodes:
                pairs.add((i, j))
    row_ptr, col = O.structure(*n)
    got = {(i, int(c)) for i in range(rows) for c in col[row_ptr[i]:row_ptr[i + 1]]}
    assert got == pairs
    # columns strictly ascending in every row
    for i in range(rows):
        seg = col[row_ptr[i]:row_ptr[i + 1]]
        assert np.all(np.diff(seg) > 0)


def test_row_length_classes():
    """Row length = c(ix) c(iy) c(iz), c = 2 on a boundary plane, else 3."""
    nx, ny, nz = 5, 4, 3
    row_ptr, _ = O.structure(nx, ny, nz)
    lens = np.diff(row_ptr)
    k = 0
    for iz in range(nz + 1):
        for iy in range(ny + 1):
            for ix in range(nx + 1):
                c = [2 if (i == 0 or i == m) else 3 for i, m in ((ix, nx), (iy, ny), (iz, nz))]
                assert lens[k] == c[0] * c[1] * c[2]
                k += 1
