"""Pins for the oracle's RCB partition, ownership and externals (G15; P:29, P:44-48;
S:61-100).

Independent references: SPEC's worked RCB examples, the cover/disjointness and ownership
totality invariants, and the distributed-SpMV property: every column of every owned row is
owned or external, so a rank's local SpMV reproduces the global rows bit-for-bit.
"""
import itertools

import numpy as np
import pytest

import oracle as O


def test_rcb_spec_examples():
    assert O.rcb(4, 4, 4, 1).tolist() == [[0, 0, 0, 4, 4, 4]]
    assert O.rcb(4, 4, 4, 2).tolist() == [[0, 0, 0, 2, 4, 4], [2, 0, 0, 4, 4, 4]]
    b4 = O.rcb(4, 4, 4, 4).tolist()
    assert b4 == [[0, 0, 0, 2, 2, 4], [0, 2, 0, 2, 4, 4], [2, 0, 0, 4, 2, 4],
                  [2, 2, 0, 4, 4, 4]]


def test_rcb_bench_configs():
    # 400^3 at p=8 gives 2x2x2 boxes of 200^3; weak scaling gives 300^3 boxes
    b = O.rcb(400, 400, 400, 8)
    assert all((r[3] - r[0], r[4] - r[1], r[5] - r[2]) == (200, 200, 200) for r in b)
    for n, p in [((600, 300, 300), 2), ((600, 600, 300), 4), ((600, 600, 600), 8)]:
        b = O.rcb(*n, p)
        assert all((r[3] - r[0], r[4] - r[1], r[5] - r[2]) == (300, 300, 300) for r in b)


def test_rcb_rejects_too_many_ranks():
    with pytest.raises(ValueError):
        O.rcb(2, 1, 1, 3)
    with pytest.raises(ValueError):
        O.rcb(3, 3, 1, 9 + 1)


@pytest.mark.parametrize("n,p", [((4, 4, 4), 3), ((6, 5, 4), 5), ((5, 5, 5), 8),
                                 ((7, 3, 2), 6)])
def test_cover_ownership(n, p):
    b = O.rcb(*n, p)
    cover = np.zeros(n[::-1], dtype=int)
    for r in b:
        cover[r[2]:r[5], r[1]:r[4], r[0]:r[3]] += 1
    assert np.all(cover == 1)
    counts = np.zeros(p, dtype=int)
    for iz, iy, ix in itertools.product(range(n[2] + 1), range(n[1] + 1), range(n[0] + 1)):
        o = O.owner(b, ix, iy, iz)
        assert 0 <= o < p
        counts[o] += 1
    owned_total = sum(O.owned(*n, b, r).size for r in range(p))
    assert owned_total == (n[0] + 1) * (n[1] + 1) * (n[2] + 1)


def test_load_balance_power_of_two():
    b = O.rcb(8, 8, 8, 8)
    vols = [(r[3] - r[0]) * (r[4] - r[1]) * (r[5] - r[2]) for r in b]
    assert max(vols) == min(vols) == 64


def test_externals_examples():
    b = O.rcb(2, 2, 2, 1)
    assert O.externals(2, 2, 2, b, 0).size == 0
    b = O.rcb(2, 2, 2, 2)                           # split at x-element 1
    e0 = O.externals(2, 2, 2, b, 0)
    assert sorted(e0.tolist()) == [2 + 3 * (iy + 3 * iz) for iz in range(3) for iy in range(3)]
    e1 = O.externals(2, 2, 2, b, 1)
    assert sorted(e1.tolist()) == [1 + 3 * (iy + 3 * iz) for iz in range(3) for iy in range(3)]


@pytest.mark.parametrize("n,p", [((4, 4, 4), 2), ((5, 4, 3), 4), ((6, 6, 6), 8),
                                 ((5, 5, 4), 3)])
def test_distributed_spmv_bit_equal(n, p):
    """halo-filled local SpMV on every rank == global SpMV, bit for bit."""
    s = O.assemble(*n)
    x = np.random.default_rng(3).uniform(-1, 1, s.rows)
    y = O.spmv(s.row_ptr, s.col, s.val, x)
    b = O.rcb(*n, p)
    seen = np.zeros(s.rows, dtype=int)
    for r in range(p):
        own = O.owned(*n, b, r)
        ext = O.externals(*n, b, r)
        # external order: owner rank ascending, then global id ascending
        owners = [O.owner(b, g % (n[0] + 1), (g // (n[0] + 1)) % (n[1] + 1),
                          g // ((n[0] + 1) * (n[1] + 1))) for g in ext]
        assert all(o != r for o in owners)
        assert list(zip(owners, ext.tolist())) == sorted(zip(owners, ext.tolist()))
        local = {int(g): k for k, g in enumerate(np.concatenate([own, ext]))}
        xl = x[np.concatenate([own, ext])]
        rp, cols, vals = [0], [], []
        for g in own:
            for k in range(s.row_ptr[g], s.row_ptr[g + 1]):
                cols.append(local[int(s.col[k])])      # KeyError = missing external
                vals.append(s.val[k])
            rp.append(len(cols))
        yl = O.spmv(np.array(rp), np.array(cols), np.array(vals), xl)
        assert np.array_equal(yl, y[own])
        seen[own] += 1
    assert np.all(seen == 1)
