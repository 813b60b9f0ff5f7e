"""GPU verification (C8) and the rooted collectives that carry it
(§3.2): minife_verify's device series against the oracle's series, its FE values
against the oracle's converged CG solution (bit-identical), the O(h^2) bound, and the same
answers from RCB parts (host combination) and from a RANK ctx (ncclReduce to rank 0)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
M = pytest.importorskip("paper_1505_08023_b200")

PROBES = [(0.5, 0.5, 0.5), (0.2, 0.5, 0.5), (0.8, 0.5, 0.5), (0.5, 0.2, 0.5), (0.6, 0.3, 0.7),
          (0.9, 0.5, 0.5), (0.0, 0.5, 0.5), (1.0, 0.5, 0.5), (0.5, 0.0, 0.3)]
NTERMS = 200


def gids_of(n):
    N = n + 1
    out = []
    for p in PROBES:
        ix, iy, iz = (int(round(c * n)) for c in p)
        out.append(ix + N * (iy + N * iz))
    return np.array(out, dtype=np.int64)


def coords(n, gid):
    N = n + 1
    return gid % N / n, gid // N % N / n, gid // (N * N) / n


def reference(n):
    s = O.assemble(n, n, n)
    r = O.cg(s.row_ptr, s.col, s.val, s.b, 3000, 1e-12)
    assert r.converged
    return r


def check(g, n, oracle_cg):
    gids = gids_of(n)
    fe, ex, mx = g.verify(gids, NTERMS)
    assert np.array_equal(fe, oracle_cg.x[gids])                 # FE values: bit-identical
    for i, gid in enumerate(gids):
        assert abs(ex[i] - O.analytic(*coords(n, gid), NTERMS)) <= 1e-13
    err = np.abs(fe - ex)
    assert mx == err.max()
    h = 1.0 / n
    interior = [i for i, p in enumerate(PROBES) if 0 < p[0] < 1 and 0 < p[1] < 1 and 0 < p[2] < 1]
    assert np.all(err[interior] <= 2 * h * h)                     # O(h^2)
    # the centre: u = 1/6 exactly (six-face superposition)
    assert abs(ex[0] - 1.0 / 6.0) <= 1e-13
    return fe, ex, mx


@pytest.mark.parametrize("n", [10, 20])
def test_verify_single(n):
    o = reference(n)
    with M.Minife(n, n, n) as g:
        g.assemble()
        r = g.cg_solve(3000, 1e-12)
        assert r.converged and r.iterations == o.iters
        check(g, n, o)


@pytest.mark.parametrize("parts", [2, 5])
def test_verify_partitioned(parts):
    n = 20
    o = reference(n)
    with M.Minife(n, n, n, virtual=parts) as g:
        g.assemble()
        g.cg_solve(3000, 1e-12)
        check(g, n, o)
        t = g.gather_times()
        assert t.shape == (parts, 2) and np.all(t[:, 1] > 0)


def test_verify_rank_mode_rooted_reduce():
    n = 20
    o = reference(n)
    uid = M.nccl_unique_id()
    with M.Minife(n, n, n, rank=(0, 1, 0, uid)) as g:
        g.assemble()
        g.cg_solve(3000, 1e-12)
        check(g, n, o)                      # ncclReduce(SUM) + ncclReduce(MAX) to rank 0
        t = g.gather_times()                # rooted gather (send/recv to rank 0)
        assert t.shape == (1, 2) and t[0, 1] > 0


def test_verify_errors():
    with M.Minife(4, 4, 4) as g:
        g.assemble()
        with pytest.raises(M.MinifeError):
            g.verify([0], 10)               # no solve yet
        g.cg_solve(10, 0.0)
        with pytest.raises(M.MinifeError):
            g.verify([5 ** 3], 10)          # gid out of range
