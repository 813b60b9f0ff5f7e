"""CPU checks of the product library: it loads, exports every symbol include/minife.h
declares, fails cleanly without a GPU, and its host-side RCB/halo plan (G15; S:61-100,
S:293-296) matches the oracle's brute-force partition exactly (integer work: bit-exact).
"""
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_1505_08023_b200 as M

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "minife.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(minife_[a-z_0-9]+)\s*\(", src))


def test_every_declared_symbol_is_exported_and_bound():
    decl = declared_symbols()
    assert len(decl) >= 20
    lib = M._lib
    for name in decl:
        assert hasattr(lib, name), name          # dlsym succeeds
        assert name in M.SIGNATURES, name        # and the binding marshals it


def test_strerror_and_version():
    assert M.minife_strerror(0) == b"ok"
    assert b"SPD" in M.minife_strerror(M.MINIFE_ENOTSPD)
    assert M.minife_strerror(999) == b"unknown status"
    assert b"sm_100a" in M.minife_version()


def test_no_gpu_is_a_clean_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(M.MinifeError) as e:
        M.Minife(4, 4, 4)
    assert e.value.status in (M.MINIFE_ENODEV, M.MINIFE_ECUDA)


def test_invalid_arguments():
    import ctypes
    h = ctypes.c_void_p()
    assert M.minife_create(0, 4, 4, 1, ctypes.byref(h)) == M.MINIFE_EINVAL
    assert M.minife_create(4, 4, 4, 0, ctypes.byref(h)) == M.MINIFE_EINVAL
    assert M.minife_create_virtual(4, 4, 4, 0, ctypes.byref(h)) == M.MINIFE_EINVAL
    assert M.minife_assemble(None) == M.MINIFE_EINVAL
    assert M.minife_cg_solve(None, 10, 0.0, None) == M.MINIFE_EINVAL
    M.minife_destroy(None)                        # NULL-safe
    with pytest.raises(M.MinifeError):
        M.plan(2, 1, 1, 3, 0)                     # RCB leaf without elements


@pytest.mark.parametrize("n,p", [((4, 4, 4), 1), ((4, 4, 4), 2), ((5, 4, 3), 4),
                                 ((6, 6, 6), 8), ((5, 5, 4), 3), ((7, 3, 2), 6),
                                 ((9, 4, 5), 5)])
def test_plan_matches_oracle_partition(n, p):
    boxes = O.rcb(*n, p)
    total_owned = 0
    for r in range(p):
        L = M.plan_lists(*n, p, r)
        info = L["info"]
        assert list(info.box) == boxes[r].tolist()
        own = O.owned(*n, boxes, r)
        assert info.rows == own.size
        total_owned += info.rows
        # owned set is the box reported in info.own, enumerated in ascending id
        NX, NY = n[0] + 1, n[1] + 1
        lo, hi = info.own[:3], info.own[3:]
        box_ids = [ix + NX * (iy + NY * iz) for iz in range(lo[2], hi[2] + 1)
                   for iy in range(lo[1], hi[1] + 1) for ix in range(lo[0], hi[0] + 1)]
        assert np.array_equal(np.array(box_ids, dtype=np.int64), own)
        # externals: same ids in the same (owner, gid) slot order
        assert np.array_equal(L["ext_gids"], O.externals(*n, boxes, r))
        # nnz of the owned rows: closed form == oracle structure
        rp, _ = O.structure(*n)
        assert info.nnz == int(np.sum(rp[own + 1] - rp[own]))
    assert total_owned == (n[0] + 1) * (n[1] + 1) * (n[2] + 1)


@pytest.mark.parametrize("n,p", [((4, 4, 4), 2), ((5, 4, 3), 4), ((6, 6, 6), 8),
                                 ((5, 5, 4), 3)])
def test_halo_lists_consistent(n, p):
    """r sends to s exactly what s expects from r, in the same order."""
    lists = [M.plan_lists(*n, p, r) for r in range(p)]
    NX, NY = n[0] + 1, n[1] + 1
    for r in range(p):
        Lr = lists[r]
        own_r = O.owned(*n, O.rcb(*n, p), r)
        send_off = np.concatenate([[0], np.cumsum(Lr["send_cnt"])])
        for k, s in enumerate(Lr["nbr"]):
            Ls = lists[s]
            ks = list(Ls["nbr"]).index(r)               # neighbor relation is symmetric
            recv_off = int(np.sum(Ls["recv_cnt"][:ks]))
            expect = Ls["ext_gids"][recv_off:recv_off + Ls["recv_cnt"][ks]]
            sent = own_r[Lr["send_idx"][send_off[k]:send_off[k + 1]]]
            assert np.array_equal(sent, expect)


@pytest.mark.parametrize("n,p", [((4, 4, 4), 1), ((6, 6, 6), 2), ((9, 4, 5), 5),
                                 ((6, 6, 6), 8), ((40, 8, 6), 2), ((12, 40, 9), 4)])
def test_interior_slices_match_brute_force(n, p):
    """DESIGN §7 overlap split: a SELL-32 slice of owned rows is interior iff none of its rows
    has a 27-point neighbour owned by another rank (brute force over the oracle's structure
    and ownership)."""
    boxes = O.rcb(*n, p)
    rp, col = O.structure(*n)
    for r in range(p):
        info = M.plan(*n, p, r)
        own = O.owned(*n, boxes, r)
        owned_set = np.zeros(rp.size - 1, dtype=bool)
        owned_set[own] = True
        reads_halo = np.array([not owned_set[col[rp[g]:rp[g + 1]]].all() for g in own])
        slices = [reads_halo[i:i + 32] for i in range(0, own.size, 32)]
        interior = sum(1 for s in slices if not s.any())
        assert info.interior_slices == interior
        if p == 1:
            assert interior == info.slices
