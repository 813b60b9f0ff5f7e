"""GPU parity at the configs' FULL sizes against stored oracle references (tests/golden/).

The references are written by ``tools/make_golden.py``, which runs ONLY the C oracle
(structure Fig 3.6, assembly Fig 3.7/C2, Dirichlet C3, CRS SpMV Fig 3.1/C4 on the seeded
vector C7, 200 CG iterations C6 from x0 = 0, tol = 0) and stores the residual history as hex
floats plus SHA-256 digests of row_ptr, col, val, b, the SpMV output y and the final x.

Here the CUDA path runs the same configuration through the C ABI, in the launch
configurations the bench uses (SINGLE 300^3 and 400^3; RCB parts of the strong- and
weak-scaling meshes as VIRTUAL parts, which run exactly the per-rank code of a torchrun
rank), and its outputs are hashed the same way: the bar is bit-identity (IEEE ==; the
digests fold -0.0 into +0.0), which is inside every north-star tolerance
(SpMV 1e-12 relative, history 1e-8 over 50 iterations, x 1e-9 max-abs).
"""
import hashlib
import json
import os

import numpy as np
import pytest

import minife_inputs

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

M = pytest.importorskip("paper_1505_08023_b200")

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CHUNK = 1 << 21


def load(n):
    path = os.path.join(GOLDEN, f"minife_{n[0]}x{n[1]}x{n[2]}.json")
    if not os.path.exists(path):
        pytest.skip(f"no golden reference {os.path.basename(path)} (tools/make_golden.py)")
    with open(path) as f:
        return json.load(f)


def sha_f64(a):
    h = hashlib.sha256()
    for i in range(0, a.size, 1 << 24):
        h.update(np.ascontiguousarray(a[i:i + (1 << 24)], dtype="<f8") + 0.0)
    return h.hexdigest()


def matrix_digests(g, rows):
    """SHA-256 of the canonical global CSR (row_ptr, col, val) exported from the device in
    chunks of rows (minife_export_rows), in the oracle's byte layout."""
    h_rp, h_col, h_val = hashlib.sha256(), hashlib.sha256(), hashlib.sha256()
    h_rp.update(np.zeros(1, dtype="<i8").tobytes())
    off = 0
    lane = np.arange(27, dtype=np.int32)[None, :]
    for s in range(0, rows, CHUNK):
        gids = np.arange(s, min(rows, s + CHUNK), dtype=np.int64)
        cols, vals, lens = g.export_rows(gids)
        assert lens.min() >= 8 and lens.max() <= 27
        keep = lane < lens[:, None]
        h_col.update(np.ascontiguousarray(cols[keep], dtype="<i8").tobytes())
        h_val.update((np.ascontiguousarray(vals[keep], dtype="<f8") + 0.0).tobytes())
        rp = off + np.cumsum(lens, dtype=np.int64)
        off = int(rp[-1])
        h_rp.update(rp.astype("<i8").tobytes())
    return {"row_ptr": h_rp.hexdigest(), "col": h_col.hexdigest(), "val": h_val.hexdigest()}


def check(g, gold, matrix=True, spmv=True):
    rows = gold["rows"]
    info = g.get_info()
    assert info.rows == rows and info.nnz == gold["nnz"]
    g.assemble()
    sha = gold["sha256"]
    if matrix:
        got = matrix_digests(g, rows)
        for k in ("row_ptr", "col", "val"):
            assert got[k] == sha[k], f"{k} differs from the oracle"
    assert sha_f64(g.rhs()) == sha["b"], "rhs b differs from the oracle"
    if spmv:
        seed = gold["spmv"]["seed"]
        y = g.spmv(minife_inputs.uniform_pm1(rows, seed))
        for gid, hx in gold["spmv"]["y_samples"].items():
            assert y[int(gid)] == float.fromhex(hx), f"y[{gid}]"
        assert sha_f64(y) == sha[f"spmv_y_seed{seed}"], "SpMV output differs from the oracle"
        del y
    cg = gold["cg"]
    r = g.cg_solve(cg["max_iters"], cg["tol"])
    assert r.status == cg["status"]
    assert r.iterations == cg["iterations"] and r.converged == cg["converged"]
    h = g.history()
    ho = np.array([float.fromhex(v) for v in cg["hist_hex"]])
    k = min(51, ho.size)
    assert np.all(np.abs(h[:k] - ho[:k]) <= 1e-8 * np.abs(ho[:k]))        # north star
    bad = np.nonzero(h != ho)[0]
    assert bad.size == 0, f"history differs first at k = {bad[:1]}"
    x = g.solution()
    for gid, hx in cg["x_samples"].items():
        assert x[int(gid)] == float.fromhex(hx), f"x[{gid}]"
    assert sha_f64(x) == sha["x"], "final x differs from the oracle"


def test_300cubed_bench_config():
    """configs[2] in the bench's launch configuration (SINGLE, SYM, graph, deferred x)."""
    gold = load((300, 300, 300))
    with M.Minife(300, 300, 300) as g:
        check(g, gold)


def test_300cubed_seg_format():
    gold = load((300, 300, 300))
    with M.Minife(300, 300, 300, fmt=M.FMT_SEG) as g:
        check(g, gold, matrix=False)


@pytest.mark.parametrize("parts", [2, 8])
def test_300cubed_partitioned(parts):
    gold = load((300, 300, 300))
    with M.Minife(300, 300, 300, virtual=parts) as g:
        check(g, gold, matrix=parts == 2, spmv=parts == 8)


def test_400cubed_single():
    """configs[3]'s strong-scaling base point on one GPU."""
    gold = load((400, 400, 400))
    with M.Minife(400, 400, 400) as g:
        check(g, gold)


@pytest.mark.parametrize("parts", [2, 4, 8])
def test_400cubed_strong_scaling_parts(parts):
    """configs[3]: the RCB parts of 400^3 over 2/4/8 ranks (VIRTUAL parts run each rank's
    kernels, plans and exchange protocol)."""
    gold = load((400, 400, 400))
    with M.Minife(400, 400, 400, virtual=parts) as g:
        check(g, gold, matrix=False, spmv=parts == 8)


def test_weak_scaling_600x300x300():
    """configs[4] at 2 GPUs: 600x300x300 in 2 RCB parts of 300^3 nodes' worth each."""
    gold = load((600, 300, 300))
    with M.Minife(600, 300, 300, virtual=2) as g:
        check(g, gold)


def test_weak_scaling_600x300x300_device_protocol():
    """configs[4] at 2 GPUs through the device-initiated protocol of MULTI/RANK ctxs (halo
    pushed into the deferred-x ring, in-kernel reductions), on one GPU as 2 virtual parts."""
    gold = load((600, 300, 300))
    with M.Minife(600, 300, 300, virtual=2) as g:
        g.set_transport(M.TRANSPORT_DEVICE)
        check(g, gold, matrix=False)


def test_weak_scaling_600x600x300():
    """configs[4] at 4 GPUs: 600x600x300 in 4 RCB parts."""
    gold = load((600, 600, 300))
    with M.Minife(600, 600, 300, virtual=4) as g:
        check(g, gold, matrix=False)
