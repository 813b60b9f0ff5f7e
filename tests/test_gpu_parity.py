"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bar: integer/index work bit-exact; floating point compared with IEEE ==
(zero error), which is inside every north-star tolerance (SpMV 1e-12 relative per entry,
history 1e-8 relative over the first 50 iterations, x 1e-9 max-abs) -- SURVEY §8(c) shows a
weaker contract cannot meet those on this problem.  Each comparison also asserts the
north-star tolerance itself, so a failure says which bar broke.
"""
import numpy as np
import pytest

import minife_inputs
import oracle as O

pytestmark = pytest.mark.gpu

M = pytest.importorskip("paper_1505_08023_b200")

MESHES = [(1, 1, 1), (2, 2, 2), (10, 10, 10), (23, 17, 9), (7, 1, 3), (33, 32, 31)]


def _same(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return a.shape == b.shape and bool(np.all((a == b) | (np.isnan(a) & np.isnan(b))))


_oracle_cache = {}


def oracle_system(n):
    if n not in _oracle_cache:
        _oracle_cache[n] = O.assemble(*n)
    return _oracle_cache[n]


def oracle_cg(n, iters, tol):
    key = ("cg", n, iters, tol)
    if key not in _oracle_cache:
        s = oracle_system(n)
        _oracle_cache[key] = O.cg(s.row_ptr, s.col, s.val, s.b, iters, tol)
    return _oracle_cache[key]


def check_matrix(g, s):
    rp, col, val = g.export_csr()
    assert np.array_equal(rp, s.row_ptr)          # pattern: bit-exact
    assert np.array_equal(col, s.col)             # indices: bit-exact
    assert _same(val, s.val)                      # values: IEEE ==
    assert _same(g.rhs(), s.b)


def check_spmv(g, s, seed):
    x = minife_inputs.uniform_pm1(s.rows, seed)
    y = g.spmv(x)
    yo = O.spmv(s.row_ptr, s.col, s.val, x)
    rel = np.abs(y - yo) / np.maximum(np.abs(yo), 1e-300)
    assert np.all((rel <= 1e-12) | (y == yo))     # north-star bar
    assert _same(y, yo)                           # canonical-arithmetic bar


def check_cg(g, n, iters, tol):
    r = g.cg_solve(iters, tol)
    o = oracle_cg(n, iters, tol)
    assert r.status == o.status
    assert r.iterations == o.iters and r.converged == o.converged
    h = g.history()
    k = min(51, h.size)
    assert np.all(np.abs(h[:k] - o.hist[:k]) <= 1e-8 * np.abs(o.hist[:k]))   # north star
    assert _same(h, o.hist)
    x = g.solution()
    assert np.abs(x - o.x).max() <= 1e-9                                       # north star
    assert _same(x, o.x)


FORMATS = [M.FMT_SEG, M.FMT_CRS]
ALL_FORMATS = FORMATS + [M.FMT_SYM]         # every process model


@pytest.mark.parametrize("fmt", ALL_FORMATS)
@pytest.mark.parametrize("n", MESHES)
def test_single_gpu_matrix_spmv_cg(n, fmt):
    s = oracle_system(n)
    with M.Minife(*n, fmt=fmt) as g:
        g.assemble()
        info = g.get_info()
        assert info.rows == s.rows and info.nnz == s.nnz
        check_matrix(g, s)
        for seed in (12345, 1, 2):
            check_spmv(g, s, seed)
        check_cg(g, n, 200, 0.0)
        check_cg(g, n, 200, 1e-8)
        check_cg(g, n, 7, 0.0)          # graph re-capture with another iteration count


@pytest.mark.parametrize("fmt", ALL_FORMATS)
@pytest.mark.parametrize("n", [(800, 3, 3), (3, 3, 800), (2, 900, 2), (61, 1, 97)])
def test_elongated_meshes(n, fmt):
    """Lines much longer / shorter than a tile (SYM mirror boxes, segment runs, SELL tails)
    and too many rows for the single-launch solvers: the multi-kernel path."""
    s = oracle_system(n)
    with M.Minife(*n, fmt=fmt) as g:
        g.assemble()
        check_matrix(g, s)
        check_spmv(g, s, 2)
        check_cg(g, n, 200, 0.0)


@pytest.mark.parametrize("fmt", ALL_FORMATS)
@pytest.mark.parametrize("n,p", [((10, 10, 10), 2), ((23, 17, 9), 3), ((10, 10, 10), 4),
                                 ((12, 11, 10), 8), ((33, 32, 31), 5), ((3, 2, 2), 4),
                                 ((1, 1, 12), 4), ((12, 1, 1), 3), ((40, 3, 2), 6)])
@pytest.mark.parametrize("transport", [0, 1, 2, 3])
def test_virtual_ranks_bit_identical(n, p, fmt, transport):
    """P10 / S:394: any partition gives bitwise the 1-rank (= oracle) results.  transport 1
    runs the multi-GPU wire protocol (pack -> per-neighbor receive blocks -> unpack), 2 the
    device-initiated push (each sender stores into the receivers' halo columns), 3 the whole
    device-initiated protocol of MULTI/RANK ctxs (push + halo flags + in-kernel reductions
    through every part's inbox, no host-launched collective)."""
    s = oracle_system(n)
    with M.Minife(*n, virtual=p, fmt=fmt) as g:
        g.set_transport(transport)
        g.assemble()
        assert g.get_info().nparts == p
        check_matrix(g, s)
        check_spmv(g, s, 12345)
        check_cg(g, n, 200, 0.0)
        check_cg(g, n, 100, 1e-10)


@pytest.mark.parametrize("fmt", [M.FMT_SEG, M.FMT_SYM])
@pytest.mark.parametrize("n,p", [((40, 8, 6), 2), ((12, 40, 9), 4), ((33, 32, 31), 8)])
@pytest.mark.parametrize("transport", [0, 1, 2, 3])
def test_overlapped_halo_split_bit_identical(n, p, transport, fmt):
    """SEG parts store interior slices first; the interior SpMV runs while the halo
    is in flight on a second stream, the boundary slices after it lands.  SYM parts compute
    the halo values of p_(k+1) ahead of K7 and exchange them while K7 runs.  Results are
    bitwise the oracle's (graph mode and profile mode, which runs the unsplit sequence)."""
    s = oracle_system(n)
    with M.Minife(*n, virtual=p, fmt=fmt) as g:
        g.set_transport(transport)
        g.assemble()
        parts = [g.part_info(q) for q in range(p)]
        if p <= 4 and fmt == M.FMT_SEG:   # at p = 8 every slice of these parts touches an x cut
            assert any(0 < q.interior_slices < q.slices for q in parts)
        check_matrix(g, s)
        check_spmv(g, s, 1)
        check_cg(g, n, 200, 0.0)
        t = g.cg_profile(200)
        assert t.spmv_ms > 0
        check_cg(g, n, 200, 0.0)


def _solver_variant(n, fmt, options):
    """One mesh through the library with the given ctx options; bitwise the oracle for a
    200-iteration solve, a tolerance stop and an odd iteration count."""
    s = oracle_system(n)
    with M.Minife(*n, fmt=fmt, options=options) as g:
        g.assemble()
        for iters, tol in ((200, 0.0), (200, 1e-8), (7, 0.0)):
            r = g.cg_solve(iters, tol)
            o = oracle_cg(n, iters, tol)
            assert (r.status, r.iterations, r.converged) == (o.status, o.iters, o.converged)
            assert _same(g.history(), o.hist)
            assert _same(g.solution(), o.x)


@pytest.mark.parametrize("small", [0, 1, 2])
@pytest.mark.parametrize("n,fmt", [((10, 10, 10), M.FMT_SYM), ((10, 10, 10), M.FMT_SEG),
                                   ((23, 17, 9), M.FMT_SYM), ((7, 1, 3), M.FMT_SEG)])
def test_single_launch_solvers_bit_identical(n, fmt, small):
    """option small_solver = 1 one-CTA solver, 2 one-cluster solver
    (DSMEM), 0 the three-kernel graph -- each bitwise the oracle."""
    if small == 1 and (n[0] + 1) * (n[1] + 1) * (n[2] + 1) > 2048:
        pytest.skip("one-CTA solver holds <= 2048 rows")
    _solver_variant(n, fmt, {"small_solver": small})


@pytest.mark.parametrize("xdef", [2, 5, 8])
@pytest.mark.parametrize("n,fmt", [((23, 17, 9), M.FMT_SYM), ((33, 32, 31), M.FMT_SEG),
                                   ((7, 1, 3), M.FMT_SYM)])
def test_x_every_second_iteration_bit_identical(n, fmt, xdef):
    """the deferred x update, every X iterations from a ring of X p buffers (forced
    at any size with option x_defer = X, the multi-kernel path with small_solver = 0): 200
    iterations, a tolerance stop and an odd count (7) leave nothing pending -- bitwise the
    oracle."""
    _solver_variant(n, fmt, {"x_defer": xdef, "small_solver": 0})


@pytest.mark.parametrize("n", [(23, 17, 9), (33, 32, 31)])
def test_sym_fallback_kernel_bit_identical(n):
    """The L1-gather SYM SpMV (`k_spmv_sym`, used where tensor maps are unavailable; option
    sym_kernel = 0 selects it) through the three-kernel path: bitwise the oracle."""
    _solver_variant(n, M.FMT_SYM, {"sym_kernel": 0, "small_solver": 0})


@pytest.mark.parametrize("opts", [{"x_late": 0}, {"cluster_dd": 0, "small_solver": 2},
                                  {"graph": 0}, {"spmv_impl": 0}, {"val_evict_first": 1},
                                  {"x_prefetch": 1, "small_solver": 0},
                                  {"snake": 1, "small_solver": 0},
                                  {"snake": 1, "band_rows": 1000, "small_solver": 0},
                                  {"symm_nw": 11, "small_solver": 0},
                                  {"symm_nw": 11, "band_rows": 1000, "small_solver": 0},
                                  {"symm_nw": 11, "snake": 1, "small_solver": 0}])
def test_other_options_bit_identical(opts):
    fmt = M.FMT_SEG if "spmv_impl" in opts else M.FMT_SYM
    _solver_variant((10, 10, 10), fmt, opts)
    _solver_variant((23, 17, 9), fmt, opts)


@pytest.mark.parametrize("fold", [1, 0])
def test_device_comm_dead_peer_fails_with_ecomm_then_recovers(fold):
    """Fault injection: one virtual part never signals (option comm_fault_part).  Its peers'
    spins time out after comm_timeout_ms and the solve fails with MINIFE_ECOMM instead of
    hanging; with the fault cleared the next solve on the same ctx is bitwise the oracle."""
    n, p = (12, 11, 10), 3
    with M.Minife(*n, virtual=p, options={"fold_comm": fold, "comm_timeout_ms": 50}) as g:
        g.set_transport(M.TRANSPORT_DEVICE)
        g.assemble()
        g.set_option("comm_fault_part", 1)
        with pytest.raises(M.MinifeError) as e:
            r = g.cg_solve(20, 0.0)
            assert r.status == M.MINIFE_ECOMM     # (raised by the binding on ECOMM)
        assert e.value.status == M.MINIFE_ECOMM
        g.set_option("comm_fault_part", -1)
        check_cg(g, n, 200, 0.0)


@pytest.mark.parametrize("band", [1000, 4000])
def test_band_order_bit_identical_across_reassembly(band):
    """The band-major SYM tile order (forced at a small mesh with option band_rows) is bitwise
    the oracle, also when the ctx re-assembles between solves (the captured graph holds the
    order's device pointer: it must survive re-assembly) and when the option changes."""
    n = (33, 32, 31)
    s = oracle_system(n)
    with M.Minife(*n, options={"band_rows": band, "small_solver": 0}) as g:
        for rep in range(3):
            g.assemble()
            check_cg(g, n, 200, 0.0)
            check_spmv(g, s, 3)
        g.set_option("band_rows", 0)              # natural order: the order buffer goes away
        g.assemble()
        check_cg(g, n, 200, 0.0)
        g.set_option("band_rows", band)
        g.assemble()
        check_cg(g, n, 100, 1e-10)
        g.set_option("symm_nw", 11)              # narrower tiles: a new order, a new graph
        g.assemble()
        check_cg(g, n, 200, 0.0)
        check_spmv(g, s, 2)


def test_option_errors():
    with M.Minife(3, 3, 3) as g:
        for name, v in (("no_such_option", 1), ("x_defer", 9), ("graph", 2), ("small_solver", -2),
                        ("symm_nw", 12), ("symm_nw", 0)):
            with pytest.raises(M.MinifeError) as e:
                g.set_option(name, v)
            assert e.value.status == M.MINIFE_EINVAL


def test_cluster_solver_after_spmv_leftovers():
    """The one-cluster solver right after SpMV launches that fill every SM's shared memory
    with other data: 20 solves, each bitwise the oracle (a fresh process: the race this guards
    against showed up in one)."""
    import os
    import subprocess
    import sys
    env = dict(os.environ)
    here = os.path.dirname(os.path.abspath(__file__))
    out = subprocess.run([sys.executable, os.path.join(here, "_cluster_after_spmv.py")], env=env,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]


def test_timing_window_inside_the_solve():
    """minife_set_timing_window: events around the SpMVs of a range of iterations are part of
    the solve graph; the results stay bitwise the oracle's; the window needs a solve that ran
    through it."""
    n = (33, 32, 31)
    with M.Minife(*n) as g:
        g.assemble()
        g.set_timing_window(5, 10)
        with pytest.raises(M.MinifeError):
            g.timing_window()                        # no solve yet
        check_cg(g, n, 200, 0.0)
        spmv_ms, iter_ms = g.timing_window()
        assert 0.0 < spmv_ms < iter_ms < 50.0
        g.set_timing_window(150, 100)                # beyond the solve
        check_cg(g, n, 200, 0.0)
        with pytest.raises(M.MinifeError):
            g.timing_window()
        g.set_timing_window(1, 0)                    # removed
        check_cg(g, n, 30, 0.0)


def test_plan_on_device_matches_host_plan():
    n, p = (12, 11, 10), 8
    with M.Minife(*n, virtual=p) as g:
        for r in range(p):
            a = g.part_info(r)
            b = M.plan(*n, p, r)
            assert (a.rows, a.externals, a.nnz, a.n_neighbors, a.send_total,
                    a.interior_slices) == \
                   (b.rows, b.externals, b.nnz, b.n_neighbors, b.send_total, b.interior_slices)
        g.set_format(M.FMT_CRS)          # plan's sell_entries is the CRS-format count
        g.assemble()
        for r in range(p):
            assert g.part_info(r).sell_entries == M.plan(*n, p, r).sell_entries


@pytest.mark.parametrize("fmt", ALL_FORMATS)
def test_rank_mode_world1_nccl_path(fmt):
    """SPMD entry point with a 1-rank NCCL communicator (exercises NCCL + graph capture)."""
    n = (10, 10, 10)
    uid = M.nccl_unique_id()
    with M.Minife(*n, rank=(0, 1, 0, uid), fmt=fmt) as g:
        g.assemble()
        check_matrix(g, oracle_system(n))
        check_cg(g, n, 200, 0.0)


@pytest.mark.parametrize("graph", [1, 0])
@pytest.mark.parametrize("n", [(10, 10, 10), (23, 17, 9)])
def test_rank_mode_world1_device_comm(n, graph):
    """RANK ctx built through the CUDA-IPC exchange (NCCL all-gather of the handles, transport
    agreement) with the device-initiated reductions forced at world 1: every dot goes through
    k_acc_push -> inbox -> flag-waiting consumers.  Bitwise the oracle, graph and eager."""
    uid = M.nccl_unique_id()
    with M.Minife(*n, rank=(0, 1, 0, uid), options={"device_comm": 1, "graph": graph,
                                                    "small_solver": 0}) as g:
        g.assemble()
        check_cg(g, n, 200, 0.0)
        check_cg(g, n, 100, 1e-10)
        info = g.get_info()
        assert info.kernel_launches > 0 and info.comm == 2


@pytest.mark.parametrize("fold", [1, 0])
def test_device_comm_launch_count_has_no_host_collective(fold):
    """VIRTUAL parts on the device protocol: every kernel of the solve is ours (the count the
    library reports equals the kernels it enqueued) and the solve is bitwise the oracle --
    with the accumulator pushes and the halo wait folded into the producing kernels' last
    CTAs (fold_comm = 1, default) and as separate launches (0)."""
    n, p = (12, 11, 10), 4
    with M.Minife(*n, virtual=p, options={"fold_comm": fold}) as g:
        assert g.get_info().comm == 0
        g.set_transport(M.TRANSPORT_DEVICE)
        assert g.get_info().comm == 2
        g.assemble()
        before = g.get_info().kernel_launches
        check_cg(g, n, 50, 0.0)
        launched = g.get_info().kernel_launches - before
        parts = [g.part_info(q) for q in range(p)]
        assert all(q.n_neighbors > 0 for q in parts)
        if fold:
            # per part: init_vectors, push of r_0, init_finalize, halo init (p_1); per
            # iteration: SpMV, K6, push of r_(k+1), K7 (no push after the last K6)
            assert launched == p * (4 + 4 * 50 - 1)
        else:
            # + the separate accumulator pushes: one at init, two per iteration
            assert launched == p * (5 + 6 * 50 - 1)


@pytest.mark.parametrize("fold", [1, 0])
@pytest.mark.parametrize("xdef", [2, 5, 8])
@pytest.mark.parametrize("n,p", [((23, 17, 9), 3), ((12, 11, 10), 8), ((40, 8, 6), 2)])
def test_device_comm_deferred_x_bit_identical(n, p, xdef, fold):
    """The device protocol with the deferred-x ring (halo of p_(k+1) pushed into the ring
    buffer it lives in): 200 iterations, a tolerance stop and an odd count -- bitwise the
    oracle."""
    s = oracle_system(n)
    with M.Minife(*n, virtual=p, options={"x_defer": xdef, "fold_comm": fold}) as g:
        g.set_transport(M.TRANSPORT_DEVICE)
        g.assemble()
        for iters, tol in ((200, 0.0), (200, 1e-8), (7, 0.0)):
            r = g.cg_solve(iters, tol)
            o = oracle_cg(n, iters, tol)
            assert (r.status, r.iterations, r.converged) == (o.status, o.iters, o.converged)
            assert _same(g.history(), o.hist)
            assert _same(g.solution(), o.x)


@pytest.mark.parametrize("fmt", ALL_FORMATS)
@pytest.mark.parametrize("n,p", [((10, 10, 10), 2), ((23, 17, 9), 3), ((12, 11, 10), 8)])
def test_device_comm_unfolded_bit_identical(n, p, fmt):
    """The device protocol with separate k_acc_push / k_halo_wait launches (fold_comm = 0):
    bitwise the oracle, graph and profile mode."""
    s = oracle_system(n)
    with M.Minife(*n, virtual=p, fmt=fmt, options={"fold_comm": 0}) as g:
        g.set_transport(M.TRANSPORT_DEVICE)
        g.assemble()
        check_spmv(g, s, 7)
        check_cg(g, n, 200, 0.0)
        check_cg(g, n, 100, 1e-10)
        g.cg_profile(50)
        check_cg(g, n, 200, 0.0)


def test_errors_and_states():
    with M.Minife(4, 4, 4) as g:
        with pytest.raises(M.MinifeError) as e:
            g.cg_solve(10, 0.0)
        assert e.value.status == M.MINIFE_ESTATE
        g.assemble()
        with pytest.raises(M.MinifeError):
            g.cg_solve(0, 0.0)
        with pytest.raises(M.MinifeError):
            g.cg_solve(10, float("nan"))
        with pytest.raises(M.MinifeError):
            g.cg_solve(10, -1.0)
        g.assemble()                      # idempotent
        check_matrix(g, oracle_system((4, 4, 4)))


def test_all_dirichlet_mesh_converges_in_one_iteration():
    # 1x1x1: every node constrained -> A = I, b = v; CG stops at k = 1 with x = b
    with M.Minife(1, 1, 1) as g:
        g.assemble()
        r = g.cg_solve(200, 0.0)
        assert r.iterations == 1 and r.converged == 1
        assert np.array_equal(g.solution(), g.rhs())


def test_spmv_device_and_user_stream():
    import torch
    n = (16, 15, 14)
    s = oracle_system(n)
    x = minife_inputs.uniform_pm1(s.rows, 7)
    yo = O.spmv(s.row_ptr, s.col, s.val, x)
    with M.Minife(*n) as g:
        g.assemble()
        st = torch.cuda.Stream()
        g.set_stream(st.cuda_stream)
        xd = torch.from_numpy(x).cuda()
        yd = torch.empty_like(xd)
        g.spmv_device(xd.data_ptr(), yd.data_ptr(), st.cuda_stream)
        st.synchronize()
        assert _same(yd.cpu().numpy(), yo)
        check_cg(g, n, 50, 0.0)           # solve launched on the torch stream
        g.set_stream(None)


def test_profile_mode_matches_graph_mode():
    n = (20, 20, 20)
    with M.Minife(*n) as g:
        g.assemble()
        g.cg_solve(200, 0.0)
        h1, x1 = g.history(), g.solution()
        t = g.cg_profile(200)
        assert t.spmv_ms > 0 and t.update_xr_ms > 0 and t.update_p_ms > 0
        assert _same(g.history(), h1) and _same(g.solution(), x1)


@pytest.mark.parametrize("n", [(1, 1, 1), (10, 10, 10), (23, 17, 9), (33, 32, 31)])
def test_fused_scheme_bit_identical(n):
    """the fused two-kernel iteration performs C6 exactly."""
    s = oracle_system(n)
    with M.Minife(*n, fmt=M.FMT_SEG) as g:      # the fused scheme runs on FMT_SEG
        g.set_scheme(M.SCHEME_FUSED)
        g.assemble()
        check_cg(g, n, 200, 0.0)
        check_cg(g, n, 200, 1e-8)       # stop inside the fused prologue -> pending x update
        check_cg(g, n, 7, 0.0)          # odd count: p_K in the second buffer
        check_cg(g, n, 8, 0.0)
        t = g.cg_profile(50)
        assert t.update_p_launches == 1 and t.spmv_ms > 0
        check_cg(g, n, 50, 0.0)
        g.set_scheme(M.SCHEME_3K)
        check_cg(g, n, 200, 0.0)
        check_spmv(g, s, 12345)


def test_format_switch_keeps_results():
    n = (14, 13, 12)
    s = oracle_system(n)
    with M.Minife(*n) as g:
        assert g.get_info().format == M.FMT_SYM     # default
        g.set_format(M.FMT_SEG)
        g.assemble()
        seg_info = g.get_info()
        # nns = number of maximal consecutive-column runs of the oracle's CRS rows
        nns = sum(1 + int(np.sum(np.diff(s.col[s.row_ptr[i]:s.row_ptr[i + 1]]) != 1))
                  for i in range(s.rows))
        assert seg_info.local_nns == nns
        g.set_format(M.FMT_CRS)
        with pytest.raises(M.MinifeError):
            g.cg_solve(5, 0.0)                 # unassembled after a format switch
        g.assemble()
        check_matrix(g, s)
        check_cg(g, n, 60, 0.0)
        g.set_format(M.FMT_SEG)
        g.assemble()
        check_matrix(g, s)
        check_cg(g, n, 60, 0.0)
        g.set_format(M.FMT_SYM)
        g.assemble()
        check_matrix(g, s)
        check_cg(g, n, 60, 0.0)
    with M.Minife(*n, virtual=2) as g:
        assert g.get_info().format == M.FMT_SYM     # default everywhere: ghost rows hold
        g.assemble()                                # the halo's mirrors
        check_matrix(g, s)
        check_cg(g, n, 60, 0.0)


@pytest.mark.slow
@pytest.mark.parametrize("fmt", ALL_FORMATS)
def test_100cubed_full_parity(fmt):
    """configs[1] at full size: matrix, SpMV and the 200-iteration CG, element by element."""
    n = (100, 100, 100)
    s = oracle_system(n)
    with M.Minife(*n, fmt=fmt) as g:
        g.assemble()
        check_matrix(g, s)
        check_spmv(g, s, 12345)
        check_cg(g, n, 200, 0.0)


@pytest.mark.slow
@pytest.mark.parametrize("parts,transport", [(2, None), (4, "device")])
def test_100cubed_partitioned_snake_order(parts, transport):
    """configs[1] in RCB parts of 40-80 MB of matrix each, where the SYM SpMV alternates its
    tile order every iteration (snake order, automatic for 48-400 MB): bitwise the oracle,
    through the default and the device-initiated transports."""
    n = (100, 100, 100)
    with M.Minife(*n, virtual=parts) as g:
        if transport == "device":
            g.set_transport(M.TRANSPORT_DEVICE)
        g.assemble()
        check_cg(g, n, 200, 0.0)


@pytest.mark.slow
def test_300cubed_sampled_parity():
    """configs[2] at full size, in the bench's launch configuration: sampled rows of A and y
    against the oracle's per-row routine, and p-independence of the whole CG (P10)."""
    n = (300, 300, 300)
    rows = 301 ** 3
    rng = np.random.default_rng(0)
    gids = np.unique(np.concatenate([rng.integers(0, rows, 400),
                                     [0, 1, 300, 301, rows // 2, rows - 1, rows - 302]]))
    x = minife_inputs.uniform_pm1(rows, 12345)
    results = []
    for fmt in (M.FMT_SYM, M.FMT_SEG):
        with M.Minife(*n, fmt=fmt) as g:
            g.assemble()
            cols, vals, lens = g.export_rows(gids)
            y = g.spmv(x)
            for i, gid in enumerate(gids):
                oc, ov, ob = O.row(*n, int(gid))
                assert lens[i] == oc.size
                assert np.array_equal(cols[i, :lens[i]], oc)
                assert _same(vals[i, :lens[i]], ov)
                yo = O.spmv(np.array([0, oc.size]), oc, ov, x)[0]
                assert y[gid] == yo
            r1 = g.cg_solve(200, 0.0)
            assert r1.iterations == 200
            results.append((g.history(), g.solution()))
    with M.Minife(*n, virtual=2) as g2:
        g2.assemble()
        r2 = g2.cg_solve(200, 0.0)
        assert r2.iterations == 200
        for h1, x1 in results:
            assert _same(g2.history(), h1)
            assert _same(g2.solution(), x1)
