"""paper_1505_08023_b200 — B200-native MiniFE CG hot path (arxiv 1505.08023).

Thin ctypes binding of the C ABI in ``include/minife.h`` (argument marshalling only: every
step of the method runs in the sm_100a kernels of ``csrc/``).  There is no CPU fallback: if
``lib/libminife_b200.so`` is missing, importing this package raises.

The module-level functions carry the C names (``minife_create`` ...); ``Minife`` is a small
RAII wrapper over them that numpy-allocates the output buffers.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MINIFE_LIB_PATH: an alternative build of the same library (A/B experiments only)
LIB_PATH = os.environ.get("MINIFE_LIB_PATH") or os.path.join(_HERE, "lib", "libminife_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not built: run `python paper_1505_08023_b200/build.py` "
        "(or __graft_entry__.build()); there is no CPU fallback")


def _torch_nccl_path() -> str:
    """The NCCL torch was built against (nvidia-nccl wheel), found without importing torch."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    for loc in (spec.submodule_search_locations or []) if spec else []:
        cand = os.path.join(loc, "lib", "libnccl.so.2")
        if os.path.exists(cand):
            return cand
    return ""


os.environ.setdefault("MINIFE_NCCL_LIB", _torch_nccl_path())
_lib = ctypes.CDLL(LIB_PATH)

MINIFE_OK, MINIFE_EINVAL, MINIFE_ESTATE, MINIFE_ECUDA, MINIFE_ENCCL = 0, 1, 2, 3, 4
MINIFE_ENOMEM, MINIFE_ENOTSPD, MINIFE_EDIVERGED, MINIFE_ENODEV = 5, 6, 7, 8
MINIFE_ECOMM = 9
MODE_SINGLE, MODE_VIRTUAL, MODE_MULTI, MODE_RANK = 0, 1, 2, 3
FMT_CRS, FMT_SEG, FMT_SYM = 0, 1, 2
SCHEME_3K, SCHEME_FUSED = 0, 1
TRANSPORT_DIRECT, TRANSPORT_WIRE, TRANSPORT_PUSH, TRANSPORT_DEVICE = 0, 1, 2, 3


class minife_part_info(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("box", ctypes.c_int32 * 6), ("own", ctypes.c_int32 * 6),
                ("n_neighbors", ctypes.c_int32), ("device", ctypes.c_int32),
                ("rows", ctypes.c_int64), ("externals", ctypes.c_int64),
                ("nnz", ctypes.c_int64), ("slices", ctypes.c_int64),
                ("sell_entries", ctypes.c_int64), ("send_total", ctypes.c_int64),
                ("interior_slices", ctypes.c_int64)]


class minife_info(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("mode", ctypes.c_int32), ("nparts", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("assembled", ctypes.c_int32),
                ("rows", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("local_rows", ctypes.c_int64), ("local_nnz", ctypes.c_int64),
                ("max_part_rows", ctypes.c_int64), ("max_part_nnz", ctypes.c_int64),
                ("max_part_externals", ctypes.c_int64), ("sell_entries", ctypes.c_int64),
                ("device_bytes", ctypes.c_int64), ("format", ctypes.c_int32),
                ("comm", ctypes.c_int32), ("local_nns", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64)]


class minife_cg_result(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("iterations", ctypes.c_int32),
                ("converged", ctypes.c_int32), ("max_iters", ctypes.c_int32),
                ("norm_b", ctypes.c_double), ("final_rel_residual", ctypes.c_double),
                ("seconds", ctypes.c_double), ("flops", ctypes.c_double),
                ("bytes", ctypes.c_double)]


class minife_kernel_times(ctypes.Structure):
    _fields_ = [("spmv_ms", ctypes.c_double), ("update_xr_ms", ctypes.c_double),
                ("update_p_ms", ctypes.c_double), ("comm_ms", ctypes.c_double),
                ("spmv_launches", ctypes.c_int32), ("update_xr_launches", ctypes.c_int32),
                ("update_p_launches", ctypes.c_int32), ("iterations", ctypes.c_int32)]


_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_D = ctypes.c_double
_PP = ctypes.POINTER(ctypes.c_void_p)

# name -> (restype, argtypes); this table is also the list of exported symbols the CPU test
# checks against include/minife.h
SIGNATURES = {
    "minife_create": (_I, [_I, _I, _I, _I, _PP]),
    "minife_create_virtual": (_I, [_I, _I, _I, _I, _PP]),
    "minife_nccl_unique_id": (_I, [_P]),
    "minife_create_rank": (_I, [_I, _I, _I, _I, _I, _I, _P, _PP]),
    "minife_destroy": (None, [_P]),
    "minife_set_stream": (_I, [_P, _P]),
    "minife_strerror": (ctypes.c_char_p, [_I]),
    "minife_last_error": (ctypes.c_char_p, [_P]),
    "minife_set_format": (_I, [_P, _I]),
    "minife_set_scheme": (_I, [_P, _I]),
    "minife_set_transport": (_I, [_P, _I]),
    "minife_set_option": (_I, [_P, ctypes.c_char_p, _I64]),
    "minife_assemble": (_I, [_P]),
    "minife_cg_solve": (_I, [_P, _I, _D, ctypes.POINTER(minife_cg_result)]),
    "minife_cg_profile": (_I, [_P, _I, ctypes.POINTER(minife_kernel_times)]),
    "minife_spmv": (_I, [_P, _P, _P]),
    "minife_spmv_device": (_I, [_P, _P, _P, _P]),
    "minife_get_info": (_I, [_P, ctypes.POINTER(minife_info)]),
    "minife_get_timings": (_I, [_P, ctypes.POINTER(_D), ctypes.POINTER(_D)]),
    "minife_verify": (_I, [_P, _I64, _P, _I, _P, _P, ctypes.POINTER(_D)]),
    "minife_gather_times": (_I, [_P, _P]),
    "minife_get_part_info": (_I, [_P, _I, ctypes.POINTER(minife_part_info)]),
    "minife_export_csr": (_I, [_P, _P, _P, _P]),
    "minife_export_rows": (_I, [_P, _I64, _P, _P, _P, _P]),
    "minife_get_rhs": (_I, [_P, _P]),
    "minife_get_solution": (_I, [_P, _P]),
    "minife_get_history": (_I, [_P, _P, _I, ctypes.POINTER(ctypes.c_int)]),
    "minife_get_owned_ids": (_I, [_P, _P]),
    "minife_plan": (_I, [_I, _I, _I, _I, _I, ctypes.POINTER(minife_part_info)]),
    "minife_plan_lists": (_I, [_I, _I, _I, _I, _I, _P, _P, _P, _P, _P]),
    "minife_bandwidth_probe": (_I, [_I, _I64, _I, ctypes.POINTER(_D), ctypes.POINTER(_D)]),
    "minife_probe_l2_read_gbs": (_D, []),
    "minife_probe_write_gbs": (_D, []),
    "minife_dot": (_I, [_I, _I64, _P, _P, ctypes.POINTER(_D)]),
    "minife_set_timing_window": (_I, [_P, _I, _I]),
    "minife_get_timing_window": (_I, [_P, ctypes.POINTER(_D), ctypes.POINTER(_D)]),
    "minife_exact_round": (_I, [_I, _P, ctypes.POINTER(_D)]),
    "minife_version": (ctypes.c_char_p, []),
}

for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args
    globals()[_name] = _f


class MinifeError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        self.status = status
        msg = f"{where}: {minife_strerror(status).decode()} (status {status})"
        if detail:
            msg += f": {detail}"
        super().__init__(msg)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def plan(nx: int, ny: int, nz: int, world: int, rank: int) -> minife_part_info:
    """Host-only RCB plan of one part (no GPU needed)."""
    out = minife_part_info()
    st = minife_plan(nx, ny, nz, world, rank, ctypes.byref(out))
    if st != MINIFE_OK:
        raise MinifeError(st, "minife_plan")
    return out


def plan_lists(nx: int, ny: int, nz: int, world: int, rank: int) -> dict:
    """Host-only halo lists of one part: externals, neighbors, recv/send counts, send idx."""
    info = plan(nx, ny, nz, world, rank)
    ext = np.zeros(info.externals, dtype=np.int64)
    nbr = np.zeros(info.n_neighbors, dtype=np.int32)
    rc = np.zeros(info.n_neighbors, dtype=np.int64)
    sc = np.zeros(info.n_neighbors, dtype=np.int64)
    si = np.zeros(info.send_total, dtype=np.int32)
    st = minife_plan_lists(nx, ny, nz, world, rank, _ptr(ext), _ptr(nbr), _ptr(rc), _ptr(sc),
                           _ptr(si))
    if st != MINIFE_OK:
        raise MinifeError(st, "minife_plan_lists")
    return {"info": info, "ext_gids": ext, "nbr": nbr, "recv_cnt": rc, "send_cnt": sc,
            "send_idx": si}


def bandwidth_probe(device: int = 0, nbytes: int = 8 << 30, reps: int = 5):
    """(read GB/s, copy GB/s) of the library's pure-read and copy stream kernels."""
    r, c = ctypes.c_double(0.0), ctypes.c_double(0.0)
    st = minife_bandwidth_probe(device, nbytes, reps, ctypes.byref(r), ctypes.byref(c))
    if st != MINIFE_OK:
        raise MinifeError(st, "minife_bandwidth_probe")
    return r.value, c.value


ACC_WORDS = 72


def dot(u: np.ndarray, v: np.ndarray, device: int = 0) -> float:
    """Exactly rounded dot product on the device (C5; the CG dots' own code path)."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    if u.shape != v.shape or u.ndim != 1:
        raise ValueError("u and v must be 1-D of equal length")
    out = ctypes.c_double(0.0)
    st = minife_dot(device, u.size, _ptr(u), _ptr(v), ctypes.byref(out))
    if st != MINIFE_OK:
        raise MinifeError(st, "minife_dot")
    return out.value


def exact_round(words, device: int = 0) -> float:
    """RN(sum_i words[i] 2^(32 i - 1074)) by the device's accumulator rounding step."""
    w = np.zeros(ACC_WORDS, dtype=np.int64)
    src = np.asarray(words, dtype=np.int64)
    w[:src.size] = src
    out = ctypes.c_double(0.0)
    st = minife_exact_round(device, _ptr(w), ctypes.byref(out))
    if st != MINIFE_OK:
        raise MinifeError(st, "minife_exact_round")
    return out.value


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = minife_nccl_unique_id(buf)
    if st != MINIFE_OK:
        raise MinifeError(st, "minife_nccl_unique_id")
    return buf.raw


class Minife:
    """RAII wrapper: Minife(nx, ny, nz, ngpu=1 | virtual=p | rank=(r, w, dev, uid))."""

    def __init__(self, nx: int, ny: int, nz: int, ngpu: int = 1, virtual: int | None = None,
                 rank: tuple | None = None, fmt: int | None = None,
                 options: dict | None = None):
        h = ctypes.c_void_p()
        if rank is not None:
            r, w, dev, uid = rank
            st = minife_create_rank(nx, ny, nz, r, w, dev, ctypes.c_char_p(uid),
                                    ctypes.byref(h))
        elif virtual is not None:
            st = minife_create_virtual(nx, ny, nz, virtual, ctypes.byref(h))
        else:
            st = minife_create(nx, ny, nz, ngpu, ctypes.byref(h))
        if st != MINIFE_OK:
            raise MinifeError(st, "minife_create")
        self.h = h
        if fmt is not None:
            self._check(minife_set_format(self.h, fmt), "minife_set_format")
        for k, v in (options or {}).items():
            self.set_option(k, v)
        self.info = self.get_info()

    # -- lifecycle -------------------------------------------------------------------------
    def close(self):
        if getattr(self, "h", None):
            minife_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except TypeError:       # interpreter shutdown: module globals already cleared
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, st, where):
        if st != MINIFE_OK:
            raise MinifeError(st, where, minife_last_error(self.h).decode())

    # -- queries ---------------------------------------------------------------------------
    def get_info(self) -> minife_info:
        out = minife_info()
        self._check(minife_get_info(self.h, ctypes.byref(out)), "minife_get_info")
        return out

    def timings(self):
        """(assemble ms, solve ms) of the last calls: device time, max over the ctx's parts."""
        a, s = ctypes.c_double(0.0), ctypes.c_double(0.0)
        self._check(minife_get_timings(self.h, ctypes.byref(a), ctypes.byref(s)),
                    "minife_get_timings")
        return a.value, s.value

    def part_info(self, part: int) -> minife_part_info:
        out = minife_part_info()
        self._check(minife_get_part_info(self.h, part, ctypes.byref(out)),
                    "minife_get_part_info")
        return out

    @property
    def io_rows(self) -> int:
        """Length of host vectors in this ctx's I/O (global rows, or owned rows in RANK)."""
        i = self.get_info()
        return i.local_rows if i.mode == MODE_RANK else i.rows

    # -- hot path --------------------------------------------------------------------------
    def set_stream(self, stream_handle: int | None):
        self._check(minife_set_stream(self.h, ctypes.c_void_p(stream_handle or 0)),
                    "minife_set_stream")

    def set_format(self, fmt: int):
        """FMT_SYM (default: BCRS segments + upper-triangle values), FMT_SEG (the paper's BCRS
        on SELL-32) or FMT_CRS (one index per entry); the ctx becomes unassembled."""
        self._check(minife_set_format(self.h, fmt), "minife_set_format")
        self.info = self.get_info()

    def set_transport(self, transport: int):
        """VIRTUAL ctxs: TRANSPORT_DIRECT (default), TRANSPORT_WIRE (the NCCL-mode protocol),
        TRANSPORT_PUSH (device halo push) or TRANSPORT_DEVICE (push + in-kernel reductions:
        the device-initiated protocol of MULTI/RANK ctxs)."""
        self._check(minife_set_transport(self.h, transport), "minife_set_transport")

    def set_option(self, name: str, value: int):
        """Per-ctx execution option (minife.h: x_defer, small_solver, graph, ...)."""
        self._check(minife_set_option(self.h, name.encode(), int(value)), "minife_set_option")

    def set_scheme(self, scheme: int):
        """SCHEME_3K (default) or SCHEME_FUSED (one part + FMT_SEG); bit-identical results."""
        self._check(minife_set_scheme(self.h, scheme), "minife_set_scheme")

    def assemble(self):
        self._check(minife_assemble(self.h), "minife_assemble")
        self.info = self.get_info()

    def cg_solve(self, max_iters: int = 200, tol: float = 0.0) -> minife_cg_result:
        res = minife_cg_result()
        st = minife_cg_solve(self.h, max_iters, tol, ctypes.byref(res))
        if st not in (MINIFE_OK, MINIFE_ENOTSPD, MINIFE_EDIVERGED):
            self._check(st, "minife_cg_solve")
        return res

    def set_timing_window(self, first_iter: int, n_iters: int):
        """Time the SpMV of iterations [first_iter, first_iter + n_iters) inside later solves."""
        self._check(minife_set_timing_window(self.h, first_iter, n_iters),
                    "minife_set_timing_window")

    def timing_window(self):
        """(SpMV ms, iteration ms) averaged over the window of the last solve."""
        a, b = ctypes.c_double(0.0), ctypes.c_double(0.0)
        self._check(minife_get_timing_window(self.h, ctypes.byref(a), ctypes.byref(b)),
                    "minife_get_timing_window")
        return a.value, b.value

    def cg_profile(self, max_iters: int = 200) -> minife_kernel_times:
        out = minife_kernel_times()
        st = minife_cg_profile(self.h, max_iters, ctypes.byref(out))
        if st not in (MINIFE_OK, MINIFE_ENOTSPD, MINIFE_EDIVERGED):
            self._check(st, "minife_cg_profile")
        return out

    def spmv(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.size != self.io_rows:
            raise ValueError(f"x has {x.size} entries, expected {self.io_rows}")
        y = np.empty_like(x)
        self._check(minife_spmv(self.h, _ptr(x), _ptr(y)), "minife_spmv")
        return y

    def spmv_device(self, x_ptr: int, y_ptr: int, stream_handle: int | None = None):
        self._check(minife_spmv_device(self.h, ctypes.c_void_p(x_ptr), ctypes.c_void_p(y_ptr),
                                       ctypes.c_void_p(stream_handle or 0)),
                    "minife_spmv_device")

    # -- getters ---------------------------------------------------------------------------
    def export_csr(self):
        i = self.get_info()
        rows = i.local_rows if i.mode == MODE_RANK else i.rows
        nnz = i.local_nnz if i.mode == MODE_RANK else i.nnz
        rp = np.zeros(rows + 1, dtype=np.int64)
        col = np.zeros(nnz, dtype=np.int64)
        val = np.zeros(nnz, dtype=np.float64)
        self._check(minife_export_csr(self.h, _ptr(rp), _ptr(col), _ptr(val)),
                    "minife_export_csr")
        return rp, col, val

    def export_rows(self, gids):
        gids = np.ascontiguousarray(gids, dtype=np.int64)
        n = gids.size
        cols = np.zeros(27 * max(n, 1), dtype=np.int64)
        vals = np.zeros(27 * max(n, 1), dtype=np.float64)
        lens = np.zeros(max(n, 1), dtype=np.int32)
        self._check(minife_export_rows(self.h, n, _ptr(gids), _ptr(cols), _ptr(vals),
                                       _ptr(lens)), "minife_export_rows")
        return cols.reshape(-1, 27)[:n], vals.reshape(-1, 27)[:n], lens[:n]

    def rhs(self) -> np.ndarray:
        b = np.zeros(self.io_rows, dtype=np.float64)
        self._check(minife_get_rhs(self.h, _ptr(b)), "minife_get_rhs")
        return b

    def solution(self) -> np.ndarray:
        x = np.zeros(self.io_rows, dtype=np.float64)
        self._check(minife_get_solution(self.h, _ptr(x)), "minife_get_solution")
        return x

    def history(self, cap: int = 100000) -> np.ndarray:
        h = np.zeros(cap, dtype=np.float64)
        n = ctypes.c_int(0)
        self._check(minife_get_history(self.h, _ptr(h), cap, ctypes.byref(n)),
                    "minife_get_history")
        return h[: n.value].copy()

    def verify(self, gids, nterms: int = 200):
        """(u_fe, u_exact, max |error|) at probe nodes (rank 0 / one-process ctxs)."""
        gids = np.ascontiguousarray(gids, dtype=np.int64)
        fe = np.zeros(max(gids.size, 1))
        ex = np.zeros(max(gids.size, 1))
        mx = ctypes.c_double(0.0)
        self._check(minife_verify(self.h, gids.size, _ptr(gids), nterms, _ptr(fe), _ptr(ex),
                                  ctypes.byref(mx)), "minife_verify")
        return fe[:gids.size], ex[:gids.size], mx.value

    def gather_times(self) -> np.ndarray:
        """Per-rank (assembly ms, solve ms) of the last calls, gathered to rank 0."""
        i = self.get_info()
        n = i.world if i.mode == MODE_RANK else max(i.nparts, 1)
        out = np.zeros(2 * n)
        self._check(minife_gather_times(self.h, _ptr(out)), "minife_gather_times")
        return out.reshape(n, 2)

    def owned_ids(self) -> np.ndarray:
        out = np.zeros(self.get_info().local_rows, dtype=np.int64)
        self._check(minife_get_owned_ids(self.h, _ptr(out)), "minife_get_owned_ids")
        return out


__all__ = ["Minife", "MinifeError", "plan", "plan_lists", "nccl_unique_id", "LIB_PATH",
           "SIGNATURES"] + list(SIGNATURES)
