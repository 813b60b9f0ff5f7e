"""CPU oracle for the MiniFE CG hot path (arxiv 1505.08023) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1505_08023_b200``) never imports it and shares no code with it.

This module is argument marshalling (ctypes + numpy) around ``minife_oracle.c``; every
step of the method runs in that plain, single-threaded C99 file (binary64, built with
``-O2 -ffp-contract=off``).  Citations (P:n = PAPER.md line n, S:n = SPEC.md line n,
C0..C8 / G1..G20 = DESIGN.md §3 readings) are in the C source beside each function.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "minife_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OR_OK, OR_EINVAL, OR_ENOTSPD, OR_EDIVERGED = 0, 1, 6, 7

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, -O2 -ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
             "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.or_node_id.restype = ctypes.c_int64
        L.or_node_id.argtypes = [ctypes.c_int64] * 6
        L.or_element_matrix.restype = None
        L.or_element_matrix.argtypes = [ctypes.c_double] * 3 + [_f64p]
        L.or_structure_nnz.restype = ctypes.c_int64
        L.or_structure_nnz.argtypes = [ctypes.c_int] * 3
        L.or_structure.restype = ctypes.c_int
        L.or_structure.argtypes = [ctypes.c_int] * 3 + [_i64p, _i64p]
        L.or_assemble.restype = ctypes.c_int
        L.or_assemble.argtypes = [ctypes.c_int] * 3 + [_i64p, _i64p, _f64p, _f64p]
        L.or_impose_dirichlet.restype = ctypes.c_int
        L.or_impose_dirichlet.argtypes = [ctypes.c_int] * 3 + [_i64p, _i64p, _f64p, _f64p]
        L.or_row.restype = ctypes.c_int
        L.or_row.argtypes = [ctypes.c_int] * 3 + [ctypes.c_int64, _i64p, _f64p,
                                                  ctypes.POINTER(ctypes.c_double)]
        L.or_spmv.restype = None
        L.or_spmv.argtypes = [ctypes.c_int64, _i64p, _i64p, _f64p, _f64p, _f64p]
        L.or_dot.restype = ctypes.c_double
        L.or_dot.argtypes = [ctypes.c_int64, _f64p, _f64p]
        L.or_cg.restype = ctypes.c_int
        L.or_cg.argtypes = [ctypes.c_int64, _i64p, _i64p, _f64p, _f64p, ctypes.c_int,
                            ctypes.c_double, _f64p, _f64p, ctypes.POINTER(ctypes.c_int),
                            ctypes.POINTER(ctypes.c_int)]
        L.or_analytic.restype = ctypes.c_double
        L.or_analytic.argtypes = [ctypes.c_double] * 3 + [ctypes.c_int]
        L.or_rcb.restype = ctypes.c_int
        L.or_rcb.argtypes = [ctypes.c_int] * 4 + [_i32p]
        L.or_owner.restype = ctypes.c_int
        L.or_owner.argtypes = [ctypes.c_int, _i32p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.or_externals.restype = ctypes.c_int64
        L.or_externals.argtypes = [ctypes.c_int] * 4 + [_i32p, ctypes.c_int,
                                                         ctypes.c_void_p]
        L.or_owned.restype = ctypes.c_int64
        L.or_owned.argtypes = [ctypes.c_int] * 4 + [_i32p, ctypes.c_int, ctypes.c_void_p]
        _lib = L
    return _lib


# ------------------------------------------------------------------------------------------
# thin wrappers
# ------------------------------------------------------------------------------------------

def node_id(nodes, ix, iy, iz) -> int:
    return int(lib().or_node_id(nodes[0], nodes[1], nodes[2], ix, iy, iz))


def element_matrix(hx: float, hy: float, hz: float) -> np.ndarray:
    K = np.zeros(64, dtype=np.float64)
    lib().or_element_matrix(hx, hy, hz, K)
    return K.reshape(8, 8)


def structure(nx: int, ny: int, nz: int):
    rows = (nx + 1) * (ny + 1) * (nz + 1)
    nnz = int(lib().or_structure_nnz(nx, ny, nz))
    row_ptr = np.zeros(rows + 1, dtype=np.int64)
    col = np.zeros(nnz, dtype=np.int64)
    st = lib().or_structure(nx, ny, nz, row_ptr, col)
    if st != OR_OK:
        raise ValueError(f"or_structure status {st}")
    return row_ptr, col


class System:
    """Assembled global system (CSR, rows in global id order) after Dirichlet (C2, C3)."""

    def __init__(self, nx, ny, nz, row_ptr, col, val, b, val_pre_bc=None, b_pre_bc=None):
        self.nx, self.ny, self.nz = nx, ny, nz
        self.row_ptr, self.col, self.val, self.b = row_ptr, col, val, b
        self.val_pre_bc, self.b_pre_bc = val_pre_bc, b_pre_bc

    @property
    def rows(self):
        return self.row_ptr.size - 1

    @property
    def nnz(self):
        return int(self.row_ptr[-1])


def assemble(nx: int, ny: int, nz: int, keep_pre_bc: bool = False) -> System:
    row_ptr, col = structure(nx, ny, nz)
    val = np.zeros(col.size, dtype=np.float64)
    b = np.zeros(row_ptr.size - 1, dtype=np.float64)
    st = lib().or_assemble(nx, ny, nz, row_ptr, col, val, b)
    if st != OR_OK:
        raise ValueError(f"or_assemble status {st}")
    pre_v = val.copy() if keep_pre_bc else None
    pre_b = b.copy() if keep_pre_bc else None
    lib().or_impose_dirichlet(nx, ny, nz, row_ptr, col, val, b)
    return System(nx, ny, nz, row_ptr, col, val, b, pre_v, pre_b)


def row(nx: int, ny: int, nz: int, gid: int):
    cols = np.zeros(27, dtype=np.int64)
    vals = np.zeros(27, dtype=np.float64)
    b = ctypes.c_double(0.0)
    n = lib().or_row(nx, ny, nz, gid, cols, vals, ctypes.byref(b))
    if n < 0:
        raise ValueError("row out of range")
    return cols[:n].copy(), vals[:n].copy(), b.value


def spmv(row_ptr, col, val, x) -> np.ndarray:
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int64)
    val = np.ascontiguousarray(val, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros(row_ptr.size - 1, dtype=np.float64)
    lib().or_spmv(row_ptr.size - 1, row_ptr, col, val, x, y)
    return y


def dot(u, v) -> float:
    u = np.ascontiguousarray(u, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    assert u.size == v.size
    return float(lib().or_dot(u.size, u, v))


class CgResult:
    def __init__(self, status, x, hist, iters, converged):
        self.status, self.x, self.iters, self.converged = status, x, iters, converged
        self.hist = hist[: iters + 1].copy()


def cg(row_ptr, col, val, b, max_iters: int = 200, tol: float = 0.0) -> CgResult:
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int64)
    val = np.ascontiguousarray(val, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    m = row_ptr.size - 1
    x = np.zeros(m, dtype=np.float64)
    hist = np.zeros(max_iters + 1, dtype=np.float64)
    iters = ctypes.c_int(0)
    conv = ctypes.c_int(0)
    st = lib().or_cg(m, row_ptr, col, val, b, max_iters, tol, x, hist, ctypes.byref(iters),
                     ctypes.byref(conv))
    return CgResult(st, x, hist, iters.value, conv.value)


def analytic(x: float, y: float, z: float, nterms: int = 300) -> float:
    return float(lib().or_analytic(x, y, z, nterms))


def rcb(nx: int, ny: int, nz: int, p: int) -> np.ndarray:
    boxes = np.zeros(6 * max(p, 1), dtype=np.int32)
    st = lib().or_rcb(nx, ny, nz, p, boxes)
    if st != OR_OK:
        raise ValueError(f"or_rcb status {st}")
    return boxes.reshape(p, 6)


def owner(boxes: np.ndarray, ix: int, iy: int, iz: int) -> int:
    b = np.ascontiguousarray(boxes, dtype=np.int32).reshape(-1)
    return int(lib().or_owner(b.size // 6, b, ix, iy, iz))


def owned(nx, ny, nz, boxes, rank) -> np.ndarray:
    b = np.ascontiguousarray(boxes, dtype=np.int32).reshape(-1)
    p = b.size // 6
    n = lib().or_owned(nx, ny, nz, p, b, rank, None)
    out = np.zeros(n, dtype=np.int64)
    lib().or_owned(nx, ny, nz, p, b, rank, out.ctypes.data)
    return out


def externals(nx, ny, nz, boxes, rank) -> np.ndarray:
    b = np.ascontiguousarray(boxes, dtype=np.int32).reshape(-1)
    p = b.size // 6
    n = lib().or_externals(nx, ny, nz, p, b, rank, None)
    out = np.zeros(n, dtype=np.int64)
    lib().or_externals(nx, ny, nz, p, b, rank, out.ctypes.data)
    return out
