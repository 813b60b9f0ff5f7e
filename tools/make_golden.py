"""Golden oracle references for the full-size configs (tests/golden/minife_*.json).

Calls ONLY ``oracle/`` (the plain C oracle) and ``minife_inputs`` (the seeded-vector module,
which holds none of the method's arithmetic); nothing here touches the CUDA path.  For one
mesh it runs the oracle's whole pipeline in the paper's module order (Fig 1.1):
structure (Fig 3.6), assembly (Fig 3.7, C2), Dirichlet (C3), one CRS SpMV on the seeded
vector (Fig 3.1, C4, C7 seed 12345) and 200 CG iterations from x0 = 0 with tol = 0 (C6,
BASELINE configs), and writes

  - the residual-norm history hist[0..200] as hex floats (bit-exact),
  - SHA-256 of row_ptr (int64), col (int64, global ids), val, b, x and the SpMV output y
    (float64, little endian; each float array hashed after adding +0.0, which folds -0.0
    into +0.0 -- the parity tests compare floats with IEEE ==),
  - a few x / y values at fixed ids as hex floats (diagnostics when a hash differs),
  - the oracle source's SHA-256 and the wall time of each phase.

    python tools/make_golden.py 300 300 300 [--iters 200]

Memory: CSR with int64 columns, 16 B per stored entry + ~6 vectors (400^3: ~33 GB;
600x600x300: ~52 GB).  Wall time on one core: ~2.2 ns per nnz per CG iteration.
"""
from __future__ import annotations

import argparse
import ctypes
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import minife_inputs  # noqa: E402
import oracle as O  # noqa: E402

CHUNK = 1 << 24


def sha_int(a: np.ndarray) -> str:
    h = hashlib.sha256()
    for i in range(0, a.size, CHUNK):
        h.update(np.ascontiguousarray(a[i:i + CHUNK], dtype="<i8").tobytes())
    return h.hexdigest()


def sha_f64(a: np.ndarray) -> str:
    h = hashlib.sha256()
    for i in range(0, a.size, CHUNK):
        c = np.ascontiguousarray(a[i:i + CHUNK], dtype="<f8") + 0.0   # -0.0 -> +0.0
        h.update(c.tobytes())
    return h.hexdigest()


def sample_ids(nx: int, ny: int, nz: int) -> list[int]:
    NX, NY, NZ = nx + 1, ny + 1, nz + 1
    rows = NX * NY * NZ
    pts = [(1, 1, 1), (nx // 2, ny // 2, nz // 2), (nx - 1, ny // 2, nz // 2),
           (nx // 4, ny // 3, nz // 5), (nx - 1, 1, nz - 1), (nx // 2, 1, nz // 2)]
    ids = sorted({ix + NX * (iy + NY * iz) for ix, iy, iz in pts} | {0, rows - 1})
    return ids


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("nx", type=int)
    ap.add_argument("ny", type=int)
    ap.add_argument("nz", type=int)
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--seed", type=int, default=minife_inputs.DEFAULT_SEED)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    nx, ny, nz = a.nx, a.ny, a.nz
    out = a.out or os.path.join(ROOT, "tests", "golden", f"minife_{nx}x{ny}x{nz}.json")
    L = O.lib()
    t = {}
    rows = (nx + 1) * (ny + 1) * (nz + 1)
    nnz = int(L.or_structure_nnz(nx, ny, nz))
    g = {"mesh": [nx, ny, nz], "rows": rows, "nnz": nnz,
         "generated_by": "tools/make_golden.py (oracle/ only: or_structure, or_assemble, "
                         "or_impose_dirichlet, or_spmv, or_cg)",
         "oracle_source_sha256": hashlib.sha256(open(O._SRC, "rb").read()).hexdigest(),
         "hash_convention": "sha256 of the little-endian array bytes; float arrays after "
                            "adding +0.0 (signed zeros folded: IEEE == semantics)"}
    sha = {}

    t0 = time.time()
    row_ptr = np.zeros(rows + 1, dtype=np.int64)
    col = np.zeros(nnz, dtype=np.int64)
    assert L.or_structure(nx, ny, nz, row_ptr, col) == O.OR_OK
    t["structure_s"] = time.time() - t0
    sha["row_ptr"] = sha_int(row_ptr)
    sha["col"] = sha_int(col)
    print(f"structure {t['structure_s']:.1f}s", flush=True)

    t0 = time.time()
    val = np.zeros(nnz, dtype=np.float64)
    b = np.zeros(rows, dtype=np.float64)
    assert L.or_assemble(nx, ny, nz, row_ptr, col, val, b) == O.OR_OK
    t["assemble_s"] = time.time() - t0
    t0 = time.time()
    assert L.or_impose_dirichlet(nx, ny, nz, row_ptr, col, val, b) == O.OR_OK
    t["dirichlet_s"] = time.time() - t0
    sha["val"] = sha_f64(val)
    sha["b"] = sha_f64(b)
    print(f"assembly {t['assemble_s']:.1f}s dirichlet {t['dirichlet_s']:.1f}s", flush=True)

    ids = sample_ids(nx, ny, nz)
    x_in = minife_inputs.uniform_pm1(rows, a.seed)
    y = np.zeros(rows, dtype=np.float64)
    t0 = time.time()
    L.or_spmv(rows, row_ptr, col, val, x_in, y)
    t["spmv_s"] = time.time() - t0
    sha[f"spmv_y_seed{a.seed}"] = sha_f64(y)
    g["spmv"] = {"seed": a.seed, "y_samples": {str(i): float(y[i]).hex() for i in ids}}
    del x_in, y
    print(f"spmv {t['spmv_s']:.2f}s", flush=True)

    x = np.zeros(rows, dtype=np.float64)
    hist = np.zeros(a.iters + 1, dtype=np.float64)
    iters = ctypes.c_int(0)
    conv = ctypes.c_int(0)
    t0 = time.time()
    st = L.or_cg(rows, row_ptr, col, val, b, a.iters, 0.0, x, hist, ctypes.byref(iters),
                 ctypes.byref(conv))
    t["cg_s"] = time.time() - t0
    sha["x"] = sha_f64(x)
    g["cg"] = {"max_iters": a.iters, "tol": 0.0, "status": int(st), "iterations": iters.value,
               "converged": conv.value,
               "hist_hex": [float(v).hex() for v in hist[:iters.value + 1]],
               "x_samples": {str(i): float(x[i]).hex() for i in ids}}
    print(f"cg {t['cg_s']:.1f}s ({t['cg_s'] / max(iters.value, 1):.2f} s/iteration)", flush=True)
    g["sha256"] = sha
    g["oracle_wall_s"] = t
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        json.dump(g, f, indent=1)
        f.write("\n")
    print("wrote", out)


if __name__ == "__main__":
    main()
