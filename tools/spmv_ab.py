"""A/B timing of SpMV / CG-iteration kernels for one format and ctx options.

    python tools/spmv_ab.py N FORMAT [--parity] [--opt NAME=VALUE ...]

Prints one JSON line: per-launch SpMV ms, update ms per iteration, graph ms per iteration.
--parity additionally checks one CG solve's history against a 2-part virtual SEG solve
(partition independence, bit-exact) -- a property, not an oracle comparison.
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1505_08023_b200 as M  # noqa: E402

n = int(sys.argv[1])
fmt = {"seg": M.FMT_SEG, "sym": M.FMT_SYM, "crs": M.FMT_CRS}[sys.argv[2]]
scheme = M.SCHEME_FUSED if "--fused" in sys.argv else M.SCHEME_3K
opts = {}
for i, a in enumerate(sys.argv):
    if a == "--opt":
        k, v = sys.argv[i + 1].split("=")
        opts[k] = int(v)
iters = 200
g = M.Minife(n, n, n, options=opts)
g.set_format(fmt)
g.set_scheme(scheme)
g.assemble()
for _ in range(2):
    r = g.cg_solve(iters, 0.0)
t = []
for _ in range(3):
    r = g.cg_solve(iters, 0.0)
    t.append(r.seconds)
p = g.cg_profile(iters)
out = {"n": n, "fmt": sys.argv[2], "options": opts,
       "spmv_ms": p.spmv_ms / p.spmv_launches,
       "upd_ms": (p.update_xr_ms + p.update_p_ms) / p.iterations,
       "iter_ms": min(t) * 1e3 / iters}
if "--parity" in sys.argv:
    h1 = g.history(iters + 1).copy()
    x1 = g.solution().copy()
    g.close()
    v = M.Minife(n, n, n, virtual=2)
    v.assemble()
    v.cg_solve(iters, 0.0)
    out["parity_vs_virtual2"] = bool(np.array_equal(h1, v.history(iters + 1)) and
                                     np.array_equal(x1, v.solution()))
print(json.dumps(out), flush=True)
