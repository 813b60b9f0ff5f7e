"""Timeline of one CG solve from a -DSYMM_TRACE build (tools/build_flags.sh trace -DSYMM_TRACE):

    MINIFE_LIB_PATH=paper_1505_08023_b200/lib/alt_trace.so python tools/trace_mid.py N [--opt K=V]

Per iteration k in 50..57: each kernel's span (earliest CTA entry .. latest CTA exit, ns of
%globaltimer) and the gaps between kernels; then, for the solve's last SpMV, the per-CTA
phases (entry -> setup, -> first tile's run starts, -> first tile folded, -> last tile, ->
expansion flush, -> accumulator merge) as medians and maxima over the CTAs."""
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1505_08023_b200 as M  # noqa: E402

n = int(sys.argv[1])
opts = {}
for i, a in enumerate(sys.argv):
    if a == "--opt":
        k, v = sys.argv[i + 1].split("=")
        opts[k] = int(v)
lib = M._lib
g = M.Minife(n, n, n, options=opts)
g.assemble()
for _ in range(2):
    g.cg_solve(200, 0.0)
kt = (ctypes.c_ulonglong * (256 * 6))()
assert lib.minife_dbg_kt(kt, 1) == 0
r = g.cg_solve(200, 0.0)
assert lib.minife_dbg_kt(kt, 0) == 0
a = np.array(kt, dtype=np.uint64).reshape(256, 3, 2).astype(np.int64)
rows = []
for k in range(50, 58):
    s, k6, k7 = a[k]
    nxt = a[k + 1][0]
    rows.append({"k": k, "spmv": int(s[1] - s[0]), "gap_s_k6": int(k6[0] - s[1]),
                 "k6": int(k6[1] - k6[0]), "gap_k6_k7": int(k7[0] - k6[1]),
                 "k7": int(k7[1] - k7[0]), "gap_k7_s": int(nxt[0] - k7[1]),
                 "iter": int(nxt[0] - s[0])})
tr = (ctypes.c_ulonglong * (1024 * 8))()
assert lib.minife_dbg_symm_trace(tr, 1024 * 8) == 0
t = np.array(tr, dtype=np.uint64).reshape(1024, 8).astype(np.int64)
t = t[t[:, 0] > 0]
t = t[t[:, 0] >= t[:, 0].max() - 10**7]          # this solve's last launch
t0 = t[:, 0].min()
ph = {}
names = ["entry", "setup", "first_runs", "first_fold", "last_tile", "flush", "merge",
         "warp0_flushed"]
for j in range(8):
    ph[names[j] + "_from_t0"] = [int(np.median(t[:, j] - t0)), int((t[:, j] - t0).max())]
k6 = (ctypes.c_ulonglong * (2048 * 16))()
assert lib.minife_dbg_k6_trace(k6, 2048 * 16) == 0
u = np.array(k6, dtype=np.uint64).reshape(2048, 16).astype(np.int64)
u = u[u[:, 0] > 0]
u = u[u[:, 0] >= u[:, 0].max() - 10**7]
u0 = u[:, 0].min()
k6ph = {}
for j, nm in enumerate(["entry", "done_read", "acc_in", "prologue", "loop", "flush", "merge",
                        "finalized", "unused", "loop_all"]):
    k6ph[nm] = [int(np.median(u[:, j] - u0)), int((u[:, j] - u0).max())]
print(json.dumps({"n": n, "options": opts, "solve_ms": r.seconds * 1e3, "ctas": len(t),
                  "iters": rows, "symm_last_launch": ph, "k6_ctas": len(u),
                  "k6_last_launch": k6ph}))
