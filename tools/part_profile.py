"""Per-kernel-class times of a solve, one part vs VIRTUAL parts (the multi-rank code path: a
part with a halo runs the SYM-ext kernels that every rank of a torchrun job runs).

    python tools/part_profile.py NX NY NZ P [TRANSPORT]
TRANSPORT (VIRTUAL parts): 0 direct copies (default), 1 wire protocol, 2 push, 3 device-initiated
protocol (push + in-kernel reductions).  Prints ms per iteration by class, summed over the
parts, and per part.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1505_08023_b200 as M  # noqa: E402

nx, ny, nz, p = (int(v) for v in sys.argv[1:5])
tr = int(sys.argv[5]) if len(sys.argv) > 5 and not sys.argv[5].startswith("--") else 0
opts = {}
for i, a in enumerate(sys.argv):
    if a == "--opt":
        k, v = sys.argv[i + 1].split("=")
        opts[k] = int(v)
g = M.Minife(nx, ny, nz, virtual=p, options=opts) if p > 1 else M.Minife(nx, ny, nz, options=opts)
if p > 1:
    g.set_transport(tr)
g.assemble()
for _ in range(2):
    g.cg_solve(200, 0.0)
t = min(g.cg_solve(200, 0.0).seconds for _ in range(3))
pr = g.cg_profile(200)
it = pr.iterations
print(json.dumps({"mesh": [nx, ny, nz], "parts": p, "transport": tr, "options": opts, "iter_ms": t * 1e3 / 200,
                  "per_iter_ms": {"spmv": pr.spmv_ms / it, "update_xr": pr.update_xr_ms / it,
                                  "update_p": pr.update_p_ms / it, "comm": pr.comm_ms / it},
                  "per_part_spmv_ms": pr.spmv_ms / max(1, pr.spmv_launches)}))
