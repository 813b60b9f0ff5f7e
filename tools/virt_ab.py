"""Per-iteration time of a VIRTUAL (p parts on one GPU) solve:
    python tools/virt_ab.py N P FMT [TRANSPORT]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1505_08023_b200 as M  # noqa: E402

n, p = int(sys.argv[1]), int(sys.argv[2])
fmt = {"seg": M.FMT_SEG, "sym": M.FMT_SYM, "crs": M.FMT_CRS}[sys.argv[3]]
g = M.Minife(n, n, n, virtual=p, fmt=fmt)
tr = int(sys.argv[4]) if len(sys.argv) > 4 else 0
g.set_transport(tr)
g.assemble()
for _ in range(2):
    g.cg_solve(200, 0.0)
t = min(g.cg_solve(200, 0.0).seconds for _ in range(3))
print(json.dumps({"n": n, "parts": p, "fmt": sys.argv[3], "transport": tr,
                  "iter_ms": t * 1e3 / 200}))
