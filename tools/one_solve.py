"""One 200-iteration solve at N^3 (a target for ncu --launch-skip captures of one iteration's
kernels):  python tools/one_solve.py N [--opt k=v]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1505_08023_b200 as M  # noqa: E402

n = int(sys.argv[1])
opts = {}
for i, a in enumerate(sys.argv):
    if a == "--opt":
        k, v = sys.argv[i + 1].split("=")
        opts[k] = int(v)
g = M.Minife(n, n, n, options=opts)
g.assemble()
r = g.cg_solve(200, 0.0)
print(r.iterations, r.status)
