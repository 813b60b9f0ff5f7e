"""Small end-to-end run of every kernel family for compute-sanitizer (no pytest overhead)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import minife_inputs
import paper_1505_08023_b200 as M

for n, kw in [((5, 4, 3), {}), ((5, 4, 3), {"fmt": M.FMT_CRS}), ((6, 5, 4), {"virtual": 3}),
              ((6, 5, 4), {"virtual": 3, "fmt": M.FMT_CRS})]:
    with M.Minife(*n, **kw) as g:
        g.assemble()
        x = minife_inputs.uniform_pm1(g.io_rows, 1)
        g.spmv(x)
        g.cg_solve(30, 0.0)
        g.cg_solve(30, 1e-6)
        g.cg_profile(10)
        g.solution(); g.history(); g.export_csr(); g.export_rows([0, 5, 17])
with M.Minife(7, 6, 5) as g:
    g.set_scheme(M.SCHEME_FUSED)
    g.assemble()
    g.cg_solve(25, 0.0)
    g.cg_solve(25, 1e-5)
print("sanitize workload done")
