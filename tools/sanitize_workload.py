"""Small end-to-end run of every kernel family for compute-sanitizer (no pytest overhead).
Run with the environment it needs to reach each path, e.g.
    compute-sanitizer --tool memcheck python tools/sanitize_workload.py
(the script sets the solver-selection toggles itself, per process, below)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
# multi-kernel path at small sizes (so the SpMV / update kernels run), x-every-2 forced
os.environ.setdefault("MINIFE_SMALL", os.environ.get("SAN_SMALL", "0"))
os.environ.setdefault("MINIFE_X2", "2")
import minife_inputs  # noqa: E402
import paper_1505_08023_b200 as M  # noqa: E402

cases = [((5, 4, 3), {}), ((5, 4, 3), {"fmt": M.FMT_SEG}), ((5, 4, 3), {"fmt": M.FMT_CRS}),
         ((40, 3, 2), {}), ((6, 5, 4), {"virtual": 3}), ((6, 5, 4), {"virtual": 3, "fmt": M.FMT_SEG}),
         ((6, 5, 4), {"virtual": 3, "fmt": M.FMT_CRS})]
for n, kw in cases:
    for transport in ((0, 1, 2) if "virtual" in kw else (None,)):
        with M.Minife(*n, **kw) as g:
            if transport is not None:
                g.set_transport(transport)
            g.assemble()
            x = minife_inputs.uniform_pm1(g.io_rows, 1)
            g.spmv(x)
            g.cg_solve(30, 0.0)
            g.cg_solve(31, 1e-6)
            g.cg_profile(10)
            g.solution(); g.history(); g.export_csr(); g.export_rows([0, 5, 17])
with M.Minife(7, 6, 5, fmt=M.FMT_SEG) as g:
    g.set_scheme(M.SCHEME_FUSED)
    g.assemble()
    g.cg_solve(25, 0.0)
    g.cg_solve(25, 1e-5)
u = minife_inputs.uniform_pm1(1000, 3)
M.dot(u, u)
M.exact_round([1, 2, 3])
print("sanitize workload done")
