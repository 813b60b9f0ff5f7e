"""Subprocess helper for test_gpu_parity: run one mesh through the library with the
single-launch solver selection given by MINIFE_SMALL (read once per process) and compare
with the oracle bit for bit.  Prints 'ok' on success."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import paper_1505_08023_b200 as M  # noqa: E402

n = tuple(int(v) for v in sys.argv[1:4])
fmt = {"seg": M.FMT_SEG, "sym": M.FMT_SYM}[sys.argv[4]]
s = O.assemble(*n)
with M.Minife(*n, fmt=fmt) as g:
    g.assemble()
    for iters, tol in ((200, 0.0), (200, 1e-8), (7, 0.0)):
        r = g.cg_solve(iters, tol)
        o = O.cg(s.row_ptr, s.col, s.val, s.b, iters, tol)
        assert (r.status, r.iterations, r.converged) == (o.status, o.iters, o.converged)
        assert np.array_equal(g.history(), o.hist)
        assert np.array_equal(g.solution(), o.x)
print("ok")
