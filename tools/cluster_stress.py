"""Repeat the single-launch cluster solver (MINIFE_SMALL=2) against the oracle many times in one
process; report every run that is not bit-identical (race hunting).

    MINIFE_SMALL=2 python tools/cluster_stress.py NX NY NZ FMT REPS
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import paper_1505_08023_b200 as M  # noqa: E402

n = tuple(int(v) for v in sys.argv[1:4])
fmt = {"seg": M.FMT_SEG, "sym": M.FMT_SYM}[sys.argv[4]]
reps = int(sys.argv[5])
s = O.assemble(*n)
o = O.cg(s.row_ptr, s.col, s.val, s.b, 200, 0.0)
bad = []
with M.Minife(*n, fmt=fmt) as g:
    g.assemble()
    for rep in range(reps):
        r = g.cg_solve(200, 0.0)
        h = g.history()
        x = g.solution()
        if not (np.array_equal(h, o.hist) and np.array_equal(x, o.x)):
            d = np.nonzero(h != o.hist)[0]
            bad.append({"rep": rep, "first_hist_diff": int(d[0]) if d.size else None,
                        "x_diffs": int(np.count_nonzero(x != o.x))})
print(json.dumps({"n": n, "fmt": sys.argv[4], "reps": reps, "bad": bad[:20], "nbad": len(bad)}))
