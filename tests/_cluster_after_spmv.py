"""Subprocess helper for test_gpu_parity: the single-launch cluster solver (option small_solver = 2) run
right after large SpMV launches that leave their data in every SM's shared memory, repeatedly,
each solve compared with the oracle bit for bit (the solver must not read shared memory it has
not written: a fresh-process race of this kind was fixed, profiles/r01/session3 §5).  Prints
'ok' on success."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import paper_1505_08023_b200 as M  # noqa: E402

n = (23, 17, 9)
s = O.assemble(*n)
o = O.cg(s.row_ptr, s.col, s.val, s.b, 200, 0.0)
big = M.Minife(60, 60, 60, fmt=M.FMT_SYM)
big.assemble()
rows = big.io_rows
x = torch.rand(rows + 64, dtype=torch.float64, device="cuda") * 1e300   # loud garbage
y = torch.empty_like(x)
stream = torch.cuda.current_stream().cuda_stream
with M.Minife(*n, fmt=M.FMT_SYM, options={"small_solver": 2}) as g:
    g.assemble()
    for rep in range(20):
        for _ in range(3):
            big.spmv_device(x.data_ptr(), y.data_ptr(), stream)
        torch.cuda.synchronize()
        r = g.cg_solve(200, 0.0)
        assert r.iterations == 200, (rep, r.iterations)
        assert np.array_equal(g.history(), o.hist), rep
        assert np.array_equal(g.solution(), o.x), rep
big.close()
print("ok")
