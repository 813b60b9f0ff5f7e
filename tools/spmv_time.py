"""Time minife_spmv_device (y = A x, no dot) in a loop: per-launch ms via CUDA events.

    python tools/spmv_time.py N FORMAT [reps]
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1505_08023_b200 as M  # noqa: E402

n = int(sys.argv[1])
fmt = {"seg": M.FMT_SEG, "sym": M.FMT_SYM, "crs": M.FMT_CRS}[sys.argv[2]]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
g = M.Minife(n, n, n, fmt=fmt)
g.assemble()
rows = g.io_rows
x = torch.rand(rows + 64, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(5):
        g.spmv_device(x.data_ptr(), y.data_ptr(), s.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        g.spmv_device(x.data_ptr(), y.data_ptr(), s.cuda_stream)
    e1.record(s)
    s.synchronize()
print(json.dumps({"n": n, "fmt": sys.argv[2], "ms": e0.elapsed_time(e1) / reps,
                  "env": {k: v for k, v in os.environ.items() if k.startswith("MINIFE_S")}}))
