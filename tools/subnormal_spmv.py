import json, os, sys
import torch
sys.path.insert(0, os.getcwd())
import paper_1505_08023_b200 as M
n = 300
g = M.Minife(n, n, n, fmt=M.FMT_SYM); g.assemble()
rows = g.io_rows
s = torch.cuda.Stream()
out = {}
for name, scale in (("normal", 1.0), ("subnormal", 1e-310), ("mixed_1pct", None), ("tiny_1e-200", 1e-200)):
    x = torch.rand(rows + 64, dtype=torch.float64, device="cuda")
    if scale is None:
        m = torch.rand(rows + 64, device="cuda") < 0.1
        x = torch.where(m, x * 1e-310, x)
    else:
        x = x * scale
    y = torch.empty_like(x)
    with torch.cuda.stream(s):
        for _ in range(5):
            g.spmv_device(x.data_ptr(), y.data_ptr(), s.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(20):
            g.spmv_device(x.data_ptr(), y.data_ptr(), s.cuda_stream)
        e1.record(s)
        s.synchronize()
    out[name] = round(e0.elapsed_time(e1) / 20, 4)
print(json.dumps(out))
