"""Is the SpMV's speed data-dependent through the power cap?  Back-to-back SpMV launches at
300^3 on x = 0, a 10 %-nonzero x and a dense random x, with nvidia-smi clock/power samples.

    python tools/power_spmv.py
"""
import json
import os
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1505_08023_b200 as M  # noqa: E402

g = M.Minife(300, 300, 300, fmt=M.FMT_SYM)
g.assemble()
rows = g.io_rows
s = torch.cuda.Stream()
out = {}
for name in ("zeros", "sparse10", "dense", "zeros", "dense"):
    if name == "zeros":
        x = torch.zeros(rows + 64, dtype=torch.float64, device="cuda")
    elif name == "sparse10":
        x = torch.rand(rows + 64, dtype=torch.float64, device="cuda")
        x[: int(rows * 0.9)] = 0.0
    else:
        x = torch.rand(rows + 64, dtype=torch.float64, device="cuda") * 2 - 1
    y = torch.empty_like(x)
    samples, stop = [], [False]

    def smp():
        while not stop[0]:
            r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw",
                                "--format=csv,noheader,nounits"], capture_output=True, text=True)
            samples.append(r.stdout.strip())
            time.sleep(0.1)
    with torch.cuda.stream(s):
        for _ in range(200):                         # ~0.2 s of warm-up at this load
            g.spmv_device(x.data_ptr(), y.data_ptr(), s.cuda_stream)
        s.synchronize()
        th = threading.Thread(target=smp)
        th.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(1000):
            g.spmv_device(x.data_ptr(), y.data_ptr(), s.cuda_stream)
        e1.record(s)
        s.synchronize()
        stop[0] = True
        th.join()
    out.setdefault(name, []).append({"ms": round(e0.elapsed_time(e1) / 1000, 4),
                                     "clock_power": samples[1::2][:6]})
print(json.dumps(out))
