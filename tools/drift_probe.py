"""Is the late-solve SpMV slowdown the exact dot or the data?  (300^3 by default)

    python tools/drift_probe.py [N]

Times, on the same ctx: (1) the CG solve's own SpMV (with the exact pAp epilogue) at
iterations 51, 121, 181 (timing window, as bench.py); (2) the plain SpMV (no dot, same kernel
without the epilogue) on the solution vectors x_51, x_121, x_181 of those solves, on x = 0 and
on a dense uniform[-1,1] x -- 1000 back-to-back launches each (the power cap reaches its
steady state), CUDA events; SM clock sampled by nvidia-smi during each run."""
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1505_08023_b200 as M  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300


def clocks(stop, out):
    while not stop.is_set():
        try:
            v = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw",
                                "--format=csv,noheader,nounits", "-i", "0"],
                               capture_output=True, text=True, timeout=5).stdout.split(",")
            out.append((float(v[0]), float(v[1])))
        except Exception:
            pass
        time.sleep(0.05)


g = M.Minife(n, n, n)
g.assemble()
rows = g.get_info().rows
res = {"n": n, "dot_spmv_ms": {}, "plain_spmv_ms": {}, "plain_sm_mhz": {}, "plain_power_w": {}}
xs = {}
for k0 in (51, 121, 181):
    g.set_timing_window(k0, 8)
    g.cg_solve(200, 0.0)
    g.cg_solve(200, 0.0)
    s, _ = g.timing_window()
    res["dot_spmv_ms"][k0] = s
    g.cg_solve(k0, 0.0)
    xs[f"x_{k0}"] = g.solution().copy()
xs["zeros"] = np.zeros(rows)
xs["uniform"] = np.random.default_rng(7).uniform(-1.0, 1.0, rows)
stream = torch.cuda.Stream()
y = torch.empty(rows, dtype=torch.float64, device="cuda")
for name, xv in xs.items():
    x = torch.from_numpy(xv).cuda()
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for _ in range(50):
            g.spmv_device(x.data_ptr(), y.data_ptr(), stream.cuda_stream)
        stop, smp = threading.Event(), []
        th = threading.Thread(target=clocks, args=(stop, smp))
        th.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(1000):
            g.spmv_device(x.data_ptr(), y.data_ptr(), stream.cuda_stream)
        e1.record(stream)
    stream.synchronize()
    stop.set()
    th.join()
    res["plain_spmv_ms"][name] = e0.elapsed_time(e1) / 1000
    if smp:
        res["plain_sm_mhz"][name] = float(np.median([c for c, _ in smp]))
        res["plain_power_w"][name] = float(np.median([w for _, w in smp]))
    res.setdefault("nonzero_frac", {})[name] = float(np.count_nonzero(xv)) / rows
print(json.dumps(res))
