"""Per-iteration time inside the timed 300^3 solve at several positions of the timing window
(minife_set_timing_window), with nvidia-smi SM clock samples: does the iteration time drift
over a solve, and does it follow the clock?

    python tools/tw_drift.py [N]
"""
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1505_08023_b200 as M  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
g = M.Minife(n, n, n)
g.assemble()
for _ in range(3):
    g.cg_solve(200, 0.0)
clk = []
stop = False


def sample():
    while not stop:
        try:
            o = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw",
                                "--format=csv,noheader,nounits"], capture_output=True,
                               text=True, timeout=5).stdout.strip()
            clk.append(o)
        except Exception:
            pass
        time.sleep(0.05)


th = threading.Thread(target=sample)
th.start()
out = {}
for k0 in (2, 25, 51, 101, 151, 191):
    g.set_timing_window(k0, 8)
    r = []
    for _ in range(3):
        res = g.cg_solve(200, 0.0)
        s, it = g.timing_window()
        r.append((round(s, 4), round(it, 4), round(res.seconds * 1e3 / 200, 4)))
    out[k0] = r
stop = True
th.join()
print(json.dumps({"n": n, "window_spmv_iter_avg_ms": out, "clock_power_samples": clk[::4]}))
