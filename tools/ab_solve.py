"""A/B timing of whole 200-iteration solves (device time) for the library at MINIFE_LIB_PATH.

    MINIFE_LIB_PATH=... python tools/ab_solve.py NX NY NZ [REPS] [--opt NAME=VALUE ...]
Prints one JSON line: median / min solve ms over REPS timed solves after 2 warm-up solves,
plus the SpMV window at iterations 51..58 and 181..188."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1505_08023_b200 as M  # noqa: E402

nx, ny, nz = (int(v) for v in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 and not sys.argv[4].startswith("--") else 5
opts = {}
for i, a in enumerate(sys.argv):
    if a == "--opt":
        k, v = sys.argv[i + 1].split("=")
        opts[k] = int(v)
g = M.Minife(nx, ny, nz, options=opts)
g.assemble()
out = {"lib": os.path.basename(M.LIB_PATH), "mesh": [nx, ny, nz], "options": opts}
for k0 in (51, 181):
    g.set_timing_window(k0, 8)
    for _ in range(2):
        g.cg_solve(200, 0.0)
    t = [g.cg_solve(200, 0.0).seconds * 1e3 for _ in range(reps)]
    try:
        s, it = g.timing_window()
    except M.MinifeError:                  # single-launch solvers: no window inside
        s = it = 0.0
    out[f"w{k0}"] = {"spmv_ms": s, "iter_ms": it}
    out.setdefault("solve_ms", []).extend(t)
out["median_ms"] = statistics.median(out["solve_ms"])
out["min_ms"] = min(out["solve_ms"])
print(json.dumps(out), flush=True)
