"""A/B of the device assembly (minife_get_timings) for the library at MINIFE_LIB_PATH.

    MINIFE_LIB_PATH=... python tools/ab_asm.py N [FMT]
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1505_08023_b200 as M  # noqa: E402

n = int(sys.argv[1])
fmt = {"sym": M.FMT_SYM, "seg": M.FMT_SEG}[sys.argv[2] if len(sys.argv) > 2 else "sym"]
g = M.Minife(n, n, n, fmt=fmt)
t = []
for i in range(12):
    g.assemble()
    if i >= 2:
        t.append(g.timings()[0])
print(json.dumps({"lib": os.path.basename(M.LIB_PATH), "n": n, "median_ms": statistics.median(t),
                  "min_ms": min(t)}), flush=True)
