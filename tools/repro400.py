"""Repro helper: one 400^3 solve in the bench's configuration with toggles.
    python tools/repro400.py N STREAM(0/1) TW(0/1) BAND(-1/0) [FMT]"""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1505_08023_b200 as M
n = int(sys.argv[1]); use_stream, tw, band = (int(v) for v in sys.argv[2:5])
g = M.Minife(n, n, n, options={"band_rows": band})
g.set_format(M.FMT_SYM)
g.set_scheme(M.SCHEME_3K)
s = torch.cuda.Stream()
if use_stream:
    g.set_stream(s.cuda_stream)
if tw:
    g.set_timing_window(51, 8)
with torch.cuda.stream(s):
    for i in range(2):
        g.assemble()
        r = g.cg_solve(200, 0.0)
        print("solve", i, r.status, r.iterations, flush=True)
print("ok", flush=True)
