"""Exact-dot flush statistics per iteration (a -DFLUSH_STATS build:
tools/build_flags.sh fstats -DFLUSH_STATS):

    MINIFE_LIB_PATH=paper_1505_08023_b200/lib/alt_fstats.so python tools/flush_stats.py N K1 K2 ..

For the SYM SpMV (pAp) and K6 (rr): warp flush calls, those with a nonzero value, lanes sent to
the slow path (value > 128 bits below the warp's largest), mean warp sums per nonzero call.
Counts of iteration K = counts(solve of K iterations) - counts(solve of K - 1)."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1505_08023_b200 as M  # noqa: E402

n = int(sys.argv[1])
ks = [int(v) for v in sys.argv[2:]] or [2, 51, 181]
lib = M._lib
g = M.Minife(n, n, n, options={"small_solver": 0})
g.assemble()
buf = (ctypes.c_ulonglong * 8)()


def counts(K):
    assert lib.minife_dbg_flush_stats(buf, 1) == 0
    g.cg_solve(K, 0.0)
    assert lib.minife_dbg_flush_stats(buf, 0) == 0
    return [int(v) for v in buf]


for K in ks:
    a, b = counts(K), counts(K - 1)
    d = [x - y for x, y in zip(a, b)]
    out = {"n": n, "iteration": K}
    for kk, name in ((0, "spmv"), (1, "k6")):
        nzc, slow, sums, calls = d[4 * kk:4 * kk + 4]
        out[name] = {"calls": calls, "nonzero_calls": nzc, "slow_lanes": slow,
                     "mean_sums": round(sums / nzc, 2) if nzc else 0.0}
    print(json.dumps(out), flush=True)
