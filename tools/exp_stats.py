"""How often the SYM SpMV's exact pAp expansion needs its second tier or the shared-memory
atomics, per iteration (a -DEXP_STATS build: tools/build_flags.sh stats -DEXP_STATS):

    MINIFE_LIB_PATH=paper_1505_08023_b200/lib/alt_stats.so python tools/exp_stats.py N K1 K2 ...

Counts of iteration K = counts(solve of K iterations) - counts(solve of K - 1)."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1505_08023_b200 as M  # noqa: E402

n = int(sys.argv[1])
ks = [int(v) for v in sys.argv[2:]] or [2, 51, 121, 181, 200]
lib = M._lib
g = M.Minife(n, n, n)
g.assemble()
buf = (ctypes.c_ulonglong * 4)()


def counts(K):
    assert lib.minife_dbg_exp_stats(buf, 1) == 0
    g.cg_solve(K, 0.0)
    assert lib.minife_dbg_exp_stats(buf, 0) == 0
    return [int(v) for v in buf[:3]]


out = {"n": n, "per_iteration": {}}
for K in ks:
    a, b = counts(K), counts(K - 1)
    d = [x - y for x, y in zip(a, b)]
    out["per_iteration"][K] = {"adds": d[0], "second_tier": d[1], "spills": d[2],
                               "second_tier_frac": d[1] / max(d[0], 1),
                               "spill_frac": d[2] / max(d[0], 1)}
print(json.dumps(out))
