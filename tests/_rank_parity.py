"""torchrun helper for test_gpu_multi: every rank builds its RANK ctx (RCB part), solves, and
rank 0 compares the gathered owned rows of x and the history with the oracle bit for bit.
Usage: torchrun --nproc-per-node N tests/_rank_parity.py NX NY NZ DEVICE_COMM GRAPH
Prints 'ok' on rank 0 on success."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1505_08023_b200 as M  # noqa: E402

nx, ny, nz, devcomm, graph = (int(v) for v in sys.argv[1:6])
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("gloo")
obj = [M.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
results = []
with M.Minife(nx, ny, nz, rank=(rank, world, local, obj[0]),
              options={"device_comm": devcomm, "graph": graph}) as g:
    g.assemble()
    for iters, tol in ((200, 0.0), (200, 1e-8)):
        r = g.cg_solve(iters, tol)
        results.append((r.status, r.iterations, r.converged, g.history(), g.owned_ids(),
                        g.solution()))
gathered = [None] * world
dist.all_gather_object(gathered, results)
if rank == 0:
    import oracle as O
    s = O.assemble(nx, ny, nz)
    for j, (iters, tol) in enumerate(((200, 0.0), (200, 1e-8))):
        o = O.cg(s.row_ptr, s.col, s.val, s.b, iters, tol)
        x = np.full(s.rows, np.nan)
        for res in gathered:
            st, it, conv, h, ids, xl = res[j]
            assert (st, it, conv) == (o.status, o.iters, o.converged)
            assert np.array_equal(h, o.hist)
            x[ids] = xl
        assert np.array_equal(x, o.x)
    print("ok", flush=True)
dist.destroy_process_group()
