"""World-size-2 (and 4) CPU run of the N>1 host path over torch.distributed/gloo.

Each process is one rank: it takes its RCB plan from the product library (host-only
minife_plan_lists), exchanges its halo with point-to-point send/recv exactly as the NCCL path
does (pack send lists in neighbor order, receive into the contiguous per-owner external
blocks), runs the local SpMV on its owned rows with the oracle's row values, and rank 0
gathers y.  The gathered y must equal the oracle's global SpMV bit for bit, and the
received externals must equal the owners' values.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, mesh, q):
    import sys
    sys.path.insert(0, ROOT)
    import minife_inputs
    import oracle as O
    import paper_1505_08023_b200 as M

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L = M.plan_lists(*mesh, world, rank)
        info = L["info"]
        NX, NY = mesh[0] + 1, mesh[1] + 1
        lo, hi = list(info.own[:3]), list(info.own[3:])
        owned = np.array([ix + NX * (iy + NY * iz) for iz in range(lo[2], hi[2] + 1)
                          for iy in range(lo[1], hi[1] + 1) for ix in range(lo[0], hi[0] + 1)],
                         dtype=np.int64)
        # this rank's owned values of the seeded global vector (counter-based generator)
        x_owned = minife_inputs.uniform_pm1(0, 12345, idx=owned.astype(np.uint64))
        x_local = np.concatenate([x_owned, np.zeros(info.externals)])
        # halo exchange: pack per neighbor, isend/irecv into the contiguous external blocks
        send_off = np.concatenate([[0], np.cumsum(L["send_cnt"])]).astype(int)
        recv_off = np.concatenate([[0], np.cumsum(L["recv_cnt"])]).astype(int)
        reqs, bufs = [], []
        for k, nb in enumerate(L["nbr"]):
            buf = torch.from_numpy(x_owned[L["send_idx"][send_off[k]:send_off[k + 1]]].copy())
            bufs.append(buf)
            reqs.append(dist.isend(buf, int(nb)))
        recvs = []
        for k, nb in enumerate(L["nbr"]):
            rb = torch.zeros(int(L["recv_cnt"][k]), dtype=torch.float64)
            recvs.append((k, rb))
            reqs.append(dist.irecv(rb, int(nb)))
        for r in reqs:
            r.wait()
        for k, rb in recvs:
            x_local[info.rows + recv_off[k]:info.rows + recv_off[k + 1]] = rb.numpy()
        expect_ext = minife_inputs.uniform_pm1(0, 12345, idx=L["ext_gids"].astype(np.uint64))
        assert np.array_equal(x_local[info.rows:], expect_ext)
        # local SpMV with local column ids (owned box index / external slot)
        slot = {int(g): i for i, g in enumerate(np.concatenate([owned, L["ext_gids"]]))}
        y = np.zeros(info.rows)
        for i, gid in enumerate(owned):
            cols, vals, _ = O.row(*mesh, int(gid))
            lc = np.array([slot[int(c)] for c in cols], dtype=np.int64)
            y[i] = O.spmv(np.array([0, lc.size]), lc, vals, x_local)[0]
        # gather to rank 0 (sizes differ per rank: pad to the max)
        n_max = torch.tensor([info.rows])
        dist.all_reduce(n_max, op=dist.ReduceOp.MAX)
        pad = np.zeros(int(n_max), dtype=np.float64)
        pad[:info.rows] = y
        gid_pad = np.full(int(n_max), -1, dtype=np.int64)
        gid_pad[:info.rows] = owned
        ys = [torch.zeros(int(n_max), dtype=torch.float64) for _ in range(world)]
        gs = [torch.zeros(int(n_max), dtype=torch.int64) for _ in range(world)]
        dist.all_gather(ys, torch.from_numpy(pad))
        dist.all_gather(gs, torch.from_numpy(gid_pad))
        if rank == 0:
            rows = NX * NY * (mesh[2] + 1)
            yg = np.full(rows, np.nan)
            for yr, gr in zip(ys, gs):
                m = gr.numpy() >= 0
                yg[gr.numpy()[m]] = yr.numpy()[m]
            s = O.assemble(*mesh)
            x = minife_inputs.uniform_pm1(rows, 12345)
            yo = O.spmv(s.row_ptr, s.col, s.val, x)
            q.put(bool(np.array_equal(yg, yo)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mesh", [(2, (9, 8, 7)), (4, (8, 7, 6)), (3, (7, 7, 5))])
def test_distributed_halo_spmv_gloo(world, mesh):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mesh, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=10) is True
