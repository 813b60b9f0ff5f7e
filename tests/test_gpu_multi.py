"""Multi-GPU parity (needs >= 2 GPUs; skipped on one): the real N > 1 code paths -- RANK ctxs
under torchrun (CUDA-IPC device comm and the NCCL transport, graph and eager) and one MULTI
ctx driving every GPU -- bitwise the oracle.  On one GPU the same kernels and protocols run as
VIRTUAL parts (test_gpu_parity.py: TRANSPORT_DEVICE, TRANSPORT_WIRE)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.gpu2]

torch = pytest.importorskip("torch")
M = pytest.importorskip("paper_1505_08023_b200")
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
need2 = pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
HERE = os.path.dirname(os.path.abspath(__file__))


@need2
@pytest.mark.parametrize("devcomm,graph", [(-1, 1), (-1, 0), (0, 1), (0, 0)])
@pytest.mark.parametrize("n", [(23, 17, 9), (40, 40, 40)])
def test_rank_mode_torchrun(n, devcomm, graph):
    world = min(NGPU, 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", "--master-port=29571",
           os.path.join(HERE, "_rank_parity.py"), *map(str, n), str(devcomm), str(graph)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=HERE)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]


@need2
@pytest.mark.parametrize("devcomm", [-1, 0])
@pytest.mark.parametrize("n", [(23, 17, 9), (40, 40, 40)])
def test_multi_mode(n, devcomm):
    import oracle as O
    s = O.assemble(*n)
    with M.Minife(*n, ngpu=min(NGPU, 4), options={"device_comm": devcomm}) as g:
        g.assemble()
        rp, col, val = g.export_csr()
        assert np.array_equal(col, s.col) and np.array_equal(val, s.val)
        for iters, tol in ((200, 0.0), (200, 1e-8)):
            r = g.cg_solve(iters, tol)
            o = O.cg(s.row_ptr, s.col, s.val, s.b, iters, tol)
            assert (r.status, r.iterations, r.converged) == (o.status, o.iters, o.converged)
            assert np.array_equal(g.history(), o.hist)
            assert np.array_equal(g.solution(), o.x)
