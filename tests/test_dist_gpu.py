"""The row-sharded driver on the CUDA path under a real 2-rank process group: two
processes share the one GPU of a gpurun box (gloo carries the broadcast of B -- NCCL
needs one device per rank), each runs ``dgemm_rowsharded`` with its default compute
(``paper_2603_10634_b200.dgemm`` -> oz2_dgemm_ex, the same kernels as bench.py), whole or
in column panels overlapped with the broadcast.  Every shard, and every panel of it, must
equal the oracle on the same sub-problem bit for bit (block-local exponents, R13/Q20)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

M, K, NCOL, NMOD = 600, 520, 700, 13


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, panels, mode, out_q):
    try:
        import torch
        import torch.distributed as dist
        import paper_2603_10634_b200 as P
        from synth import gen_host
        from paper_2603_10634_b200.dist import dgemm_rowsharded, row_block

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        A = gen_host(M, K, "phi", phi=1.0, seed=31)
        r0, r1 = row_block(M, rank, world)
        A_local = torch.from_numpy(np.asfortranarray(A[r0:r1])).cuda()
        A_local = A_local.t().contiguous().t()                     # column-major
        if rank == 0:
            Bh = gen_host(K, NCOL, "phi", phi=1.0, seed=32)
            B = torch.from_numpy(np.ascontiguousarray(Bh.T)).cuda().t()   # column-major
        else:
            B = torch.zeros((NCOL, K), dtype=torch.float64, device="cuda").t()
        assert P.oz2_set_mode(mode) == 0
        C = dgemm_rowsharded(A_local, B, num_moduli=NMOD, panels=panels)
        torch.cuda.synchronize()
        out_q.put((rank, r0, r1, C.cpu().numpy(), B.cpu().numpy(), None))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:          # report instead of hanging the parent
        import traceback
        out_q.put((rank, 0, 0, None, None, traceback.format_exc()))


@pytest.mark.parametrize("panels,mode", [(1, "accurate"), (3, "accurate"), (3, "fast")])
def test_rowsharded_cuda_two_ranks(panels, mode):
    import torch
    import torch.multiprocessing as mp
    from oracle import scheme
    from synth import gen_host
    from paper_2603_10634_b200.dist import col_panels

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, panels, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for r in results:
        assert r[5] is None, r[5]
    assert all(p.exitcode == 0 for p in procs)
    A = gen_host(M, K, "phi", phi=1.0, seed=31)
    B = gen_host(K, NCOL, "phi", phi=1.0, seed=32)
    exact = A @ B
    pans = col_panels(NCOL, panels)
    for rank, r0, r1, C_local, Bseen, _ in results:
        assert np.array_equal(Bseen, B)
        for j0, j1 in pans:
            want = scheme.dgemm(A[r0:r1], B[:, j0:j1], NMOD, mode=mode).C
            assert np.array_equal(C_local[:, j0:j1], want), (rank, j0)
        rel = np.linalg.norm(C_local - exact[r0:r1]) / np.linalg.norm(exact[r0:r1])
        assert rel < 1e-15
