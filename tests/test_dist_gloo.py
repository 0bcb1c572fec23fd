"""World-size-2 gloo tests of the row-sharded driver on CPU: the partition, the broadcast
of B (whole, or in column panels overlapped with the per-panel calls), and per-shard /
per-panel results equal to the oracle on the same sub-problem (the per-block compute is
injected here; on GPUs it is oz2_dgemm over NCCL -- tests/test_dist_gpu.py runs the CUDA
path under a 2-rank process group on one device)."""
import os
import socket

import numpy as np
import pytest

from paper_2603_10634_b200.dist import col_panels, row_block


def test_row_block_partition():
    for m in [0, 1, 7, 64, 1000]:
        for world in [1, 2, 3, 8]:
            blocks = [row_block(m, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == m
            for (a0, a1), (b0, b1) in zip(blocks, blocks[1:]):
                assert a1 == b0
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1


def test_col_panels():
    assert col_panels(1000, 1) == [(0, 1000)]
    assert col_panels(200, 4) == [(0, 200)]
    for n in [257, 1000, 4096, 32768, 5000]:
        for p in [2, 3, 4, 8]:
            pans = col_panels(n, p)
            assert pans[0][0] == 0 and pans[-1][1] == n and len(pans) <= p
            assert all(b == c for (_, b), (c, _) in zip(pans, pans[1:]))
            assert all((b - a) % 256 == 0 for a, b in pans[:-1])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


M, K, NCOL, NMOD = 24, 40, 600, 12


def _worker(rank, world, port, panels, out_q):
    import torch
    import torch.distributed as dist
    from oracle import scheme
    from synth import gen_host
    from paper_2603_10634_b200.dist import dgemm_rowsharded, row_block

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A = gen_host(M, K, "phi", phi=1.0, seed=3, order="C")
    r0, r1 = row_block(M, rank, world)
    A_local = torch.from_numpy(A[r0:r1].copy())
    # column-major B (the layout the panelled broadcast needs)
    if rank == 0:
        B = torch.from_numpy(np.ascontiguousarray(gen_host(K, NCOL, "phi", phi=1.0, seed=4).T)).t()
    else:
        B = torch.zeros((NCOL, K), dtype=torch.float64).t()     # filled by the broadcast
    calls = []

    def oracle_gemm(A_, B_, alpha, beta, C, num_moduli):
        calls.append(B_.shape[1])
        C.copy_(torch.from_numpy(scheme.dgemm(A_.numpy(), B_.numpy(), num_moduli).C))
        return C

    C_local = dgemm_rowsharded(A_local, B, num_moduli=NMOD, gemm_fn=oracle_gemm, panels=panels)
    out_q.put((rank, r0, r1, C_local.numpy().copy(), B.numpy().copy(), calls))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("panels", [1, 3])
def test_rowsharded_gloo_world2(panels):
    import torch.multiprocessing as mp
    from oracle import scheme
    from synth import gen_host

    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, panels, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    A = gen_host(M, K, "phi", phi=1.0, seed=3, order="C")
    B = gen_host(K, NCOL, "phi", phi=1.0, seed=4)
    exact = A @ B
    pans = col_panels(NCOL, panels)
    for rank, r0, r1, C_local, Bseen, calls in results:
        assert np.array_equal(Bseen, B)                       # broadcast delivered B
        assert calls == [b - a for a, b in pans]              # one call per panel
        for j0, j1 in pans:                                   # per-block oracle (R13, Q20)
            want = scheme.dgemm(A[r0:r1], B[:, j0:j1], NMOD).C
            assert np.array_equal(C_local[:, j0:j1], want)
        rel = np.linalg.norm(C_local - exact[r0:r1]) / np.linalg.norm(exact[r0:r1])
        assert rel < 1e-14
    assert sorted(r[0] for r in results) == [0, 1]
