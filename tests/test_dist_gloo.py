"""World-size-2 gloo test of the row-sharded driver on CPU: the partition, the broadcast
of B, and per-shard results equal to the oracle on the same sub-problem (the per-shard
compute is injected; on GPUs it is oz2_dgemm over NCCL)."""
import os
import socket

import numpy as np
import pytest

from paper_2603_10634_b200.dist import row_block


def test_row_block_partition():
    for m in [0, 1, 7, 64, 1000]:
        for world in [1, 2, 3, 8]:
            blocks = [row_block(m, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == m
            for (a0, a1), (b0, b1) in zip(blocks, blocks[1:]):
                assert a1 == b0
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    import torch
    import torch.distributed as dist
    from oracle import scheme
    from synth import gen_host
    from paper_2603_10634_b200.dist import dgemm_rowsharded, row_block

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, k, n, N = 24, 40, 10, 12
    A = gen_host(m, k, "phi", phi=1.0, seed=3, order="C")
    r0, r1 = row_block(m, rank, world)
    A_local = torch.from_numpy(A[r0:r1].copy())
    if rank == 0:
        B = torch.from_numpy(gen_host(k, n, "phi", phi=1.0, seed=4, order="C"))
    else:
        B = torch.zeros((k, n), dtype=torch.float64)     # filled by the broadcast

    def oracle_gemm(A_, B_, alpha, beta, C, num_moduli):
        return torch.from_numpy(scheme.dgemm(A_.numpy(), B_.numpy(), num_moduli).C)

    C_local = dgemm_rowsharded(A_local, B, num_moduli=N, gemm_fn=oracle_gemm)
    out_q.put((rank, r0, r1, C_local.numpy(), B.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_rowsharded_gloo_world2():
    import torch.multiprocessing as mp
    from oracle import scheme
    from synth import gen_host

    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    A = gen_host(24, 40, "phi", phi=1.0, seed=3, order="C")
    B = gen_host(40, 10, "phi", phi=1.0, seed=4, order="C")
    full = scheme.dgemm(A, B, 12).C
    exact = A @ B
    for rank, r0, r1, C_local, Bseen in results:
        assert np.array_equal(Bseen, B)                       # broadcast delivered B
        want = scheme.dgemm(A[r0:r1], B, 12).C                # per-shard oracle
        assert np.array_equal(C_local, want)
        # same accuracy class as the unsharded call (block-local nu, R13)
        rel = np.linalg.norm(C_local - exact[r0:r1]) / np.linalg.norm(exact[r0:r1])
        assert rel < 1e-14
    assert sorted(r[0] for r in results) == [0, 1]
    assert np.allclose(np.vstack([r[3] for r in sorted(results)]), full, rtol=1e-13, atol=0)
