"""Row-sharded multi-GPU driver (north_star: "C is partitioned by output row blocks
across the GPUs of one box, with B broadcast over NVLink via NCCL and no other
collective").

Every rank owns the row block [r0, r1) of A and C; B lives on ``src`` and is broadcast
(``torch.distributed.broadcast``: NCCL over NVLink 5 / NVSwitch on GPUs, gloo in the CPU
tests); each rank then runs the single-GPU pipeline (``oz2_dgemm``) on its block.  The
scaling exponent nu of a column becomes block-local (its maximum is taken over the rank's
rows only), so results are certified per shard but not bitwise equal to the unsharded
call (R13).
"""


def row_block(m: int, rank: int, world: int):
    """[r0, r1) rows of an m-row matrix owned by `rank` (balanced, contiguous)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(m, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def dgemm_rowsharded(A_local, B, alpha=1.0, beta=0.0, C_local=None, num_moduli=13, src=0,
                     group=None, gemm_fn=None):
    """C_local <- alpha A_local @ B + beta C_local on every rank after broadcasting B.

    ``B`` must be allocated with the full k x n shape on every rank (its contents matter
    only on ``src``).  ``gemm_fn(A, B, alpha, beta, C, num_moduli)`` defaults to the
    CUDA path (``paper_2603_10634_b200.dgemm``)."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        # collectives need contiguous storage: broadcast whichever of B / B^T is contiguous
        buf = B if B.is_contiguous() else B.t()
        if not buf.is_contiguous():
            raise ValueError("B must be row- or column-major contiguous")
        dist.broadcast(buf, src=src, group=group)
    if gemm_fn is None:
        from .oz2 import dgemm
        gemm_fn = dgemm
    return gemm_fn(A_local, B, alpha=alpha, beta=beta, C=C_local, num_moduli=num_moduli)
