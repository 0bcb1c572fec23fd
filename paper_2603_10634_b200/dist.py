"""Row-sharded multi-GPU driver (north_star: "C is partitioned by output row blocks
across the GPUs of one box, with B broadcast over NVLink via NCCL and no other
collective").

Every rank owns the row block [r0, r1) of A and C; B lives on ``src`` and is broadcast
(``torch.distributed.broadcast``: NCCL over NVLink 5 / NVSwitch on GPUs, gloo in the CPU
tests); each rank then runs the single-GPU pipeline (``oz2_dgemm``) on its block.  The
scaling exponent nu of a column becomes block-local (its maximum is taken over the rank's
rows only), so results are certified per shard but not bitwise equal to the unsharded
call (R13).

Overlap: with ``panels`` > 1 and a column-major B, B is broadcast in
column panels, all enqueued asynchronously up front (NCCL runs them in order on its own
stream), and the rank's call for panel p -- C[:, panel p] = A_local B[:, panel p], a
complete emulation of that block (prescale, bound GEMM, exponents, digits, residue GEMMs,
CRT) -- waits only for panel p's broadcast, so it runs while panels p+1.. are in flight.
Only the first panel's transfer is exposed.  Each panel is its own Ozaki-II call, so mu
becomes panel-local as well (its row maximum is over the panel's columns): every block is
certified on its own (the paper's blocked call; SPEC gemm_blocked S:371-379),
with at least the accuracy of the unpanelled call (a smaller maximum gives a larger mu).
A's conversion is repeated once per panel (m_local k elements, a few ms at config 5).
"""


def row_block(m: int, rank: int, world: int):
    """[r0, r1) rows of an m-row matrix owned by `rank` (balanced, contiguous)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(m, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def col_panels(n: int, panels: int, align: int = 256):
    """[(j0, j1)] column panels of an n-column matrix: `panels` near-equal pieces, all but
    the last a multiple of `align` (the residue GEMM's 256-column tile)."""
    if panels <= 1 or n <= align:
        return [(0, n)]
    w = -(-n // panels)
    w = -(-w // align) * align
    out, j = [], 0
    while j < n:
        out.append((j, min(n, j + w)))
        j += w
    return out


def dgemm_rowsharded(A_local, B, alpha=1.0, beta=0.0, C_local=None, num_moduli=13, src=0,
                     group=None, gemm_fn=None, panels=1):
    """C_local <- alpha A_local @ B + beta C_local on every rank after broadcasting B.

    ``B`` must be allocated with the full k x n shape on every rank (its contents matter
    only on ``src``).  ``gemm_fn(A, B, alpha, beta, C, num_moduli)`` defaults to the
    CUDA path (``paper_2603_10634_b200.dgemm``).  ``panels`` > 1 overlaps the broadcast of
    B's later column panels with the calls on the earlier ones (B column-major only;
    otherwise one broadcast).  Returns C_local."""
    import torch
    import torch.distributed as dist
    if gemm_fn is None:
        from .oz2 import dgemm
        gemm_fn = dgemm
    m, k = A_local.shape
    n = B.shape[1]
    if C_local is None:
        C_local = torch.empty((n, m), dtype=B.dtype, device=B.device).t()
        beta = 0.0
    multi = dist.is_initialized() and dist.get_world_size(group) > 1
    colmajor = B.stride(0) == 1 and B.stride(1) == k
    pans = col_panels(n, panels) if (multi and colmajor) else [(0, n)]
    if multi and len(pans) == 1:
        # collectives need contiguous storage: broadcast whichever of B / B^T is contiguous
        buf = B if B.is_contiguous() else B.t()
        if not buf.is_contiguous():
            raise ValueError("B must be row- or column-major contiguous")
        dist.broadcast(buf, src=src, group=group)
        gemm_fn(A_local, B, alpha=alpha, beta=beta, C=C_local, num_moduli=num_moduli)
        return C_local
    works = []
    if multi:
        for j0, j1 in pans:
            # a column range of a column-major B is one contiguous block (B^T rows j0..j1)
            works.append(dist.broadcast(B.t()[j0:j1], src=src, group=group, async_op=True))
    for p, (j0, j1) in enumerate(pans):
        if works:
            works[p].wait()          # NCCL: the current stream waits; the host does not
        gemm_fn(A_local, B[:, j0:j1], alpha=alpha, beta=beta, C=C_local[:, j0:j1],
                num_moduli=num_moduli)
    return C_local
