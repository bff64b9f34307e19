"""Block-row partition of a large GEMM across ranks (north star:
"partitioned across the 8xB200 box by block-rows of A and C, which needs no
communication beyond an optional NCCL all-gather of C").

Rank p owns rows [p*M/P, (p+1)*M/P) of A and C; B is replicated; each rank
plans its own LCMA on (M/P, N, K).  The only collective is the optional
all-gather of the contiguous C row blocks, which *is* row-major C.
"""
from __future__ import annotations


def row_block(M: int, world: int, rank: int):
    """[r0, r1) rows of rank `rank`; blocks differ by at most one row."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, extra = divmod(M, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def allgather_rows(C_local, M: int, group=None):
    """All-gather the equal-size row blocks of C (torch.distributed, NCCL over
    NVLink on GPUs, gloo on CPU).  Requires M divisible by the world size."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if M % world:
        raise ValueError("all-gather of C needs M divisible by the world size")
    out = torch.empty((M,) + tuple(C_local.shape[1:]), dtype=C_local.dtype, device=C_local.device)
    dist.all_gather_into_tensor(out, C_local.contiguous(), group=group)
    return out


def band_rows(rows: int, n_bands: int, align: int = 256):
    """Split [0, rows) into <= n_bands contiguous bands of `align`-multiple
    height (the last band takes the remainder)."""
    if rows < 1 or n_bands < 1:
        raise ValueError("rows and n_bands must be >= 1")
    per = -(-rows // n_bands)                  # ceil(rows / n_bands)
    step = -(-per // align) * align            # rounded up to the alignment
    out, r = [], 0
    while r < rows:
        out.append((r, min(rows, r + step)))
        r += step
    return out


def gemm_allgather_overlapped(compute_band, C_local, C_full, bands, group=None, comm_stream=None):
    """All-gather of C overlapped with the compute of later row bands
    (SURVEY 8(f) item 3).

    compute_band(r0, r1) enqueues rows [r0, r1) of this rank's block C_local on
    the current stream.  After each band the same band of every rank is
    gathered into C_full (rank q's rows start at q * C_local.shape[0]) on
    `comm_stream` (a side CUDA stream; None on CPU), so band c's transfer
    overlaps band c+1's compute.  Returns after the current stream has been
    ordered after every gather."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    ml = C_local.shape[0]
    if C_full.shape[0] != ml * world:
        raise ValueError("C_full must hold world * rows_per_rank rows")
    cuda = C_local.is_cuda
    works = []
    for r0, r1 in bands:
        compute_band(r0, r1)
        outs = [C_full[q * ml + r0:q * ml + r1] for q in range(world)]
        if cuda:
            ev = torch.cuda.Event()
            ev.record()
            with torch.cuda.stream(comm_stream):
                comm_stream.wait_event(ev)
                works.append(dist.all_gather(outs, C_local[r0:r1], group=group, async_op=True))
        else:
            dist.all_gather(outs, C_local[r0:r1], group=group)
    for w in works:
        w.wait()
    if cuda:
        torch.cuda.current_stream().wait_stream(comm_stream)
