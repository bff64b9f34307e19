"""Block-row partition of a large GEMM across ranks (north star:
"partitioned across the 8xB200 box by block-rows of A and C, which needs no
communication beyond an optional NCCL all-gather of C").

Plain partition: rank p owns rows [p*M/P, (p+1)*M/P) of A and C; B is
replicated; each rank plans its own LCMA on (M/P, N, K).  The only collective
is the optional all-gather of the contiguous C row blocks, which *is*
row-major C.

Banded partition (the overlapped all-gather of SURVEY 8(f) 3): the rows are
cut into `bands` bands of P*h rows and rank p owns rows
[(c*P + p)*h, (c*P + p + 1)*h) of every band c.  Each rank computes its
bands one after the other; band c of all ranks is then one contiguous block
of C, so a single all_gather_into_tensor lands it in place (no staging copy,
no strided views) while band c+1 is being computed.
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


def band_height(M: int, world: int, bands: int) -> int:
    """Rows per (rank, band) of the banded partition; M must split evenly."""
    if world < 1 or bands < 1 or M < 1:
        raise ValueError("M, world and bands must be >= 1")
    if M % (world * bands):
        raise ValueError("banded partition needs M divisible by world * bands")
    return M // (world * bands)


def banded_rows(M: int, world: int, rank: int, bands: int):
    """Global row ranges [r0, r1) that rank `rank` owns, band by band."""
    if not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    h = band_height(M, world, bands)
    return [((c * world + rank) * h, (c * world + rank + 1) * h) for c in range(bands)]


def gemm_allgather_banded(compute_band, C_local, C_full, bands: int, group=None, comm_stream=None):
    """All-gather of C overlapped with the compute of later bands.

    C_local holds this rank's bands stacked ([bands * h, N], band c at rows
    c*h .. c*h+h); compute_band(c) enqueues band c into it on the current
    stream.  After band c, all_gather_into_tensor(C_full[c*P*h:(c+1)*P*h],
    C_local[c*h:(c+1)*h]) runs on `comm_stream` (a side CUDA stream; None on
    CPU), so band c's transfer overlaps band c+1's compute.  Returns after the
    current stream has been ordered after every gather."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if C_local.shape[0] % bands:
        raise ValueError("C_local rows must be bands * h")
    h = C_local.shape[0] // bands
    if C_full.shape[0] != h * bands * world:
        raise ValueError("C_full must hold world * bands * h rows")
    cuda = C_local.is_cuda
    works = []
    for c in range(bands):
        compute_band(c)
        dst = C_full[c * world * h:(c + 1) * world * h]
        src = C_local[c * h:(c + 1) * h]
        if cuda:
            ev = torch.cuda.Event()
            ev.record()
            with torch.cuda.stream(comm_stream):
                comm_stream.wait_event(ev)
                works.append(dist.all_gather_into_tensor(dst, src, group=group, async_op=True))
        else:
            dist.all_gather_into_tensor(dst, src, group=group)
    for w in works:
        w.wait()
    if cuda:
        torch.cuda.current_stream().wait_stream(comm_stream)
