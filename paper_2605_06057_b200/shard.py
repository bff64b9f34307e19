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
