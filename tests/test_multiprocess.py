"""N>1 path on CPU: world_size-2 gloo processes split the product by block-rows
(paper_2605_06057_b200.shard), compute their shard with the oracle and
all-gather C; the gathered matrix equals the single-process product."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_06057_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, M, N, K, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from paper_2605_06057_b200 import inputs
    A, B = inputs.operands(M, N, K, 2, 61, 62, dist="int", lo=-2, hi=2)
    r0, r1 = shard.row_block(M, world, rank)
    Cl = O.lcma_i64(A[r0:r1].to(torch.int64).numpy(), B.to(torch.int64).numpy(), O.strassen()).C
    C = shard.allgather_rows(torch.from_numpy(Cl), M)
    if rank == 0:
        out.put(C.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_row_block_partition():
    for M in (1, 7, 8192, 32768):
        for P in (1, 2, 3, 8):
            blocks = [shard.row_block(M, P, p) for p in range(P)]
            assert blocks[0][0] == 0 and blocks[-1][1] == M
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard.row_block(10, 2, 2)


def test_gloo_world2_block_rows_allgather():
    M, N, K = 96, 64, 48
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, M, N, K, q)) for r in range(2)]
    for p in procs:
        p.start()
    C = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    import oracle as O
    from paper_2605_06057_b200 import inputs
    A, B = inputs.operands(M, N, K, 2, 61, 62, dist="int", lo=-2, hi=2)
    assert np.array_equal(C, O.gemm_i64(A.to(torch.int64).numpy(), B.to(torch.int64).numpy()))


def _worker_overlap(rank, world, port, M, N, K, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from paper_2605_06057_b200 import inputs
    A, B = inputs.operands(M, N, K, 2, 71, 72, dist="int", lo=-2, hi=2)
    r0, r1 = shard.row_block(M, world, rank)
    Ai, Bi = A[r0:r1].to(torch.int64).numpy(), B.to(torch.int64).numpy()
    C_local = torch.zeros(r1 - r0, N, dtype=torch.int64)
    C_full = torch.full((M, N), -999, dtype=torch.int64)
    order = []

    def compute_band(b0, b1):
        order.append((b0, b1))
        C_local[b0:b1] = torch.from_numpy(O.gemm_i64(Ai[b0:b1], Bi))

    bands = shard.band_rows(r1 - r0, 3, align=8)
    shard.gemm_allgather_overlapped(compute_band, C_local, C_full, bands)
    assert order == bands
    if rank == 0:
        out.put(C_full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_band_rows():
    assert shard.band_rows(4096, 4) == [(0, 1024), (1024, 2048), (2048, 3072), (3072, 4096)]
    assert shard.band_rows(1000, 3, align=256) == [(0, 512), (512, 1000)]
    assert shard.band_rows(100, 8, align=256) == [(0, 100)]
    with pytest.raises(ValueError):
        shard.band_rows(0, 2)


def test_gloo_world2_overlapped_band_allgather():
    # cfg5's all-gather of C in row bands: every band of every
    # rank lands at its row offset; the result equals the single-process GEMM
    M, N, K = 96, 40, 24
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_overlap, args=(r, 2, port, M, N, K, q)) for r in range(2)]
    for p in procs:
        p.start()
    C = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    import oracle as O
    from paper_2605_06057_b200 import inputs
    A, B = inputs.operands(M, N, K, 2, 71, 72, dist="int", lo=-2, hi=2)
    assert np.array_equal(C, O.gemm_i64(A.to(torch.int64).numpy(), B.to(torch.int64).numpy()))
