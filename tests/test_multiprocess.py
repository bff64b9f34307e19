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


def _worker_banded(rank, world, port, M, N, K, bands, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from paper_2605_06057_b200 import inputs
    A, B = inputs.operands(M, N, K, 2, 71, 72, dist="int", lo=-2, hi=2)
    Bi = B.to(torch.int64).numpy()
    rows = shard.banded_rows(M, world, rank, bands)
    h = shard.band_height(M, world, bands)
    C_local = torch.zeros(bands * h, N, dtype=torch.int64)
    C_full = torch.full((M, N), -999, dtype=torch.int64)
    order = []

    def compute_band(c):
        # this rank's band c = global rows rows[c] (the oracle stands in for
        # the GPU kernel: the test covers partition, order and placement)
        order.append(c)
        r0, r1 = rows[c]
        C_local[c * h:(c + 1) * h] = torch.from_numpy(O.gemm_i64(A[r0:r1].to(torch.int64).numpy(), Bi))

    shard.gemm_allgather_banded(compute_band, C_local, C_full, bands)
    assert order == list(range(bands))
    if rank == 0:
        out.put(C_full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_banded_partition():
    # every row owned exactly once; band c of all ranks is one contiguous block
    for (M, P, bands) in [(96, 2, 3), (32768, 8, 2), (32768, 2, 4), (64, 1, 4)]:
        h = shard.band_height(M, P, bands)
        owned = sorted(r for p in range(P) for r0, r1 in shard.banded_rows(M, P, p, bands) for r in range(r0, r1))
        assert owned == list(range(M))
        for c in range(bands):
            starts = sorted(shard.banded_rows(M, P, p, bands)[c][0] for p in range(P))
            assert starts == [c * P * h + p * h for p in range(P)]
    with pytest.raises(ValueError):
        shard.band_height(100, 3, 2)


@pytest.mark.parametrize("bands", [1, 3])
def test_gloo_world2_banded_overlapped_allgather(bands):
    # cfg5's all-gather of C overlapped band by band with
    # all_gather_into_tensor straight into C: equals the single-process GEMM
    M, N, K = 96, 40, 24
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_banded, args=(r, 2, port, M, N, K, bands, q)) for r in range(2)]
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
