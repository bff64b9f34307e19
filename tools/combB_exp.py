"""Combine-B bandwidth at several shapes (precombine_b alone), vs a plain copy."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs


def t(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for (M, N, K) in ((8192, 14336, 4096), (32768, 28672, 8192), (8192, 28672, 8192), (8192, 28672 + 256, 8192),
                  (8192, 16384, 8192), (8192, 32768, 8192)):
    for bl in (0, 1):
        A, B = inputs.operands(256, N, K, L.BF16, 1, 2, b_layout=bl)
        B = B.cuda()
        for algo in ("strassen",):
            p = L.Plan(M, N, K, dtype=L.BF16, algo=algo, b_layout=bl)
            Bt = torch.empty(p.btilde_bytes // 2, dtype=torch.bfloat16, device="cuda")
            us = t(lambda: p.precombine_b(B, Bt))
            by = B.numel() * 2 + Bt.numel() * 2
            cp = torch.empty_like(Bt)
            src = torch.empty_like(Bt)
            uc = t(lambda: cp.copy_(src))
            print(f"K={K} N={N} bl={bl} {algo}: {us:8.1f} us  {by / us / 1e6:6.2f} TB/s   "
                  f"(copy of Bt size: {2 * Bt.numel() * 2 / uc / 1e6:5.2f} TB/s)", flush=True)
            del Bt, cp, src
        del B
        torch.cuda.empty_cache()
