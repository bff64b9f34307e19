"""Classical / Strassen kernel time for B K-major (b_layout 1) vs MN-major (b_layout 0)."""
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


for (M, N, K) in ((8192, 14336, 4096), (8192, 8192, 8192)):
    for bl in (0, 1):
        A, B = inputs.operands(M, N, K, 0, 1, 2, b_layout=bl)
        A, B = A.cuda(), B.cuda()
        for algo in ("classical", "strassen"):
            p = L.Plan(M, N, K, dtype=0, algo=algo, b_layout=bl, b_static=(algo != "classical"))
            C = p.empty_c(); ws = p.workspace()
            if algo == "classical":
                us = t(lambda: p.gemm(A, B, C, ws))
            else:
                Bt = p.precombine_b(B)
                us = t(lambda: p.gemm_precombined(A, Bt, C, ws))
            print(f"{M}x{N}x{K} bl={bl} {algo:10s} {us:8.1f} us {2*M*N*K/us/1e6:7.1f} TF", flush=True)
        if bl == 1:
            us = t(lambda: torch.nn.functional.linear(A, B))
        else:
            us = t(lambda: torch.matmul(A, B))
        print(f"{M}x{N}x{K} bl={bl} cublas     {us:8.1f} us {2*M*N*K/us/1e6:7.1f} TF (context)", flush=True)
