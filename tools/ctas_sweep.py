"""Classical / Strassen GEMM time vs number of persistent CTAs (is the
mainloop limited by a shared resource?)."""
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


M, N, K = 8192, 14336, 4096
A, B = inputs.operands(M, N, K, 0, 1, 2)
A, B = A.cuda(), B.cuda()
for algo in ("classical", "strassen"):
    for ctas in (148, 140, 132, 120, 100, 80):
        p = L.Plan(M, N, K, dtype=0, algo=algo, num_ctas=ctas, b_static=(algo != "classical"))
        C = p.empty_c(); ws = p.workspace()
        if algo == "classical":
            us = t(lambda: p.gemm(A, B, C, ws))
        else:
            Bt = p.precombine_b(B)
            us = t(lambda: p.gemm_precombined(A, Bt, C, ws))
        print(f"{algo:10s} ctas={ctas:4d} {us:8.1f} us  {2*M*N*K/us/1e6:7.1f} TF  "
              f"per-SM {2*M*N*K/us/1e6/ctas:6.2f}", flush=True)
