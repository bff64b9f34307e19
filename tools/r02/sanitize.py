"""Small fused-LCMA and classical calls for compute-sanitizer (memcheck /
racecheck / synccheck): split groups, TMA-store epilogue, in-place operands."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs
for algo, (M, N, K), ctas, dt in (("strassen", (1024, 1536, 512), 10, L.BF16), ("classical", (768, 1024, 512), 6, L.BF16),
                                  ("strassen", (1024, 1024, 512), 8, L.FP8)):
    A, B = inputs.operands(M, N, K, dt, 1, 2, b_layout=1)
    p = L.Plan(M, N, K, dtype=dt, algo=algo, b_layout=1, num_ctas=ctas)
    for _ in range(2):
        C = p.gemm(A.cuda(), B.cuda())
    torch.cuda.synchronize()
    print(algo, dt, "ok", float(C.float().abs().sum()))
