"""One GEMM launch per algorithm for ncu captures (cfg2 shape unless given).
usage: python tools/ncu_one.py ALGO [static] [M N K] [bl]   (DT=4: FP8)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs

algo = sys.argv[1]
static = len(sys.argv) > 2 and sys.argv[2] == "static"
M, N, K = [int(v) for v in sys.argv[3:6]] if len(sys.argv) > 5 else (8192, 14336, 4096)
bl = int(sys.argv[6]) if len(sys.argv) > 6 else 1
dt = int(os.environ.get("DT", "0"))
A, B = inputs.operands(M, N, K, dt, 1, 2, b_layout=bl)
A, B = A.cuda(), B.cuda()
p = L.Plan(M, N, K, dtype=dt, algo=algo, b_layout=bl, b_static=static)
C = p.empty_c(); ws = p.workspace()
Bt = p.precombine_b(B) if static else None
for _ in range(3):
    p.gemm_precombined(A, Bt, C, ws) if static else p.gemm(A, B, C, ws)
torch.cuda.synchronize()
