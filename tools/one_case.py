"""Run one configuration a few times (for ncu)."""
import sys, os, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs
ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=8192); ap.add_argument("--N", type=int, default=14336)
ap.add_argument("--K", type=int, default=4096); ap.add_argument("--algo", default="strassen")
ap.add_argument("--variant", default="auto"); ap.add_argument("--b_layout", type=int, default=0)
ap.add_argument("--dtype", type=int, default=0); ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--schedule", type=int, default=0); ap.add_argument("--static_b", type=int, default=0)
a = ap.parse_args()
A, B = inputs.operands(a.M, a.N, a.K, a.dtype, 1, 2, b_layout=a.b_layout)
A, B = A.cuda(), B.cuda()
p = L.Plan(a.M, a.N, a.K, dtype=a.dtype, algo=a.algo, variant=a.variant, b_layout=a.b_layout, schedule=a.schedule)
C = p.empty_c(); ws = p.workspace()
Bt = p.precombine_b(B) if a.static_b else None
for _ in range(a.reps):
    if Bt is not None: p.gemm_precombined(A, Bt, C, ws)
    else: p.gemm(A, B, C, ws)
torch.cuda.synchronize()
print("ok", p.info["scheme"], p.info["waves"])
