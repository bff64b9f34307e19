"""Context only: cuBLAS kernel name/time at cfg2 next to our classical kernel
(cuBLAS is never on the product path)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs

M, N, K = 8192, 14336, 4096
A, B = inputs.operands(M, N, K, 0, 1, 2)
A, B = A.cuda(), B.cuda()
p = L.Plan(M, N, K, dtype=0, algo="classical")
C = p.empty_c(); ws = p.workspace()
fs = {"cublas": lambda: torch.matmul(A, B), "ours": lambda: p.gemm(A, B, C, ws)}
for name, f in fs.items():
    for _ in range(5): f()
torch.cuda.synchronize()
if os.environ.get("NCU_ONE"):
    fs[os.environ["NCU_ONE"]]()
    torch.cuda.synchronize()
    sys.exit(0)
with profile(activities=[ProfilerActivity.CUDA]) as pr:
    for name, f in fs.items():
        for _ in range(5): f()
    torch.cuda.synchronize()
for e in pr.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        print(f"{e.time_range.elapsed_us():8.1f} us {e.name[:120]}")
