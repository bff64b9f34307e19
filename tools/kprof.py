"""Per-kernel device times via torch.profiler (CUPTI), back-to-back runs."""
import sys, os, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs

def prof(M, N, K, algo, static_b=False, reps=10, dtype=0, b_layout=0, **kw):
    A, B = inputs.operands(M, N, K, dtype, 1, 2, b_layout=b_layout)
    A, B = A.cuda(), B.cuda()
    p = L.Plan(M, N, K, dtype=dtype, algo=algo, b_layout=b_layout, **kw)
    C = p.empty_c(); ws = p.workspace()
    Bt = p.precombine_b(B) if (static_b and algo != "classical") else None
    f = (lambda: p.gemm_precombined(A, Bt, C, ws)) if Bt is not None else (lambda: p.gemm(A, B, C, ws))
    for _ in range(5): f()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as pr:
        for _ in range(reps): f()
        torch.cuda.synchronize()
    tot = {}
    for e in pr.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            tot.setdefault(e.name, []).append(e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total)
    fl = 2.0 * M * N * K
    s = 0.0
    print(f"== {algo} {kw} static_b={static_b} shape={M}x{N}x{K}")
    for k, v in tot.items():
        avg = sum(v) / reps
        s += avg
        print(f"   {avg:9.1f} us  x{len(v)//reps}  {k[:90]}")
    print(f"   total {s:.1f} us -> {fl / s / 1e6:.1f} TFLOP/s effective")

if __name__ == "__main__":
    M, N, K = 8192, 14336, 4096
    prof(M, N, K, "classical")
    prof(M, N, K, "strassen")
    prof(M, N, K, "strassen", static_b=True)
    prof(M, N, K, "strassen", variant="unfused")
    prof(M, N, K, "strassen2", static_b=True)
