"""Per-launch device times, in launch order, via torch.profiler (CUPTI)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs


def seq(M, N, K, algo, static_b=False, reps=3, dtype=0, **kw):
    A, B = inputs.operands(M, N, K, dtype, 1, 2)
    A, B = A.cuda(), B.cuda()
    p = L.Plan(M, N, K, dtype=dtype, algo=algo, **kw)
    C = p.empty_c(); ws = p.workspace()
    Bt = p.precombine_b(B) if static_b else None
    f = (lambda: p.gemm_precombined(A, Bt, C, ws)) if Bt is not None else (lambda: p.gemm(A, B, C, ws))
    for _ in range(3): f()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as pr:
        for _ in range(reps): f()
        torch.cuda.synchronize()
    evs = [e for e in pr.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    print(f"== {algo} {kw} static_b={static_b} {M}x{N}x{K}")
    for e in evs:
        print(f"   t={e.time_range.start:14.1f} dur={e.time_range.elapsed_us():9.1f} us  {e.name[:60]}")


if __name__ == "__main__":
    M, N, K = 32768, 28672, 8192
    seq(M, N, K, "strassen")
    seq(M, N, K, "strassen", static_b=True)
    seq(M, N, K, "classical")
    seq(M, N, K, "strassen")
