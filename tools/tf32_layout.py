"""tf32 classical vs Strassen at the cfg3 corner for both B layouts (interleaved)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs

def timed(f, reps=1):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps

M, N, K = [int(v) for v in (sys.argv[1:4] or ["16384", "14336", "14336"])]
for bl in (0, 1):
    A, B = inputs.operands(M, N, K, L.TF32, 301, 302, b_layout=bl)
    A, B = A.cuda(), B.cuda()
    fns, keep = {}, []
    for algo in ("classical", "strassen"):
        p = L.Plan(M, N, K, dtype=L.TF32, algo=algo, b_layout=bl)
        C, ws = p.empty_c(), p.workspace()
        fns[algo] = (lambda p=p, C=C, ws=ws: p.gemm(A, B, C, ws)); keep += [p, C, ws]
    res = {n: [] for n in fns}
    for rnd in range(5):
        for n in (list(fns) if rnd % 2 == 0 else list(fns)[::-1]):
            res[n].append(timed(fns[n]))
    fl = 2.0 * M * N * K
    med = {n: statistics.median(v) for n, v in res.items()}
    print(f"tf32 {M}x{N}x{K} bl={bl}: " + " ".join(f"{n}={fl/(ms*1e-3)/1e12:.1f}TF" for n, ms in med.items()) +
          f" ratio={med['classical']/med['strassen']:.3f}", flush=True)
    del fns, keep, A, B
    torch.cuda.empty_cache()
