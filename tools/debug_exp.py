"""Classical kernel time with epilogue parts disabled (LCMA_DEBUG bits:
1 = no global traffic, 2 = no TMEM loads)."""
import os, sys
os.environ.setdefault("LCMA_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)).split("/tools")[0], "paper_2605_06057_b200", "liblcma_diag.so"))  # env knobs: -DLCMA_DIAG build
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


M, N, K = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (8192, 14336, 4096))]
BL = int(os.environ.get("BL", "1"))
A, B = inputs.operands(M, N, K, 0, 1, 2, b_layout=BL)
A, B = A.cuda(), B.cuda()
for algo in ("classical", "strassen"):
    p = L.Plan(M, N, K, dtype=0, algo=algo, b_layout=BL, b_static=(algo != "classical"))
    C = p.empty_c(); ws = p.workspace()
    Bt = p.precombine_b(B) if algo != "classical" else None
    for dbg in sys.argv[4:] or ("0", "4", "1", "5"):
        os.environ["LCMA_DEBUG"] = dbg
        f = (lambda: p.gemm(A, B, C, ws)) if Bt is None else (lambda: p.gemm_precombined(A, Bt, C, ws))
        us = t(f)
        print(f"{M}x{N}x{K} bl={BL} {algo:10s} debug={dbg} {us:8.1f} us {2*M*N*K/us/1e6:7.1f} TF", flush=True)
    os.environ["LCMA_DEBUG"] = "0"
