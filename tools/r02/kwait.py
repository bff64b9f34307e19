"""MMA-warp operand wait by k-block position inside a product (LCMA_STATS,
-DLCMA_DIAG build): are the stalls at product starts (new Ã_r / B̃_r panels
missing L2) or spread evenly?  usage: kwait.py M N K"""
import ctypes, os, sys
os.environ.setdefault("LCMA_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)).split("/tools")[0],
                                               "paper_2605_06057_b200", "liblcma_diag.so"))
os.environ["LCMA_STATS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs

M, N, K = [int(v) for v in sys.argv[1:4]]
A, B = inputs.operands(M, N, K, 0, 1, 2, b_layout=1)
A, B = A.cuda(), B.cuda()
lo = [0, 1, 2, 3, 4, 8, 16, 32]
hi = [1, 2, 3, 4, 8, 16, 32, 1 << 20]
for algo, dbg, sched in (("classical", "", 1), ("classical", "1", 1), ("strassen", "", 1), ("strassen", "1", 1),
                         ("strassen", "", 5), ("classical", "", 5)):
    os.environ.pop("LCMA_DEBUG", None)
    if dbg:
        os.environ["LCMA_DEBUG"] = dbg
    st = algo != "classical"
    p = L.Plan(M, N, K, algo=algo, b_layout=1, b_static=st, schedule=sched)
    C = p.empty_c(); ws = p.workspace()
    Bt = p.precombine_b(B) if st else None
    for _ in range(3):
        (p.gemm_precombined(A, Bt, C, ws) if st else p.gemm(A, B, C, ws))
    torch.cuda.synchronize()
    n = 1024 * 16
    buf = (ctypes.c_ulonglong * n)()
    L.lib().lcma_debug_stats(buf, n)
    s = np.array(buf[:p.info["ctas"] * 16]).reshape(-1, 16).astype(float)[0::2]   # leaders
    tot = s[:, 3].sum()
    nK = p.info["Kb"] // p.info["BK"] if st else -(-K // p.info["BK"])
    prods = p.info["groups"] * p.info["R"]
    per_kb = []
    for b in range(8):
        width = max(0, min(hi[b], nK) - lo[b])
        per_kb.append(s[:, 8 + b].sum() / max(1, prods * width) if width else float("nan"))
    print(f"{algo:9s} dbg={dbg or '-'} sched={sched} nK={nK} mma_loop_cyc/leader={tot/len(s):.0f} "
          f"full_wait={s[:, 2].sum()/tot*100:.1f}% tempty_wait={s[:, 1].sum()/tot*100:.1f}%", flush=True)
    print("   wait cycles per k-block by position [0,1,2,3,4-7,8-15,16-31,32+]:",
          " ".join(f"{v:.0f}" for v in per_kb), flush=True)
    del C, ws, Bt, p
    torch.cuda.empty_cache()
