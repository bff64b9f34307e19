"""CTA end-time distribution of the GEMM kernel (LCMA_STATS, diag build):
how long the slowest pairs (split-tail owners / contributors) run past the
median.  usage: tail.py M N K [algo ...]"""
import ctypes, os, sys
os.environ.setdefault("LCMA_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)).split("/tools")[0],
                                               "paper_2605_06057_b200", "liblcma_diag.so"))
os.environ["LCMA_STATS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs

M, N, K = [int(v) for v in sys.argv[1:4]]
algos = sys.argv[4:] or ["strassen", "classical"]
A, B = inputs.operands(M, N, K, 0, 1, 2, b_layout=1)
A, B = A.cuda(), B.cuda()
for algo in algos:
    p = L.Plan(M, N, K, algo=algo, b_layout=1, b_static=(algo != "classical"))
    C = p.empty_c(); ws = p.workspace()
    Bt = p.precombine_b(B) if algo != "classical" else None
    f = (lambda: p.gemm_precombined(A, Bt, C, ws)) if Bt is not None else (lambda: p.gemm(A, B, C, ws))
    for _ in range(3): f()
    torch.cuda.synchronize()
    n = 1024 * 16
    buf = (ctypes.c_ulonglong * n)()
    L.lib().lcma_debug_stats(buf, n)
    sa = np.array(buf[:p.info["ctas"] * 16]).reshape(-1, 16).astype(float)
    t0 = sa[:, 6].min()
    ends = np.sort((sa[:, 7] - t0) / 1e3)
    sched = [p.schedule(c) for c in range(0, p.info["ctas"], 2)]
    roles = [sum(1 for u in s if u[3] == 1) for s in sched]
    print(f"{algo}: ctas {p.info['ctas']} groups {p.info['groups']} split {p.info['split_groups']}  CTA end "
          f"p10/p50/p90/max {np.percentile(ends,10):.1f}/{np.percentile(ends,50):.1f}/{np.percentile(ends,90):.1f}/{ends.max():.1f} us")
    e_pair = (sa[0::2, 7] - t0) / 1e3
    own = [i for i, r in enumerate(roles) if r]
    print("   owner pairs end:", np.round(e_pair[own], 1).tolist())
    print("   slowest pairs:", np.argsort(e_pair)[-6:].tolist(), np.round(np.sort(e_pair)[-6:], 1).tolist())
