"""Where the fused GEMM's time goes per CTA pair: kernel start -> first MMA,
MMA span, last MMA -> CTA end (LCMA_TIMELINE + LCMA_STATS, diag build).
usage: span.py M N K [algo]"""
import ctypes, os, sys
os.environ.setdefault("LCMA_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)).split("/tools")[0],
                                               "paper_2605_06057_b200", "liblcma_diag.so"))
os.environ["LCMA_STATS"] = "1"
os.environ["LCMA_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs

M, N, K = [int(v) for v in sys.argv[1:4]]
algo = sys.argv[4] if len(sys.argv) > 4 else "strassen"
A, B = inputs.operands(M, N, K, 0, 1, 2, b_layout=1)
A, B = A.cuda(), B.cuda()
p = L.Plan(M, N, K, algo=algo, b_layout=1, b_static=(algo != "classical"))
C = p.empty_c(); ws = p.workspace()
Bt = p.precombine_b(B) if algo != "classical" else None
f = (lambda: p.gemm_precombined(A, Bt, C, ws)) if Bt is not None else (lambda: p.gemm(A, B, C, ws))
for _ in range(3): f()
torch.cuda.synchronize()
ctas = p.info["ctas"]
st = (ctypes.c_ulonglong * (1024 * 16))()
L.lib().lcma_debug_stats(st, 1024 * 16)
sa = np.array(st[:ctas * 16]).reshape(-1, 16).astype(float)
n = ctas * 512 * 4
tl = (ctypes.c_ulonglong * n)()
L.lib().lcma_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_longlong]
L.lib().lcma_debug_timeline(tl, n)
t = np.array(tl[:n], dtype=np.float64).reshape(ctas, 512, 4)[0::2]
k0 = sa[:, 6].min()
start = (sa[0::2, 6] - k0) / 1e3
end = (sa[0::2, 7] - k0) / 1e3
cnt = (t[:, :, 1] > 0).sum(1)
first = np.array([(t[i, 0, 0] - k0) / 1e3 for i in range(len(t))])
last = np.array([(t[i, cnt[i] - 1, 1] - k0) / 1e3 for i in range(len(t))])
lastrel = np.array([(t[i, cnt[i] - 1, 3] - k0) / 1e3 for i in range(len(t))])
for name, v in (("CTA start", start), ("first MMA slot", first), ("last MMA issued", last),
                ("last acc released", lastrel), ("CTA end", end), ("products", cnt)):
    print(f"{algo} {name:18s} p10 {np.percentile(v,10):9.1f}  p50 {np.percentile(v,50):9.1f}  p90 {np.percentile(v,90):9.1f}  max {v.max():9.1f}")
print("end - last release p50/max", np.percentile(end - lastrel, 50).round(1), (end - lastrel).max().round(1))
