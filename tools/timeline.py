"""Per-product timeline of the fused GEMM (LCMA_TIMELINE=1): where the MMA
warp waits for the epilogue to release an accumulator slot, by product
position inside the group.  usage: python tools/timeline.py [algo] [M N K]"""
import ctypes, os, sys
os.environ.setdefault("LCMA_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)).split("/tools")[0], "paper_2605_06057_b200", "liblcma_diag.so"))  # env knobs: -DLCMA_DIAG build
os.environ["LCMA_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs

algo = sys.argv[1] if len(sys.argv) > 1 else "strassen"
M, N, K = [int(v) for v in sys.argv[2:5]] if len(sys.argv) > 4 else (8192, 14336, 4096)
DT = int(os.environ.get("DT", "0"))
A, B = inputs.operands(M, N, K, DT, 1, 2, b_layout=1)
A, B = A.cuda(), B.cuda()
p = L.Plan(M, N, K, dtype=DT, algo=algo, b_layout=1, b_static=(algo != "classical"))
C = p.empty_c(); ws = p.workspace()
Bt = p.precombine_b(B) if algo != "classical" else None
f = (lambda: p.gemm_precombined(A, Bt, C, ws)) if Bt is not None else (lambda: p.gemm(A, B, C, ws))
for _ in range(4): f()
torch.cuda.synchronize()
ctas = p.info["ctas"]
n = ctas * 512 * 4
buf = (ctypes.c_ulonglong * n)()
L.lib().lcma_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_longlong]
assert L.lib().lcma_debug_timeline(buf, n) == 0
t = np.array(buf[:n], dtype=np.float64).reshape(ctas, 512, 4)
R = 1 if algo == "classical" else {"strassen": 7, "laderman": 23, "strassen2": 49}[algo]
lead = t[0::2]                                  # leader CTAs carry the MMA stamps
nprod = int((lead[:, :, 1] > 0).sum(1).min())
t0 = lead[:, :nprod, 0]; t1 = lead[:, :nprod, 1]
wait_slot = t0[:, 1:] - t1[:, :-1]             # MMA idle between products (ns)
prod = t1 - t0                                 # MMA issue time per product (ns)
e_start = lead[:, :nprod, 2]; e_rel = lead[:, :nprod, 3]
epi = e_rel - e_start                          # epilogue time to release (ns), half 0 start .. half 1 release
print(f"{algo} {M}x{N}x{K}: {nprod} products per leader CTA; MMA issue per product median {np.median(prod)/1e3:.2f} us")
print(f"MMA slot waits: total per CTA median {np.median(wait_slot.sum(1))/1e3:.1f} us of {np.median(t1[:, -1]-t0[:, 0])/1e3:.1f} us")
for pos in range(R):
    ks = [k for k in range(1, nprod) if k % R == pos]
    if not ks: continue
    w_ = wait_slot[:, [k - 1 for k in ks]]
    e_ = epi[:, [k for k in ks]]
    print(f"  position {pos}: slot wait before it median {np.median(w_)/1e3:6.2f} us (p90 {np.percentile(w_,90)/1e3:6.2f}); "
          f"epilogue-to-release median {np.median(e_)/1e3:6.2f} us (p90 {np.percentile(e_,90)/1e3:6.2f})")
# MMA issue time per product position and by round (where the mean exceeds the median)
print("MMA issue time by position (us): " + "  ".join(
    f"{pos}: p50 {np.median(prod[:, pos::R])/1e3:.2f} mean {np.mean(prod[:, pos::R])/1e3:.2f}" for pos in range(min(R, nprod))))
nr = nprod // R
if nr > 1:
    per_round = [np.mean(prod[:, k * R:(k + 1) * R]) / 1e3 for k in range(nr)]
    print("mean MMA issue per product by round (us):", " ".join(f"{v:.2f}" for v in per_round))
