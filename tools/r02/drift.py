"""Round-2 probe: drift between CTA pairs of the persistent schedule.  For
lockstep round p (whole groups), the MMA start stamp of its first product on
every leader CTA (LCMA_TIMELINE=1); prints the spread (max - min) per round in
units of the median round duration.  usage: drift.py algo M N K"""
import ctypes, os, sys
os.environ.setdefault("LCMA_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)).split("/tools")[0], "paper_2605_06057_b200", "liblcma_diag.so"))  # env knobs: -DLCMA_DIAG build
os.environ["LCMA_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs

algo = sys.argv[1]
M, N, K = [int(v) for v in sys.argv[2:5]]
A, B = inputs.operands(M, N, K, 0, 1, 2, b_layout=1)
A, B = A.cuda(), B.cuda()
st = algo != "classical"
p = L.Plan(M, N, K, algo=algo, b_layout=1, b_static=st)
C = p.empty_c(); ws = p.workspace()
Bt = p.precombine_b(B) if st else None
f = (lambda: p.gemm_precombined(A, Bt, C, ws)) if st else (lambda: p.gemm(A, B, C, ws))
for _ in range(3): f()
torch.cuda.synchronize()
ctas = p.info["ctas"]
n = ctas * 512 * 4
buf = (ctypes.c_ulonglong * n)()
L.lib().lcma_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_longlong]
assert L.lib().lcma_debug_timeline(buf, n) == 0
t = np.array(buf[:n], dtype=np.float64).reshape(ctas, 512, 4)
R = p.info["R"]
lead = t[0::2]
nprod = int((lead[:, :, 1] > 0).sum(1).min())
t0 = lead[:, :nprod, 0]
base = t0[:, 0].min()
starts = t0[:, ::R] - base            # start of each round per pair
rd = np.median(np.diff(starts, axis=1))
spread = starts.max(0) - starts.min(0)
print(f"{algo} {M}x{N}x{K}: pairs {lead.shape[0]} rounds {starts.shape[1]} median round {rd/1e3:.1f} us")
for q in list(range(0, starts.shape[1], max(1, starts.shape[1] // 12))) + [starts.shape[1] - 1]:
    print(f"  round {q:4d}: spread {spread[q]/1e3:8.1f} us = {spread[q]/rd:5.2f} rounds; p10-p90 "
          f"{(np.percentile(starts[:, q], 90) - np.percentile(starts[:, q], 10))/1e3:8.1f} us")
