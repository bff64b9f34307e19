"""Which part of the fused Combine-H epilogue slows the Strassen mainloop?
LCMA_DEBUG bits (diag build, results wrong): 1 no epilogue traffic at all
(TMEM loads only), 2 no TMEM loads, 128 no C stores, 256 no L2 partial
traffic, 512 no shared-memory partial work, 1024 no register partial work.
Interleaved rounds; prints us per call and the MMA-loop cycles / operand wait
(LCMA_STATS).  usage: epi_ablate.py M N K"""
import ctypes, os, statistics, sys
os.environ.setdefault("LCMA_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)).split("/tools")[0],
                                               "paper_2605_06057_b200", "liblcma_diag.so"))
os.environ["LCMA_STATS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs

M, N, K = [int(v) for v in sys.argv[1:4]] if len(sys.argv) > 3 else (8192, 14336, 4096)
A, B = inputs.operands(M, N, K, 0, 1, 2, b_layout=1)
A, B = A.cuda(), B.cuda()
p = L.Plan(M, N, K, algo="strassen", b_layout=1, b_static=True)
C = p.empty_c(); ws = p.workspace(); Bt = p.precombine_b(B)
pc = L.Plan(M, N, K, algo="classical", b_layout=1); Cc = pc.empty_c(); wc = pc.workspace()
arms = [("cls", 0, True), ("clsNoC", 128, True), ("clsMain", 1, True), ("full", 0, False), ("mainloop", 1, False), ("noC", 128, False), ("noL2", 256, False),
        ("noSmem", 512, False), ("noReg", 1024, False), ("noAll4", 128 | 256 | 512 | 1024, False),
        ("noTmemLd", 2 | 1, False), ("coalC", 2048, False), ("clsCoalC", 2048, True)]
res = {a[0]: [] for a in arms}
cyc = {a[0]: [] for a in arms}
for rnd in range(5):
    for j in range(len(arms)):
        name, dbg, cls = arms[(j + rnd) % len(arms)]
        os.environ["LCMA_DEBUG"] = str(dbg)
        f = (lambda: pc.gemm(A, B, Cc, wc)) if cls else (lambda: p.gemm_precombined(A, Bt, C, ws))
        f(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): f()
        e1.record(); e1.synchronize()
        res[name].append(e0.elapsed_time(e1) / 5 * 1e3)
        n = 1024 * 16
        buf = (ctypes.c_ulonglong * n)()
        L.lib().lcma_debug_stats(buf, n)
        s = np.array(buf[:p.info["ctas"] * 16]).reshape(-1, 16).astype(float)[0::2]
        sa = np.array(buf[:p.info["ctas"] * 16]).reshape(-1, 16).astype(float)
        ghz = np.median(sa[:, 5] / np.maximum(1.0, sa[:, 7] - sa[:, 6]))      # SM cycles / ns over the kernel
        t0 = sa[:, 6].min()
        ends = (sa[:, 7] - t0) / 1e3
        # MMA-loop end per leader (us): start + loop cycles / clock
        cyc[name].append((s[:, 3].mean(), s[:, 2].sum() / s[:, 3].sum(), ghz, np.median(ends), ends.max(),
                          np.percentile(ends, 10)))
for name, _, _ in arms:
    us = statistics.median(res[name])
    c = statistics.median(x[0] for x in cyc[name]); w = statistics.median(x[1] for x in cyc[name])
    g = statistics.median(x[2] for x in cyc[name])
    e50 = statistics.median(x[3] for x in cyc[name]); emax = statistics.median(x[4] for x in cyc[name])
    e10 = statistics.median(x[5] for x in cyc[name])
    print(f"{name:9s} {us:8.1f} us   mma_loop_cyc {c:10.0f}   operand_wait {w*100:5.1f} %   sm_clock {g:5.3f} GHz"
          f"   CTA end p10/p50/max {e10:6.1f}/{e50:6.1f}/{emax:6.1f} us", flush=True)
