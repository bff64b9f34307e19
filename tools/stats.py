"""Per-role wait-cycle breakdown of the tcgen05 kernel (LCMA_STATS=1)."""
import sys, os, ctypes
os.environ.setdefault("LCMA_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)).split("/tools")[0], "paper_2605_06057_b200", "liblcma_diag.so"))  # env knobs: -DLCMA_DIAG build
os.environ["LCMA_STATS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs
def run(M, N, K, algo, static_b=True, env=None, **kw):
    for k in ("LCMA_DEBUG",): os.environ.pop(k, None)
    if env: os.environ.update(env)
    A, B = inputs.operands(M, N, K, 0, 1, 2)
    A, B = A.cuda(), B.cuda()
    p = L.Plan(M, N, K, algo=algo, **kw)
    C = p.empty_c(); ws = p.workspace()
    Bt = p.precombine_b(B) if (algo != "classical" and static_b) else None
    for _ in range(3):
        (p.gemm_precombined(A, Bt, C, ws) if Bt is not None else p.gemm(A, B, C, ws))
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (1024 * 16))()
    L.lib().lcma_debug_stats(buf, 1024 * 16)
    s = np.array(buf[:p.info["ctas"] * 16]).reshape(-1, 16).astype(float)
    tot = s[:, 3].mean()
    print(f"{algo:10s} {env or ''} total_cyc={tot:.0f} mma_wait_tempty={s[:,1].mean()/tot*100:.1f}% "
          f"mma_wait_full={s[:,2].mean()/tot*100:.1f}% prod_wait_empty={s[:,0].mean()/tot*100:.1f}% "
          f"epi_wait_tfull={s[:,4].mean()/s[:,5].mean()*100:.1f}%", flush=True)
M, N, K = 8192, 14336, 4096
run(M, N, K, "classical")
run(M, N, K, "classical", env={"LCMA_DEBUG": "1"})
run(M, N, K, "strassen")
run(M, N, K, "strassen", env={"LCMA_DEBUG": "1"})
run(M, N, K, "strassen2")

def timeline(M, N, K, algo):
    A, B = inputs.operands(M, N, K, 0, 1, 2)
    A, B = A.cuda(), B.cuda()
    p = L.Plan(M, N, K, algo=algo)
    C = p.empty_c(); ws = p.workspace()
    for _ in range(3): p.gemm(A, B, C, ws)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (1024 * 16))()
    L.lib().lcma_debug_stats(buf, 1024 * 16)
    s = np.array(buf[:p.info["ctas"] * 16]).reshape(-1, 16)
    t0 = s[:, 6].min()
    st = (s[:, 6] - t0) / 1000.0; en = (s[:, 7] - t0) / 1000.0
    print(f"{algo} cg={p.info['cta_group']} start_us min/med/max {st.min():.1f}/{np.median(st):.1f}/{st.max():.1f}  end_us {en.min():.1f}/{np.median(en):.1f}/{en.max():.1f} mma_cyc_med {np.median(s[:,3]):.0f} sm_GHz {np.median(s[:,5]/(s[:,7]-s[:,6])):.3f}", flush=True)
    print("  sorted starts:", np.round(np.sort(st)[::8], 1).tolist())
timeline(8192, 14336, 4096, "classical")
buf = (ctypes.c_ulonglong * (1024 * 16))()
L.lib().lcma_debug_stats(buf, 1024 * 16)
s = np.array(buf[:148 * 16]).reshape(-1, 16)
np.set_printoptions(linewidth=200)
print(s[:6])
t0 = s[:, 6].min()
print("end-start us per CTA (first 10):", ((s[:10, 7] - s[:10, 6]) / 1000).round(1).tolist())
