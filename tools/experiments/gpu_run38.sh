ROUNDS=5 timeout 600 python tools/cmp.py 8192 14336 4096 cl:classical st:strassen sts:strassen:s pf:strassen:variant=producer pfs:strassen:s:variant=producer
ROUNDS=3 timeout 900 python tools/cmp.py 32768 28672 8192 cl:classical sts:strassen:s pfs:strassen:s:variant=producer
LCMA_STATS=1 timeout 300 python - <<'PY'
import ctypes, numpy as np, torch, sys
sys.path.insert(0, ".")
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs
M, N, K = 8192, 14336, 4096
A, B = inputs.operands(M, N, K, 0, 1, 2, b_layout=1)
A, B = A.cuda(), B.cuda()
for v in ("fused_h", "producer"):
    p = L.Plan(M, N, K, algo="strassen", b_layout=1, b_static=True, variant=v)
    C = p.empty_c(); ws = p.workspace(); Bt = p.precombine_b(B)
    for _ in range(3): p.gemm_precombined(A, Bt, C, ws)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (1024 * 8))()
    L.lib().lcma_debug_stats(buf, 1024 * 8)
    s = np.array(buf[:p.info["ctas"] * 8]).reshape(-1, 8).astype(float)
    tot = s[:, 3].mean()
    print(v, "mma_wait_full %.1f%%" % (s[:, 2].mean() / tot * 100), "prod_wait_empty %.1f%%" % (s[:, 0].mean() / tot * 100), "mma_wait_tempty %.1f%%" % (s[:,1].mean()/tot*100))
PY
