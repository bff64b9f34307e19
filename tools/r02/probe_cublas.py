"""Context probe (round 2): co-resident cluster counts for cluster sizes 2/4/8
and cuBLAS (torch.matmul, context only, never on the product path) vs our
classical and Strassen kernels at cfg2 and the cfg5 shape, interleaved."""
import os, sys, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs

lib = L.lib()
for cs in (2, 4, 8):
    print("max_clusters", cs, lib.lcma_debug_max_clusters(cs), flush=True)


def timed(f, reps):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps


for (M, N, K, reps) in ((8192, 14336, 4096, 5), (32768, 28672, 8192, 1)):
    A, B = inputs.operands(M, N, K, 0, 1, 2, b_layout=1)
    A, B = A.cuda(), B.cuda()
    pc = L.Plan(M, N, K, algo="classical", b_layout=1); Cc = pc.empty_c()
    ps = L.Plan(M, N, K, algo="strassen", b_layout=1); Cs = ps.empty_c(); ws = ps.workspace()
    pt = L.Plan(M, N, K, algo="strassen", b_layout=1, b_static=True); Ct = pt.empty_c(); wt = pt.workspace()
    Bt = pt.precombine_b(B)
    Bk = B.t()   # N x K storage -> K x N view for torch (nn.Linear layout)
    arms = {"cublas": lambda: torch.matmul(A, Bk), "classical": lambda: pc.gemm(A, B, Cc),
            "strassen": lambda: ps.gemm(A, B, Cs, ws), "strassen_static": lambda: pt.gemm_precombined(A, Bt, Ct, wt)}
    res = {k: [] for k in arms}
    for rnd in range(7):
        ks = list(arms)
        for j in range(len(ks)):
            k = ks[(j + rnd) % len(ks)]
            res[k].append(timed(arms[k], reps))
    fl = 2.0 * M * N * K
    out = {k: round(fl / statistics.median(v) / 1e9, 1) for k, v in res.items()}
    print(json.dumps({"shape": [M, N, K], "TFLOPs": out}), flush=True)
    del A, B, Cc, Cs, ws, Ct, wt, Bt
    torch.cuda.empty_cache()
