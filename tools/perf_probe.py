"""Quick perf probe: effective TFLOP/s of classical vs LCMA variants (CUDA events)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs

def bench(fn, reps=20, warm=5):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts)//2]

def case(M, N, K, dtype=L.BF16, b_layout=0):
    A, B = inputs.operands(M, N, K, dtype, 1, 2, b_layout=b_layout)
    A, B = A.cuda(), B.cuda()
    fl = 2.0 * M * N * K
    res = {}
    Bm = B if b_layout == 0 else B.t()
    t = bench(lambda: torch.matmul(A, Bm)); res["torch.matmul"] = fl / t / 1e9
    for name, kw in [("classical", dict(algo="classical")),
                     ("strassen_fusedH", dict(algo="strassen", variant="fused_h")),
                     ("strassen_unfused", dict(algo="strassen", variant="unfused")),
                     ("strassen2_fusedH", dict(algo="strassen2", variant="fused_h")),
                     ("strassen_paper_sched", dict(algo="strassen", variant="fused_h", schedule=2))]:
        p = L.Plan(M, N, K, dtype=dtype, b_layout=b_layout, **kw)
        C = p.empty_c(); ws = p.workspace()
        t = bench(lambda: p.gemm(A, B, C, ws))
        res[name] = fl / t / 1e9
        if "fusedH" in name and "strassen" in name:
            Bt = p.precombine_b(B)
            t2 = bench(lambda: p.gemm_precombined(A, Bt, C, ws))
            res[name + "_staticB"] = fl / t2 / 1e9
    print(json.dumps({"shape": [M, N, K], "dtype": dtype, "b_layout": b_layout, "TFLOPs_eff": {k: round(v, 1) for k, v in res.items()}}), flush=True)

case(8192, 14336, 4096)
case(8192, 14336, 4096, b_layout=1)
case(8192, 8192, 8192)
