"""First-contact GPU probe: one small classical tcgen05 GEMM, then growing."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs

def run(M, N, K, dtype=L.BF16, algo="classical", b_layout=0, out=L.FP32, variant="auto", num_ctas=0, dist="int"):
    A, B = inputs.operands(M, N, K, dtype, 1, 2, dist=dist, b_layout=b_layout)
    Ad, Bd = A.cuda(), B.cuda()
    p = L.Plan(M, N, K, dtype=dtype, algo=algo, out_dtype=out, b_layout=b_layout, variant=variant, num_ctas=num_ctas)
    C = p.gemm(Ad, Bd)
    torch.cuda.synchronize()
    Bf = B.double() if b_layout == 0 else B.double().t()
    ref = A.double() @ Bf
    err = (C.double().cpu() - ref).abs().max().item()
    print(f"{algo:10s} v={variant:8s} M={M} N={N} K={K} dt={dtype} bl={b_layout} maxerr={err} info waves={p.info['waves']}", flush=True)
    return err

t0 = time.time()
run(128, 256, 64)
run(128, 256, 64, b_layout=1)
run(256, 512, 128)
run(256, 512, 128, b_layout=1)
run(300, 264, 200)
run(1024, 1024, 1024)
run(256, 512, 256, algo="strassen", variant="unfused")
run(256, 512, 256, algo="strassen")
run(512, 1024, 512, algo="strassen", b_layout=1)
print("done", time.time() - t0)
