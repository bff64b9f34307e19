import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs
for bl in (1, 0):
    for (M, N, K) in [(128, 256, 32), (128, 256, 64), (256, 256, 32)]:
        A, B = inputs.operands(M, N, K, 2, 1, 2, dist="int", b_layout=bl)
        p = L.Plan(M, N, K, dtype=L.TF32, algo="classical", b_layout=bl)
        C = p.gemm(A.cuda(), B.cuda()).cpu().double()
        Bd = B.double() if bl == 0 else B.double().t()
        ref = A.double() @ Bd
        err = (C - ref).abs().max().item()
        # test hypotheses: maybe operand pairs are transposed within 8x8 etc.
        print(f"bl={bl} {M}x{N}x{K} maxerr={err} C[0,:4]={C[0,:4].tolist()} ref={ref[0,:4].tolist()}", flush=True)
        if bl == 0 and err > 0:
            # compare to A @ B' for alternative B interpretations
            for name, alt in [("B with rows/cols swapped in 32-blocks", None)]:
                pass
