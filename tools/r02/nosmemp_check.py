"""Exactness of the diag-only no-shared-partial 7-stage variant (LCMA_NOSMEMP=1)."""
import os, sys
os.environ.setdefault("LCMA_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)).split("/tools")[0], "paper_2605_06057_b200", "liblcma_diag.so"))
os.environ["LCMA_NOSMEMP"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2605_06057_b200 as L
import oracle as O
from paper_2605_06057_b200 import inputs
for M, N, K in ((1024, 1536, 8192), (1000, 1048, 6200)):
    A, B = inputs.operands(M, N, K, 0, 3, 4, dist="int", b_layout=1, lo=-2, hi=2)
    p = L.Plan(M, N, K, algo="strassen", b_layout=1, out_dtype=L.FP32, num_ctas=12)
    C = p.gemm(A.cuda(), B.cuda()).cpu().numpy()
    ref = O.gemm_i64(A.to(torch.int64).numpy(), B.t().to(torch.int64).numpy())
    print(M, N, K, "exact" if np.array_equal(C, ref) else "MISMATCH")
