"""Subprocess helper of tests/test_gpu_parity.py::test_partial_homes_exact_diag_build:
runs against LCMA_LIB = the -DLCMA_DIAG build, whose launch-time knobs select
the non-default C_ij partial homes, and checks every placement exactly
against the int64 oracle (whole and split groups)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle as O
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs

assert os.environ.get("LCMA_LIB", "").endswith("liblcma_diag.so")
ENVS = [{}, {"LCMA_QFULL": "1"}, {"LCMA_REG_PARTIAL": "0"}, {"LCMA_SMEM_PARTIAL": "0"},
        {"LCMA_REG_PARTIAL": "0", "LCMA_SMEM_PARTIAL": "0"}, {"LCMA_SERPENTINE": "1"}, {"LCMA_ORDER": "0"}]
CASES = [("strassen", (1536, 2304, 512), 0, (-2, 2)), ("strassen", (1536, 2304, 512), 10, (-2, 2)),
         ("laderman", (1000, 808, 520), 0, (-1, 1)), ("strassen2", (1024, 1024, 512), 0, (-1, 1))]
SCH = {"strassen": O.strassen, "laderman": O.laderman, "strassen2": O.strassen2}
KEYS = sorted({k for e in ENVS for k in e})
for env in ENVS:
    for k in KEYS:
        os.environ.pop(k, None)
    os.environ.update(env)
    for algo, (M, N, K), ctas, (lo, hi) in CASES:
        for schedule in (1, 5):
            if "LCMA_SERPENTINE" in env and schedule == 5:
                continue          # serpentine rounds exist in the static schedule only
            A, B = inputs.operands(M, N, K, 0, M + 7, N + K, dist="int", lo=lo, hi=hi)
            plan = L.Plan(M, N, K, algo=algo, out_dtype=L.FP32, variant="fused_h", num_ctas=ctas,
                          schedule=schedule)
            C = plan.gemm(A.cuda(), B.cuda()).cpu().numpy()
            ref = O.gemm_i64(A.to(torch.int64).numpy(), B.to(torch.int64).numpy())
            bad = np.argwhere(C != ref)
            assert bad.size == 0, (env, algo, ctas, schedule, len(bad))
    print("ok", env, flush=True)
print("homes ok")
