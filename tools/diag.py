import sys, os, json, subprocess
os.environ.setdefault("LCMA_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)).split("/tools")[0], "paper_2605_06057_b200", "liblcma_diag.so"))  # env knobs: -DLCMA_DIAG build
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs
from tools.perf_probe import bench
M, N, K = 8192, 14336, 4096
A, B = inputs.operands(M, N, K, 0, 1, 2)
A, B = A.cuda(), B.cuda()
fl = 2.0 * M * N * K
out = {}
for name, kw, env in [("classical", dict(algo="classical"), {}),
                      ("classical_noepi", dict(algo="classical"), {"LCMA_DEBUG": "1"}),
                      ("strassen", dict(algo="strassen"), {}),
                      ("strassen_noepi", dict(algo="strassen"), {"LCMA_DEBUG": "1"}),
                      ("strassen_hint", dict(algo="strassen"), {"LCMA_PARTIAL_HINT": "1"}),
                      ("strassen_swz4", dict(algo="strassen"), {"LCMA_SWZ": "4"}),
                      ("strassen_swz32", dict(algo="strassen"), {"LCMA_SWZ": "32"}),
                      ("strassen_unfusedGEMM", dict(algo="strassen", variant="unfused"), {})]:
    os.environ.pop("LCMA_DEBUG", None); os.environ.pop("LCMA_PARTIAL_HINT", None); os.environ.pop("LCMA_SWZ", None)
    os.environ.update(env)
    p = L.Plan(M, N, K, **kw)
    C = p.empty_c(); ws = p.workspace()
    Bt = p.precombine_b(B) if kw["algo"] != "classical" else None
    f = (lambda: p.gemm_precombined(A, Bt, C, ws)) if Bt is not None else (lambda: p.gemm(A, B, C, ws))
    t = bench(f)
    out[name] = dict(ms=round(t, 4), eff_tflops=round(fl / t / 1e9, 1))
    print(name, out[name], flush=True)
