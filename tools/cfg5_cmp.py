"""Interleaved classical vs Strassen (per call / B offline) at cfg5 shapes."""
import os, sys, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs

def timed(f, reps):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps

for M in [int(v) for v in (sys.argv[1:] or ["16384", "32768"])]:
    N, K = 28672, 8192
    A, B = inputs.operands(M, N, K, 0, 510, 502, b_layout=1)
    A, B = A.cuda(), B.cuda()
    fns = {}
    keep = []
    for name, kw in (("classical", dict(algo="classical")), ("strassen", dict(algo="strassen")),
                     ("strassen_sb", dict(algo="strassen", b_static=True))):
        p = L.Plan(M, N, K, dtype=0, b_layout=1, **kw)
        C = p.empty_c(); ws = p.workspace()
        if kw.get("b_static"):
            Bt = p.precombine_b(B); keep.append(Bt)
            fns[name] = (lambda p=p, Bt=Bt, C=C, ws=ws: p.gemm_precombined(A, Bt, C, ws))
        else:
            fns[name] = (lambda p=p, C=C, ws=ws: p.gemm(A, B, C, ws))
        keep += [p, C, ws]
    res = {n: [] for n in fns}
    names = list(fns)
    for rnd in range(7):
        for j in range(len(names)):
            n = names[(j + rnd) % len(names)]
            res[n].append(timed(fns[n], 2))
    fl = 2.0 * M * N * K
    med = {n: statistics.median(v) for n, v in res.items()}
    out = {n: round(fl / (ms * 1e-3) / 1e12, 1) for n, ms in med.items()}
    out.update({n + "_vs_classical": round(med["classical"] / med[n], 4) for n in names if n != "classical"})
    print(M, N, K, json.dumps(out), flush=True)
    del fns, keep, A, B
    torch.cuda.empty_cache()
