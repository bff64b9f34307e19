"""cfg3 sweep (BASELINE.json configs[2]): M = 4096..16384 step 2048, (N,K) in
{(4096,4096), (14336,4096), (4096,14336), (14336,14336)}, fp16 and tf32.
Every candidate (classical, Strassen, Strassen^2, Laderman; fused Combine H,
Combine B per call) is timed with CUDA events; the Decision Module's choice
(calibrated B200 model and the paper's model) is scored by regret =
t(chosen) / t(best measured).  Writes profiles/r01_cfg3_decision.json."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs

ALGOS = ["classical", "strassen", "strassen2", "laderman"]
NAME = {"classical": "classical", "strassen-2x2x2-r7": "strassen", "strassen2-4x4x4-r49": "strassen2",
        "laderman-3x3x3-r23": "laderman"}


def timeit(f, reps=5, warm=2):
    for _ in range(warm):
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        f()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / reps


def main():
    quick = "--quick" in sys.argv
    Ms = [4096, 10240, 16384] if quick else list(range(4096, 16385, 2048))
    NKs = [(4096, 4096), (14336, 4096), (4096, 14336), (14336, 14336)]
    rows = []
    for dtype in (L.FP16, L.TF32):
        for (N, K) in NKs:
            for M in Ms:
                A, B = inputs.operands(M, N, K, dtype, 301, 302)
                A, B = A.cuda(), B.cuda()
                t = {}
                for algo in ALGOS:
                    p = L.Plan(M, N, K, dtype=dtype, algo=algo)
                    C = p.empty_c()
                    ws = p.workspace()
                    t[algo] = timeit(lambda: p.gemm(A, B, C, ws))
                    del ws, C, p
                # Combine B offline (static weights): for model fitting only
                ps = L.Plan(M, N, K, dtype=dtype, algo="strassen", b_static=True)
                Cs, wss = ps.empty_c(), ps.workspace()
                Bts = ps.precombine_b(B)
                t_sb = timeit(lambda: ps.gemm_precombined(A, Bts, Cs, wss))
                del ps, Cs, wss, Bts
                auto = L.Plan(M, N, K, dtype=dtype, algo="auto")
                paper = L.Plan(M, N, K, dtype=dtype, algo="auto", decision_model=1)
                best = min(t, key=t.get)
                ch, chp = NAME[auto.info["scheme"]], NAME[paper.info["scheme"]]
                row = {"dtype": {1: "fp16", 2: "tf32"}[dtype], "M": M, "N": N, "K": K,
                       "ms": {k: round(v, 4) for k, v in t.items()},
                       "eff_tflops": {k: round(2 * M * N * K / v / 1e9, 1) for k, v in t.items()},
                       "best": best, "auto_b200": ch, "auto_paper": chp,
                       "regret_b200": round(t[ch] / t[best], 4), "regret_paper": round(t[chp] / t[best], 4),
                       "pred_speedup_b200": round(auto.info["speedup_pred"], 4),
                       "strassen_static_b_ms": round(t_sb, 4)}
                rows.append(row)
                print(json.dumps(row), flush=True)
                del A, B
                torch.cuda.empty_cache()
    n = len(rows)
    summ = {
        "cases": n,
        "b200_model_correct": sum(r["auto_b200"] == r["best"] for r in rows),
        "paper_model_correct": sum(r["auto_paper"] == r["best"] for r in rows),
        "b200_mean_regret": sum(r["regret_b200"] for r in rows) / n,
        "paper_mean_regret": sum(r["regret_paper"] for r in rows) / n,
        "b200_max_regret": max(r["regret_b200"] for r in rows),
        "paper_max_regret": max(r["regret_paper"] for r in rows),
        "lcma_best_cases": sum(r["best"] != "classical" for r in rows),
    }
    print(json.dumps(summ), flush=True)
    os.makedirs("profiles", exist_ok=True)
    out = os.environ.get("CFG3_OUT", "gpurun_out/r01_cfg3_decision.json")
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    with open(out, "w") as f:
        json.dump({"summary": summ, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
