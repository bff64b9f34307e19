"""BASELINE cfg4: Laderman <3,3,3;23> and Strassen^2 <4,4,4;49> at 12288^3 bf16
(with Strassen and classical for context).  Reports interleaved median times,
the rank / memory-overhead trade-off (workspace, B~ bytes, live partial tiles)
and the tile plan.  ABL_ONE=<algo> runs a single launch for ncu.
usage: python tools/cfg4.py > profiles/r01c_cfg4.json"""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs

M = N = K = 12288
A, B = inputs.operands(M, N, K, 0, 401, 402, b_layout=1)
A, B = A.cuda(), B.cuda()
arms = {}
for algo in ("classical", "strassen", "laderman", "strassen2"):
    if os.environ.get("ABL_ONE") and os.environ["ABL_ONE"] != algo:
        continue
    for static in ((False, True) if algo != "classical" else (False,)):
        p = L.Plan(M, N, K, dtype=0, algo=algo, b_layout=1, b_static=static)
        C = p.empty_c()
        ws = p.workspace()
        if static:
            Bt = p.precombine_b(B)
            f = (lambda p=p, Bt=Bt, C=C, ws=ws: p.gemm_precombined(A, Bt, C, ws))
        else:
            f = (lambda p=p, C=C, ws=ws: p.gemm(A, B, C, ws))
        arms[algo + ("_static_b" if static else "")] = (f, p.info)
if os.environ.get("ABL_ONE"):
    f, _ = arms[os.environ["ABL_ONE"]]
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    sys.exit(0)


def timed(f, reps=3):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


names = list(arms)
res = {n: [] for n in names}
for rnd in range(5):
    for j in range(len(names)):
        n = names[(j + rnd) % len(names)]
        res[n].append(timed(arms[n][0]))
fl = 2.0 * M * N * K
out = {"shape": [M, N, K], "dtype": "bf16", "b_layout": "NxK",
       "timing": "median of 5 interleaved rounds x 3 calls, CUDA events", "arms": {}}
cl = statistics.median(res["classical"])
for n in names:
    ms = statistics.median(res[n])
    i = arms[n][1]
    out["arms"][n] = {
        "ms": ms, "eff_tflops": fl / (ms * 1e-3) / 1e12, "vs_classical": cl / ms,
        "real_mma_tflop": 2.0 * i["R"] * i["Mb"] * i["Nb"] * i["Kb"] / 1e12 if i["R"] > 1 else fl / 1e12,
        "R": i["R"], "scheme": i["scheme"].decode() if isinstance(i["scheme"], bytes) else i["scheme"],
        "Mb_Nb_Kb": [i["Mb"], i["Nb"], i["Kb"]], "tile": [i["BM"], i["BN"], i["BK"]],
        "cta_group": i["cta_group"], "groups": i["groups"], "waves": i["waves"],
        "workspace_MiB": i["workspace_bytes"] / 2 ** 20, "btilde_MiB": i["btilde_bytes"] / 2 ** 20,
        "partial_slots_per_cta": i["partial_slots"],
        "partial_MiB_live": i["partial_slots"] * 128 * i["BN"] * 4 * i["ctas"] / 2 ** 20,
    }
print(json.dumps(out, indent=1))
