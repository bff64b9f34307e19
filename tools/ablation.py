"""Execution-Module ablation on B200 (the paper's step-wise
study P:475-491): Alg. 1 -> Group-Parallel -> Split-Group -> Cache-Aware ->
product order (partials in L2) -> on-chip partial homes (registers, shared
memory), the producer-fused combine variant, plus diagnostics (mainloop only;
producer-side combine traffic).  Interleaved timing (median of rounds).

usage: python tools/ablation.py [M N K] [--static]   -> JSON on stdout
       ABL_ONE=<name> python tools/ablation.py ...   -> one launch (for ncu)
"""
import json, os, statistics, sys
os.environ.setdefault("LCMA_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)).split("/tools")[0], "paper_2605_06057_b200", "liblcma_diag.so"))  # env knobs: -DLCMA_DIAG build
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs

args = [a for a in sys.argv[1:] if not a.startswith("--")]
M, N, K = [int(v) for v in args[:3]] if len(args) >= 3 else (8192, 14336, 4096)
static = "--static" in sys.argv
ALGO = os.environ.get("ABL_ALGO", "strassen")

# name -> (plan kwargs, env)
STEPS = {
    "classical": (dict(algo="classical"), {}),
    "alg1_unfused": (dict(algo=ALGO, variant="unfused"), {}),
    "group_parallel": (dict(algo=ALGO, schedule=3), {"LCMA_ORDER": "0", "LCMA_DISCARD": "0"}),
    "split_group_paper": (dict(algo=ALGO, schedule=2), {"LCMA_ORDER": "0", "LCMA_DISCARD": "0"}),
    "cache_aware_lockstep": (dict(algo=ALGO, schedule=1), {"LCMA_ORDER": "0", "LCMA_DISCARD": "0"}),
    "product_order_slots_discard": (dict(algo=ALGO, schedule=1),
                                    {"LCMA_REG_PARTIAL": "0", "LCMA_SMEM_PARTIAL": "0"}),
    "onchip_partial_homes": (dict(algo=ALGO, schedule=1), {}),
    "variant3_producer_combine": (dict(algo=ALGO, variant="producer"), {}),
    "diag_mainloop_only": (dict(algo=ALGO), {"LCMA_DEBUG": "1"}),
    "diag_producer_combine_traffic": (dict(algo=ALGO), {"LCMA_DEBUG": "33"}),
    "diag_classical_mainloop_only": (dict(algo="classical"), {"LCMA_DEBUG": "1"}),
}
ENV_KEYS = {k for _, e in STEPS.values() for k in e}

A, B = inputs.operands(M, N, K, 0, 1, 2, b_layout=1)
A, B = A.cuda(), B.cuda()
runs = {}
for name, (kw, env) in STEPS.items():
    if os.environ.get("ABL_ONE") and name != os.environ["ABL_ONE"]:
        continue
    st = static and kw["algo"] != "classical"
    p = L.Plan(M, N, K, dtype=0, b_layout=1, b_static=st, **kw)
    C = p.empty_c(); ws = p.workspace()
    Bt = p.precombine_b(B) if st else None
    f = (lambda p=p, C=C, ws=ws, Bt=Bt: p.gemm_precombined(A, Bt, C, ws)) if st else \
        (lambda p=p, C=C, ws=ws: p.gemm(A, B, C, ws))
    runs[name] = (f, env, p.info)


def setenv(env):
    for k in ENV_KEYS:
        os.environ.pop(k, None)
    os.environ.update(env)


if os.environ.get("ABL_ONE"):
    f, env, _ = runs[os.environ["ABL_ONE"]]
    setenv(env)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    sys.exit(0)


def timed(f, reps=5):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


res = {n: [] for n in runs}
names = list(runs)
for rnd in range(5):
    for j in range(len(names)):
        n = names[(j + rnd) % len(names)]
        f, env, _ = runs[n]
        setenv(env)
        res[n].append(timed(f))
# clock / power under sustained load per step (the paper's L2 thrash
# lowered the H20's clock from 1.80 to 1.61 GHz): each arm runs back to back
# for ~1 s while nvidia-smi samples SM clock and board power every 50 ms
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler
import time
power = {}
for n in names:
    f, env, _ = runs[n]
    setenv(env)
    f(); torch.cuda.synchronize()
    smp = ClockSampler(torch.cuda.current_device())
    smp.start()
    time.sleep(0.2)
    t_end = time.time() + 1.0
    while time.time() < t_end:
        for _ in range(8):
            f()
        torch.cuda.synchronize()
    smp.stop()
    vals = []
    for ln in smp.lines:
        parts = [x.strip() for x in ln.split(",")]
        try:
            vals.append((float(parts[0]), float(parts[2])))
        except (ValueError, IndexError):
            pass
    load = vals[len(vals) // 4:] or vals
    power[n] = {"sm_mhz_median": statistics.median(v[0] for v in load) if load else None,
                "power_w_median": statistics.median(v[1] for v in load) if load else None,
                "samples": len(load)}
setenv({})
fl = 2.0 * M * N * K
out = {"shape": [M, N, K], "algo": ALGO, "b_static": static, "b_layout": "NxK",
       "timing": "median of 5 interleaved rounds x 5 calls, CUDA events", "steps": {}}
for n in names:
    ms = statistics.median(res[n])
    info = runs[n][2]
    out["steps"][n] = {"ms": ms, "eff_tflops": fl / (ms * 1e-3) / 1e12,
                       "waves": info.get("waves"), "split_groups": info.get("split_groups"),
                       "env": runs[n][1], **power.get(n, {})}
print(json.dumps(out, indent=1))
