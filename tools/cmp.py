"""Interleaved timing of several (algo, static-B, LCMA_* env) arms on one shape.
usage: python tools/cmp.py M N K arm [arm ...]
  arm = name:algo[:s][:variant=NAME][:sched=S][:swz=H][:ENV=v,ENV2=w]
  (s = B precombined offline; ENV knobs need a -DLCMA_DIAG build via LCMA_LIB)
Prints per-arm median time, effective TFLOP/s and the ratio to the first arm."""
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


M, N, K = [int(v) for v in sys.argv[1:4]]
dtype = int(os.environ.get("DT", "0"))
bl = int(os.environ.get("BL", "1"))
rounds = int(os.environ.get("ROUNDS", "7"))
reps = int(os.environ.get("REPS", "3"))
A, B = inputs.operands(M, N, K, dtype, 1, 2, b_layout=bl)
A, B = A.cuda(), B.cuda()
arms = []
keys = set()
for spec in sys.argv[4:]:
    parts = spec.split(":")
    name, algo = parts[0], parts[1]
    static = "s" in parts[2:]
    variant = next((q.split("=", 1)[1] for q in parts[2:] if q.startswith("variant=")), "auto")
    # plan fields: sched=<schedule>, swz=<raster_rows>
    kw = {}
    for q in parts[2:]:
        for key, field in (("sched=", "schedule"), ("swz=", "raster_rows")):
            if q.startswith(key):
                kw[field] = int(q.split("=", 1)[1])
    envp = [q for q in parts[2:] if "=" in q and not q.startswith(("variant=", "sched=", "swz="))]
    env = dict(kv.split("=") for kv in (envp[-1].split(",") if envp else []))
    keys |= set(env)
    p = L.Plan(M, N, K, dtype=dtype, algo=algo, b_layout=bl, b_static=static, variant=variant, **kw)
    C = p.empty_c(); ws = p.workspace()
    Bt = p.precombine_b(B) if static else None
    f = (lambda p=p, Bt=Bt, C=C, ws=ws: p.gemm_precombined(A, Bt, C, ws)) if static else \
        (lambda p=p, C=C, ws=ws: p.gemm(A, B, C, ws))
    arms.append((name, env, f, (p, C, ws, Bt)))


def setenv(env):
    for k in keys: os.environ.pop(k, None)
    os.environ.update(env)


res = {a[0]: [] for a in arms}
for rnd in range(rounds):
    for j in range(len(arms)):
        name, env, f, _ = arms[(j + rnd) % len(arms)]
        setenv(env)
        res[name].append(timed(f, reps))
fl = 2.0 * M * N * K
base = statistics.median(res[arms[0][0]])
for name, env, _, _ in arms:
    ms = statistics.median(res[name])
    print(json.dumps({"shape": [M, N, K], "arm": name, "env": env, "us": round(ms * 1e3, 1),
                      "TF": round(fl / ms / 1e9, 1), "speedup_vs_first": round(base / ms, 4)}), flush=True)
