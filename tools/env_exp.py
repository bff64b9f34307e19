"""Interleaved timing of one plan under several LCMA_* environment settings.
usage: python tools/env_exp.py ALGO [static] M N K  'ENV1=a,ENV2=b' 'ENV3=c' ..."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


algo = sys.argv[1]
static = sys.argv[2] == "static"
M, N, K = [int(v) for v in sys.argv[3:6]]
envs = [dict(kv.split("=") for kv in e.split(",") if kv) for e in (sys.argv[6:] or [""])]
A, B = inputs.operands(M, N, K, 0, 1, 2, b_layout=1)
A, B = A.cuda(), B.cuda()
keys = sorted({k for e in envs for k in e})
res = {i: [] for i in range(len(envs))}
plans = []
for i, e in enumerate(envs):
    for k in keys: os.environ.pop(k, None)
    os.environ.update(e)
    p = L.Plan(M, N, K, dtype=0, algo=algo, b_layout=1, b_static=static)
    C = p.empty_c(); ws = p.workspace()
    Bt = p.precombine_b(B) if static else None
    plans.append((p, C, ws, Bt))
for rnd in range(5):
    for i, e in enumerate(envs):
        for k in keys: os.environ.pop(k, None)
        os.environ.update(e)
        p, C, ws, Bt = plans[i]
        f = (lambda: p.gemm_precombined(A, Bt, C, ws)) if static else (lambda: p.gemm(A, B, C, ws))
        res[i].append(t(f))
for i, e in enumerate(envs):
    us = statistics.median(res[i])
    print(f"{algo} static={static} {M}x{N}x{K} {e}: {us:9.1f} us  {2*M*N*K/us/1e6:7.1f} TF", flush=True)
