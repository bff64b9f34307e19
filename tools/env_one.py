"""Median time of one plan in a fresh process under the current LCMA_* env.
usage: python tools/env_one.py ALGO static|dyn M N K [rounds]"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs

algo, mode = sys.argv[1], sys.argv[2]
M, N, K = [int(v) for v in sys.argv[3:6]]
rounds = int(sys.argv[6]) if len(sys.argv) > 6 else 7
A, B = inputs.operands(M, N, K, 0, 1, 2, b_layout=1)
A, B = A.cuda(), B.cuda()
p = L.Plan(M, N, K, dtype=0, algo=algo, b_layout=1, b_static=(mode == "static"))
C = p.empty_c(); ws = p.workspace()
Bt = p.precombine_b(B) if mode == "static" else None
f = (lambda: p.gemm_precombined(A, Bt, C, ws)) if Bt is not None else (lambda: p.gemm(A, B, C, ws))
for _ in range(3): f()
torch.cuda.synchronize()
ts = []
for _ in range(rounds):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): f()
    e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1) / 3 * 1e3)
env = {k: v for k, v in os.environ.items() if k.startswith("LCMA_")}
us = statistics.median(ts)
print(f"{algo} {mode} {M}x{N}x{K} {env}: median {us:9.1f} us ({2*M*N*K/us/1e6:7.1f} TF) min {min(ts):9.1f}", flush=True)
