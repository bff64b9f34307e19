import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.kprof import prof
import paper_2605_06057_b200 as L
for dt in (0, 1, 2):
    M, N, K = 16384, 28672, 8192
    print("=== dtype", dt, M, N, K, flush=True)
    prof(M, N, K, "classical", reps=4, dtype=dt)
    prof(M, N, K, "strassen", reps=4, dtype=dt)
    prof(M, N, K, "strassen", static_b=True, reps=4, dtype=dt)
    p = L.Plan(M, N, K, dtype=dt, algo="auto", b_static=True)
    print("auto(static):", p.info["scheme"], round(p.info["speedup_pred"], 3), flush=True)
