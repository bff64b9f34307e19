import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.kprof import prof
import paper_2605_06057_b200 as L
for (M, N, K) in [(12288, 12288, 12288), (16384, 28672, 8192)]:
    print("=== shape", M, N, K, flush=True)
    prof(M, N, K, "classical", reps=3)
    prof(M, N, K, "strassen", reps=3)
    prof(M, N, K, "strassen", static_b=True, reps=3)
    prof(M, N, K, "strassen", variant="unfused", reps=3)
    prof(M, N, K, "laderman", static_b=True, reps=3)
    prof(M, N, K, "strassen2", static_b=True, reps=3)
    print(L.decide(M, N, K), flush=True)
