import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.kprof import prof
M, N, K = 8192, 14336, 4096
for env in ({"LCMA_OLD_COMBINE": "1"}, {}):
    os.environ.pop("LCMA_OLD_COMBINE", None); os.environ.update(env)
    print(env, flush=True)
    prof(M, N, K, "strassen")
    prof(M, N, K, "laderman", static_b=True)
    prof(M, N, K, "strassen2", static_b=True)
