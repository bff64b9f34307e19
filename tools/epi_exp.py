import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.kprof import prof
M, N, K = 8192, 14336, 4096
for env in [{"LCMA_ORDER": "0", "LCMA_DISCARD": "0"}, {"LCMA_ORDER": "1", "LCMA_DISCARD": "0"},
            {"LCMA_ORDER": "0", "LCMA_DISCARD": "1"}, {"LCMA_ORDER": "1", "LCMA_DISCARD": "1"}]:
    os.environ.update(env)
    print(env, flush=True)
    prof(M, N, K, "strassen", static_b=True)
    prof(M, N, K, "laderman", static_b=True)
    prof(M, N, K, "strassen2", static_b=True)
