import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.kprof import prof
M, N, K = 8192, 14336, 4096
for dbg in ("0", "1", "2", "4", "8", "6", "14"):
    os.environ["LCMA_DEBUG"] = dbg
    print("debug", dbg, flush=True)
    prof(M, N, K, "strassen", static_b=True)
