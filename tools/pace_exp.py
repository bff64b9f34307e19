import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.kprof import prof
M, N, K = 8192, 14336, 4096
for ns in ("0", "500", "1000", "2000", "4000"):
    os.environ["LCMA_PACE_NS"] = ns
    print("pace", ns, flush=True)
    prof(M, N, K, "strassen", static_b=True)
