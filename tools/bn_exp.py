import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.kprof import prof
M, N, K = 8192, 14336, 4096
for bn in ("256", "128"):
    os.environ["LCMA_BN"] = bn
    print("BN", bn)
    prof(M, N, K, "classical")
    prof(M, N, K, "classical", b_layout=1)
    prof(M, N, K, "strassen", static_b=True)
    prof(M, N, K, "strassen", variant="unfused", static_b=True)
