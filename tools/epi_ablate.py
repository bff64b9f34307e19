import os, sys
os.environ.setdefault("LCMA_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)).split("/tools")[0], "paper_2605_06057_b200", "liblcma_diag.so"))  # env knobs: -DLCMA_DIAG build
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.kprof import prof
M, N, K = 8192, 14336, 4096
for dbg in ("0", "1", "2", "4", "8", "6", "14"):
    os.environ["LCMA_DEBUG"] = dbg
    print("debug", dbg, flush=True)
    prof(M, N, K, "strassen", static_b=True)
