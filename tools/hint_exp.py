import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.kprof import prof
M, N, K = 8192, 14336, 4096
for env in [{}, {"LCMA_PARTIAL_HINT": "1"}, {"LCMA_OPERAND_HINT": "1"}, {"LCMA_PARTIAL_HINT": "1", "LCMA_OPERAND_HINT": "1"}, {"LCMA_OPERAND_HINT": "2"}]:
    for k in ("LCMA_PARTIAL_HINT", "LCMA_OPERAND_HINT"): os.environ.pop(k, None)
    os.environ.update(env)
    print(env)
    prof(M, N, K, "strassen", static_b=True)
    if env.get("LCMA_OPERAND_HINT"): prof(M, N, K, "classical")
