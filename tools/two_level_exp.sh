for shape in "12288 12288 12288" "8192 14336 4096"; do
python tools/env_one.py classical dyn $shape 3 2>&1 | grep median
python tools/env_one.py strassen2 dyn $shape 3 2>&1 | grep median
python - <<PY 2>&1 | grep median
import os, sys, statistics
sys.path.insert(0, ".")
import torch, paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs
M,N,K=[int(v) for v in "$shape".split()]
A,B=inputs.operands(M,N,K,0,1,2,b_layout=1); A,B=A.cuda(),B.cuda()
for static in (False, True):
    p=L.Plan(M,N,K,dtype=0,algo="strassen2",b_layout=1,variant="two_level",b_static=static)
    C=p.empty_c(); ws=p.workspace()
    if static:
        Bt=p.precombine_b(B); f=lambda: p.gemm_precombined(A,Bt,C,ws)
    else:
        f=lambda: p.gemm(A,B,C,ws)
    for _ in range(3): f()
    torch.cuda.synchronize(); ts=[]
    for _ in range(5):
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record(); [f() for _ in range(3)]; e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1)/3*1e3)
    print("two_level static=%s %s median %.1f us" % (static, "$shape", statistics.median(ts)))
PY
done
