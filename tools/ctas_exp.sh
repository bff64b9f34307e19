for c in 148 136 124 112; do
python - <<PY 2>&1 | grep median
import os, sys, statistics
sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import torch, paper_2605_06057_b200 as L
from paper_2605_06057_b200 import inputs
M,N,K=8192,14336,4096
A,B=inputs.operands(M,N,K,0,1,2,b_layout=1); A,B=A.cuda(),B.cuda()
p=L.Plan(M,N,K,dtype=0,algo="strassen",b_layout=1,b_static=True,num_ctas=$c)
C=p.empty_c(); ws=p.workspace(); Bt=p.precombine_b(B)
f=lambda: p.gemm_precombined(A,Bt,C,ws)
for _ in range(3): f()
torch.cuda.synchronize(); ts=[]
for _ in range(7):
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record(); [f() for _ in range(3)]; e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1)/3*1e3)
print("ctas $c median", statistics.median(ts))
PY
done
