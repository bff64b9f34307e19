import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
torch.cuda.init()
import paper_2605_06057_b200 as L
p = L.Plan(8192, 14336, 4096, algo="classical")
print("pairs ctas", p.info["ctas"])
