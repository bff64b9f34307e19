"""Combine A+B time inside a tf32 / bf16 Strassen call (per-kernel CUPTI times)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.kseq import seq
seq(8192, 14336, 4096, "strassen", dtype=2, reps=2)
seq(8192, 14336, 4096, "strassen", dtype=0, reps=2)
