"""Seeded synthetic inputs shared by tests, bench.py and the oracle harness.

Holds none of the method's arithmetic: it only draws matrices.  Recipes
(DESIGN.md section "Inputs"): U[-1,1) (default, the paper states no
distribution -- S:521), U[0,1) (positive mean, makes the normwise gate
sensitive), and small integers for exact parity ([-2,2] for Strassen,
{-1,0,1} for Laderman / Strassen^2 so every intermediate stays < 2^21).
Values are drawn in fp32 from a seeded torch.Generator on the CPU and cast
(RN) to the storage dtype; the oracle receives host copies of the exact same
values.
"""
from __future__ import annotations

import torch

_TORCH_DT = {0: torch.bfloat16, 1: torch.float16, 2: torch.float32, 3: torch.float32,
             4: torch.bfloat16}   # 4 = FP8 path: bf16 inputs


def seed_for(cfg: int, idx: int, which: str) -> int:
    """s_A = 100*cfg + 2*i + 1, s_B = 100*cfg + 2*i + 2."""
    return 100 * cfg + 2 * idx + (1 if which == "A" else 2)


def matrix(rows: int, cols: int, dtype_code: int, seed: int, dist: str = "uniform",
           lo: int = -2, hi: int = 2) -> torch.Tensor:
    g = torch.Generator(device="cpu")
    g.manual_seed(seed)
    if dist == "uniform":
        x = torch.rand((rows, cols), generator=g, dtype=torch.float32) * 2.0 - 1.0
    elif dist == "uniform_coarse":
        # U[-1,1) with |x| < 2^-8 set to 0: after the bf16 cast every value
        # has an exponent in [-8, -1], so fp32 sums of a few of them are exact
        # (the FP8 tests compare quantized bytes bit for bit)
        x = torch.rand((rows, cols), generator=g, dtype=torch.float32) * 2.0 - 1.0
        x = torch.where(x.abs() < 2.0 ** -8, torch.zeros_like(x), x)
    elif dist == "positive":
        x = torch.rand((rows, cols), generator=g, dtype=torch.float32)
    elif dist == "int":
        x = torch.randint(lo, hi + 1, (rows, cols), generator=g, dtype=torch.int32).to(torch.float32)
    else:
        raise ValueError(dist)
    return x.to(_TORCH_DT[dtype_code])


def operands(M: int, N: int, K: int, dtype_code: int, seed_a: int, seed_b: int,
             dist: str = "uniform", b_layout: int = 0, lo: int = -2, hi: int = 2):
    """A (M x K) and B (K x N if b_layout == 0, else N x K), host tensors."""
    A = matrix(M, K, dtype_code, seed_a, dist, lo, hi)
    B = matrix(K, N, dtype_code, seed_b, dist, lo, hi) if b_layout == 0 else \
        matrix(N, K, dtype_code, seed_b, dist, lo, hi)
    return A, B
