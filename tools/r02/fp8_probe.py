"""FP8 bring-up probe: exact small cases that separate the block-scale
semantics (per-row A scales, per-column B scales, pair halves)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_2605_06057_b200 as L
import oracle as O

torch.manual_seed(0)


def run(M, N, K, algo, A, B):
    p = L.Plan(M, N, K, dtype=L.FP8, algo=algo, b_layout=1, out_dtype=L.FP32)
    C = p.gemm(A.cuda(), B.cuda())
    torch.cuda.synchronize()
    return C.cpu().double().numpy(), p


def report(name, got, ref):
    bad = np.argwhere(got != ref)
    print(f"{name}: bad {len(bad)} / {ref.size}", flush=True)
    if len(bad):
        rows = np.unique(bad[:, 0]); cols = np.unique(bad[:, 1])
        print("  bad rows", rows[:20], "... n", len(rows), " bad cols", cols[:20], "... n", len(cols))
        i, j = bad[0]
        with np.errstate(divide="ignore", invalid="ignore"):
            ratio = got[bad[:, 0], bad[:, 1]] / ref[bad[:, 0], bad[:, 1]]
        print("  first", (i, j), got[i, j], ref[i, j], "ratios", np.unique(np.round(ratio, 4))[:12])


for algo in ("classical", "strassen"):
    for (M, N, K) in ((256, 128, 128), (512, 256, 256), (600, 520, 400)):
        Mx, Nx, Kx = (2 * M, 2 * N, 2 * K) if algo == "strassen" else (M, N, K)
        A = torch.randint(-2, 3, (Mx, Kx)).to(torch.bfloat16)
        B = torch.randint(-2, 3, (Nx, Kx)).to(torch.bfloat16)     # N x K
        ref = A.double().numpy() @ B.double().numpy().T
        got, p = run(Mx, Nx, Kx, algo, A, B)
        report(f"{algo} {Mx}x{Nx}x{Kx} ints", got, ref)
        # per-row scales of A (powers of two by row), per-column scales of B
        rs = torch.tensor([2.0 ** ((i % 7) - 3) for i in range(Mx)])
        cs = torch.tensor([2.0 ** ((j % 5) - 2) for j in range(Nx)])
        A2 = (A.float() * rs[:, None]).to(torch.bfloat16)
        got, _ = run(Mx, Nx, Kx, algo, A2, B)
        report(f"{algo} row-scaled A", got, A2.double().numpy() @ B.double().numpy().T)
        B2 = (B.float() * cs[:, None]).to(torch.bfloat16)
        got, _ = run(Mx, Nx, Kx, algo, A, B2)
        report(f"{algo} col-scaled B", got, A.double().numpy() @ B2.double().numpy().T)
        # k-block varying scales
        ks = torch.tensor([2.0 ** ((k // 128) % 3 - 1) for k in range(Kx)])
        A3 = (A.float() * ks[None, :]).to(torch.bfloat16)
        got, _ = run(Mx, Nx, Kx, algo, A3, B)
        report(f"{algo} k-scaled A", got, A3.double().numpy() @ B.double().numpy().T)
print("probe done")

# quantized B~ bytes vs the oracle (inputs whose fp32 combine sums are exact)
M, N, K = 512, 512, 512
B = torch.empty(N, K).uniform_(-1, 1)
B[B.abs() < 2 ** -8] = 0
B = B.to(torch.bfloat16)
p = L.Plan(M, N, K, dtype=L.FP8, algo="strassen", b_layout=1)
Bt = p.precombine_b(B.cuda()).cpu()
R, Nb, Kb = 7, p.info["Nb"], p.info["Kb"]
q = Bt[:R * Nb * Kb].view(torch.float8_e4m3fn).float().double().numpy().reshape(R, Nb, Kb)
sf = Bt[R * Nb * Kb:R * Nb * Kb + R * Nb * (Kb // 128) * 4].numpy().reshape(R, Nb // 128, Kb // 128, 512)
Qo, Eo = O.combine_b_fp8(B.double().numpy().T, O.strassen(), (p.info["Mb"], Kb, Nb))
print("B~ values equal:", np.array_equal(q, Qo), "mismatches", int((q != Qo).sum()))
n = np.arange(Nb)
e_gpu = np.stack([sf[:, n // 128, kb, (n % 32) * 16 + (n % 128 // 32) * 4].astype(np.int64) - 127
                  for kb in range(Kb // 128)], axis=2)
print("scales equal:", np.array_equal(e_gpu, Eo), "mismatches", int((e_gpu != Eo).sum()))
