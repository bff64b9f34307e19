"""GPU parity of the FP8 E4M3 path (reading 23)
through the C ABI against the CPU oracle.

* quantized operands: the combine kernels' E4M3 bytes and UE8M0 scale chunks
  equal oracle.combine_b_fp8 / combine_a_fp8_rows bit for bit (inputs whose
  fp32 combine sums are exact);
* exact mode: small-integer inputs are represented exactly by the 1 x 128
  quantization, so C (fp32) equals A.B exactly for every scheme;
* float mode: C equals the oracle's FP8 emulation (exact quantized products,
  fp64 sums) up to fp32 accumulation (eps_rel <= 1e-5, ~500x below the E4M3
  error itself), and meets the FP8 gate eps_norm <= 0.1 / sqrt(K) against
  the exact GEMM;
* full size (cfg2 shape): sampled rows against the emulation, bf16 output
  within one bf16 rounding.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2605_06057_b200 import inputs

pytestmark = pytest.mark.gpu

L = pytest.importorskip("paper_2605_06057_b200")

SCHEMES = {"classical": lambda: O.standard(1, 1, 1), "strassen": O.strassen, "strassen2": O.strassen2,
           "laderman": O.laderman}
INT_RANGE = {"classical": (-4, 4), "strassen": (-2, 2), "strassen2": (-1, 1), "laderman": (-1, 1)}


def fp8_gate(s, K):
    """FP8 normwise gate (reading 23): 0.1 / sqrt(K) for the
    classical product, scaled by sqrt(T / mkn) with T = sum_r nnz(U_r)
    nnz(V_r) nnz(W_r) the elementary product terms the scheme's C entries
    carry (each carries an independent quantization error; mkn for the
    classical block product): Strassen sqrt(32/8) = 2, Strassen^2 4."""
    T = sum(int((s.U[r] != 0).sum()) * int((s.V[r] != 0).sum()) * int((s.W[r] != 0).sum())
            for r in range(s.R))
    return 0.1 * np.sqrt(T / (s.m * s.k * s.n)) / np.sqrt(K)


def _ext(plan):
    return plan.info["Mb"], plan.info["Kb"], plan.info["Nb"]


def _scales_from_chunks(buf, R, rows, Kb):
    """UE8M0 chunk bytes [R][rows/128][Kb/128][512] -> exponents [R][rows][Kb/128]."""
    sf = buf.reshape(R, rows // 128, Kb // 128, 512)
    n = np.arange(rows)
    off = (n % 32) * 16 + (n % 128 // 32) * 4
    out = np.empty((R, rows, Kb // 128), np.int64)
    for kb in range(Kb // 128):
        for j in range(4):                                   # the four 32-K slots agree
            e = sf[:, n // 128, kb, off + j].astype(np.int64) - 127
            if j == 0:
                out[:, :, kb] = e
            else:
                assert np.array_equal(out[:, :, kb], e)
    return out


def _split_q(buf, R, rows, Kb):
    q = torch.from_numpy(buf[:R * rows * Kb].copy()).view(torch.float8_e4m3fn).float().double().numpy()
    e = _scales_from_chunks(buf[R * rows * Kb:R * rows * Kb + R * rows * (Kb // 128) * 4], R, rows, Kb)
    return q.reshape(R, rows, Kb), e


@pytest.mark.parametrize("algo", ["classical", "strassen", "laderman", "strassen2"])
def test_fp8_quantized_b_bitexact(algo):
    M, N, K = 520, 600, 704
    A, B = inputs.operands(M, N, K, L.FP8, 41, 42, dist="uniform_coarse", b_layout=1)
    plan = L.Plan(M, N, K, dtype=L.FP8, algo=algo, b_layout=1)
    Mb, Kb, Nb = _ext(plan)
    s = SCHEMES[algo]()
    Bt = plan.precombine_b(B.cuda()).cpu().numpy()
    q, e = _split_q(Bt, s.R, Nb, Kb)
    Qo, Eo = O.combine_b_fp8(B.double().numpy().T, s, (Mb, Kb, Nb))
    assert np.array_equal(e, Eo), int((e != Eo).sum())
    assert np.array_equal(q, Qo), int((q != Qo).sum())


@pytest.mark.parametrize("algo", ["classical", "strassen"])
def test_fp8_quantized_a_bitexact(algo):
    # Combine A with the fused quantization: read back from the
    # workspace (A~ E4M3 [R][Mb][Kb] + scale chunks at the start of the A~
    # region, lcma.h workspace layout) after a call
    M, N, K = 1000, 256, 520
    A, B = inputs.operands(M, N, K, L.FP8, 43, 44, dist="uniform_coarse", b_layout=1)
    plan = L.Plan(M, N, K, dtype=L.FP8, algo=algo, b_layout=1)
    Mb, Kb, Nb = _ext(plan)
    s = SCHEMES[algo]()
    ws = plan.workspace()
    plan.gemm(A.cuda(), B.cuda(), workspace=ws)
    torch.cuda.synchronize()
    off = plan.workspace_region(0)
    buf = ws.cpu().numpy()[off:]
    q, e = _split_q(buf, s.R, Mb, Kb)
    Qo, Eo = O.combine_a_fp8_rows(A.double().numpy(), s, np.arange(Mb), (Mb, Kb, Nb))
    assert np.array_equal(e, Eo) and np.array_equal(q, Qo)


@pytest.mark.parametrize("algo,shape", [
    ("classical", (256, 128, 128)), ("classical", (600, 520, 400)), ("classical", (1300, 1104, 1032)),
    ("strassen", (512, 256, 256)), ("strassen", (1200, 1040, 800)), ("strassen", (2100, 1800, 1304)),
    ("laderman", (780, 800, 904)), ("strassen2", (1024, 1024, 1024))])
def test_fp8_exact_small_int(algo, shape):
    M, N, K = shape
    lo, hi = INT_RANGE[algo]
    A, B = inputs.operands(M, N, K, L.FP8, M + 3, N + K, dist="int", b_layout=1, lo=lo, hi=hi)
    plan = L.Plan(M, N, K, dtype=L.FP8, algo=algo, b_layout=1, out_dtype=L.FP32)
    C = plan.gemm(A.cuda(), B.cuda()).cpu().double().numpy()
    Ad, Bd = A.double().numpy(), B.double().numpy().T
    ref = Ad @ Bd
    # the oracle's FP8 workflow at the GPU's extents is exact here too
    rows = np.array([0, M // 2, M - 1])
    assert np.array_equal(O.lcma_rows_fp8(Ad, Bd, SCHEMES[algo](), rows, _ext(plan)), ref[rows])
    bad = np.argwhere(C != ref)
    assert bad.size == 0, f"{len(bad)} mismatches, first {bad[:3].tolist()}"


@pytest.mark.parametrize("algo,shape,dist", [
    ("classical", (600, 520, 400), "uniform"), ("classical", (1000, 1048, 1032), "positive"),
    ("strassen", (1200, 1040, 800), "uniform"), ("strassen", (1000, 1048, 1032), "positive"),
    ("laderman", (780, 800, 904), "uniform"), ("strassen2", (1024, 1024, 1024), "uniform")])
def test_fp8_matches_emulation(algo, shape, dist):
    M, N, K = shape
    A, B = inputs.operands(M, N, K, L.FP8, 7 * M + 1, 5 * N + 2, dist=dist, b_layout=1)
    plan = L.Plan(M, N, K, dtype=L.FP8, algo=algo, b_layout=1, out_dtype=L.FP32)
    C = plan.gemm(A.cuda(), B.cuda()).cpu().double().numpy()
    Ad, Bd = A.double().numpy(), B.double().numpy().T
    rows = np.unique(np.linspace(0, M - 1, 48).astype(np.int64))
    em = O.lcma_rows_fp8(Ad, Bd, SCHEMES[algo](), rows, _ext(plan))
    # fp32 accumulation of exact E4M3 products: far below the E4M3 error
    assert O.eps_rel(C[rows], em) <= 1e-5
    # the FP8 gate against the exact product (reading 23)
    ref = O.gemm_rows_f64(Ad, Bd, rows)
    e = O.eps_norm(C[rows], ref, Ad[rows], Bd)
    assert e <= fp8_gate(SCHEMES[algo](), K), e


def test_fp8_bf16_output_and_static_b():
    M, N, K = 1200, 1040, 800
    A, B = inputs.operands(M, N, K, L.FP8, 51, 52, b_layout=1)
    for algo in ("classical", "strassen"):
        p = L.Plan(M, N, K, dtype=L.FP8, algo=algo, b_layout=1)          # C bf16
        C = p.gemm(A.cuda(), B.cuda())
        assert C.dtype == torch.bfloat16
        Bt = p.precombine_b(B.cuda())
        C2 = p.gemm_precombined(A.cuda(), Bt)
        assert torch.equal(C, C2)                  # offline quantized B~ == per call, bitwise
        pf = L.Plan(M, N, K, dtype=L.FP8, algo=algo, b_layout=1, out_dtype=L.FP32)
        Cf = pf.gemm(A.cuda(), B.cuda()).cpu().double().numpy()
        # one RN rounding of the fp32 result (ties aside): within half a bf16 ulp
        d = np.abs(C.float().cpu().double().numpy() - Cf)
        assert np.all(d <= np.abs(Cf) * 2.0 ** -8 + 1e-30)


def test_fp8_full_size_cfg2_sampled():
    # BASELINE cfg2 shape, the launch configuration bench.py times (B~ offline)
    M, N, K = 8192, 14336, 4096
    A, B = inputs.operands(M, N, K, L.FP8, 201, 202, b_layout=1)
    Ad, Bd = A.double().numpy(), B.double().numpy().T
    rows = np.array([0, 1, 4095, 4096, 6000, 8191])
    for algo in ("strassen", "classical"):
        p = L.Plan(M, N, K, dtype=L.FP8, algo=algo, b_layout=1)
        Bt = p.precombine_b(B.cuda())
        C = p.gemm_precombined(A.cuda(), Bt).cpu()[rows].double().numpy()
        em = O.lcma_rows_fp8(Ad, Bd, SCHEMES[algo](), rows, _ext(p))
        d = np.abs(C - em)
        assert np.all(d <= np.abs(em) * 2.0 ** -8 + 1e-3 * np.abs(em).max()), float(d.max())
        assert O.eps_rel(C, em) < 4e-3
        assert O.eps_norm(C, O.gemm_rows_f64(Ad, Bd, rows), Ad[rows], Bd) <= fp8_gate(SCHEMES[algo](), K)


def test_fp8_gate_term_counts():
    assert np.isclose(fp8_gate(O.standard(1, 1, 1), 100), 0.01)
    assert np.isclose(fp8_gate(O.strassen(), 100), 0.02)          # T = 32 (hand count), mkn = 8
    assert np.isclose(fp8_gate(O.strassen2(), 100), 0.04)         # T = 32^2, mkn = 64


def test_fp8_api_rules():
    with pytest.raises(L.LcmaError):
        L.Plan(512, 512, 512, dtype=L.FP8, algo="strassen", b_layout=0)        # B must be N x K
    with pytest.raises(L.LcmaError):
        L.Plan(512, 512, 512, dtype=L.FP8, algo="strassen", b_layout=1, variant="producer")
    p = L.Plan(512, 512, 512, dtype=L.FP8, algo="strassen", b_layout=1)
    assert p.info["BN"] == 128 and p.info["BK"] == 128 and p.btilde_bytes == 7 * 256 * 256 + 7 * 256 * 2 * 4
