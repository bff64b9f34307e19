"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Exact mode: small-integer inputs, fp32 C -> bit-exact equality with the int64
oracle (every intermediate < 2^21).  Float mode:
the BASELINE.json normwise gates plus eps_rel against the oracle's
dtype-faithful emulation at the plan's block extents.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2605_06057_b200 import inputs

pytestmark = pytest.mark.gpu

L = pytest.importorskip("paper_2605_06057_b200")

SCHEMES = {"strassen": O.strassen, "strassen2": O.strassen2, "laderman": O.laderman}
INT_RANGE = {"classical": (-4, 4), "strassen": (-2, 2), "strassen2": (-1, 1), "laderman": (-1, 1)}


def _b_dense(B, b_layout):
    return B if b_layout == 0 else B.t()


def _exact_case(M, N, K, algo, dtype=0, b_layout=0, variant="auto", **kw):
    lo, hi = INT_RANGE[algo]
    A, B = inputs.operands(M, N, K, dtype, M + 7, N + K, dist="int", b_layout=b_layout, lo=lo, hi=hi)
    plan = L.Plan(M, N, K, dtype=dtype, algo=algo, out_dtype=L.FP32, b_layout=b_layout,
                  variant=variant, **kw)
    C = plan.gemm(A.cuda(), B.cuda()).cpu().numpy()
    Ai = A.to(torch.int64).numpy()
    Bi = _b_dense(B, b_layout).to(torch.int64).numpy()
    ref = O.gemm_i64(Ai, Bi)
    if algo != "classical":
        # the method mirror at the GPU's block extents (Alg. 1, exact)
        lc = O.lcma_i64(Ai, Bi, SCHEMES[algo](), extents=(plan.info["Mb"], plan.info["Kb"], plan.info["Nb"]))
        assert np.array_equal(lc.C, ref)
        assert np.abs(ref).max() < 2 ** 21
    bad = np.argwhere(C != ref)
    assert bad.size == 0, f"{len(bad)} mismatches, first {bad[:3].tolist()}"
    return plan


@pytest.mark.parametrize("b_layout", [0, 1])
@pytest.mark.parametrize("shape", [(128, 256, 64), (256, 512, 128), (300, 264, 200),
                                   (1000, 1048, 520), (2304, 2560, 1024)])
def test_classical_exact_bf16(shape, b_layout):
    _exact_case(*shape, "classical", b_layout=b_layout)


@pytest.mark.parametrize("dtype", [1, 2])
def test_classical_exact_fp16_tf32(dtype):
    _exact_case(520, 776, 392, "classical", dtype=dtype)
    _exact_case(520, 776, 392, "classical", dtype=dtype, b_layout=1)


@pytest.mark.parametrize("variant", ["fused_h", "unfused"])
@pytest.mark.parametrize("b_layout", [0, 1])
@pytest.mark.parametrize("algo,shape", [
    ("strassen", (512, 512, 512)), ("strassen", (300, 264, 200)), ("strassen", (1000, 1560, 776)),
    ("strassen2", (1024, 1024, 512)), ("strassen2", (700, 1032, 264)),
    ("laderman", (768, 1536, 384)), ("laderman", (1000, 808, 520))])
def test_lcma_exact(algo, shape, b_layout, variant):
    _exact_case(*shape, algo, b_layout=b_layout, variant=variant)


@pytest.mark.parametrize("b_layout", [0, 1])
@pytest.mark.parametrize("shape", [(1024, 1024, 512), (700, 1032, 264), (2048, 3072, 1024)])
def test_two_level_exact(shape, b_layout):
    # Strassen^2 as Strassen o Strassen: inner fused GEMMs write the outer H_q
    # in fp32, the outer Combine H runs as an HBM pass (LCMA_VARIANT_TWO_LEVEL)
    plan = _exact_case(*shape, "strassen2", b_layout=b_layout, variant="two_level")
    assert plan.info["variant"] == L.VARIANT["two_level"] and plan.info["partial_slots"] == 2


def test_two_level_float_and_static_b():
    for dtype, gate in ((0, 2e-2), (1, 3e-3), (2, 3e-3)):
        e, er, er_emu, fv = _float_case(1032, 1544, 1032, "strassen2", dtype, variant="two_level")
        assert e <= gate and fv <= gate
        assert er <= 3.0 * er_emu + 1e-6, (er, er_emu)
    M, N, K = 1536, 2048, 1024
    A, B = inputs.operands(M, N, K, 0, 11, 12, b_layout=1)
    A, B = A.cuda(), B.cuda()
    p1 = L.Plan(M, N, K, dtype=L.BF16, algo="strassen2", b_layout=1, variant="two_level")
    p2 = L.Plan(M, N, K, dtype=L.BF16, algo="strassen2", b_layout=1, variant="two_level", b_static=True)
    assert torch.equal(p1.gemm(A, B), p2.gemm_precombined(A, p2.precombine_b(B)))
    with pytest.raises(L.LcmaError, match="NOT_SUPPORTED"):
        L.Plan(M, N, K, dtype=L.BF16, algo="laderman", variant="two_level")


@pytest.mark.parametrize("dtype", [1, 2])
def test_lcma_exact_fp16_tf32(dtype):
    _exact_case(512, 1024, 384, "strassen", dtype=dtype)
    _exact_case(1000, 520, 392, "strassen", dtype=dtype, b_layout=1)


@pytest.mark.parametrize("num_ctas,schedule", [(6, 0), (10, 0), (14, 2), (2, 0), (148, 2)])
def test_split_groups_exact(num_ctas, schedule):
    # forces tail groups split over several CTAs (segments merged by the owner)
    plan = _exact_case(1536, 2304, 512, "strassen", num_ctas=num_ctas, schedule=schedule)
    assert plan.info["split_groups"] > 0 or plan.info["groups"] % (plan.info["ctas"] // plan.info["cta_group"]) == 0
    _exact_case(1024, 1536, 256, "laderman", num_ctas=num_ctas, schedule=schedule)


def test_precombined_b_matches_oracle_intermediates():
    # Combine B (Eq. 4) materialised by lcma_precombine_b == oracle Bt, bitwise
    M, N, K = 520, 776, 392
    for b_layout in (0, 1):
        A, B = inputs.operands(M, N, K, 0, 3, 4, dist="int", b_layout=b_layout, lo=-2, hi=2)
        plan = L.Plan(M, N, K, dtype=L.BF16, algo="strassen", out_dtype=L.FP32, b_layout=b_layout)
        Bt = plan.precombine_b(B.cuda())
        Mb, Nb, Kb = plan.info["Mb"], plan.info["Nb"], plan.info["Kb"]
        lc = O.lcma_i64(A.to(torch.int64).numpy(), _b_dense(B, b_layout).to(torch.int64).numpy(),
                        O.strassen(), extents=(Mb, Kb, Nb), intermediates=True)
        g = Bt[: 7 * Kb * Nb * 2].view(torch.bfloat16).float().cpu().numpy()
        g = g.reshape(7, Kb, Nb) if b_layout == 0 else g.reshape(7, Nb, Kb).transpose(0, 2, 1)
        assert np.array_equal(g, lc.Bt.astype(np.float32))
        # and the precombined GEMM equals the full one bitwise
        Ad = A.cuda()
        C1 = plan.gemm(Ad, B.cuda())
        C2 = plan.gemm_precombined(Ad, Bt)
        assert torch.equal(C1, C2)


def _float_case(M, N, K, algo, dtype, dist="uniform", b_layout=0, variant="auto"):
    A, B = inputs.operands(M, N, K, dtype, 31, 32, dist=dist, b_layout=b_layout)
    plan = L.Plan(M, N, K, dtype=dtype, algo=algo, b_layout=b_layout, variant=variant)
    C = plan.gemm(A.cuda(), B.cuda()).double().cpu().numpy()
    Ad = A.double().numpy()
    Bd = _b_dense(B, b_layout).double().numpy()
    ref = O.gemm_f64(Ad, Bd)
    e = O.eps_norm(C, ref, Ad, Bd)
    er = O.eps_rel(C, ref)
    fmt = {0: "bf16", 1: "fp16", 2: "tf32"}[dtype]
    out_fmt = {0: "bf16", 1: "fp16", 2: "fp32"}[dtype]
    if algo == "classical":
        if dtype == 2:   # the tf32 MMA truncates raw fp32 operands (reading 7)
            emu = O.gemm_f64(O.round_to(Ad, "tf32_rz"), O.round_to(Bd, "tf32_rz"))
        else:
            emu = O.round_to(ref, out_fmt)
    else:
        emu = O.lcma_f64(Ad, Bd, SCHEMES[algo](), extents=(plan.info["Mb"], plan.info["Kb"], plan.info["Nb"]),
                         fmt_in=fmt, fmt_out=out_fmt).C
    er_emu = O.eps_rel(emu, ref)
    return e, er, er_emu, O.freivalds(C, Ad, Bd)


@pytest.mark.parametrize("algo", ["classical", "strassen", "strassen2", "laderman"])
@pytest.mark.parametrize("dtype,gate", [(0, 2e-2), (1, 3e-3), (2, 3e-3)])
@pytest.mark.parametrize("dist", ["uniform", "positive"])
def test_float_tolerance(algo, dtype, gate, dist):
    e, er, er_emu, fv = _float_case(1032, 1544, 1032, algo, dtype, dist=dist)
    assert e <= gate
    assert er <= 3.0 * er_emu + 1e-6, (er, er_emu)     # within 3x the dtype-faithful emulation
    assert fv <= gate


def test_fp32_cfg1_simt():
    # cfg1: Strassen one level, 256^3, true fp32 (BASELINE gate 1e-5)
    for algo in ("strassen", "classical"):
        A, B = inputs.operands(256, 256, 256, L.FP32, 101, 102)
        plan = L.Plan(256, 256, 256, dtype=L.FP32, algo=algo)
        C = plan.gemm(A.cuda(), B.cuda()).double().cpu().numpy()
        ref = O.gemm_f64(A.double().numpy(), B.double().numpy())
        assert O.eps_norm(C, ref, A.double().numpy(), B.double().numpy()) <= 1e-5
    _exact_case(256, 256, 256, "strassen", dtype=L.FP32)
    _exact_case(300, 264, 200, "strassen2", dtype=L.FP32)


def test_determinism_bitwise():
    A, B = inputs.operands(1536, 2304, 1024, 0, 41, 42)
    Ad, Bd = A.cuda(), B.cuda()
    for algo in ("strassen", "laderman", "classical"):
        plan = L.Plan(1536, 2304, 1024, dtype=L.BF16, algo=algo, num_ctas=20)
        C1 = plan.gemm(Ad, Bd).clone()
        for _ in range(3):
            assert torch.equal(plan.gemm(Ad, Bd), C1)


def test_cfg2_full_size_sampled():
    # BASELINE cfg2 at full size in the bench configuration: sampled rows vs the
    # fp64 oracle, Freivalds over all of C, and an exact-integer run.
    M, N, K = 8192, 14336, 4096
    A, B = inputs.operands(M, N, K, 0, 201, 202)
    plan = L.Plan(M, N, K, dtype=L.BF16, algo="strassen")
    C = plan.gemm(A.cuda(), B.cuda())
    rng = np.random.default_rng(0)
    Mb = plan.info["Mb"]
    rows = np.unique(np.concatenate([rng.choice(M, 48, replace=False),
                                     [0, 127, 128, 255, 256, Mb - 1, Mb, Mb + 1, M - 1]]))
    Ad = A.double().numpy()
    Bd = B.double().numpy()
    ref = O.gemm_rows_f64(Ad, Bd, rows)
    got = C[torch.from_numpy(rows).cuda()].double().cpu().numpy()
    _assert_vs_emulation(got, ref, O.gemm_rows_f64(np.abs(Ad), np.abs(Bd), rows),
                         _emulated_rows(Ad, Bd, rows, plan, "strassen", ref))
    assert O.freivalds(C.double().cpu().numpy(), Ad, Bd, trials=2) < 2e-2
    # exact integer mode at full size
    Ai, Bi = inputs.operands(M, N, K, 0, 203, 204, dist="int", lo=-1, hi=1)
    plan = L.Plan(M, N, K, dtype=L.BF16, algo="strassen", out_dtype=L.FP32)
    Ci = plan.gemm(Ai.cuda(), Bi.cuda())
    refi = O.gemm_rows_f64(Ai.double().numpy(), Bi.double().numpy(), rows)
    assert np.array_equal(Ci[torch.from_numpy(rows).cuda()].double().cpu().numpy(), refi)


def _sampled_rows(M, Mb, n=24, seed=0):
    rng = np.random.default_rng(seed)
    edges = [0, 127, 128, 255, 256, Mb - 1, Mb, Mb + 1, 2 * Mb - 1, M - 1]
    return np.unique(np.concatenate([rng.choice(M, n, replace=False), [r for r in edges if 0 <= r < M]]))


def _emulated_rows(Ad, Bd, rows, plan, algo, ref):
    """The oracle's dtype-faithful emulation of the same rows (bf16 operands,
    one RN rounding of each combined operand and of C, exact products and
    sums): the expected error level of a correct kernel (DESIGN reading 20)."""
    if algo == "classical":
        return O.round_to(ref, "bf16")
    return O.lcma_rows_f64(Ad, Bd, SCHEMES[algo](), rows,
                           extents=(plan.info["Mb"], plan.info["Kb"], plan.info["Nb"]),
                           fmt_in="bf16", fmt_out="bf16")


def _assert_vs_emulation(got, ref, absAB, emu):
    """Componentwise and normwise error of the GPU rows within 2x those of the
    emulation on the same rows (DESIGN reading 20: GPU and emulation round at
    the same points; what differs is fp32 vs exact accumulation, <= K*2^-24
    relative, and C ties, <= one bf16 ulp), plus the 1e-2 eps_rel sanity gate."""
    comp = (np.abs(got - ref) / absAB).max()
    comp_emu = (np.abs(emu - ref) / absAB).max()
    er, er_emu = O.eps_rel(got, ref), O.eps_rel(emu, ref)
    print(f"componentwise {comp:.3e} (emulation {comp_emu:.3e}), eps_rel {er:.3e} (emulation {er_emu:.3e})")
    assert er < 1e-2
    assert comp <= 2.0 * comp_emu, (comp, comp_emu)
    assert er <= 2.0 * er_emu, (er, er_emu)


def _check_rows(C, A, B, b_layout, rows, plan, algo):
    """Sampled rows of C against the fp64 oracle (row-restricted naive GEMM)
    and the dtype-faithful emulation of the same rows."""
    Ad = A.double().numpy()
    Bd = _b_dense(B, b_layout).double().numpy()
    ref = O.gemm_rows_f64(Ad, Bd, rows)
    got = C[torch.from_numpy(rows).to(C.device)].double().cpu().numpy()
    absAB = O.gemm_rows_f64(np.abs(Ad), np.abs(Bd), rows)
    _assert_vs_emulation(got, ref, absAB, _emulated_rows(Ad, Bd, rows, plan, algo, ref))


@pytest.mark.parametrize("algo", ["strassen", "classical"])
def test_cfg2_bench_layout_sampled(algo):
    # the exact launch configuration bench.py times: cfg2, B stored N x K
    M, N, K = 8192, 14336, 4096
    A, B = inputs.operands(M, N, K, 0, 510, 502, b_layout=1)
    plan = L.Plan(M, N, K, dtype=L.BF16, algo=algo, b_layout=1)
    C = plan.gemm(A.cuda(), B.cuda())
    rows = _sampled_rows(M, plan.info["Mb"])
    _check_rows(C, A, B, 1, rows, plan, algo)
    Ai, Bi = inputs.operands(M, N, K, 0, 503, 504, dist="int", lo=-1, hi=1, b_layout=1)
    plan = L.Plan(M, N, K, dtype=L.BF16, algo=algo, out_dtype=L.FP32, b_layout=1)
    Ci = plan.gemm(Ai.cuda(), Bi.cuda())
    refi = O.gemm_rows_f64(Ai[torch.from_numpy(rows)].double().numpy(), Bi.t().double().numpy(),
                           np.arange(len(rows)))
    assert np.array_equal(Ci[torch.from_numpy(rows).cuda()].double().cpu().numpy(), refi)


@pytest.mark.parametrize("algo", ["laderman", "strassen2"])
def test_cfg4_full_size_sampled(algo):
    # BASELINE cfg4: Laderman <3,3,3;23> and Strassen^2 <4,4,4;49> at 12288^3 bf16
    M = N = K = 12288
    A, B = inputs.operands(M, N, K, 0, 401, 402, b_layout=1)
    plan = L.Plan(M, N, K, dtype=L.BF16, algo=algo, b_layout=1)
    C = plan.gemm(A.cuda(), B.cuda())
    rows = _sampled_rows(M, plan.info["Mb"], n=16)
    _check_rows(C, A, B, 1, rows, plan, algo)
    assert O.freivalds(C.double().cpu().numpy(), A.double().numpy(), B.t().double().numpy(), trials=1) < 2e-2
    Ai, Bi = inputs.operands(M, N, K, 0, 403, 404, dist="int", lo=-1, hi=1, b_layout=1)
    plan = L.Plan(M, N, K, dtype=L.BF16, algo=algo, out_dtype=L.FP32, b_layout=1)
    Ci = plan.gemm(Ai.cuda(), Bi.cuda())
    refi = O.gemm_rows_f64(Ai[torch.from_numpy(rows)].double().numpy(), Bi.t().double().numpy(),
                           np.arange(len(rows)))
    assert np.array_equal(Ci[torch.from_numpy(rows).cuda()].double().cpu().numpy(), refi)


def test_cfg5_full_shape_static_b_sampled():
    # BASELINE cfg5 shape on one GPU (the bench's large_llama_ffn line): Strassen
    # with B precombined offline, sampled rows vs the fp64 oracle
    M, N, K = 32768, 28672, 8192
    A, B = inputs.operands(M, N, K, 0, 510, 502, b_layout=1)
    plan = L.Plan(M, N, K, dtype=L.BF16, algo="strassen", b_layout=1, b_static=True)
    Bt = plan.precombine_b(B.cuda())
    C = plan.gemm_precombined(A.cuda(), Bt)
    rows = _sampled_rows(M, plan.info["Mb"], n=12)
    _check_rows(C, A, B, 1, rows, plan, "strassen")


def test_cuda_graph_capture_and_streams():
    # lcma_gemm only enqueues (no allocation, no host sync): capturable in a
    # CUDA graph; replay equals eager; concurrent plans on two streams
    M, N, K = 1536, 2304, 1024
    A, B = inputs.operands(M, N, K, 0, 81, 82, b_layout=1)
    A, B = A.cuda(), B.cuda()
    for algo in ("classical", "strassen", "laderman", "strassen2"):
        plan = L.Plan(M, N, K, dtype=L.BF16, algo=algo, b_layout=1)
        ws = plan.workspace()
        ref = plan.gemm(A, B, workspace=ws).clone()
        C = plan.empty_c()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            plan.gemm(A, B, C, ws, stream=s)
        for _ in range(3):
            C.zero_()
            g.replay()
        torch.cuda.synchronize()
        assert torch.equal(C, ref), algo
    p1 = L.Plan(M, N, K, dtype=L.BF16, algo="strassen", b_layout=1)
    p2 = L.Plan(M, N, K, dtype=L.BF16, algo="classical", b_layout=1)
    r1, r2 = p1.gemm(A, B).clone(), p2.gemm(A, B).clone()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    C1, C2 = p1.empty_c(), p2.empty_c()
    torch.cuda.synchronize()
    for _ in range(4):
        with torch.cuda.stream(s1):
            p1.gemm(A, B, C1, stream=s1)
        with torch.cuda.stream(s2):
            p2.gemm(A, B, C2, stream=s2)
    torch.cuda.synchronize()
    assert torch.equal(C1, r1) and torch.equal(C2, r2)


@pytest.mark.parametrize("seed", range(16))
def test_random_shapes_exact(seed):
    # fuzz: random ragged shapes, algorithms, layouts, variants, schedules,
    # CTA counts -- bit-exact against the int64 oracle
    rng = np.random.default_rng(1000 + seed)
    algo = ["strassen", "laderman", "strassen2", "classical"][seed % 4]
    M = int(rng.integers(1, 1400)); N = int(rng.integers(1, 180)) * 8; K = int(rng.integers(1, 160)) * 8
    kw = dict(b_layout=int(rng.integers(0, 2)))
    if algo != "classical":
        kw["variant"] = ["fused_h", "unfused"][int(rng.integers(0, 2))]
        if kw["variant"] == "fused_h":
            kw["schedule"] = int(rng.choice([0, 2, 3]))
            kw["num_ctas"] = int(rng.choice([0, 2, 8, 20, 64]))
    _exact_case(M, N, K, algo, **kw)


def test_error_paths():
    # C ABI (raw pointers): alignment, workspace size, aliasing
    plan = L.Plan(256, 512, 256, dtype=L.BF16, algo="strassen")
    A = torch.zeros(256 * 256 + 8, dtype=torch.bfloat16, device="cuda")
    B = torch.zeros(256, 512, dtype=torch.bfloat16, device="cuda")
    C = torch.empty(256, 512, dtype=torch.bfloat16, device="cuda")
    ws = plan.workspace()
    lib = L.lib()
    st = torch.cuda.current_stream().cuda_stream

    def raw(a, b, c, w, nbytes):
        return lib.lcma_gemm(plan._h, a, b, c, w, nbytes, st)

    assert raw(A.data_ptr() + 2, B.data_ptr(), C.data_ptr(), ws.data_ptr(), ws.numel()) == 3   # MISALIGNED
    assert raw(A.data_ptr(), B.data_ptr(), C.data_ptr(), ws.data_ptr(), 16) == 7               # WORKSPACE
    assert raw(A.data_ptr(), B.data_ptr(), A.data_ptr(), ws.data_ptr(), ws.numel()) == 1       # C aliases A
    assert "overlap" in lib.lcma_last_error().decode()
    with pytest.raises(L.LcmaError, match="MISALIGNED"):
        L.Plan(256, 500, 256, dtype=L.BF16)
    # the Python binding checks what the raw pointers cannot carry
    A2 = A[:256 * 256].view(256, 256)
    with pytest.raises(L.LcmaError, match="shape|needs"):
        plan.gemm(A2.t().contiguous()[:128], B, C)
    with pytest.raises(L.LcmaError, match="contiguous"):
        plan.gemm(A2.t(), B, C)
    with pytest.raises(L.LcmaError, match="dtype"):
        plan.gemm(A2.half(), B, C)
    with pytest.raises(L.LcmaError, match="CUDA"):
        plan.gemm(A2.cpu(), B, C)
    with pytest.raises(L.LcmaError, match="workspace"):
        plan.gemm(A2, B, C, workspace=torch.zeros(16, dtype=torch.uint8, device="cuda"))


def test_fake_multi_gpu_block_rows():
    # block-row partition on one GPU: shards planned independently, stacked == full
    from paper_2605_06057_b200 import shard
    M, N, K, P = 2048, 1024, 512, 4
    A, B = inputs.operands(M, N, K, 0, 51, 52, dist="int", lo=-2, hi=2)
    parts = []
    for p in range(P):
        r0, r1 = shard.row_block(M, P, p)
        plan = L.Plan(r1 - r0, N, K, dtype=L.BF16, algo="strassen", out_dtype=L.FP32)
        parts.append(plan.gemm(A[r0:r1].cuda(), B.cuda()).cpu())
    C = torch.cat(parts).numpy()
    assert np.array_equal(C, O.gemm_i64(A.to(torch.int64).numpy(), B.to(torch.int64).numpy()))


def test_partial_homes_exact_diag_build():
    # fused Combine H keeps live C_ij partials in epilogue registers, shared
    # memory or L2 slots; the non-default placements are diagnostic knobs of
    # the -DLCMA_DIAG build (the product build reads no environment), run in
    # a subprocess against that library: every placement must be exact
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    diag = os.path.join(os.path.dirname(here), "paper_2605_06057_b200", "liblcma_diag.so")
    assert os.path.exists(diag), "build() builds liblcma_diag.so"
    env = dict(os.environ, LCMA_LIB=diag)
    r = subprocess.run([sys.executable, os.path.join(here, "_diag_homes.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "homes ok" in r.stdout


@pytest.mark.parametrize("schedule", [1, 5, 6, 7])
@pytest.mark.parametrize("algo,shape,ctas", [("strassen", (1536, 2304, 512), 0), ("strassen", (1536, 2304, 512), 10),
                                             ("strassen", (2560, 3072, 256), 6), ("laderman", (1000, 808, 520), 4),
                                             ("classical", (2304, 2560, 256), 8), ("classical", (1000, 1048, 520), 0)])
def test_dynamic_vs_static_schedule_exact(schedule, algo, shape, ctas):
    # schedule 5: whole groups and split-tail segments drawn from the workspace
    # ticket counters at run time; 6: static whole groups, run-time tail;
    # 1 (default): the static lockstep assignment.  Exact every
    # ways; repeated calls on one workspace check that the counter is back at
    # zero after every launch (a stale counter would skip or repeat groups)
    plan = _exact_case(*shape, algo, schedule=schedule, num_ctas=ctas)
    lo, hi = INT_RANGE[algo]
    A, B = inputs.operands(*shape, 0, 5, 6, dist="int", lo=lo, hi=hi)
    A, B = A.cuda(), B.cuda()
    ws = plan.workspace()
    C1 = plan.gemm(A, B, workspace=ws).clone()
    for _ in range(4):
        assert torch.equal(plan.gemm(A, B, workspace=ws), C1)
    assert ws[:8].view(torch.int32).tolist() == [0, 0]      # counters reset by the last tickets


@pytest.mark.parametrize("b_layout", [0, 1])
@pytest.mark.parametrize("shape,dtype,ctas", [((512, 512, 512), 0, 0), ((1024, 1560, 768), 0, 0),
                                              ((1536, 2304, 512), 0, 10), ((1024, 1032, 768), 1, 0),
                                              ((1024, 1024, 1024), 1, 0), ((1536, 2048, 512), 0, 10)])
def test_producer_fused_combine_a_exact(shape, dtype, ctas, b_layout):
    # variant 3: Combine A (and, for B stored N x K with exactly tiled N, K,
    # Combine B) inside the GEMM producer path: the one or two nonzero blocks
    # are loaded by TMA and summed in shared memory before the MMAs; exact
    # against the int64 oracle, whole and split groups
    _exact_case(*shape, "strassen", dtype=dtype, b_layout=b_layout, variant="producer", num_ctas=ctas)


def test_producer_fused_rejects():
    # non-dividing M / K, or more than two A blocks per product (Laderman)
    for args in ((1000, 512, 512, "strassen"), (512, 512, 520, "strassen"), (768, 768, 768, "laderman")):
        with pytest.raises(L.LcmaError):
            L.Plan(args[0], args[1], args[2], algo=args[3], variant="producer")


@pytest.mark.parametrize("algo,shape", [("strassen", (1024, 1024, 512)), ("strassen", (2048, 1536, 1024)),
                                        ("laderman", (768, 768, 384))])
def test_inplace_single_term_operands_exact(algo, shape):
    # exactly tiled shapes, B stored N x K: the single-term A~_r / B~_r are read
    # in place from A / B (reading 25); per call and with B~ offline
    # (A in place only), exact against the int64 oracle
    M, N, K = shape
    plan = _exact_case(M, N, K, algo, b_layout=1)
    assert plan.info["Mb"] * (2 if algo == "strassen" else 3) == M
    lo, hi = INT_RANGE[algo]
    A, B = inputs.operands(M, N, K, 0, M + 7, N + K, dist="int", b_layout=1, lo=lo, hi=hi)
    sp = L.Plan(M, N, K, dtype=0, algo=algo, out_dtype=L.FP32, b_layout=1, b_static=True)
    Bt = sp.precombine_b(B.cuda())
    C = sp.gemm_precombined(A.cuda(), Bt).cpu().numpy()
    ref = O.gemm_i64(A.to(torch.int64).numpy(), B.t().to(torch.int64).numpy())
    assert np.array_equal(C, ref)
