"""Pins for the oracle's naive GEMM, rounding helpers and Algorithm-1
evaluator (CPU)."""
import numpy as np
import pytest
import torch

import oracle as O


def test_naive_gemm_worked_example():
    # [[1,2],[3,4]] x [[5,6],[7,8]] = [[19,22],[43,50]]
    A = np.array([[1, 2], [3, 4]])
    B = np.array([[5, 6], [7, 8]])
    assert O.gemm_i64(A, B).tolist() == [[19, 22], [43, 50]]
    assert O.gemm_f64(A, B).tolist() == [[19, 22], [43, 50]]


def test_naive_gemm_identity_and_library():
    rng = np.random.default_rng(1)
    A = rng.standard_normal((7, 7))
    assert np.array_equal(O.gemm_f64(A, np.eye(7)), A)          # S:176 A*I = A
    # small-integer inputs: exact, equal to numpy's integer matmul (library routine)
    for (M, N, K) in [(1, 1, 1), (5, 3, 9), (33, 17, 65), (64, 64, 64)]:
        Ai = rng.integers(-50, 50, (M, K))
        Bi = rng.integers(-50, 50, (K, N))
        assert np.array_equal(O.gemm_i64(Ai, Bi), Ai @ Bi)
        assert np.array_equal(O.gemm_f64(Ai, Bi), (Ai @ Bi).astype(np.float64))
    with pytest.raises(ValueError):
        O.gemm_f64(np.zeros((2, 3)), np.zeros((4, 2)))


def test_gemm_rows_matches_full():
    rng = np.random.default_rng(2)
    A = rng.uniform(-1, 1, (40, 23))
    B = rng.uniform(-1, 1, (23, 31))
    rows = [0, 7, 39, 12]
    assert np.array_equal(O.gemm_rows_f64(A, B, rows), O.gemm_f64(A, B)[rows])


def test_rounding_matches_torch_and_numpy():
    rng = np.random.default_rng(3)
    x32 = rng.uniform(-4, 4, 20000).astype(np.float32)
    x32 = np.concatenate([x32, np.float32([1.00390625, 1.01171875, -3.0078125, 1e-30, 6e4])])
    bf = torch.from_numpy(x32).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(O.round_to(x32.astype(np.float64), "bf16"), bf)
    f16 = x32.astype(np.float16).astype(np.float64)
    y = O.round_to(x32.astype(np.float64), "fp16")
    assert np.array_equal(y, f16)
    # fp16 subnormal and overflow
    assert O.round_to(np.array([2.0 ** -20, 70000.0]), "fp16").tolist() == [2.0 ** -20, np.inf]
    # tf32: 10 stored mantissa bits, ties away from zero (cvt.rna.tf32.f32)
    t = O.round_to(np.array([1 + 2.0 ** -11, 1 + 3 * 2.0 ** -11, -(1 + 2.0 ** -11), 1 + 2.0 ** -12]), "tf32")
    assert t.tolist() == [1 + 2.0 ** -10, 1 + 2 * 2.0 ** -10, -(1 + 2.0 ** -10), 1.0]
    z = O.round_to(np.array([1 + 3 * 2.0 ** -11, -(1 + 2.0 ** -11), 1.9999999]), "tf32_rz")
    assert z.tolist() == [1 + 2.0 ** -10, -1.0, 2 - 2.0 ** -10]
    assert np.array_equal(O.round_to(x32.astype(np.float64) * 1.0000001, "fp32"),
                          (x32.astype(np.float64) * 1.0000001).astype(np.float32).astype(np.float64))


SCHEMES = [O.strassen, O.laderman, O.strassen2, lambda: O.standard(2, 2, 2),
           lambda: O.standard(2, 3, 2)]


@pytest.mark.parametrize("make", SCHEMES)
def test_lcma_equals_naive_exact_random_shapes(make):
    # S:259 / S:536: Algorithm 1 == naive GEMM bit-exactly in int64, random
    # shapes M,N,K in [1,128] incl. non-divisible.
    s = make()
    rng = np.random.default_rng(100 + s.R)
    n_shapes = 50 if s.R < 49 else 12
    for _ in range(n_shapes):
        M, N, K = (int(v) for v in rng.integers(1, 129, 3))
        A = rng.integers(-3, 4, (M, K))
        B = rng.integers(-3, 4, (K, N))
        assert np.array_equal(O.lcma_i64(A, B, s).C, O.gemm_i64(A, B)), (M, N, K)


def test_laderman_100x50x30():
    # 100x50x30 integers, Laderman -> bit-equal to naive
    rng = np.random.default_rng(7)
    A = rng.integers(-9, 10, (100, 30))
    B = rng.integers(-9, 10, (30, 50))
    s = O.laderman()
    assert np.array_equal(O.lcma_i64(A, B, s).C, A @ B)
    r = O.lcma_f64(A, B, s)
    assert np.array_equal(r.C, (A @ B).astype(np.float64))


def test_lcma_larger_extents_still_exact():
    # any extents >= ceil(.) give an exact LCMA (reading 6)
    rng = np.random.default_rng(8)
    s = O.strassen()
    A = rng.integers(-2, 3, (37, 29))
    B = rng.integers(-2, 3, (29, 45))
    for ext in [(19, 15, 23), (32, 16, 64), (128, 64, 128)]:
        assert np.array_equal(O.lcma_i64(A, B, s, extents=ext).C, A @ B)
        assert np.array_equal(O.lcma_f64(A, B, s, extents=ext).C, (A @ B).astype(float))
    with pytest.raises(ValueError):
        O.lcma_i64(A, B, s, extents=(10, 15, 23))


def test_counters_match_cost_table():
    # S:228, S:241, S:260 and Table "cost_model" for a divisible
    # shape: Combine-A adds = (12-7)*(M/2)(K/2) etc.
    s = O.strassen()
    M = N = K = 512
    rng = np.random.default_rng(9)
    A = rng.integers(-1, 2, (M, K)).astype(np.float64)
    B = rng.integers(-1, 2, (K, N)).astype(np.float64)
    c = O.lcma_f64(A, B, s).counters
    h = M // 2
    assert c["combineA_adds"] == (12 - 7) * h * h
    assert c["combineB_adds"] == (12 - 7) * h * h
    assert c["combineH_adds"] == (12 - 4) * h * h
    assert c["gemm_mults"] == 7 * h ** 3                  # ratio 7/8 vs M*N*K
    assert c["gemm_mults"] * 8 == 7 * M * N * K
    assert c["A_loads"] == 12 * h * h                     # Alg. 1 reads A ||U||_0 (M/m)(K/k)
    assert c["H_stores"] == 7 * h * h


def test_counters_standard_scheme():
    s = O.standard(2, 2, 2)
    M = N = K = 64
    A = np.ones((M, K))
    B = np.ones((K, N))
    c = O.lcma_f64(A, B, s).counters
    assert c["combineA_adds"] == 0 and c["combineB_adds"] == 0
    assert c["combineH_adds"] == (8 - 4) * 32 * 32                   # (k-1)*MN, reading 20


def test_precision_direction_downcast_h():
    # P:518 / S:541: fused (fp32/fp64 on-chip H) error <= staged with H
    # downcast to the working precision; Strassen, uniform[-1,1], 512^3.
    rng = np.random.default_rng(10)
    M = N = K = 512
    A = O.round_to(rng.uniform(-1, 1, (M, K)), "bf16")
    B = O.round_to(rng.uniform(-1, 1, (K, N)), "bf16")
    ref = O.gemm_f64(A, B)
    s = O.strassen()
    fused = O.lcma_f64(A, B, s, fmt_in="bf16", fmt_h="fp32", fmt_out="bf16").C
    staged = O.lcma_f64(A, B, s, fmt_in="bf16", fmt_h="bf16", fmt_out="bf16").C
    e_f = np.mean(np.abs(fused - ref) / (np.abs(ref) + 1e-3))
    e_s = np.mean(np.abs(staged - ref) / (np.abs(ref) + 1e-3))
    assert e_f <= e_s


def test_zero_inputs():
    s = O.strassen()
    assert not O.lcma_f64(np.zeros((5, 6)), np.zeros((6, 7)), s).C.any()


@pytest.mark.parametrize("scheme", ["strassen", "laderman", "strassen2"])
def test_lcma_rows_matches_full_evaluator(scheme):
    # the row-restricted Algorithm 1 (sampled full-size checks) equals the
    # whole evaluator's rows: exactly on integer-valued inputs (ragged shape,
    # GPU-like padded extents), and within fp64 summation order on floats with
    # the bf16 rounding points (C rounded once: at most one bf16 ulp apart)
    s = getattr(O, scheme)()
    rng = np.random.default_rng(21)
    M, N, K = 70, 52, 38
    ext = (-(-M // s.m) + 3, -(-K // s.k) + 1, -(-N // s.n) + 2)
    rows = np.array([0, 1, ext[0] - 1, ext[0], M - 1, 33])
    Ai = rng.integers(-3, 4, (M, K)).astype(np.float64)
    Bi = rng.integers(-3, 4, (K, N)).astype(np.float64)
    got = O.lcma_rows_f64(Ai, Bi, s, rows, extents=ext)
    assert np.array_equal(got, O.gemm_f64(Ai, Bi)[rows])
    assert np.array_equal(got, O.lcma_f64(Ai, Bi, s, extents=ext).C[rows])
    A = rng.uniform(-1, 1, (M, K))
    B = rng.uniform(-1, 1, (K, N))
    full = O.lcma_f64(A, B, s, extents=ext, fmt_in="bf16", fmt_out="bf16").C[rows]
    got = O.lcma_rows_f64(A, B, s, rows, extents=ext, fmt_in="bf16", fmt_out="bf16")
    assert np.all(np.abs(got - full) <= 2.0 ** -7 * np.abs(full) + 1e-300)
    assert np.mean(got == full) > 0.95
