"""Pins for the oracle's FP8 E4M3 path ("1 x 128 block-wise scaling
for FP8E4M3", P:471 quantization fused into Combine A; reading 23).
CPU only: the rounding is checked against torch's float8_e4m3fn cast (an
independent library routine), the scale rule against its closed forms, the
evaluator against exact GEMM on inputs the quantization represents exactly
and against the E4M3 error bound on random inputs."""
import numpy as np
import pytest
import torch

import oracle as O


def test_round_e4m3_hand_values():
    # max normal, RN-even ties in [1, 2) (spacing 1/8), subnormal spacing 2^-9
    cases = {448.0: 448.0, 464.0: 448.0, 1e9: 448.0, 1.0625: 1.0, 1.1875: 1.25, 1.0624: 1.0,
             0.015625: 0.015625, 2.0 ** -10: 0.0, 3 * 2.0 ** -11: 2.0 ** -9, 2.0 ** -9: 2.0 ** -9,
             -3.3: -3.25, 17.0: 16.0, 19.0: 20.0, 0.0: 0.0, 240.0: 240.0, 232.0: 224.0}
    got = O.round_e4m3(np.array(list(cases)))
    assert got.tolist() == list(cases.values())


def test_round_e4m3_matches_torch_on_every_bf16_in_range():
    # every finite bf16 bit pattern with |x| <= 448: torch's cast is RN-even
    bits = torch.arange(0, 1 << 16, dtype=torch.int32).to(torch.int16)
    v = bits.view(torch.bfloat16).float()
    v = v[torch.isfinite(v) & (v.abs() <= 448)]
    ref = v.to(torch.float8_e4m3fn).float().double().numpy()
    got = O.round_e4m3(v.double().numpy())
    assert np.array_equal(got, ref)


def test_round_e4m3_matches_torch_on_random_fp64():
    rng = np.random.default_rng(5)
    x = rng.uniform(-448, 448, 200000) * np.exp2(rng.integers(-14, 1, 200000))
    ref = torch.from_numpy(x).float().to(torch.float8_e4m3fn).double().numpy()
    # fp64 -> fp32 first (torch path) can only change values within 2^-24 relative,
    # far from an E4M3 rounding boundary except at exact ties: compare where x is
    # exactly an fp32 value
    x32 = x.astype(np.float32).astype(np.float64)
    assert np.array_equal(O.round_e4m3(x32), ref)


def test_scale_exponent_closed_forms():
    amax = np.array([448.0, 449.0, 1.0, 1.75, np.nextafter(1.75, 2), 0.0, 448 * 2.0 ** -20,
                     896.0, 897.0, 224.0, 224.000001, 2.0 ** -140])
    want = [0, 1, -8, -8, -7, 0, -20, 1, 2, -1, 0, -127]
    assert O.scale_exponent(amax).tolist() == want


def test_scale_exponent_is_minimal():
    rng = np.random.default_rng(7)
    amax = rng.uniform(0, 1, 5000) * np.exp2(rng.integers(-30, 30, 5000))
    amax = amax[amax > 0]
    e = O.scale_exponent(amax)
    assert np.all(amax <= np.ldexp(448.0, e))          # fits
    assert np.all(amax > np.ldexp(448.0, e - 1))       # the smallest that fits


def test_quantize_1x128_block_values():
    x = np.zeros((1, 128))
    x[0, :4] = [3.0, -1.0, 0.1, 2.9]
    Q, e = O.quantize_1x128(x)
    assert e.tolist() == [[-7]]
    # 3*128 = 384, -128, 12.8 -> 13 (spacing 1 in [8, 16)), 371.2 -> 384 (spacing 32 in [256, 448])
    assert Q[0, :4].tolist() == [384.0, -128.0, 13.0, 384.0]
    assert np.all(Q[0, 4:] == 0)


def test_quantize_1x128_invariants_and_error_bound():
    rng = np.random.default_rng(9)
    X = rng.uniform(-1, 1, (64, 512)) * np.exp2(rng.integers(-8, 8, (64, 1)))
    X[3, 128:256] = 0.0                                 # an all-zero block
    Q, e = O.quantize_1x128(X)
    assert e[3, 1] == 0 and np.all(Q[3, 128:256] == 0)
    blk = np.abs(Q.reshape(64, 4, 128)).max(axis=2)
    nz = blk > 0
    assert np.all(blk <= 448) and np.all(blk[nz] > 224)   # the minimal scale uses the top binade
    D = O.dequantize_1x128(Q, e)
    # RN to 3 mantissa bits: |x - q| <= 2^-4 |x| for normals, <= 2^-10 * 2^e below 2^-6 * 2^e
    bound = np.maximum(np.abs(X) * 2.0 ** -4, np.repeat(np.ldexp(2.0 ** -10, e), 128, axis=1))
    assert np.all(np.abs(D - X) <= bound * (1 + 1e-12))
    # values already on the E4M3 x 2^e grid with amax = 448 * 2^e are kept exactly
    G = O.round_e4m3(rng.uniform(-448, 448, (8, 256)))
    G[:, 0] = 448.0
    G[:, 128] = -448.0
    G = G * 2.0 ** -5
    Q2, e2 = O.quantize_1x128(G)
    assert np.all(e2 == -5) and np.array_equal(O.dequantize_1x128(Q2, e2), G)
    with pytest.raises(ValueError):
        O.quantize_1x128(np.zeros((2, 100)))


def test_fp8_lcma_exact_on_representable_inputs():
    # small integers: every combined block has amax <= 4, its scaled values are
    # integers times a power of two with <= 2 significant bits -> exact in E4M3,
    # so the FP8 workflow returns A.B exactly (Strassen, classical, Laderman)
    rng = np.random.default_rng(11)
    M, N, K = 40, 24, 256
    A = rng.integers(-2, 3, (M, K)).astype(np.float64)
    B = rng.integers(-2, 3, (K, N)).astype(np.float64)
    ref = A @ B
    for s, ext in ((O.strassen(), (20, 128, 12)), (O.standard(1, 1, 1), (40, 256, 24))):
        got = O.lcma_rows_fp8(A, B, s, np.arange(M), ext)
        assert np.array_equal(got, ref), s.name
    A1 = rng.integers(-1, 2, (M, 384)).astype(np.float64)
    B1 = rng.integers(-1, 2, (384, N)).astype(np.float64)
    got = O.lcma_rows_fp8(A1, B1, O.laderman(), np.arange(M), (14, 128, 8))
    assert np.array_equal(got, A1 @ B1)


def test_fp8_lcma_detects_a_dropped_term():
    # the exactness above is a real pin: a wrong sign in one W entry breaks it
    rng = np.random.default_rng(12)
    A = rng.integers(-2, 3, (16, 256)).astype(np.float64)
    B = rng.integers(-2, 3, (256, 16)).astype(np.float64)
    s = O.strassen()
    s.W = s.W.copy()
    s.W[4, 0, 0] = -s.W[4, 0, 0]
    got = O.lcma_rows_fp8(A, B, s, np.arange(16), (8, 128, 8))
    assert not np.array_equal(got, A @ B)


def test_fp8_lcma_error_bound_random():
    # U[-1,1) inputs: each quantized operand element is within 2^-4 of its
    # block's amax; the errors of the K terms of a dot product have random
    # signs, so normwise eps_norm ~ 2^-4 * c / sqrt(K) with c ~ 1 for the
    # classical path and ~1.5 for Strassen (sums of two blocks, Combine H):
    # the FP8 gate of DESIGN.md reading 23 is eps_norm <= 0.1 / sqrt(K)
    rng = np.random.default_rng(13)
    M, N, K = 32, 48, 512
    A = rng.uniform(-1, 1, (M, K))
    B = rng.uniform(-1, 1, (K, N))
    ref = A @ B
    for s, ext in ((O.standard(1, 1, 1), (32, 512, 48)), (O.strassen(), (16, 256, 24))):
        got = O.lcma_rows_fp8(A, B, s, np.arange(M), ext)
        e = O.eps_norm(got, ref, A, B)
        assert 1e-4 < e < 0.1 / np.sqrt(K), (s.name, e)
    # fp32 / bf16 output rounding on top
    got = O.lcma_rows_fp8(A, B, O.strassen(), [0, 31], (16, 256, 24), fmt_out="bf16")
    assert np.array_equal(got, O.round_to(got, "bf16"))


def test_combine_b_fp8_layout():
    # B~_r stored N x K; scales per (column, 128-block of K)
    rng = np.random.default_rng(14)
    B = rng.uniform(-1, 1, (256, 64))
    Q, E = O.combine_b_fp8(B, O.strassen(), (64, 128, 32))
    assert Q.shape == (7, 32, 128) and E.shape == (7, 32, 1)
    # r = 1 (0-based): B~ = B11; column n of B11 is B[:128, n]
    q1, e1 = O.quantize_1x128(B[:128, :32].T)
    assert np.array_equal(Q[1], q1) and np.array_equal(E[1], e1)
