"""Pins for the oracle's Decision Module (Sec. III-C) and schedule
simulator.  Values are the paper's, SPEC's worked numbers, or
closed forms derived in the test comments."""
import math

import numpy as np
import pytest

import oracle as O


def test_gemm_intensity_fixed_points():
    assert O.gemm_intensity(4096, 4096, 4096) == pytest.approx(2730.6667, abs=1e-3)
    for n in (1, 7, 100, 4096):
        assert O.gemm_intensity(n, n, n) == pytest.approx(2 * n / 3)
    assert O.gemm_intensity(1, 1, 1) == pytest.approx(2 / 3)


def test_std_gemm_memory_bound():
    hw = O.Profile(100.0, 1.0, 1.0)          # FLOPS_x / beta = 100
    assert O.std_gemm_memory_bound(64, 64, 64, hw)
    assert not O.std_gemm_memory_bound(4096, 4096, 4096, hw)
    # "<=" at equality (reading 13): 2N/3 == 100 at N=150
    assert O.std_gemm_memory_bound(150, 150, 150, hw)


def test_combine_a_intensity_strassen():
    # Table cell (||U||_0 - R)/(mk + R) = 5/11
    s = O.strassen()
    hw = O.Profile(1e15, 1e12, 1e12)
    a = O.stage_costs(s, 1024, 1024, 1024, hw)[0]
    assert a.flops / a.mem == pytest.approx(5 / 11)
    b = O.stage_costs(s, 1024, 2048, 512, hw)[1]
    assert b.flops / b.mem == pytest.approx(5 / 11)
    g = O.stage_costs(s, 1024, 1024, 1024, hw, fused=False)[2]
    # GEMM stage AI = 2MNK/(nMK + mNK + kMN) (Table row 4) = 2N/6 for square/2x2x2
    assert g.flops / g.mem == pytest.approx(2 * 1024 ** 3 / (3 * 2 * 1024 ** 2))
    h = O.stage_costs(s, 1024, 1024, 1024, hw, fused=False)[3]
    assert h.flops / h.mem == pytest.approx((12 - 4) / (7 + 4))   # (||W||-mn)/(R+mn)


def test_condition_closed_forms_strassen_square():
    # fused LHS = 2N^3(1/8) / (2N^2(1+7/4) + N^2) = N/26 ; unfused = N/33
    s = O.strassen()
    for N in (512, 1000, 4096):
        assert O.lcma_condition_lhs(s, N, N, N, fused=True) == pytest.approx(N / 26)
        assert O.lcma_condition_lhs(s, N, N, N, fused=False) == pytest.approx(N / 33)


def test_strassen_crossover_2600():
    # S:415 / S:540: ratio 100 -> crossover at N = 2600
    s = O.strassen()
    hw = O.Profile(100.0, 1.0, 1.0)
    assert O.lcma_beneficial(s, 4096, 4096, 4096, hw)
    assert not O.lcma_beneficial(s, 1024, 1024, 1024, hw)
    assert O.lcma_beneficial(s, 2601, 2601, 2601, hw)
    assert not O.lcma_beneficial(s, 2600, 2600, 2600, hw)


def test_standard_time_and_limits():
    # 2*4096^3 at 100 TFLOP/s -> 1.374 ms
    hw = O.Profile(100e12, 1e12, 1e12)
    assert O.estimate_time(None, 4096, 4096, 4096, hw) == pytest.approx(1.3744e-3, rel=1e-3)
    # beta -> inf: LCMA time -> (R/mnk) * standard time (combines cost flops/F+ only
    # when compute bound; with F+ -> inf too it is the GEMM stage alone)
    s = O.strassen()
    hw_inf = O.Profile(100e12, 1e30, 1e30)
    assert O.estimate_time(s, 4096, 4096, 4096, hw_inf) == pytest.approx(
        7 / 8 * O.estimate_time(None, 4096, 4096, 4096, hw_inf), rel=1e-9)


def test_select_rules():
    cat = [O.strassen(), O.strassen2(), O.laderman()]
    hw = O.Profile(100.0, 100.0, 1.0)
    d = O.select(cat, 64, 64, 64, hw)                     # memory-bound -> classical
    assert d.choice == "classical" and d.memory_bound
    d = O.select([O.standard(2, 2, 2)], 8192, 8192, 8192, hw)   # standard-only
    assert d.choice == "classical"
    d = O.select(cat, 8192, 8192, 1, hw)                  # K=1
    assert d.choice == "classical"
    # high intensity with cheap combines: rank-49 (largest mnk/R) wins
    hw = O.Profile(1.0, 1e6, 1e6)
    d = O.select(cat, 1 << 14, 1 << 14, 1 << 14, hw)
    assert d.choice == "strassen2-4x4x4-r49"
    assert d.times["strassen2-4x4x4-r49"] < d.times["strassen-2x2x2-r7"] < d.times["classical"]


def test_ceilings():
    assert O.effective_ceiling(O.strassen(), 1.0) == pytest.approx(8 / 7)
    assert O.effective_ceiling(O.strassen2(), 1.0) == pytest.approx(64 / 49)
    assert O.effective_ceiling(O.laderman(), 1.0) == pytest.approx(27 / 23)


def test_roofline_low_intensity_classical_dominates():
    cat = [O.strassen(), O.strassen2()]
    hw = O.Profile(148e12, 148e12, 2e12)     # H20-like ratio 74
    rows = O.roofline_table(cat, hw, [10, 50])
    for ai in (10, 50):
        best = max((r for r in rows if r[0] == ai), key=lambda r: r[2])
        assert best[1] == "classical"


def test_decision_coherence_random():
    # S:449/S:540 (in-regime, reading 12): beneficial <=> estimate < std;
    # fused estimate <= unfused; monotone in beta; estimate-beneficial => Eq.
    rng = np.random.default_rng(5)
    cat = [O.strassen(), O.strassen2(), O.laderman()]
    n_in_regime = 0
    for _ in range(400):
        M, N, K = (int(2 ** rng.uniform(8, 15)) * 12 for _ in range(3))
        fm = 10 ** rng.uniform(12, 15)
        beta = fm / 10 ** rng.uniform(0.5, 2.5)
        fa = beta * 10 ** rng.uniform(0.8, 1.5)     # combines memory-bound (in regime)
        hw = O.Profile(fm, fa, beta)
        t_std = O.estimate_time(None, M, N, K, hw)
        for s in cat:
            for fused in (True, False):
                cs = O.stage_costs(s, M, N, K, hw, fused)
                in_regime = (cs[0].bound == cs[1].bound == cs[3].bound == "memory"
                             and cs[2].bound == "compute")
                t = O.estimate_time(s, M, N, K, hw, fused)
                if t < t_std:
                    assert O.lcma_beneficial(s, M, N, K, hw, fused)
                if in_regime:
                    n_in_regime += 1
                    assert (t < t_std) == O.lcma_beneficial(s, M, N, K, hw, fused)
            assert O.estimate_time(s, M, N, K, hw, True) <= O.estimate_time(s, M, N, K, hw, False)
            hw2 = O.Profile(fm, fa, beta * 2)
            if O.lcma_beneficial(s, M, N, K, hw):
                assert O.lcma_beneficial(s, M, N, K, hw2)
        d = O.select(cat, M, N, K, hw)
        assert d.times[d.choice] == min(d.times.values())
    assert n_in_regime >= 200


# ------------------------------------------------------------- schedule
def test_split_group_paper_example():
    # 4096^3, 128x128 tiles, Strassen, 78 SMs: 1792 tiles, 256 groups,
    # ceil(1792/78) = 23 waves vs ceil(256/78)*7 = 28, waste 21.7 %.
    sch = O.plan_split_group(256, 7, 78)
    assert sum(len(a) for a in sch.assignments) == 1792
    assert sch.waves == 23 and sch.group_waves == 28
    assert (sch.group_waves - sch.waves) / sch.waves * 100 == pytest.approx(21.7, abs=0.05)


def test_split_group_small_cases():
    sch = O.plan_split_group(4, 7, 3)          # P:364 / S:322: 4 groups on 3 SMs
    assert sch.waves == 10 and sch.group_waves == 14
    sch = O.plan_split_group(1, 7, 1)
    assert sch.waves == 7 and sch.splits == []


def test_split_group_random_invariants():
    rng = np.random.default_rng(11)
    for _ in range(300):
        G, R, W = (int(v) for v in rng.integers(1, 513, 3))
        R = int(rng.choice([7, 23, 49, int(R % 64) + 1]))
        sch = O.plan_split_group(G, R, W)
        items = [gr for a in sch.assignments for gr in a]
        assert sorted(items) == [(g, r) for g in range(G) for r in range(R)]   # completeness
        lens = [len(a) for a in sch.assignments]
        c = -(-G * R // W)
        assert max(lens) == c and all(l <= c for l in lens)
        nonempty = [l for l in lens if l]
        assert max(nonempty) - min(nonempty[:-1] or [c]) <= 1 or len(nonempty) == 1
        assert sch.waves <= sch.group_waves
        if c >= R:                                              # <= 2 workers per group
            assert all(len(ws) == 2 for _, ws in sch.splits)
        for g, ws in sch.splits:                                # prefix on earlier worker
            assert ws == sorted(ws)


def test_cache_aware_never_worse_and_fig_c():
    sch = O.plan_split_group(4, 7, 3)
    re = O.cache_aware(sch.assignments, 7)
    assert O.r_alignment(re) >= O.r_alignment(sch.assignments)
    for a, b in zip(sch.assignments, re):
        assert sorted(a) == sorted(b)                            # same multiset per worker
    # Fig. (c): a wave where concurrent SMs process H_1 of three groups
    assert any(len({re[w][t][0] for w in range(3)}) == 3 and all(re[w][t][1] == 0 for w in range(3))
               for t in range(min(len(a) for a in re)))
    for (G, R, W) in [(256, 7, 78), (896, 7, 74), (512, 23, 74), (224, 49, 74)]:
        sch = O.plan_split_group(G, R, W)
        ff = O.reorder_full_first(sch.assignments, R)
        assert O.r_alignment(ff) > O.r_alignment(sch.assignments)
        assert O.r_alignment(O.cache_aware(sch.assignments, R)) >= O.r_alignment(ff)


def test_cache_aware_divisible_fully_aligned():
    # groups divisible by workers, no splits -> 100 % of waves r-aligned
    sch = O.plan_split_group(12, 7, 4)
    assert O.r_alignment(O.cache_aware(sch.assignments, 7)) == 1.0


# ------------------------------------------------------------- metrics
def test_metrics_detect_sign_flip_block():
    rng = np.random.default_rng(12)
    A = rng.uniform(-1, 1, (64, 256))
    B = rng.uniform(-1, 1, (256, 48))
    C = A @ B
    assert O.eps_norm(C, C, A, B) == 0.0 and O.freivalds(C, A, B) < 1e-12
    bad = C.copy()
    bad[:32, :24] *= -1
    assert O.eps_rel(bad, C) > 0.3
    assert O.freivalds(bad, A, B) > 1e-3


# ------------------------------------------------------------- metric pins
def _golden_metrics():
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "metrics_2x2.txt")
    rows = []
    for ln in open(path):
        if ln.strip() and not ln.startswith("#"):
            f = ln.split()
            rows.append((f[0], np.array([float(v) for v in f[1:5]]).reshape(2, 2), float(f[5]), float(f[6])))
    return rows


def test_metrics_hand_computed():
    # tests/golden/metrics_2x2.txt: eps_norm / eps_rel on the S:175 example,
    # hand-computed.  A squared norm, ||A B|| as the denominator, or a missing
    # factor in ||A||_F ||B||_F changes these values.
    A = np.array([[1.0, 2.0], [3.0, 4.0]])
    B = np.array([[5.0, 6.0], [7.0, 8.0]])
    Cref = O.gemm_f64(A, B)
    for name, C, en, er in _golden_metrics():
        assert O.eps_norm(C, Cref, A, B) == pytest.approx(en, rel=1e-8), name
        assert O.eps_rel(C, Cref) == pytest.approx(er, rel=1e-8), name


def test_metrics_scaling_laws():
    # eps_norm is invariant under C, Cref -> a*C, a*Cref with A -> a*A, and
    # scales as 1/(ab) when only A, B are scaled by a, b (the error fixed)
    rng = np.random.default_rng(3)
    A, B = rng.uniform(-1, 1, (9, 5)), rng.uniform(-1, 1, (5, 7))
    Cref = A @ B
    C = Cref + rng.uniform(-1e-3, 1e-3, Cref.shape)
    e = O.eps_norm(C, Cref, A, B)
    assert O.eps_norm(3 * C, 3 * Cref, 3 * A, B) == pytest.approx(e, rel=1e-12)
    assert O.eps_norm(C, Cref, 2 * A, 5 * B) == pytest.approx(e / 10, rel=1e-12)
    assert O.eps_rel(4 * C, 4 * Cref) == pytest.approx(O.eps_rel(C, Cref), rel=1e-12)


# ----------------------------------------------------------- roofline pins
def test_roofline_rows_hand_computed():
    # S:439-445 roofline rows at AI = 100 (square N = 1.5*AI = 150), Strassen
    # <2,2,2;7> (nnz 12/12/12), profile FLOPS_x = FLOPS_+ = 10, beta = 1, so
    # thr/beta = 10.  By hand from the Table, Mq = Kq = Nq = 75:
    #  A: flops 5*75^2 = 28125, mem 150^2 + 7*75^2 = 61875 -> AI .45 < 10 -> t 61875
    #  B: the same, t 61875
    #  GEMM: flops 2*7*75^3 = 5906250, mem 7*(2*75^2) + 150^2 = 101250 (fused)
    #        -> AI 58.3 > 10 -> t = 590625
    #  H: flops 8*75^2 = 45000, mem 150^2 = 22500 -> AI 2 < 10 -> t 22500
    #  total 736875 -> effective 2*150^3 / 736875 = 10800/1179
    #  unfused: GEMM mem + 7*75^2 (still compute), H mem 22500 + 39375 = 61875
    #  -> total 776250 -> effective 200/23; classical 2*150^3/10 -> effective 10.
    hw = O.Profile(10.0, 10.0, 1.0)
    rows = {(a, n): v for a, n, v in O.roofline_table([O.strassen()], hw, [100])}
    assert rows[(100, "classical")] == pytest.approx(10.0, rel=1e-12)
    assert rows[(100, "strassen-2x2x2-r7")] == pytest.approx(10800 / 1179, rel=1e-12)
    rows_u = {(a, n): v for a, n, v in O.roofline_table([O.strassen()], hw, [100], fused=False)}
    assert rows_u[(100, "strassen-2x2x2-r7")] == pytest.approx(200 / 23, rel=1e-12)


def test_roofline_compute_ceiling():
    # beta, FLOPS_+ -> infinity: every stage but the GEMM vanishes and the LCMA
    # row reaches its effective ceiling FLOPS_x * mnk / R exactly
    hw = O.Profile(1.0, 1e30, 1e30)
    cat = [O.strassen(), O.strassen2(), O.laderman()]
    # AI = 576 -> N = 864, divisible by 2, 3 and 4 (no padding)
    rows = {n: v for a, n, v in O.roofline_table(cat, hw, [576])}
    assert rows["classical"] == pytest.approx(1.0, rel=1e-12)
    assert rows[O.strassen().name] == pytest.approx(8 / 7, rel=1e-9)
    assert rows[O.strassen2().name] == pytest.approx(64 / 49, rel=1e-9)
    assert rows[O.laderman().name] == pytest.approx(27 / 23, rel=1e-9)
