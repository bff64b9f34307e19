"""CPU tests of the C-ABI library's host side (no GPU): the library loads and
exports every symbol include/lcma.h declares; its independently written
scheme tables, decision model and schedule agree with the oracle."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2605_06057_b200 as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "lcma.h")).read()
    names = set(re.findall(r"\b(lcma_[a-z_]+)\s*\(", hdr))
    assert len(names) >= 18
    lib = L.lib()
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing


@pytest.mark.parametrize("sid,make", [(1, O.strassen), (2, O.strassen2), (3, O.laderman)])
def test_library_tables_equal_oracle(sid, make):
    m, k, n, R, U, V, W = L.scheme_get(sid)
    s = make()
    assert (m, k, n, R) == (s.m, s.k, s.n, s.R)
    assert np.array_equal(U, s.U) and np.array_equal(V, s.V) and np.array_equal(W, s.W)
    assert O.brent(O.Scheme("lib", m, k, n, U, V, W))[0] == 0


def test_register_file_and_errors(tmp_path):
    s = O.laderman()
    p = tmp_path / "laderman.txt"
    p.write_text(O.scheme_to_text(s))
    sid = L.scheme_register_file(str(p))
    m, k, n, R, U, V, W = L.scheme_get(sid)
    assert np.array_equal(U, s.U) and np.array_equal(W, s.W)
    # sign flip -> SCHEME_INVALID with the failing tuple in the message
    W2 = s.W.copy()
    W2[0][np.nonzero(W2[0])[0][0], np.nonzero(W2[0])[1][0]] *= -1
    with pytest.raises(L.LcmaError, match="SCHEME_INVALID.*Brent"):
        L.scheme_register(s.U, s.V, W2)
    txt = O.scheme_to_text(O.strassen()).splitlines()
    txt[2] = "2 0"
    p.write_text("\n".join(txt))
    with pytest.raises(L.LcmaError, match="COEFF_RANGE"):
        L.scheme_register_file(str(p))
    p.write_text("2 2 2\n")
    with pytest.raises(L.LcmaError, match="PARSE.*line 1"):
        L.scheme_register_file(str(p))
    # registered scheme is usable by a plan
    sid2 = L.scheme_register(O.strassen().U, O.strassen().V, O.strassen().W, "s-copy")
    plan = L.Plan(512, 512, 512, algo="scheme", scheme_id=sid2)
    assert plan.info["R"] == 7


def test_decision_matches_oracle_random():
    rng = np.random.default_rng(3)
    cat = [O.strassen(), O.strassen2(), O.laderman()]
    names = {1: "classical", 2: "strassen-2x2x2-r7", 3: "strassen2-4x4x4-r49", 4: "laderman-3x3x3-r23"}
    for _ in range(200):
        M, N, K = (int(v) for v in rng.integers(64, 40000, 3))
        fm = 10 ** rng.uniform(12, 15.5)
        beta = fm / 10 ** rng.uniform(0, 3.5)
        fa = beta * 10 ** rng.uniform(-1, 1.5)
        for fused in (True, False):
            d = O.select(cat, M, N, K, O.Profile(fm, fa, beta), fused)
            info = L.decide(M, N, K, L.BF16, hw={"flops_mul": fm, "flops_add": fa, "beta_elems": beta},
                            fused=fused)
            assert names[info["algo"]] == d.choice
            assert info["t_pred_classical"] == pytest.approx(d.times["classical"], rel=1e-12)
            assert info["t_pred_choice"] == pytest.approx(d.times[d.choice], rel=1e-12)
            assert bool(info["memory_bound"]) == d.memory_bound


def test_decision_crossover_and_flags():
    hw = {"flops_mul": 100.0, "flops_add": 1.0, "beta_elems": 1.0}
    for n, expect in ((4096, True), (1024, False)):
        plan = L.Plan(n, n, n, algo="strassen", hw=hw)
        assert bool(plan.info["fused_condition"]) == expect      # N/26 > 100
    assert not L.Plan(64, 64, 64, hw=hw).info["lcma_condition"]


def test_plan_validation():
    with pytest.raises(L.LcmaError, match="INVALID"):
        L.Plan(0, 256, 256)
    with pytest.raises(L.LcmaError, match="MISALIGNED"):
        L.Plan(256, 256, 100)
    with pytest.raises(L.LcmaError, match="NOT_SUPPORTED"):
        L.Plan(256, 256, 256, dtype=L.FP32, algo="strassen", variant="fused_h")
    with pytest.raises(L.LcmaError, match="INVALID"):
        L.Plan(256, 256, 256, algo="scheme", scheme_id=999)


def test_plan_extents_and_workspace():
    p = L.Plan(8192, 14336, 4096, algo="strassen")
    i = p.info
    assert (i["Mb"], i["Nb"], i["Kb"]) == (4096, 7168, 2048)          # ceil extents
    assert i["Mb"] % i["BM"] == 0 and i["Nb"] % i["BN"] == 0 and i["Kb"] % i["BK"] == 0
    assert i["btilde_bytes"] == 7 * 2048 * 7168 * 2
    p2 = L.Plan(1000, 1048, 520, algo="laderman")
    i2 = p2.info
    assert 3 * i2["Mb"] >= 1000 and 3 * i2["Nb"] >= 1048 and 3 * i2["Kb"] >= 520
    # classical: only the dynamic schedule's ticket counter (256-byte region)
    assert L.Plan(256, 256, 256, algo="classical").workspace_bytes == 256
    assert L.Plan(256, 256, 256, algo="classical", schedule=4).workspace_bytes == 256


def _flatten(plan):
    W = plan.info["ctas"] // plan.info["cta_group"]
    per = []
    for w in range(W):
        items = []
        for g, r0, r1, role in plan.schedule(w):
            items += [(g, r) for r in range(r0, r1)]
        per.append(items)
    return per


def test_schedule_paper_mode_equals_oracle():
    # schedule=2 is the paper's contiguous split-group order
    for (M, N, K, algo) in [(8192, 14336, 4096, "strassen"), (4096, 4096, 4096, "strassen"),
                            (12288, 12288, 1024, "laderman")]:
        plan = L.Plan(M, N, K, algo=algo, schedule=2)
        W = plan.info["ctas"] // plan.info["cta_group"]
        sim = O.plan_split_group(plan.info["groups"], plan.info["R"], W)
        assert _flatten(plan) == sim.assignments
        assert plan.info["waves"] == sim.waves and plan.info["group_waves"] == sim.group_waves


def test_schedule_lockstep_mode_properties():
    for (M, N, K, algo, ctas) in [(8192, 14336, 4096, "strassen", 0), (1536, 2304, 512, "strassen", 6),
                                  (12288, 12288, 1024, "strassen2", 0), (2048, 3072, 512, "laderman", 10)]:
        plan = L.Plan(M, N, K, algo=algo, num_ctas=ctas)
        per = _flatten(plan)
        G, R = plan.info["groups"], plan.info["R"]
        items = sorted(x for a in per for x in a)
        assert items == [(g, r) for g in range(G) for r in range(R)]       # completeness
        assert max(len(a) for a in per) == plan.info["waves"]
        assert plan.info["waves"] == -(-G * R // len(per))                 # split-group wave count
        # lockstep rounds: every worker on the same r in each full-round wave
        W = len(per)
        q = G // W
        for t in range(q * R):
            assert len({a[t][1] for a in per}) == 1
        assert O.r_alignment(per) >= O.r_alignment(O.plan_split_group(G, R, W).assignments)


def test_schedule_group_parallel_only_mode():
    # schedule=3: whole groups round-robin, no split (the ablation step before
    # Split-Group): complete, never split, ceil(G/W)*R waves
    for (M, N, K, algo, ctas) in [(8192, 14336, 4096, "strassen", 0), (1536, 2304, 512, "strassen", 6),
                                  (2048, 3072, 512, "laderman", 10)]:
        plan = L.Plan(M, N, K, algo=algo, num_ctas=ctas, schedule=3)
        per = _flatten(plan)
        G, R = plan.info["groups"], plan.info["R"]
        assert sorted(x for a in per for x in a) == [(g, r) for g in range(G) for r in range(R)]
        assert plan.info["split_groups"] == 0
        W = len(per)
        assert plan.info["waves"] == -(-G // W) * R
        for w, a in enumerate(per):
            assert [g for g, _ in a[::R]] == list(range(w, G, W))


def test_partial_slots_product_order():
    # fused Combine H stores a C_ij partial across the boundary after product
    # position t iff first <= t < last (the last contribution goes straight to
    # the rounded C store); the product order must reach the brute-force
    # minimum for Strassen (2 of 4 C blocks: one register and one shared-memory
    # home per CTA, no L2 partial traffic)
    import itertools
    m, k, n, R, U, V, W = L.scheme_get(1)
    T = [set(np.flatnonzero(W[r].reshape(-1))) for r in range(R)]
    best = R
    for perm in itertools.permutations(range(R)):
        first, last = {}, {}
        for t, r in enumerate(perm):
            for c in T[r]:
                first.setdefault(c, t)
                last[c] = t
        best = min(best, max(sum(1 for c in first if first[c] <= t < last[c]) for t in range(R)))
    assert best == 2
    assert L.Plan(8192, 14336, 4096, algo="strassen").info["partial_slots"] == best
    for algo, mn in (("laderman", 9), ("strassen2", 16)):
        s = L.Plan(12288, 12288, 12288, algo=algo).info["partial_slots"]
        assert 1 <= s <= mn
    assert L.Plan(4096, 4096, 4096, algo="classical").info["partial_slots"] == 0
    assert L.Plan(4096, 4096, 4096, algo="strassen", variant="unfused").info["partial_slots"] == 0


def test_l2_partial_transfers_per_group():
    # fused Combine H: the two most-updated partial slots live on chip
    # (registers; shared memory for column half 0), the rest move through L2.
    # Strassen: 2 live slots -> only half of the shared-memory slot's 6 tile
    # transfers (its C_ij uses) go to L2.
    import ctypes
    f = L.lib().lcma_debug_l2_partial_tiles
    f.restype, f.argtypes = ctypes.c_double, [ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)]
    live = ctypes.c_int32()
    assert f(1, ctypes.byref(live)) == 3.0 and live.value == 2      # Strassen
    assert f(0, ctypes.byref(live)) == 0.0 and live.value == 0      # classical
    for sid in (2, 3):                                              # Strassen^2 (flat), Laderman
        m, k, n, R, U, V, W = L.scheme_get(sid)
        t = f(sid, ctypes.byref(live))
        assert 2 < live.value <= m * n
        # never more than every nonzero W entry moving through L2
        assert 0 < t <= int(np.count_nonzero(W))


def test_b200_model_two_level_and_partial_terms():
    # B200 decision model (decision_model=0): depth 2 executes two-level, so
    # its estimate carries the outer H_q fp32 round trip; fewer L2 partial
    # transfers (Strassen) must not cost more than many (Laderman) per flop
    M, N, K = 8192, 14336, 4096
    t = {a: L.Plan(M, N, K, algo=a).info["t_pred_choice"] for a in ("classical", "strassen", "strassen2", "laderman")}
    hq = 2 * 7 * (M // 2) * (N // 2) * 4 / 6.55e12          # outer H_q written + read, fp32, at HBM speed
    assert t["strassen2"] > t["strassen"] + 0.5 * hq
    # Laderman: 33 L2 partial transfers per group vs Strassen's 3
    assert t["laderman"] > t["strassen"]
    # cfg3 grid corner 16384 x 14336 x 14336 with the final kernels
    # (profiles/r02g_cfg3_decision.json): Strassen measured best in fp16
    # (1.06x), classical in tf32 -- AUTO follows both
    assert L.Plan(16384, 14336, 14336, dtype=L.FP16, algo="auto").info["scheme"].startswith("strassen-2x2x2")
    assert L.Plan(16384, 14336, 14336, dtype=L.TF32, algo="auto").info["scheme"] == "classical"
    # 16-bit cfg2: classical (measured best)
    assert L.Plan(M, N, K, dtype=L.BF16, algo="auto").info["scheme"] == "classical"


def test_producer_variant_plan_rules():
    # variant 3 (Combine A / B in the GEMM producer path, include/lcma.h):
    # Strassen on exactly tiled M, K plans; ragged M or K, or a scheme with
    # more than two A blocks in a product (Laderman), is rejected up front
    p = L.Plan(512, 512, 512, algo="strassen", variant="producer")
    assert p.info["variant"] == L.VARIANT["producer"] and p.info["cta_group"] == 2
    assert p.info["partial_slots"] == 2
    for M, N, K, algo in ((1000, 512, 512, "strassen"), (512, 512, 520, "strassen"), (768, 768, 768, "laderman")):
        with pytest.raises(L.LcmaError) as e:
            L.Plan(M, N, K, algo=algo, variant="producer")
        assert "NOT_SUPPORTED" in str(e.value)
