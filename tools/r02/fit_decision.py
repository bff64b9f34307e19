"""Refit the B200 decision model's (FLOPS_x, epilogue overhead c0, alpha)
per dtype on a cfg3 sweep (tools/cfg3_sweep.py output): the same cost
formula as decision.cpp estimate_time_b200, grid search minimising the mean
regret of the chosen algorithm.  usage: fit_decision.py sweep.json"""
import ctypes, itertools, json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_06057_b200 as L

lib = L.lib()
lib.lcma_debug_l2_partial_tiles.restype = ctypes.c_double
lib.lcma_debug_l2_partial_tiles.argtypes = [ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)]
SCH = {"strassen": (1, 2, 2, 2, 7, -1), "strassen2": (2, 4, 4, 4, 49, 1), "laderman": (3, 3, 3, 3, 23, -1)}
l2 = {k: lib.lcma_debug_l2_partial_tiles(v[0], None) for k, v in SCH.items()}


def t_lcma(name, M, N, K, e, fm, c0, alpha, beta_c, beta):
    sid, m, k, n, R, base = SCH[name]
    BK = 128.0 / e
    Mb = math.ceil(math.ceil(M / m) / 256) * 256
    Nb = math.ceil(math.ceil(N / n) / 256) * 256
    Kb = math.ceil(math.ceil(K / k) / BK) * BK
    t = (M * K + R * Mb * Kb) / beta_c + (K * N + R * Kb * Nb) / beta_c
    t_mma = 2.0 * R * Mb * Nb * Kb / fm
    if base >= 0:
        bR = 7
        partial = l2["strassen"] * 128 * 256 * 4.0
        operand = bR * (Kb / BK) * (2 * 128 * 128.0)
        rho = partial / operand
        t += t_mma * (1 + c0 + alpha * rho * rho)
        hq = 7 * math.ceil(M / 2) * math.ceil(N / 2) * 4.0
        t += (2 * hq + M * N * e) / (beta * e)
    else:
        partial = l2[name] * 128 * 256 * 4.0
        operand = R * (Kb / BK) * (2 * 128 * 128.0)
        rho = partial / operand
        t += t_mma * (1 + c0 + alpha * rho * rho)
    return t


rows = json.load(open(sys.argv[1]))["rows"]
FM = {"fp16": 1.41e15, "tf32": float(__import__("os").environ.get("FM_TF32", 0.75e15))}   # measured classical throughput (this sweep, median)
for dt, e in (("fp16", 2.0), ("tf32", 4.0)):
    rs = [r for r in rows if r["dtype"] == dt]
    best = None
    for fm in [FM[dt]]:
        for c0 in [x / 100 for x in range(-10, 31)]:
            for alpha in (0.0, 2.0, 4.0, 8.0, 16.0):
                beta_c = 4.4e12 / e
                beta = 6.55e12 / e
                reg = []
                for r in rs:
                    M, N, K = r["M"], r["N"], r["K"]
                    tc = 2.0 * M * N * K / fm
                    ch, tbest = "classical", tc
                    for name in SCH:
                        t = t_lcma(name, M, N, K, e, fm, c0, alpha, beta_c, beta)
                        if t < tbest:
                            ch, tbest = name, t
                    reg.append(r["ms"][ch] / min(r["ms"].values()))
                score = (sum(reg) / len(reg), max(reg))
                if best is None or score < best[0]:
                    best = (score, fm, c0, alpha, sum(1 for x in reg if x == 1.0))
    print(dt, "mean regret %.4f max %.4f" % best[0], "flops_mul %.3g c0 %.2f alpha %.1f correct %d/%d" %
          (best[1], best[2], best[3], best[4], len(rs)))
