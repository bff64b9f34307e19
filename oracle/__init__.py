"""CPU oracle for the LCMA hot path of arxiv/paper_2605_06057 -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` leg may import this package.  It shares no code, table,
header or constant generator with ``paper_2605_06057_b200`` (the product); the
two meet only through arrays produced by the seeded input generator module.

Citations: ``P:n`` = /root/reference/PAPER.md line n, ``S:n`` = SPEC.md line n.

Contents (each function cites the passage it follows):

* schemes      -- Strassen, Laderman, standard(m,k,n), compose, text loader
* brent        -- exact bilinear identity check (C, int64)
* gemm_*       -- naive triple-loop GEMM, Eq. (1) (C, fp64 / int64)
* lcma_*       -- Algorithm 1 evaluator, Eqs. (3)-(6) (C, fp64 / int64)
* decision     -- the Decision Module of Sec. III-C, step by step (Python)
* schedule     -- Split-Group / Cache-Aware schedule simulator (Python)
* metrics      -- error metrics of DESIGN.md (numpy fp64)

Parity pins: see tests/test_oracle_*.py; every function here is pinned by a
paper value, a closed form, an invariant or brute force.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile oracle.c (plain C, -O2, OpenMP).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        I = ctypes.c_int
        L.or_round.restype = ctypes.c_double
        L.or_round.argtypes = [ctypes.c_double, I]
        L.or_round_array.argtypes = [P, I64, I]
        L.or_gemm_f64.argtypes = [I64, I64, I64, P, P, P]
        L.or_gemm_i64.argtypes = [I64, I64, I64, P, P, P]
        L.or_gemm_rows_f64.argtypes = [I64, I64, I64, P, P, P, I64, P]
        L.or_brent.restype = I64
        L.or_brent.argtypes = [I, I, I, I, P, P, P, P, P]
        L.or_lcma_f64.restype = I
        L.or_lcma_f64.argtypes = [I64, I64, I64, I, I, I, I, P, P, P, I64, I64, I64,
                                  P, P, P, P, P, P, I, I, I, P]
        L.or_lcma_i64.restype = I
        L.or_lcma_i64.argtypes = [I64, I64, I64, I, I, I, I, P, P, P, I64, I64, I64,
                                  P, P, P, P, P, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


# =============================================================== schemes
@dataclass
class Scheme:
    """LCMA tuple <m,k,n,R,U,V,W> (Sec. II-A).

    U[r,i,l] multiplies A_{i,l} (Eq. 3), V[r,l,j] multiplies B_{l,j} (Eq. 4),
    W[r,i,j] adds H_r into C_{i,j} (Eq. 6).  0-based indices.
    """
    name: str
    m: int
    k: int
    n: int
    U: np.ndarray  # int8 R x m x k
    V: np.ndarray  # int8 R x k x n
    W: np.ndarray  # int8 R x m x n

    @property
    def R(self) -> int:
        return int(self.U.shape[0])

    def nnz(self):
        """(||U||_0, ||V||_0, ||W||_0), Table "cost_model"."""
        return (int(np.count_nonzero(self.U)), int(np.count_nonzero(self.V)),
                int(np.count_nonzero(self.W)))


def _scheme_from_products(name, m, k, n, products, outputs):
    """Build U, V, W from product strings "(a11+a22)*(b11+b22)" and output
    equations {"c11": "m1+m4-m5+m7"} (1-based names, as in the literature)."""
    R = len(products)
    U = np.zeros((R, m, k), np.int8)
    V = np.zeros((R, k, n), np.int8)
    W = np.zeros((R, m, n), np.int8)

    def terms(expr):
        expr = expr.replace(" ", "").strip("()")
        out, sign, tok = [], 1, ""
        for ch in expr + "+":
            if ch in "+-":
                if tok:
                    out.append((sign, tok))
                sign, tok = (1 if ch == "+" else -1), ""
            else:
                tok += ch
        return out

    for r, prod in enumerate(products):
        a_part, b_part = prod.split("*")
        for s, t in terms(a_part):
            assert t[0] == "a"
            U[r, int(t[1]) - 1, int(t[2]) - 1] += s
        for s, t in terms(b_part):
            assert t[0] == "b"
            V[r, int(t[1]) - 1, int(t[2]) - 1] += s
    for cname, expr in outputs.items():
        i, j = int(cname[1]) - 1, int(cname[2]) - 1
        for s, t in terms(expr):
            assert t[0] == "m"
            W[int(t[1:]) - 1, i, j] += s
    return Scheme(name, m, k, n, U, V, W)


def strassen() -> Scheme:
    """Strassen <2,2,2;7> (figure lost, classic 1969 numbering --
    DESIGN.md reading 1).  Pinned by the S:226-247 worked example and by
    "C_11 depends on H1, H4, H5, H7"."""
    products = [
        "(a11+a22)*(b11+b22)",   # H1
        "(a21+a22)*(b11)",       # H2
        "(a11)*(b12-b22)",       # H3
        "(a22)*(b21-b11)",       # H4
        "(a11+a12)*(b22)",       # H5
        "(a21-a11)*(b11+b12)",   # H6
        "(a12-a22)*(b21+b22)",   # H7
    ]
    outputs = {"c11": "m1+m4-m5+m7", "c12": "m3+m5", "c21": "m2+m4",
               "c22": "m1-m2+m3+m6"}
    return _scheme_from_products("strassen-2x2x2-r7", 2, 2, 2, products, outputs)


def laderman() -> Scheme:
    """Laderman <3,3,3;23> (P:663 names it; coefficients not printed --
    Laderman 1976 table, reading 2).  Pinned by the exhaustive
    Brent identity only ("parity unpinned" for the specific coefficients)."""
    products = [
        "(a11+a12+a13-a21-a22-a32-a33)*(b22)",   # 1
        "(a11-a21)*(-b12+b22)",                  # 2
        "(a22)*(-b11+b12+b21-b22-b23-b31+b33)",  # 3
        "(-a11+a21+a22)*(b11-b12+b22)",          # 4
        "(a21+a22)*(-b11+b12)",                  # 5
        "(a11)*(b11)",                           # 6
        "(-a11+a31+a32)*(b11-b13+b23)",          # 7
        "(-a11+a31)*(b13-b23)",                  # 8
        "(a31+a32)*(-b11+b13)",                  # 9
        "(a11+a12+a13-a22-a23-a31-a32)*(b23)",   # 10
        "(a32)*(-b11+b13+b21-b22-b23-b31+b32)",  # 11
        "(-a13+a32+a33)*(b22+b31-b32)",          # 12
        "(a13-a33)*(b22-b32)",                   # 13
        "(a13)*(b31)",                           # 14
        "(a32+a33)*(-b31+b32)",                  # 15
        "(-a13+a22+a23)*(b23+b31-b33)",          # 16
        "(a13-a23)*(b23-b33)",                   # 17
        "(a22+a23)*(-b31+b33)",                  # 18
        "(a12)*(b21)",                           # 19
        "(a23)*(b32)",                           # 20
        "(a21)*(b13)",                           # 21
        "(a31)*(b12)",                           # 22
        "(a33)*(b33)",                           # 23
    ]
    outputs = {
        "c11": "m6+m14+m19",
        "c12": "m1+m4+m5+m6+m12+m14+m15",
        "c13": "m6+m7+m9+m10+m14+m16+m18",
        "c21": "m2+m3+m4+m6+m14+m16+m17",
        "c22": "m2+m4+m5+m6+m20",
        "c23": "m14+m16+m17+m18+m21",
        "c31": "m6+m7+m8+m11+m12+m13+m14",
        "c32": "m12+m13+m14+m15+m22",
        "c33": "m6+m7+m8+m9+m23",
    }
    return _scheme_from_products("laderman-3x3x3-r23", 3, 3, 3, products, outputs)


def standard(m: int, k: int, n: int) -> Scheme:
    """Classical decomposition: one product per (i,l,j), rank m*k*n."""
    R = m * k * n
    U = np.zeros((R, m, k), np.int8)
    V = np.zeros((R, k, n), np.int8)
    W = np.zeros((R, m, n), np.int8)
    r = 0
    for i in range(m):
        for l in range(k):
            for j in range(n):
                U[r, i, l] = 1
                V[r, l, j] = 1
                W[r, i, j] = 1
                r += 1
    return Scheme(f"standard-{m}x{k}x{n}", m, k, n, U, V, W)


def compose(outer: Scheme, inner: Scheme) -> Scheme:
    """Two-level scheme ("two-level recursive Strassen"), S:70-78:
    U'[(r1,r2),(i1,i2),(l1,l2)] = U1[r1,i1,l1] * U2[r2,i2,l2] with
    r = r1*R2 + r2 and block index i = i1*m2 + i2 (outer-major, DESIGN.md
    reading 3); likewise V, W."""
    m, k, n = outer.m * inner.m, outer.k * inner.k, outer.n * inner.n
    R = outer.R * inner.R

    def kron(T1, T2):
        R1, p1, q1 = T1.shape
        R2, p2, q2 = T2.shape
        out = np.zeros((R1 * R2, p1 * p2, q1 * q2), np.int8)
        for r1 in range(R1):
            for r2 in range(R2):
                for a in range(p1):
                    for b in range(q1):
                        for c in range(p2):
                            for d in range(q2):
                                out[r1 * R2 + r2, a * p2 + c, b * q2 + d] = T1[r1, a, b] * T2[r2, c, d]
        return out

    return Scheme(f"{outer.name}*{inner.name}", m, k, n,
                  kron(outer.U, inner.U), kron(outer.V, inner.V), kron(outer.W, inner.W))


def strassen2() -> Scheme:
    """<4,4,4;49> = compose(Strassen, Strassen)."""
    s = compose(strassen(), strassen())
    s.name = "strassen2-4x4x4-r49"
    return s


class SchemeFileError(ValueError):
    pass


def load_scheme_text(text: str, name: str = "file") -> Scheme:
    """Text format of S:143-145: line 1 "m k n R"; then all "U r" blocks,
    all "V r" blocks, all "W r" blocks, each followed by its factor-matrix
    rows; '#' starts a comment.  Entries outside {-1,0,1} are rejected
    (reading 4)."""
    lines = []
    for ln, raw in enumerate(text.splitlines(), 1):
        s = raw.split("#", 1)[0].strip()
        if s:
            lines.append((ln, s))
    if not lines:
        raise SchemeFileError("empty scheme file")
    ln, head = lines[0]
    try:
        m, k, n, R = (int(x) for x in head.split())
    except Exception:
        raise SchemeFileError(f"line {ln}: expected 'm k n R'")
    U = np.zeros((R, m, k), np.int8)
    V = np.zeros((R, k, n), np.int8)
    W = np.zeros((R, m, n), np.int8)
    pos = 1
    for tag, T, rows, cols in (("U", U, m, k), ("V", V, k, n), ("W", W, m, n)):
        for r in range(R):
            if pos >= len(lines):
                raise SchemeFileError(f"unexpected end of file in {tag} block {r + 1}")
            ln, s = lines[pos]
            parts = s.split()
            if len(parts) != 2 or parts[0] != tag or parts[1] != str(r + 1):
                raise SchemeFileError(f"line {ln}: expected '{tag} {r + 1}'")
            pos += 1
            for p in range(rows):
                if pos >= len(lines):
                    raise SchemeFileError(f"unexpected end of file in {tag} {r + 1}")
                ln, s = lines[pos]
                vals = s.split()
                if len(vals) != cols:
                    raise SchemeFileError(f"line {ln}: expected {cols} entries")
                for q, v in enumerate(vals):
                    try:
                        iv = int(v)
                    except ValueError:
                        raise SchemeFileError(f"line {ln}: bad entry {v!r}")
                    if iv not in (-1, 0, 1):
                        raise SchemeFileError(f"line {ln}: coefficient {iv} outside {{-1,0,1}}")
                    T[r, p, q] = iv
                pos += 1
    if pos != len(lines):
        raise SchemeFileError(f"line {lines[pos][0]}: trailing content")
    return Scheme(name, m, k, n, U, V, W)


def scheme_to_text(s: Scheme) -> str:
    out = [f"{s.m} {s.k} {s.n} {s.R}"]
    for tag, T in (("U", s.U), ("V", s.V), ("W", s.W)):
        for r in range(s.R):
            out.append(f"{tag} {r + 1}")
            for row in T[r]:
                out.append(" ".join(str(int(v)) for v in row))
    return "\n".join(out) + "\n"


# ================================================================= brent
def brent(s: Scheme):
    """Exact Brent-equation check: returns (n_failures, first_tuple,
    n_checked).  first_tuple = (i, l, l2, j, i2, j2, observed, expected)."""
    first = np.zeros(8, np.int64)
    checked = np.zeros(1, np.int64)
    U = np.ascontiguousarray(s.U, np.int8)
    V = np.ascontiguousarray(s.V, np.int8)
    W = np.ascontiguousarray(s.W, np.int8)
    f = lib().or_brent(s.m, s.k, s.n, s.R, _p(U), _p(V), _p(W), _p(first), _p(checked))
    return int(f), tuple(int(x) for x in first), int(checked[0])


# ================================================================= gemm
def gemm_f64(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Naive fp64 i-k-j GEMM, Eq. (1) P:581."""
    A = np.ascontiguousarray(A, np.float64)
    B = np.ascontiguousarray(B, np.float64)
    M, K = A.shape
    K2, N = B.shape
    if K != K2:
        raise ValueError("dimension mismatch")
    C = np.empty((M, N), np.float64)
    lib().or_gemm_f64(M, N, K, _p(A), _p(B), _p(C))
    return C


def gemm_i64(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    A = np.ascontiguousarray(A, np.int64)
    B = np.ascontiguousarray(B, np.int64)
    M, K = A.shape
    K2, N = B.shape
    if K != K2:
        raise ValueError("dimension mismatch")
    C = np.empty((M, N), np.int64)
    lib().or_gemm_i64(M, N, K, _p(A), _p(B), _p(C))
    return C


def gemm_rows_f64(A: np.ndarray, B: np.ndarray, rows) -> np.ndarray:
    """Rows `rows` of A*B (naive fp64) -- for sampled checks at full size."""
    A = np.ascontiguousarray(A, np.float64)
    B = np.ascontiguousarray(B, np.float64)
    rows = np.ascontiguousarray(rows, np.int64)
    M, K = A.shape
    N = B.shape[1]
    C = np.empty((len(rows), N), np.float64)
    lib().or_gemm_rows_f64(M, N, K, _p(A), _p(B), _p(rows), len(rows), _p(C))
    return C


# ========================================================= Algorithm 1
FMT = {None: 0, "fp64": 0, "bf16": 1, "fp16": 2, "tf32": 3, "fp32": 4, "tf32_rz": 5}


def round_to(x: np.ndarray, fmt: str) -> np.ndarray:
    """Round fp64 values to bf16/fp16 (RN-even), tf32 (RN-away), fp32, or
    truncate to tf32 ("tf32_rz")."""
    y = np.array(x, np.float64, copy=True, order="C")
    lib().or_round_array(_p(y), y.size, FMT[fmt])
    return y


def default_extents(M, N, K, s: Scheme):
    """ceil(M/m), ceil(K/k), ceil(N/n)."""
    return -(-M // s.m), -(-K // s.k), -(-N // s.n)


@dataclass
class LcmaResult:
    C: np.ndarray
    At: np.ndarray | None = None
    Bt: np.ndarray | None = None
    H: np.ndarray | None = None
    counters: dict = field(default_factory=dict)


_COUNTER_NAMES = ("combineA_adds", "combineB_adds", "gemm_mults", "gemm_adds",
                  "combineH_adds", "A_loads", "B_loads", "H_loads", "H_stores")


def lcma_f64(A, B, s: Scheme, extents=None, fmt_in=None, fmt_h=None, fmt_out=None,
             intermediates=False) -> LcmaResult:
    """Algorithm 1 in fp64 with optional rounding points."""
    A = np.ascontiguousarray(A, np.float64)
    B = np.ascontiguousarray(B, np.float64)
    M, K = A.shape
    N = B.shape[1]
    Mb, Kb, Nb = extents if extents else default_extents(M, N, K, s)
    C = np.empty((M, N), np.float64)
    At = np.empty((s.R, Mb, Kb)) if intermediates else None
    Bt = np.empty((s.R, Kb, Nb)) if intermediates else None
    H = np.empty((s.R, Mb, Nb)) if intermediates else None
    cnt = np.zeros(9, np.int64)
    U, V, W = (np.ascontiguousarray(t, np.int8) for t in (s.U, s.V, s.W))
    rc = lib().or_lcma_f64(M, N, K, s.m, s.k, s.n, s.R, _p(U), _p(V), _p(W), Mb, Kb, Nb,
                           _p(A), _p(B), _p(C), _p(At), _p(Bt), _p(H),
                           FMT[fmt_in], FMT[fmt_h], FMT[fmt_out], _p(cnt))
    if rc != 0:
        raise ValueError("bad block extents")
    return LcmaResult(C, At, Bt, H, dict(zip(_COUNTER_NAMES, (int(c) for c in cnt))))


def lcma_rows_f64(A, B, s: Scheme, rows, extents=None, fmt_in=None, fmt_out=None) -> np.ndarray:
    """Rows `rows` of Algorithm 1 with the dtype-faithful rounding
    points of lcma_f64 (fmt_in after Combine A / B, fmt_out on C; H and the
    Combine-H sums in fp64): for sampled checks at full size, where the whole
    evaluator would take minutes.  Output row rho = i*Mb + x only needs row x
    of every A~_r (Eq. 3) and all of B~_r (Eq. 4); H_r[x, :]
    (Eq. 5) is a library matmul step; Combine H is Eq. 6.
    Zero padding outside M x K / K x N."""
    A = np.asarray(A, np.float64)
    B = np.asarray(B, np.float64)
    M, K = A.shape
    N = B.shape[1]
    Mb, Kb, Nb = extents if extents else default_extents(M, N, K, s)
    Ap = np.zeros((s.m * Mb, s.k * Kb))
    Ap[:M, :K] = A
    Bp = np.zeros((s.k * Kb, s.n * Nb))
    Bp[:K, :N] = B
    rows = np.asarray(rows, np.int64)
    out = np.zeros((len(rows), N))
    Bt = []
    for r in range(s.R):                                   # Combine B (Eq. 4)
        acc = np.zeros((Kb, Nb))
        for l in range(s.k):
            for j in range(s.n):
                if s.V[r, l, j]:
                    acc += s.V[r, l, j] * Bp[l * Kb:(l + 1) * Kb, j * Nb:(j + 1) * Nb]
        Bt.append(round_to(acc, fmt_in) if fmt_in else acc)
    for q, rho in enumerate(rows):
        i, x = divmod(int(rho), Mb)
        crow = np.zeros(s.n * Nb)
        for r in range(s.R):
            if not s.W[r, i, :].any():
                continue
            at = np.zeros(Kb)                                # Combine A (Eq. 3), row x
            for i2 in range(s.m):
                for l in range(s.k):
                    if s.U[r, i2, l]:
                        at += s.U[r, i2, l] * Ap[i2 * Mb + x, l * Kb:(l + 1) * Kb]
            if fmt_in:
                at = round_to(at, fmt_in)
            h = at @ Bt[r]                                   # Eq. 5, row x of H_r
            for j in range(s.n):                             # Eq. 6
                if s.W[r, i, j]:
                    crow[j * Nb:(j + 1) * Nb] += s.W[r, i, j] * h
        out[q] = crow[:N]          # C_ij holds columns j*Nb .. j*Nb+Nb-1: crop to N
    return round_to(out, fmt_out) if fmt_out else out


def lcma_i64(A, B, s: Scheme, extents=None, intermediates=False) -> LcmaResult:
    """Algorithm 1 in exact int64 (exact mode)."""
    A = np.ascontiguousarray(A, np.int64)
    B = np.ascontiguousarray(B, np.int64)
    M, K = A.shape
    N = B.shape[1]
    Mb, Kb, Nb = extents if extents else default_extents(M, N, K, s)
    C = np.empty((M, N), np.int64)
    At = np.empty((s.R, Mb, Kb), np.int64) if intermediates else None
    Bt = np.empty((s.R, Kb, Nb), np.int64) if intermediates else None
    H = np.empty((s.R, Mb, Nb), np.int64) if intermediates else None
    U, V, W = (np.ascontiguousarray(t, np.int8) for t in (s.U, s.V, s.W))
    rc = lib().or_lcma_i64(M, N, K, s.m, s.k, s.n, s.R, _p(U), _p(V), _p(W), Mb, Kb, Nb,
                           _p(A), _p(B), _p(C), _p(At), _p(Bt), _p(H))
    if rc != 0:
        raise ValueError("bad block extents")
    return LcmaResult(C, At, Bt, H)


# ========================================================= decision model
@dataclass
class Profile:
    """Hardware triple (FLOPS_x, FLOPS_+, beta) of P:171-175; beta in
    elements/s for the data type."""
    flops_mul: float
    flops_add: float
    beta: float


@dataclass
class StageCost:
    stage: str
    flops: float
    mem: float
    time: float
    bound: str


def gemm_intensity(M, N, K):
    """Eq. stdgemm left side: 2MNK / (MK + NK + MN)."""
    return 2.0 * M * N * K / (M * K + N * K + M * N)


def std_gemm_memory_bound(M, N, K, hw: Profile) -> bool:
    """Eq. stdgemm: memory bound iff AI <= FLOPS_x / beta ("<=", reading 13)."""
    return gemm_intensity(M, N, K) <= hw.flops_mul / hw.beta


def _stage(stage, flops, mem, thr, beta):
    # compute-bound iff flops/mem > thr/beta (strict), time = flops/thr,
    # else memory-bound, time = mem/beta.
    if mem > 0 and flops / mem > thr / beta:
        return StageCost(stage, flops, mem, flops / thr, "compute")
    return StageCost(stage, flops, mem, mem / beta, "memory")


def stage_costs(s: Scheme, M, N, K, hw: Profile, fused=True):
    """Table "cost_model" with ceil quotients; the
    fused variant drops the R/mn H traffic."""
    R = s.R
    nU, nV, nW = s.nnz()
    Mq, Kq, Nq = -(-M // s.m), -(-K // s.k), -(-N // s.n)
    a = _stage("A", (nU - R) * Mq * Kq, M * K + R * Mq * Kq, hw.flops_add, hw.beta)
    b = _stage("B", (nV - R) * Kq * Nq, N * K + R * Kq * Nq, hw.flops_add, hw.beta)
    gm = R * (Mq * Kq + Kq * Nq) + (M * N if fused else R * Mq * Nq)
    g = _stage("GEMM", 2.0 * R * Mq * Nq * Kq, gm, hw.flops_mul, hw.beta)
    hm = M * N if fused else M * N + R * Mq * Nq
    h = _stage("H", (nW - s.m * s.n) * Mq * Nq, hm, hw.flops_add, hw.beta)
    return [a, b, g, h]


def estimate_time(s: Scheme | None, M, N, K, hw: Profile, fused=True) -> float:
    """Sum of per-stage times, no overlap.  s=None: the
    standard GEMM, 2MNK/FLOPS_x."""
    if s is None:
        return 2.0 * M * N * K / hw.flops_mul
    return sum(c.time for c in stage_costs(s, M, N, K, hw, fused))


def lcma_condition_lhs(s: Scheme, M, N, K, fused: bool) -> float:
    """Left side of Eq. lcma_condition or Eq. fused_condition."""
    m, k, n, R = s.m, s.k, s.n, s.R
    num = 2.0 * M * N * K * (1.0 - R / (m * n * k))
    den = M * K * (1 + R / (m * k)) + N * K * (1 + R / (n * k)) + \
        M * N * (1.0 if fused else (1 + R / (m * n)))
    return num / den


def lcma_beneficial(s: Scheme, M, N, K, hw: Profile, fused=True) -> bool:
    if s.R >= s.m * s.n * s.k:
        return False
    return lcma_condition_lhs(s, M, N, K, fused) > hw.flops_mul / hw.beta


@dataclass
class Decision:
    choice: str            # "classical" or scheme name
    times: dict            # name -> predicted seconds
    speedup: float         # t_std / t_choice
    memory_bound: bool


def select(catalog, M, N, K, hw: Profile, fused=True) -> Decision:
    """Decision Module: Eq. stdgemm early exit; else argmin of the
    estimated time over {classical} U catalog; ties -> classical, then name
    (S:427)."""
    t_std = estimate_time(None, M, N, K, hw)
    if std_gemm_memory_bound(M, N, K, hw):
        return Decision("classical", {"classical": t_std}, 1.0, True)
    times = {"classical": t_std}
    best, best_t = "classical", t_std
    for s in sorted(catalog, key=lambda s: s.name):
        if s.R >= s.m * s.k * s.n:
            continue
        t = estimate_time(s, M, N, K, hw, fused)
        times[s.name] = t
        if t < best_t:
            best, best_t = s.name, t
    return Decision(best, times, t_std / best_t, False)


def roofline_table(catalog, hw: Profile, intensities, fused=True):
    """Roofline rows: for each intensity, a square shape with
    AI_std = 2N/3 realises it; effective = 2N^3 / t_est per algorithm."""
    rows = []
    for ai in intensities:
        Nn = max(1, int(round(1.5 * ai)))
        for s in [None] + list(catalog):
            t = estimate_time(s, Nn, Nn, Nn, hw, fused)
            rows.append((ai, "classical" if s is None else s.name, 2.0 * Nn ** 3 / t))
    return rows


def effective_ceiling(s: Scheme, flops_mul: float) -> float:
    """Compute-side effective ceiling FLOPS_x * mnk / R."""
    return flops_mul * s.m * s.n * s.k / s.R


# ========================================================= schedule sim
@dataclass
class Schedule:
    assignments: list      # per worker: list of (g, r)
    waves: int
    group_waves: int
    waste: float
    splits: list           # (g, [workers...])


def plan_split_group(G: int, R: int, W: int) -> Schedule:
    """Split-Group Parallelism: tiles t = g*R + r distributed in
    contiguous chunks of capacity c = ceil(G*R/W); a group overflowing a
    worker's capacity continues on the next worker."""
    T = G * R
    c = -(-T // W)
    assign = []
    for w in range(W):
        lo, hi = w * c, min((w + 1) * c, T)
        assign.append([(t // R, t % R) for t in range(lo, hi)])
    waves = max(len(a) for a in assign)
    group_waves = -(-G // W) * R           # group-granular scheduling
    owners = {}
    for w, a in enumerate(assign):
        for g, _ in a:
            owners.setdefault(g, [])
            if w not in owners[g]:
                owners[g].append(w)
    splits = [(g, ws) for g, ws in sorted(owners.items()) if len(ws) > 1]
    return Schedule(assign, waves, group_waves, (group_waves - waves) / waves, splits)


def r_alignment(assign) -> float:
    """Fraction of waves in which every active worker processes the same r."""
    waves = max(len(a) for a in assign)
    if waves == 0:
        return 1.0
    good = 0
    for t in range(waves):
        rs = {a[t][1] for a in assign if t < len(a)}
        good += (len(rs) == 1)
    return good / waves


def reorder_rg_sorted(assign):
    """Cache-aware order (b): per-worker stable sort by (r, g)."""
    return [sorted(a, key=lambda gr: (gr[1], gr[0])) for a in assign]


def reorder_full_first(assign, R: int):
    """Cache-aware order (c) "full-first" (reading 11): each worker's
    whole groups first, in r order, then its split portions."""
    out = []
    for a in assign:
        counts = {}
        for g, _ in a:
            counts[g] = counts.get(g, 0) + 1
        whole = [gr for gr in a if counts[gr[0]] == R]
        part = [gr for gr in a if counts[gr[0]] != R]
        out.append(whole + part)
    return out


def cache_aware(assign, R: int):
    """Never lower than the input order: best of the candidates by the
    r-alignment metric, ties -> input order."""
    best, best_v = assign, r_alignment(assign)
    for cand in (reorder_full_first(assign, R), reorder_rg_sorted(assign)):
        v = r_alignment(cand)
        if v > best_v:
            best, best_v = cand, v
    return best


# ================================================================ metrics
def eps_norm(C, Cref, A, B) -> float:
    """||C - C_ref||_F / (||A||_F ||B||_F) -- the BASELINE.json gate."""
    C = np.asarray(C, np.float64)
    Cref = np.asarray(Cref, np.float64)
    return float(np.linalg.norm(C - Cref) /
                 (np.linalg.norm(np.asarray(A, np.float64)) * np.linalg.norm(np.asarray(B, np.float64))))


def eps_rel(C, Cref) -> float:
    Cref = np.asarray(Cref, np.float64)
    d = np.linalg.norm(Cref)
    return float(np.linalg.norm(np.asarray(C, np.float64) - Cref) / (d if d else 1.0))


def freivalds(C, A, B, trials=4, seed=0) -> float:
    """max over trials of ||C x - A (B x)||_2 / (||A||_F ||B||_F ||x||_2),
    x random +-1: covers all of C at O(MN + NK + MK) cost."""
    rng = np.random.default_rng(seed)
    C = np.asarray(C, np.float64)
    A = np.asarray(A, np.float64)
    B = np.asarray(B, np.float64)
    nA, nB = np.linalg.norm(A), np.linalg.norm(B)
    worst = 0.0
    for _ in range(trials):
        x = rng.choice([-1.0, 1.0], size=C.shape[1])
        r = C @ x - A @ (B @ x)
        worst = max(worst, float(np.linalg.norm(r) / (nA * nB * np.linalg.norm(x))))
    return worst


# ================================================================ FP8
# "the full BF16-to-quantized-FP8 workflow with 1 x 128 block-wise scaling for
# FP8E4M3", "fuses the quantization into the Combine A stage".
# DESIGN.md reading 23: every 1 x 128 block (one row of an operand, 128
# consecutive K elements) gets one power-of-two scale 2^e (UE8M0), the smallest
# with amax <= 448 * 2^e; the block is stored as E4M3(x / 2^e) (RN-even,
# satfinite).  B~ blocks run along K for each output column.  The oracle
# quantizes the exact (fp64) combined operand; the product and Combine H are
# exact (fp64), C is rounded once to the output type.
E4M3_MAX = 448.0


def round_e4m3(x) -> np.ndarray:
    """RN-even rounding of fp64 values to FP8 E4M3 (OCP E4M3: bias 7, 3
    mantissa bits, normals 2^-6 .. 448, subnormal spacing 2^-9, no
    infinities), saturating to +-448."""
    x = np.asarray(x, np.float64)
    a = np.abs(x)
    _, ex = np.frexp(np.where(a > 0, a, 1.0))      # a = f * 2^ex, f in [0.5, 1)
    e = np.maximum(ex - 1, -6)                      # binade exponent (subnormals share -6)
    spacing = np.ldexp(1.0, e - 3)                  # 3 mantissa bits
    y = np.round(a / spacing) * spacing             # np.round: half to even
    y = np.minimum(y, E4M3_MAX)
    return np.where(x < 0, -y, y)


def scale_exponent(amax) -> np.ndarray:
    """Smallest integer e with amax <= 448 * 2^e (0 for an all-zero block),
    clamped to the UE8M0 range [-127, 127].  Written as the definition: a
    first guess from log2, then exact comparisons move it to the minimum."""
    amax = np.asarray(amax, np.float64)
    pos = amax > 0
    safe = np.where(pos, amax, E4M3_MAX)
    e = np.ceil(np.log2(safe / E4M3_MAX)).astype(np.int64)
    for _ in range(2):
        e = np.where(safe > np.ldexp(E4M3_MAX, e), e + 1, e)            # not enough
        e = np.where(safe <= np.ldexp(E4M3_MAX, e - 1), e - 1, e)       # not the smallest
    e = np.where(pos, e, 0)
    return np.clip(e, -127, 127)


def quantize_1x128(X):
    """1 x 128 block scaling of a (rows, K) operand, K a multiple of 128:
    returns (Q, e) with Q the E4M3 values (as fp64) and e[rows, K/128] the
    scale exponents; the dequantized operand is Q * 2^e per block."""
    X = np.asarray(X, np.float64)
    rows, K = X.shape
    if K % 128:
        raise ValueError("K must be a multiple of 128 (zero-pad the block)")
    blk = X.reshape(rows, K // 128, 128)
    e = scale_exponent(np.abs(blk).max(axis=2))
    Q = round_e4m3(blk / np.ldexp(1.0, e)[..., None])
    return Q.reshape(rows, K), e


def dequantize_1x128(Q, e) -> np.ndarray:
    Q = np.asarray(Q, np.float64)
    rows, K = Q.shape
    return (Q.reshape(rows, K // 128, 128) * np.ldexp(1.0, np.asarray(e))[..., None]).reshape(rows, K)


def combine_b_fp8(B, s: Scheme, extents):
    """Combine B (Eq. 4) in exact arithmetic, then each B~_r quantized
    1 x 128 along K per column n (reading 23).  Returns (Q[R][Nb][Kb],
    e[R][Nb][Kb/128]) -- B~_r stored N x K, the nn.Linear layout."""
    B = np.asarray(B, np.float64)
    K, N = B.shape
    Mb, Kb, Nb = extents
    Bp = np.zeros((s.k * Kb, s.n * Nb))
    Bp[:K, :N] = B
    Q = np.empty((s.R, Nb, Kb))
    E = np.empty((s.R, Nb, Kb // 128), np.int64)
    for r in range(s.R):
        acc = np.zeros((Kb, Nb))
        for l in range(s.k):
            for j in range(s.n):
                if s.V[r, l, j]:
                    acc += s.V[r, l, j] * Bp[l * Kb:(l + 1) * Kb, j * Nb:(j + 1) * Nb]
        Q[r], E[r] = quantize_1x128(acc.T)
    return Q, E


def _padded_rows(X, rows, c0, width):
    """Rows `rows` of X, columns [c0, c0 + width), zero outside X."""
    out = np.zeros((len(rows), width))
    R_, C_ = X.shape
    for q, rho in enumerate(rows):
        if rho < R_ and c0 < C_:
            seg = X[rho, c0:min(c0 + width, C_)]
            out[q, :len(seg)] = seg
    return out


def combine_a_fp8_rows(A, s: Scheme, rows_x, extents):
    """Combine A (Eq. 3) for block rows x in `rows_x`, exact, then 1 x
    128 quantization along K (the quantization fused into Combine A).
    Returns (Q[R][len(rows_x)][Kb], e[R][len(rows_x)][Kb/128])."""
    A = np.asarray(A, np.float64)
    Mb, Kb, Nb = extents
    xs = np.asarray(rows_x, np.int64)
    Q = np.empty((s.R, len(xs), Kb))
    E = np.empty((s.R, len(xs), Kb // 128), np.int64)
    for r in range(s.R):
        acc = np.zeros((len(xs), Kb))
        for i in range(s.m):
            for l in range(s.k):
                if s.U[r, i, l]:
                    acc += s.U[r, i, l] * _padded_rows(A, i * Mb + xs, l * Kb, Kb)
        Q[r], E[r] = quantize_1x128(acc)
    return Q, E


def lcma_rows_fp8(A, B, s: Scheme, rows, extents, fmt_out=None, bq=None) -> np.ndarray:
    """Rows `rows` of Algorithm 1 on the FP8 path: Combine A / B
    exact then quantized 1 x 128 (reading 23), H_r = dequant(A~_r) .
    dequant(B~_r) exact (Eq. 5; a library matmul step), Combine H (Eq. 6)
    exact, C rounded once to fmt_out.  `bq` = a precomputed combine_b_fp8."""
    A = np.asarray(A, np.float64)
    M, K = A.shape
    N = np.asarray(B).shape[1]
    Mb, Kb, Nb = extents
    QB, EB = bq if bq is not None else combine_b_fp8(B, s, extents)
    Bdq = [dequantize_1x128(QB[r], EB[r]).T for r in range(s.R)]          # Kb x Nb
    rows = np.asarray(rows, np.int64)
    out = np.zeros((len(rows), N))
    xs = np.unique(rows % Mb)
    QA, EA = combine_a_fp8_rows(A, s, xs, extents)
    for q, rho in enumerate(rows):
        i, x = divmod(int(rho), Mb)
        k = int(np.searchsorted(xs, x))
        crow = np.zeros(s.n * Nb)
        for r in range(s.R):
            if not s.W[r, i, :].any():
                continue
            h = dequantize_1x128(QA[r, k:k + 1], EA[r, k:k + 1])[0] @ Bdq[r]   # Eq. 5, row x of H_r
            for j in range(s.n):                                            # Eq. 6
                if s.W[r, i, j]:
                    crow[j * Nb:(j + 1) * Nb] += s.W[r, i, j] * h
        out[q] = crow[:N]
    return round_to(out, fmt_out) if fmt_out else out
