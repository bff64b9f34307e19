/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for the LCMA hot path of
 * arxiv/paper_2605_06057 ("FalconGEMM").  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or constant with paper_2605_06057_b200/.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n.
 *
 *   or_gemm_*        C = A*B by the textbook i-k-j triple loop (Eq. 1).
 *   or_brent         Sum_r U[r,i,l] V[r,l',j] W[r,i',j'] = [i=i'][l=l'][j=j']
 *                    over every index tuple, exact int64.  This is the
 *                    algebraic condition under which Eqs. 3-6
 *                    reproduce Eq. 2 for all A, B.
 *   or_lcma          Algorithm 1 "LCMA Workflow" step by step:
 *                    stage 1 Combine A (Eq. 3), stage 2 Combine B
 *                    (Eq. 4), stage 3 H_r = At_r * Bt_r (Eq. 5),
 *                    stage 4 Combine H (Eq. 6); zero padding for the
 *                    ceil(M/m) block extents.
 *
 * Rounding modes (reading 7): an optional rounding of At/Bt to the
 * MMA input type, of H (the "downcast H" path of P:518), and of C to the
 * output type; all arithmetic in between is fp64.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- rounding */
/* fmt: 0 = none (fp64), 1 = bf16 (RN-even), 2 = fp16 (RN-even, IEEE binary16
 * range incl. subnormals and overflow to inf), 3 = tf32 (round-to-nearest,
 * ties away: cvt.rna.tf32.f32), 4 = fp32 (RN-even), 5 = tf32 truncation
 * (round toward zero: how the tf32 MMA reads raw fp32 operands). */
static double round_sig(double x, int sig_bits, int ties_away, int emin, int emax);
static double trunc_sig(double x, int sig_bits)
{
    if (x == 0.0 || !isfinite(x)) return x;
    int e;
    double f = frexp(x, &e);
    double scaled = ldexp(f, sig_bits);
    return ldexp(trunc(scaled), e - sig_bits);
}
static double round_sig(double x, int sig_bits, int ties_away, int emin, int emax)
{
    if (x == 0.0 || !isfinite(x)) return x;
    int e;
    double f = frexp(x, &e);           /* x = f * 2^e, 0.5 <= |f| < 1 */
    /* value has exponent (e-1) in the 1.xxx convention */
    int exp1 = e - 1;
    int bits = sig_bits;
    if (exp1 < emin) {                 /* subnormal: fewer significant bits */
        bits = sig_bits - (emin - exp1);
        if (bits < 0) return copysign(0.0, x);
    }
    double scaled = ldexp(f, bits);    /* |scaled| in [2^(bits-1), 2^bits) */
    double r;
    if (ties_away) {
        r = floor(fabs(scaled) + 0.5);
        r = copysign(r, scaled);
    } else {
        r = nearbyint(scaled);         /* default FE_TONEAREST = ties-to-even */
    }
    double y = ldexp(r, e - bits);
    if (fabs(y) >= ldexp(1.0, emax + 1)) return copysign(INFINITY, x);
    return y;
}

double or_round(double x, int fmt)
{
    switch (fmt) {
    case 1: return round_sig(x, 8, 0, -126, 127);
    case 2: return round_sig(x, 11, 0, -14, 15);
    case 3: return round_sig(x, 11, 1, -126, 127);
    case 4: return round_sig(x, 24, 0, -126, 127);
    case 5: return trunc_sig(x, 11);
    default: return x;
    }
}

void or_round_array(double* x, int64_t n, int fmt)
{
    for (int64_t i = 0; i < n; ++i) x[i] = or_round(x[i], fmt);
}

/* ------------------------------------------------------------- naive GEMM */
/* P:581 Eq. (1): C = A x B, A M x K, B K x N, C M x N, all row-major. */
void or_gemm_f64(int64_t M, int64_t N, int64_t K,
                 const double* A, const double* B, double* C)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < M; ++i) {
        double* c = C + i * N;
        for (int64_t j = 0; j < N; ++j) c[j] = 0.0;
        for (int64_t p = 0; p < K; ++p) {
            double a = A[i * K + p];
            const double* b = B + p * N;
            for (int64_t j = 0; j < N; ++j) c[j] += a * b[j];
        }
    }
}

void or_gemm_i64(int64_t M, int64_t N, int64_t K,
                 const int64_t* A, const int64_t* B, int64_t* C)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < M; ++i) {
        int64_t* c = C + i * N;
        for (int64_t j = 0; j < N; ++j) c[j] = 0;
        for (int64_t p = 0; p < K; ++p) {
            int64_t a = A[i * K + p];
            const int64_t* b = B + p * N;
            for (int64_t j = 0; j < N; ++j) c[j] += a * b[j];
        }
    }
}

/* Selected rows only (for sampled checks at full BASELINE sizes). */
void or_gemm_rows_f64(int64_t M, int64_t N, int64_t K,
                      const double* A, const double* B,
                      const int64_t* rows, int64_t nrows, double* Crows)
{
    (void)M;
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < nrows; ++t) {
        int64_t i = rows[t];
        double* c = Crows + t * N;
        for (int64_t j = 0; j < N; ++j) c[j] = 0.0;
        for (int64_t p = 0; p < K; ++p) {
            double a = A[i * K + p];
            const double* b = B + p * N;
            for (int64_t j = 0; j < N; ++j) c[j] += a * b[j];
        }
    }
}

/* ------------------------------------------------------------ Brent check */
/* Returns the number of failing tuples; the first one goes to first[0..5] as
 * (i, l, l2, j, i2, j2) with first[6] = observed sum, first[7] = expected.
 * U is R x m x k, V is R x k x n, W is R x m x n (row-major, int8). */
int64_t or_brent(int m, int k, int n, int R,
                 const int8_t* U, const int8_t* V, const int8_t* W,
                 int64_t* first, int64_t* checked)
{
    int64_t fails = 0, cnt = 0;
    for (int i = 0; i < m; ++i)
    for (int l = 0; l < k; ++l)
    for (int l2 = 0; l2 < k; ++l2)
    for (int j = 0; j < n; ++j)
    for (int i2 = 0; i2 < m; ++i2)
    for (int j2 = 0; j2 < n; ++j2) {
        int64_t s = 0;
        for (int r = 0; r < R; ++r)
            s += (int64_t)U[(r * m + i) * k + l] *
                 (int64_t)V[(r * k + l2) * n + j] *
                 (int64_t)W[(r * m + i2) * n + j2];
        /* A_{i,l} B_{l2,j} must land in C_{i2,j2} exactly when
         * l == l2, i == i2, j == j2 (block matrix product, Eq. 2). */
        int64_t expect = (i == i2 && l == l2 && j == j2) ? 1 : 0;
        ++cnt;
        if (s != expect) {
            if (fails == 0 && first) {
                first[0] = i; first[1] = l; first[2] = l2; first[3] = j;
                first[4] = i2; first[5] = j2; first[6] = s; first[7] = expect;
            }
            ++fails;
        }
    }
    if (checked) *checked = cnt;
    return fails;
}

/* ---------------------------------------------------- Algorithm 1 (fp64) */
/* Counters: [0] combineA adds, [1] combineB adds, [2] GEMM mults,
 * [3] GEMM adds, [4] combineH adds, [5] A elements loaded, [6] B elements
 * loaded, [7] H elements loaded, [8] H elements stored. */
typedef struct {
    int fmt_in;   /* rounding of At, Bt (MMA input type) */
    int fmt_h;    /* rounding of H before Combine H ("downcast H") */
    int fmt_out;  /* rounding of C */
} or_round_cfg;

static inline double blk_get_f64(const double* X, int64_t rows, int64_t cols,
                                 int64_t r, int64_t c)
{
    return (r < rows && c < cols) ? X[r * cols + c] : 0.0;   /* zero padding */
}

/* Computes C (M x N) from A (M x K), B (K x N) through the scheme with block
 * extents Mb >= ceil(M/m), Kb >= ceil(K/k), Nb >= ceil(N/n).  If At/Bt/H are
 * non-NULL they receive the materialised intermediates (R x Mb x Kb,
 * R x Kb x Nb, R x Mb x Nb).  Returns 0, or -1 on bad extents / OOM. */
int or_lcma_f64(int64_t M, int64_t N, int64_t K,
                int m, int k, int n, int R,
                const int8_t* U, const int8_t* V, const int8_t* W,
                int64_t Mb, int64_t Kb, int64_t Nb,
                const double* A, const double* B, double* C,
                double* At_out, double* Bt_out, double* H_out,
                int fmt_in, int fmt_h, int fmt_out, int64_t* counters)
{
    if (Mb * m < M || Kb * k < K || Nb * n < N) return -1;
    int64_t cnt[9] = {0};
    double* At = At_out ? At_out : (double*)malloc(sizeof(double) * R * Mb * Kb);
    double* Bt = Bt_out ? Bt_out : (double*)malloc(sizeof(double) * R * Kb * Nb);
    double* H  = H_out  ? H_out  : (double*)malloc(sizeof(double) * R * Mb * Nb);
    double* Cb = (double*)malloc(sizeof(double) * m * n * Mb * Nb);
    if (!At || !Bt || !H || !Cb) return -1;

    /* Stage 1: Combine A, Eq. (3): At_r = sum_{i,l} U[r,i,l] A_{i,l}; only
     * nonzero coefficients are loaded (Alg. 1 lines 2-5). */
    for (int r = 0; r < R; ++r) {
        double* a = At + (int64_t)r * Mb * Kb;
        for (int64_t t = 0; t < Mb * Kb; ++t) a[t] = 0.0;
        int first = 1;
        for (int i = 0; i < m; ++i)
        for (int l = 0; l < k; ++l) {
            int u = U[(r * m + i) * k + l];
            if (!u) continue;
            for (int64_t x = 0; x < Mb; ++x)
            for (int64_t y = 0; y < Kb; ++y)
                a[x * Kb + y] += u * blk_get_f64(A, M, K, i * Mb + x, l * Kb + y);
            cnt[5] += Mb * Kb;
            if (!first) cnt[0] += Mb * Kb;
            first = 0;
        }
        if (fmt_in) or_round_array(a, Mb * Kb, fmt_in);
    }
    /* Stage 2: Combine B, Eq. (4). */
    for (int r = 0; r < R; ++r) {
        double* b = Bt + (int64_t)r * Kb * Nb;
        for (int64_t t = 0; t < Kb * Nb; ++t) b[t] = 0.0;
        int first = 1;
        for (int l = 0; l < k; ++l)
        for (int j = 0; j < n; ++j) {
            int v = V[(r * k + l) * n + j];
            if (!v) continue;
            for (int64_t y = 0; y < Kb; ++y)
            for (int64_t z = 0; z < Nb; ++z)
                b[y * Nb + z] += v * blk_get_f64(B, K, N, l * Kb + y, j * Nb + z);
            cnt[6] += Kb * Nb;
            if (!first) cnt[1] += Kb * Nb;
            first = 0;
        }
        if (fmt_in) or_round_array(b, Kb * Nb, fmt_in);
    }
    /* Stage 3: H_r = At_r x Bt_r, Eq. (5). */
    for (int r = 0; r < R; ++r) {
        or_gemm_f64(Mb, Nb, Kb, At + (int64_t)r * Mb * Kb,
                    Bt + (int64_t)r * Kb * Nb, H + (int64_t)r * Mb * Nb);
        cnt[2] += Mb * Nb * Kb;
        cnt[3] += Mb * Nb * (Kb - 1);
        cnt[8] += Mb * Nb;
        if (fmt_h) or_round_array(H + (int64_t)r * Mb * Nb, Mb * Nb, fmt_h);
    }
    /* Stage 4: Combine H, Eq. (6): C_{i,j} = sum_r W[r,i,j] H_r (Alg. 1
     * lines 15-19: for each C block load only H_r with W != 0). */
    for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) {
        double* c = Cb + (int64_t)(i * n + j) * Mb * Nb;
        for (int64_t t = 0; t < Mb * Nb; ++t) c[t] = 0.0;
        int first = 1;
        for (int r = 0; r < R; ++r) {
            int w = W[(r * m + i) * n + j];
            if (!w) continue;
            const double* h = H + (int64_t)r * Mb * Nb;
            for (int64_t t = 0; t < Mb * Nb; ++t) c[t] += w * h[t];
            cnt[7] += Mb * Nb;
            if (!first) cnt[4] += Mb * Nb;
            first = 0;
        }
    }
    /* Crop the padded block result to M x N. */
    for (int64_t row = 0; row < M; ++row)
    for (int64_t col = 0; col < N; ++col) {
        int64_t i = row / Mb, x = row % Mb, j = col / Nb, z = col % Nb;
        double v = Cb[((int64_t)(i * n + j) * Mb + x) * Nb + z];
        C[row * N + col] = fmt_out ? or_round(v, fmt_out) : v;
    }
    if (counters) memcpy(counters, cnt, sizeof(cnt));
    if (!At_out) free(At);
    if (!Bt_out) free(Bt);
    if (!H_out) free(H);
    free(Cb);
    return 0;
}

/* --------------------------------------------------- Algorithm 1 (int64) */
static inline int64_t blk_get_i64(const int64_t* X, int64_t rows, int64_t cols,
                                  int64_t r, int64_t c)
{
    return (r < rows && c < cols) ? X[r * cols + c] : 0;
}

int or_lcma_i64(int64_t M, int64_t N, int64_t K,
                int m, int k, int n, int R,
                const int8_t* U, const int8_t* V, const int8_t* W,
                int64_t Mb, int64_t Kb, int64_t Nb,
                const int64_t* A, const int64_t* B, int64_t* C,
                int64_t* At_out, int64_t* Bt_out, int64_t* H_out)
{
    if (Mb * m < M || Kb * k < K || Nb * n < N) return -1;
    int64_t* At = At_out ? At_out : (int64_t*)malloc(sizeof(int64_t) * R * Mb * Kb);
    int64_t* Bt = Bt_out ? Bt_out : (int64_t*)malloc(sizeof(int64_t) * R * Kb * Nb);
    int64_t* H  = H_out  ? H_out  : (int64_t*)malloc(sizeof(int64_t) * R * Mb * Nb);
    if (!At || !Bt || !H) return -1;
    for (int r = 0; r < R; ++r) {                       /* Eq. (3) */
        int64_t* a = At + (int64_t)r * Mb * Kb;
        for (int64_t x = 0; x < Mb; ++x)
        for (int64_t y = 0; y < Kb; ++y) {
            int64_t s = 0;
            for (int i = 0; i < m; ++i)
            for (int l = 0; l < k; ++l) {
                int u = U[(r * m + i) * k + l];
                if (u) s += u * blk_get_i64(A, M, K, i * Mb + x, l * Kb + y);
            }
            a[x * Kb + y] = s;
        }
    }
    for (int r = 0; r < R; ++r) {                       /* Eq. (4) */
        int64_t* b = Bt + (int64_t)r * Kb * Nb;
        for (int64_t y = 0; y < Kb; ++y)
        for (int64_t z = 0; z < Nb; ++z) {
            int64_t s = 0;
            for (int l = 0; l < k; ++l)
            for (int j = 0; j < n; ++j) {
                int v = V[(r * k + l) * n + j];
                if (v) s += v * blk_get_i64(B, K, N, l * Kb + y, j * Nb + z);
            }
            b[y * Nb + z] = s;
        }
    }
    for (int r = 0; r < R; ++r)                         /* Eq. (5) */
        or_gemm_i64(Mb, Nb, Kb, At + (int64_t)r * Mb * Kb,
                    Bt + (int64_t)r * Kb * Nb, H + (int64_t)r * Mb * Nb);
    for (int64_t row = 0; row < M; ++row)               /* Eq. (6) + crop */
    for (int64_t col = 0; col < N; ++col) {
        int64_t i = row / Mb, x = row % Mb, j = col / Nb, z = col % Nb;
        int64_t s = 0;
        for (int r = 0; r < R; ++r) {
            int w = W[(r * m + i) * n + j];
            if (w) s += w * H[((int64_t)r * Mb + x) * Nb + z];
        }
        C[row * N + col] = s;
    }
    if (!At_out) free(At);
    if (!Bt_out) free(Bt);
    if (!H_out) free(H);
    return 0;
}
