// combine.cuh -- group-parallel combine kernels (Algorithm 2 stages 1-2,
// P:300-320, and the group Combine H of the unfused path, P:95-100 reordered
// per P:355-358).  Each thread owns one relative coordinate (x, y) of the
// block grid, loads the m*k (k*n) source elements A_{i,l}[x,y] exactly once
// and emits every At_r[x,y] of the group: reads of the source = 1x, writes =
// R x (Table "cost_model" memory column MK(1 + R/mk)).  HBM-bound.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <stdint.h>

namespace lcma {

constexpr int kCombMaxR = 128;
constexpr int kCombMaxPQ = 32;

enum ElemType : int { ELEM_BF16 = 0, ELEM_FP16 = 1, ELEM_FP32 = 2 };

struct CombineParams {
    const void* src;          // rows x cols row-major
    void* dst;                // [R][E0][E1] row-major
    long long rows, cols;     // true source extents (zero padding beyond)
    long long E0, E1;         // block extents (multiples of 8 along E1)
    int P, Q;                 // source block grid
    int R;
    int elem;                 // ElemType
    int round_tf32;           // fp32 outputs rounded RN-away to tf32
    int8_t coef[kCombMaxR * kCombMaxPQ];   // coef[r][p*Q + q]
    uint8_t skip[kCombMaxR];  // 1: output r not written (a single +1 source block the GEMM reads in place)
};

template <int VEC>
__device__ __forceinline__ void load_vec(const CombineParams& p, long long r, long long c, float* v) {
    if (r >= p.rows || c >= p.cols) {
#pragma unroll
        for (int e = 0; e < VEC; ++e) v[e] = 0.f;
        return;
    }
    const long long off = r * p.cols + c;
    if (p.elem == ELEM_FP32) {
        const float4* s = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.src) + off);
#pragma unroll
        for (int e = 0; e < VEC; e += 4) {
            float4 t = __ldcs(s + e / 4);
            v[e] = t.x; v[e + 1] = t.y; v[e + 2] = t.z; v[e + 3] = t.w;
        }
    } else {
        const uint16_t* s = reinterpret_cast<const uint16_t*>(p.src) + off;
        uint32_t w[VEC / 2];
        if (VEC == 8) {
            uint4 t = __ldcs(reinterpret_cast<const uint4*>(s));
            w[0] = t.x; w[1] = t.y; w[2] = t.z; w[3] = t.w;
        } else {
            uint2 t = __ldcs(reinterpret_cast<const uint2*>(s));
            w[0] = t.x; w[1] = t.y;
        }
#pragma unroll
        for (int h = 0; h < VEC / 2; ++h) {
            if (p.elem == ELEM_BF16) {
                __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&w[h]);
                float2 f = __bfloat1622float2(b);
                v[2 * h] = f.x; v[2 * h + 1] = f.y;
            } else {
                __half2 b = *reinterpret_cast<__half2*>(&w[h]);
                float2 f = __half22float2(b);
                v[2 * h] = f.x; v[2 * h + 1] = f.y;
            }
        }
    }
}

__device__ __forceinline__ float round_tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

template <int VEC>
__device__ __forceinline__ void store_vec(const CombineParams& p, long long off, const float* v) {
    if (p.elem == ELEM_FP32) {
        float4* d = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.dst) + off);
#pragma unroll
        for (int e = 0; e < VEC; e += 4) {
            float a = v[e], b = v[e + 1], c = v[e + 2], dd = v[e + 3];
            if (p.round_tf32) {
                a = round_tf32_rna(a); b = round_tf32_rna(b);
                c = round_tf32_rna(c); dd = round_tf32_rna(dd);
            }
            __stcs(d + e / 4, make_float4(a, b, c, dd));
        }
    } else {
        uint32_t w[VEC / 2];
#pragma unroll
        for (int h = 0; h < VEC / 2; ++h) {
            if (p.elem == ELEM_BF16) {
                __nv_bfloat162 b = __floats2bfloat162_rn(v[2 * h], v[2 * h + 1]);
                w[h] = *reinterpret_cast<uint32_t*>(&b);
            } else {
                __half2 b = __floats2half2_rn(v[2 * h], v[2 * h + 1]);
                w[h] = *reinterpret_cast<uint32_t*>(&b);
            }
        }
        uint16_t* d = reinterpret_cast<uint16_t*>(p.dst) + off;
        if (VEC == 8)
            __stcs(reinterpret_cast<uint4*>(d), make_uint4(w[0], w[1], w[2], w[3]));
        else
            __stcs(reinterpret_cast<uint2*>(d), make_uint2(w[0], w[1]));
    }
}

// 16-bit Group Combine with more bytes in flight: sources stay packed (8
// elements per 16-byte register quad), every thread owns U vector positions
// and issues all U*PQ streaming loads before any arithmetic; outputs are
// written with streaming (evict-first) stores.  Same arithmetic as below:
// fp32 signed sum in coefficient order, one RN rounding.
template <int PQ, int U>
__device__ __forceinline__ void combine16_body(const CombineParams& p, int bid, int nblk) {
    const long long nvec = p.E0 * (p.E1 / 8);
    const long long per_r = p.E0 * p.E1;
    const long long stride = (long long)nblk * blockDim.x * U;
    const bool bf16 = p.elem == ELEM_BF16;
    for (long long v0 = (bid * (long long)blockDim.x + threadIdx.x) * U; v0 < nvec; v0 += stride) {
        uint4 src[U][PQ];
        long long e0s[U], e1s[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long vi = v0 + u;
            const long long e0 = vi / (p.E1 / 8);
            const long long e1 = (vi - e0 * (p.E1 / 8)) * 8;
            e0s[u] = e0;
            e1s[u] = e1;
#pragma unroll
            for (int pq = 0; pq < PQ; ++pq) {
                const int pi = pq / p.Q, qi = pq - (pq / p.Q) * p.Q;
                const long long r = pi * p.E0 + e0, c = qi * p.E1 + e1;
                if (vi < nvec && r < p.rows && c < p.cols)
                    src[u][pq] = __ldcs(reinterpret_cast<const uint4*>(
                        reinterpret_cast<const uint16_t*>(p.src) + r * p.cols + c));
                else
                    src[u][pq] = make_uint4(0, 0, 0, 0);
            }
        }
        for (int r = 0; r < p.R; ++r) {
            if (p.skip[r]) continue;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (v0 + u >= nvec) continue;
                float acc[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[e] = 0.f;
#pragma unroll
                for (int pq = 0; pq < PQ; ++pq) {
                    const int cf = p.coef[r * PQ + pq];
                    if (!cf) continue;
                    const uint32_t w[4] = {src[u][pq].x, src[u][pq].y, src[u][pq].z, src[u][pq].w};
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        float2 f;
                        if (bf16) f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[h]));
                        else f = __half22float2(*reinterpret_cast<const __half2*>(&w[h]));
                        if (cf > 0) { acc[2 * h] += f.x; acc[2 * h + 1] += f.y; }
                        else { acc[2 * h] -= f.x; acc[2 * h + 1] -= f.y; }
                    }
                }
                uint32_t o[4];
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    if (bf16) {
                        __nv_bfloat162 b = __floats2bfloat162_rn(acc[2 * h], acc[2 * h + 1]);
                        o[h] = *reinterpret_cast<uint32_t*>(&b);
                    } else {
                        __half2 b = __floats2half2_rn(acc[2 * h], acc[2 * h + 1]);
                        o[h] = *reinterpret_cast<uint32_t*>(&b);
                    }
                }
                __stcs(reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p.dst) + (long long)r * per_r +
                                                e0s[u] * p.E1 + e1s[u]),
                       make_uint4(o[0], o[1], o[2], o[3]));
            }
        }
    }
}

template <int PQ, int U>
__global__ void __launch_bounds__(256, 4) group_combine16_kernel(const __grid_constant__ CombineParams p) {
    combine16_body<PQ, U>(p, blockIdx.x, gridDim.x);
}

// Combine A and Combine B of one call in a single launch (blocks [0, nA)
// take A, the rest B): one kernel boundary and one tail instead of two.
template <int PQA, int PQB>
__global__ void __launch_bounds__(256, 4) group_combine16_dual_kernel(const __grid_constant__ CombineParams pa,
                                                                     const __grid_constant__ CombineParams pb,
                                                                     int nA) {
    if ((int)blockIdx.x < nA) combine16_body<PQA, 1>(pa, blockIdx.x, nA);
    else combine16_body<PQB, 1>(pb, blockIdx.x - nA, gridDim.x - nA);
}

// Group Combine (Alg. 2 lines 2-9 / 11-18): out_r[e0][e1] =
// sum_{p,q} coef[r][p][q] * src[p*E0 + e0][q*E1 + e1], fp32 sum, one rounding.
template <int VEC, int PQ>
__global__ void __launch_bounds__(256) group_combine_kernel(const __grid_constant__ CombineParams p) {
    const long long nvec = p.E0 * (p.E1 / VEC);
    const long long per_r = p.E0 * p.E1;
    for (long long vi = blockIdx.x * (long long)blockDim.x + threadIdx.x; vi < nvec;
         vi += (long long)gridDim.x * blockDim.x) {
        const long long e0 = vi / (p.E1 / VEC);
        const long long e1 = (vi - e0 * (p.E1 / VEC)) * VEC;
        float src[PQ][VEC];
#pragma unroll
        for (int pq = 0; pq < PQ; ++pq) {
            const int pi = pq / p.Q, qi = pq - (pq / p.Q) * p.Q;
            load_vec<VEC>(p, pi * p.E0 + e0, qi * p.E1 + e1, src[pq]);
        }
        for (int r = 0; r < p.R; ++r) {
            if (p.skip[r]) continue;
            float acc[VEC];
#pragma unroll
            for (int e = 0; e < VEC; ++e) acc[e] = 0.f;
#pragma unroll
            for (int pq = 0; pq < PQ; ++pq) {
                const int c = p.coef[r * PQ + pq];
                if (c == 1) {
#pragma unroll
                    for (int e = 0; e < VEC; ++e) acc[e] += src[pq][e];
                } else if (c == -1) {
#pragma unroll
                    for (int e = 0; e < VEC; ++e) acc[e] -= src[pq][e];
                }
            }
            store_vec<VEC>(p, (long long)r * per_r + e0 * p.E1 + e1, acc);
        }
    }
}

// FP8 Group Combine with the quantization fused in (DESIGN.md
// reading 23): out_r = sum_{p,q} coef[r][p][q] * src blocks (bf16 sources,
// fp32 signed sum in coefficient order as above), then every 1 x 128 block
// of an output row is scaled by 2^-e, e the smallest integer with amax <= 448 *
// 2^e (UE8M0, clamped to [-127, 127]; 0 for an all-zero block), and stored as
// E4M3 (RN-even, satfinite).  The scale bytes go to the tcgen05 block-scale
// layout: per (r, 128-row block, 128-column block) a 512-byte chunk, byte
// (row % 32) * 16 + (row % 128 / 32) * 4 + j = e + 127 for the four 32-column
// scale slots j of the MMA (equal: one scale per 1 x 128 block).
// 16 consecutive threads own one 128-column block of a row (8 columns each):
// the amax is a 16-lane shuffle reduction.
struct CombineQ8Params {
    const uint16_t* src;      // bf16, rows x cols row-major
    uint8_t* dst;             // E4M3 [R][E0][E1]
    uint32_t* sf;             // scale chunks [R][E0/128][E1/128][128] words
    long long rows, cols;     // true source extents (zero padding beyond)
    long long E0, E1;         // block extents: E0 % 128 == 0, E1 % 128 == 0
    int P, Q, R;
    int8_t coef[kCombMaxR * kCombMaxPQ];   // coef[r][p*Q + q]
};

// smallest e with amax <= 448 * 2^e (amax >= 0, exact fp32)
__device__ __forceinline__ int ue8m0_exponent(float amax) {
    const uint32_t b = __float_as_uint(amax);
    const int ef = (int)(b >> 23) & 0xFF;
    if (b == 0u) return 0;
    if (ef == 0) return -127;                           // subnormal amax: below 448 * 2^-127
    int e = (ef - 127) - 8 + ((b & 0x7FFFFFu) > 0x600000u ? 1 : 0);   // 448 = 1.75 * 2^8
    return e < -127 ? -127 : (e > 127 ? 127 : e);
}

template <int PQ, int U>
__global__ void __launch_bounds__(256) group_combine_q8_kernel(const __grid_constant__ CombineQ8Params p) {
    const long long nvec = p.E0 * (p.E1 / 8);
    const long long per_r = p.E0 * p.E1;
    const long long nkb = p.E1 / 128;
    const int lane = threadIdx.x & 31;
    // U vectors per thread, each from its own 256-vector chunk (16 consecutive
    // lanes stay inside one 1 x 128 block): all U * PQ loads are issued before
    // any arithmetic (memory-level parallelism)
    uint4 srcs[U][PQ];
    long long e0s[U], e1s[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const long long vi = ((long long)blockIdx.x * U + u) * blockDim.x + threadIdx.x;
        const long long e0 = vi / (p.E1 / 8);
        const long long e1 = (vi - e0 * (p.E1 / 8)) * 8;
        e0s[u] = e0;
        e1s[u] = e1;
#pragma unroll
        for (int pq = 0; pq < PQ; ++pq) {
            const int pi = pq / p.Q, qi = pq - (pq / p.Q) * p.Q;
            const long long r = pi * p.E0 + e0, c = qi * p.E1 + e1;
            srcs[u][pq] = (vi < nvec && pq < p.P * p.Q && r < p.rows && c < p.cols)
                              ? __ldcs(reinterpret_cast<const uint4*>(p.src + r * p.cols + c))
                              : make_uint4(0, 0, 0, 0);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const long long vi = ((long long)blockIdx.x * U + u) * blockDim.x + threadIdx.x;
        if (vi >= nvec) break;                 // whole 256-vector chunks: uniform per warp
        const long long e0 = e0s[u], e1 = e1s[u];
        const uint4* src = srcs[u];
        for (int r = 0; r < p.R; ++r) {
            float acc[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[e] = 0.f;
#pragma unroll
            for (int pq = 0; pq < PQ; ++pq) {
                const int cf = p.coef[r * PQ + pq];
                if (!cf) continue;
                const uint32_t w[4] = {src[pq].x, src[pq].y, src[pq].z, src[pq].w};
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[h]));
                    if (cf > 0) { acc[2 * h] += f.x; acc[2 * h + 1] += f.y; }
                    else { acc[2 * h] -= f.x; acc[2 * h + 1] -= f.y; }
                }
            }
            float amax = 0.f;
#pragma unroll
            for (int e = 0; e < 8; ++e) amax = fmaxf(amax, fabsf(acc[e]));
#pragma unroll
            for (int o = 8; o >= 1; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
            const int ex = ue8m0_exponent(amax);
            // 2^-e exactly (e <= 126 keeps it a normal fp32; e = 127 needs amax > 2^135)
            const float inv = __uint_as_float((uint32_t)(127 - (ex > 126 ? 126 : ex)) << 23);
            uint32_t q[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const __nv_fp8x2_storage_t lo = __nv_cvt_float2_to_fp8x2(
                    make_float2(acc[4 * h] * inv, acc[4 * h + 1] * inv), __NV_SATFINITE, __NV_E4M3);
                const __nv_fp8x2_storage_t hi = __nv_cvt_float2_to_fp8x2(
                    make_float2(acc[4 * h + 2] * inv, acc[4 * h + 3] * inv), __NV_SATFINITE, __NV_E4M3);
                q[h] = (uint32_t)lo | ((uint32_t)hi << 16);
            }
            __stcs(reinterpret_cast<uint2*>(p.dst + (long long)r * per_r + e0 * p.E1 + e1), make_uint2(q[0], q[1]));
            if ((lane & 15) == 0) {
                const uint32_t byte = (uint32_t)(ex + 127);
                const long long chunk = ((long long)r * (p.E0 / 128) + e0 / 128) * nkb + e1 / 128;
                const int rw = (int)(e0 & 127);
                p.sf[chunk * 128 + (rw & 31) * 4 + (rw >> 5)] = byte * 0x01010101u;
            }
        }
    }
}

// Group Combine H for the unfused path: each thread owns H_r[x][z..z+3] for
// all r (read once) and produces C_ij[x][z..z+3] for all (i,j).
struct CombineHParams {
    const float* H;           // [R][Mb][Nb]
    void* C;                  // M x N, ldc
    long long M, N, Mb, Nb, ldc;
    int m, n, R;
    int out_type;             // 0 bf16, 1 fp16, 2 fp32
    int8_t Wc[kCombMaxR * kCombMaxPQ];   // W[r][i*n + j]
};

template <int MN>
__global__ void __launch_bounds__(256) group_combine_h_kernel(const __grid_constant__ CombineHParams p) {
    const long long nvec = p.Mb * (p.Nb / 4);
    for (long long vi = blockIdx.x * (long long)blockDim.x + threadIdx.x; vi < nvec;
         vi += (long long)gridDim.x * blockDim.x) {
        const long long x = vi / (p.Nb / 4);
        const long long z = (vi - x * (p.Nb / 4)) * 4;
        float acc[MN][4];
#pragma unroll
        for (int ij = 0; ij < MN; ++ij)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[ij][e] = 0.f;
        for (int r = 0; r < p.R; ++r) {
            const float4 h = __ldg(reinterpret_cast<const float4*>(p.H + ((long long)r * p.Mb + x) * p.Nb + z));
#pragma unroll
            for (int ij = 0; ij < MN; ++ij) {
                const int w = p.Wc[r * MN + ij];
                if (w) {
                    const float s = (float)w;
                    acc[ij][0] += s * h.x; acc[ij][1] += s * h.y;
                    acc[ij][2] += s * h.z; acc[ij][3] += s * h.w;
                }
            }
        }
#pragma unroll
        for (int ij = 0; ij < MN; ++ij) {
            const int i = ij / p.n, j = ij % p.n;
            const long long row = i * p.Mb + x, col = j * p.Nb + z;
            if (row >= p.M || col >= p.N) continue;
            if (p.out_type == 2) {
                *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.C) + row * p.ldc + col) =
                    make_float4(acc[ij][0], acc[ij][1], acc[ij][2], acc[ij][3]);
            } else {
                uint32_t w2[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (p.out_type == 0) {
                        __nv_bfloat162 b = __floats2bfloat162_rn(acc[ij][2 * h], acc[ij][2 * h + 1]);
                        w2[h] = *reinterpret_cast<uint32_t*>(&b);
                    } else {
                        __half2 b = __floats2half2_rn(acc[ij][2 * h], acc[ij][2 * h + 1]);
                        w2[h] = *reinterpret_cast<uint32_t*>(&b);
                    }
                }
                *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(p.C) + row * p.ldc + col) =
                    make_uint2(w2[0], w2[1]);
            }
        }
    }
}

// True-fp32 batched SIMT GEMM (dtype LCMA_FP32): H_r = At_r * Bt_r with
// At_r = A + r*sAr (rows x K, lda), Bt_r = B + r*sBr; B is K x N (ldb) or,
// with b_kmajor, N x K.  128 x 128 output tile per 256-thread block, 8 x 8
// per thread, BK = 8 staged through shared memory.
struct SimtParams {
    const float* A; const float* B; float* H;
    long long Mr, Nr, Kr;         // per-product extents
    long long lda, ldb, ldh;
    long long sAr, sBr, sHr;      // per-r strides (elements)
    int b_kmajor;
};

__global__ void __launch_bounds__(256) simt_sgemm_batched_kernel(const __grid_constant__ SimtParams p) {
    __shared__ float sA[8][128 + 4];
    __shared__ float sB[8][128 + 4];
    const int r = blockIdx.z;
    const long long m0 = (long long)blockIdx.y * 128, n0 = (long long)blockIdx.x * 128;
    const float* A = p.A + r * p.sAr;
    const float* B = p.B + r * p.sBr;
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    for (long long k0 = 0; k0 < p.Kr; k0 += 8) {
        for (int t = threadIdx.x; t < 8 * 128; t += 256) {
            const int kk = t % 8, mm = t / 8;
            const long long gm = m0 + mm, gk = k0 + kk;
            sA[kk][mm] = (gm < p.Mr && gk < p.Kr) ? A[gm * p.lda + gk] : 0.f;
            const int nn = p.b_kmajor ? t / 8 : t % 128;
            const int kb = p.b_kmajor ? t % 8 : t / 128;
            const long long gn = n0 + nn, gk2 = k0 + kb;
            float bv = 0.f;
            if (gn < p.Nr && gk2 < p.Kr) bv = p.b_kmajor ? B[gn * p.ldb + gk2] : B[gk2 * p.ldb + gn];
            sB[kb][nn] = bv;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            float a[8], b[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = sA[kk][ty * 8 + i];
#pragma unroll
            for (int j = 0; j < 8; ++j) b[j] = sB[kk][tx * 8 + j];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
    float* Hr = p.H + r * p.sHr;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const long long gm = m0 + ty * 8 + i;
        if (gm >= p.Mr) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const long long gn = n0 + tx * 8 + j;
            if (gn < p.Nr) Hr[gm * p.ldh + gn] = acc[i][j];
        }
    }
}

}  // namespace lcma
