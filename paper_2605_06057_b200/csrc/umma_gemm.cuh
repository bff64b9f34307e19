// umma_gemm.cuh -- persistent, warp-specialised tcgen05 GEMM for sm_100a that
// runs the GEMM stage of the LCMA workflow (Eq. 5) and, in the
// fused mode, Combine H (Eq. 6) as its epilogue (Algorithm 2,
// stage 3/4).  The classical GEMM ("standard GEMM") is
// the same kernel with the trivial scheme <1,1,1;1>.
//
// Roles (one CTA per SM, 384 threads):
//   warp 0      TMA producer: At_r[x, y] and Bt_r[y, z] tiles -> smem ring
//   warp 1      MMA issuer: one thread issues tcgen05.mma into TMEM
//   warp 2      TMEM allocator (512 columns = 2 fp32 accumulators of 256)
//   warps 4-11  epilogue: TMEM -> registers -> (Combine H) -> global
//
// Work decomposition (Group-Parallel Optimization): a *group* is
// the set {H_r[x,z]}_{r=1..R} of one output tile position (x,z); the CTA that
// owns a group accumulates every C_{ij}[x,z] with W[r,i,j] != 0 on chip/L2 and
// writes C once.  Scheduling: lockstep rounds of whole groups
// (all CTAs on the same r at the same time: cache-aware), then the tail of
// G mod W groups split at tile granularity over all CTAs (split-group); the
// segment holding r = 0 owns the group and merges the other segments'
// partials in a fixed order (deterministic, no atomics).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "ptx.cuh"

namespace lcma {

constexpr int kBM = 128;          // UMMA M (cta_group::1)
constexpr int kBN = 256;          // UMMA N = accumulator columns
constexpr int kStages = 4;        // smem ring depth
constexpr int kThreads = 384;     // 12 warps
constexpr int kEpiWarp0 = 4;      // first epilogue warp
constexpr int kEpiWarps = 8;
constexpr int kMaxR = 128;
constexpr int kMaxMN = 32;
constexpr int kTileBytesA = kBM * 128;    // 128 rows x 128 bytes
constexpr int kTileBytesB = kBN * 128;    // 256 rows(K-major) or 4x(BK x 128B)
constexpr int kStageBytes = kTileBytesA + kTileBytesB;
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;

enum EpiMode : int { EPI_FUSED = 0, EPI_STORE_H = 1 };
enum OutType : int { OUT_BF16 = 0, OUT_FP16 = 1, OUT_FP32 = 2 };
enum UnitRole : int { ROLE_WHOLE = 0, ROLE_OWNER = 1, ROLE_CONTRIB = 2 };

struct GemmParams {
    // problem / blocking
    int nX, nZ;            // tiles per block along M, N: Mb/kBM, Nb/kBN
    int G;                 // groups = nX * nZ
    int R;                 // products per group
    int nK;                // k-blocks per product: Kb / BK
    int BK;                // elements per 128-byte row
    int a_rows_per_r;      // row offset of At_r in the A tensor map (Mb), 0 for R == 1
    int b_rows_per_r;      // row offset of Bt_r in the B map (Nb if K-major else Kb)
    int b_mn_major;        // B operand MN-major (B stored K x N)
    int tf32;              // kind::tf32 (else kind::f16)
    uint32_t idesc;        // instruction descriptor
    // schedule
    int W;                 // CTAs
    int q;                 // lockstep rounds of whole groups
    int tail_c;            // tile capacity per CTA in the split tail
    int swz;               // raster band height (tiles) for group -> (x, z)
    // epilogue
    int epi_mode;
    int out_type;
    int m, n;              // scheme grid (C blocks)
    long long M, N;        // true C extents (crop)
    long long Mb, Nb;      // block extents: C_ij origin = (i*Mb, j*Nb)
    long long ldc;
    void* C;
    float* P;              // partial tiles: [2W][m*n][kBN/4][kBM][4] fp32
    int* flags;            // [W] split-segment ready flags
    float* H;              // EPI_STORE_H: H [R][Mb][Nb] fp32
    int8_t Wc[kMaxR * kMaxMN];   // W[r][i*n + j]
};

// ------------------------------------------------------------ scheduling
struct Unit {
    int g, r0, r1, role;
};

// Enumerates the units of CTA `w` in processing order.  Every role of the
// CTA (producer, MMA, epilogue) walks the same sequence.
struct UnitIter {
    const GemmParams& p;
    int w;
    int idx;           // lockstep round index, then tail
    long long t, t_end;  // tail tile cursor
    __device__ UnitIter(const GemmParams& p_, int w_) : p(p_), w(w_), idx(0) {
        long long Tt = (long long)(p.G - p.q * p.W) * p.R;
        t = (long long)w * p.tail_c;
        t_end = t + p.tail_c;
        if (t_end > Tt) t_end = Tt;
        if (t > Tt) t = Tt;
    }
    __device__ bool next(Unit& u) {
        if (idx < p.q) {
            u.g = idx * p.W + w;
            u.r0 = 0;
            u.r1 = p.R;
            u.role = ROLE_WHOLE;
            ++idx;
            return true;
        }
        if (t >= t_end) return false;
        long long gl = t / p.R;                // tail-local group
        int r0 = (int)(t - gl * p.R);
        long long stop = (gl + 1) * p.R;
        if (stop > t_end) stop = t_end;
        int r1 = (int)(stop - gl * p.R);
        u.g = p.q * p.W + (int)gl;
        u.r0 = r0;
        u.r1 = r1;
        u.role = (r0 == 0 && r1 == p.R) ? ROLE_WHOLE : (r0 == 0 ? ROLE_OWNER : ROLE_CONTRIB);
        t = stop;
        return true;
    }
};

// Group index -> tile coordinates: bands of `swz` tile-rows traversed
// column by column so that the W groups of a lockstep round cover a compact
// (x, z) region (operand reuse in L2).
__device__ __forceinline__ void group_xz(const GemmParams& p, int g, int& x, int& z) {
    int band_tiles = p.swz * p.nZ;
    int band = g / band_tiles;
    int within = g - band * band_tiles;
    int rows = p.nX - band * p.swz;
    if (rows > p.swz) rows = p.swz;
    x = band * p.swz + within % rows;
    z = within / rows;
}

// ------------------------------------------------------------ epilogue helpers
__device__ __forceinline__ float4 ld_cg_f4(const float* p) {
    return __ldcg(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ void st_cg_f4(float* p, float4 v) {
    __stcg(reinterpret_cast<float4*>(p), v);
}

// Store 32 consecutive fp32 values of one C row segment (cols c0..c0+31),
// cropping to N.  N is a multiple of 8 (TMA rule) so 8-element vectors are
// either fully inside or fully outside.
__device__ __forceinline__ void store_c_row(const GemmParams& p, long long row, long long c0,
                                            const float* v) {
    if (row >= p.M) return;
    if (p.out_type == OUT_FP32) {
        float* dst = reinterpret_cast<float*>(p.C) + row * p.ldc + c0;
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
            if (c0 + e < p.N)
                *reinterpret_cast<float4*>(dst + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
        }
    } else {
        uint16_t* dst = reinterpret_cast<uint16_t*>(p.C) + row * p.ldc + c0;
#pragma unroll
        for (int e = 0; e < 32; e += 8) {
            if (c0 + e < p.N) {
                uint32_t w4[4];
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    if (p.out_type == OUT_BF16) {
                        __nv_bfloat162 b = __floats2bfloat162_rn(v[e + 2 * h], v[e + 2 * h + 1]);
                        w4[h] = *reinterpret_cast<uint32_t*>(&b);
                    } else {
                        __half2 b = __floats2half2_rn(v[e + 2 * h], v[e + 2 * h + 1]);
                        w4[h] = *reinterpret_cast<uint32_t*>(&b);
                    }
                }
                *reinterpret_cast<uint4*>(dst + e) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
            }
        }
    }
}

// Partial tile layout: [kBN/4][kBM][4] floats, so that the 32 threads of a
// warp (32 consecutive rows) touch 512 contiguous bytes per float4 access.
__device__ __forceinline__ float* partial_tile(const GemmParams& p, int slot, int ij) {
    return p.P + ((size_t)slot * p.m * p.n + ij) * (size_t)(kBM * kBN);
}
__device__ __forceinline__ size_t partial_off(int row, int col4) {
    return ((size_t)col4 * kBM + row) * 4;
}

// ------------------------------------------------------------ the kernel
__global__ void __launch_bounds__(kThreads, 1)
    umma_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a,
                     const __grid_constant__ CUtensorMap tmap_b,
                     const __grid_constant__ GemmParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* empty_bar = full_bar + kStages;
    uint64_t* tfull_bar = empty_bar + kStages;   // [2]
    uint64_t* tempty_bar = tfull_bar + 2;        // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmap_a);
        ptx::tma_prefetch_desc(&tmap_b);
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&full_bar[s], 1);
            ptx::mbar_init(&empty_bar[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull_bar[a], 1);
            ptx::mbar_init(&tempty_bar[a], kEpiWarps);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 2) {
        ptx::tmem_alloc(tmem_slot, 512);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int w = blockIdx.x;

    if (warp == 0) {
        // ================================ TMA producer
        if (ptx::elect_one()) {
            const int b_bytes_chunk = p.BK * 128;   // MN-major chunk: BK rows x 128 B
            const int n_chunks = kBN / p.BK;       // MN-major: 128-byte column chunks
            int stage = 0;
            uint32_t phase = 0;
            UnitIter it(p, w);
            Unit u;
            while (it.next(u)) {
                int x, z;
                group_xz(p, u.g, x, z);
                for (int r = u.r0; r < u.r1; ++r) {
                    const int a_row = r * p.a_rows_per_r + x * kBM;
                    for (int kb = 0; kb < p.nK; ++kb) {
                        ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
                        uint8_t* sa = smem + stage * kStageBytes;
                        uint8_t* sb = sa + kTileBytesA;
                        ptx::mbar_arrive_expect_tx(&full_bar[stage], kStageBytes);
                        const int kcol = kb * p.BK;
                        ptx::tma_load_2d(sa, &tmap_a, &full_bar[stage], kcol, a_row);
                        if (!p.b_mn_major) {
                            ptx::tma_load_2d(sb, &tmap_b, &full_bar[stage], kcol,
                                             r * p.b_rows_per_r + z * kBN);
                        } else {
                            for (int c = 0; c < n_chunks; ++c)
                                ptx::tma_load_2d(sb + c * b_bytes_chunk, &tmap_b, &full_bar[stage],
                                                 z * kBN + c * p.BK,
                                                 r * p.b_rows_per_r + kcol);
                        }
                        if (++stage == kStages) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ================================ MMA issuer
        if (ptx::elect_one()) {
            const int k_steps = 4;                        // BK / UMMA_K (32 bytes per step)
            const uint32_t b_lbo = p.BK * 128;            // MN-major: chunk stride
            const uint32_t b_kstep = p.b_mn_major ? (uint32_t)(32 / (p.tf32 ? 4 : 2)) * 128u : 32u;
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            UnitIter it(p, w);
            Unit u;
            while (it.next(u)) {
                for (int r = u.r0; r < u.r1; ++r) {
                    ptx::mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
                    ptx::tc_fence_after();
                    const uint32_t d_tmem = tmem_base + acc * kBN;
                    for (int kb = 0; kb < p.nK; ++kb) {
                        ptx::mbar_wait(&full_bar[stage], phase);
                        ptx::tc_fence_after();
                        const uint32_t sa = ptx::smem_u32(smem + stage * kStageBytes);
                        const uint32_t sb = sa + kTileBytesA;
#pragma unroll
                        for (int ks = 0; ks < k_steps; ++ks) {
                            const uint64_t adesc = ptx::smem_desc_sw128(sa + ks * 32, 16, 1024);
                            const uint64_t bdesc =
                                p.b_mn_major ? ptx::smem_desc_sw128(sb + ks * b_kstep, b_lbo, 1024)
                                             : ptx::smem_desc_sw128(sb + ks * 32, 16, 1024);
                            const uint32_t accum = (kb | ks) ? 1u : 0u;
                            if (p.tf32)
                                ptx::mma_tf32_ss(d_tmem, adesc, bdesc, p.idesc, accum);
                            else
                                ptx::mma_f16_ss(d_tmem, adesc, bdesc, p.idesc, accum);
                        }
                        ptx::mma_commit(&empty_bar[stage]);       // smem slot free when MMAs done
                        if (++stage == kStages) { stage = 0; phase ^= 1; }
                    }
                    ptx::mma_commit(&tfull_bar[acc]);             // accumulator ready
                    if (++acc == 2) { acc = 0; acc_phase ^= 1; }
                }
            }
        }
    } else if (warp >= kEpiWarp0) {
        // ================================ epilogue
        const int ew = warp - kEpiWarp0;           // 0..7
        const int quarter = warp & 3;              // TMEM lane quarter
        const int half = ew >> 2;                  // column half
        const int row = quarter * 32 + lane;       // tile row owned by this thread
        const int mn = p.m * p.n;
        int acc = 0;
        uint32_t acc_phase = 0;
        UnitIter it(p, w);
        Unit u;
        while (it.next(u)) {
            int x, z;
            group_xz(p, u.g, x, z);
            // first / last contributing r of each C_ij inside this unit
            int first_r[kMaxMN], last_r[kMaxMN];
            for (int ij = 0; ij < mn; ++ij) {
                first_r[ij] = -1;
                last_r[ij] = -1;
                for (int r = u.r0; r < u.r1; ++r)
                    if (p.Wc[r * mn + ij]) {
                        if (first_r[ij] < 0) first_r[ij] = r;
                        last_r[ij] = r;
                    }
            }
            const int slot = (u.role == ROLE_CONTRIB) ? p.W + w : w;
            for (int r = u.r0; r < u.r1; ++r) {
                ptx::mbar_wait(&tfull_bar[acc], acc_phase);
                ptx::tc_fence_after();
                const uint32_t t_addr = tmem_base + ((uint32_t)(quarter * 32) << 16) +
                                        (uint32_t)(acc * kBN + half * (kBN / 2));
#pragma unroll 1
                for (int ch = 0; ch < (kBN / 2) / 32; ++ch) {
                    uint32_t raw[32];
                    ptx::tmem_ld_32x32b_x32(t_addr + ch * 32, raw);
                    ptx::tmem_wait_ld();
                    if (ch == (kBN / 2) / 32 - 1) {
                        // all TMEM reads of this accumulator are done: release it
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive(&tempty_bar[acc]);
                    }
                    const int col0 = half * (kBN / 2) + ch * 32;   // column inside the tile
                    if (p.epi_mode == EPI_STORE_H) {
                        // Algorithm 1 stage 3: H_r to main memory
                        long long hr = (long long)x * kBM + row;
                        float* dst = p.H + ((long long)r * p.Mb + hr) * p.Nb + (long long)z * kBN + col0;
#pragma unroll
                        for (int e = 0; e < 32; e += 4)
                            st_cg_f4(dst + e, make_float4(__uint_as_float(raw[e]), __uint_as_float(raw[e + 1]),
                                                          __uint_as_float(raw[e + 2]), __uint_as_float(raw[e + 3])));
                        continue;
                    }
                    // Combine H (Eq. 6): C_ij += W[r,i,j] * H_r for every nonzero W
                    for (int ij = 0; ij < mn; ++ij) {
                        const int wc = p.Wc[r * mn + ij];
                        if (!wc) continue;
                        const float sw = (float)wc;
                        float v[32];
#pragma unroll
                        for (int e = 0; e < 32; ++e) v[e] = sw * __uint_as_float(raw[e]);
                        float* pt = partial_tile(p, slot, ij);
                        if (r != first_r[ij]) {
#pragma unroll
                            for (int e = 0; e < 32; e += 4) {
                                float4 o = ld_cg_f4(pt + partial_off(row, (col0 + e) >> 2));
                                v[e] += o.x; v[e + 1] += o.y; v[e + 2] += o.z; v[e + 3] += o.w;
                            }
                        }
                        const bool final_here = (r == last_r[ij]) && (u.role == ROLE_WHOLE);
                        if (final_here) {
                            const int i = ij / p.n, j = ij - (ij / p.n) * p.n;
                            const long long crow = (long long)i * p.Mb + (long long)x * kBM + row;
                            const long long ccol = (long long)j * p.Nb + (long long)z * kBN + col0;
                            // rows / cols beyond this block's extent belong to padding
                            if ((long long)x * kBM + row < p.Mb && ccol < (long long)(j + 1) * p.Nb)
                                store_c_row(p, crow, ccol, v);
                        } else {
#pragma unroll
                            for (int e = 0; e < 32; e += 4)
                                st_cg_f4(pt + partial_off(row, (col0 + e) >> 2),
                                         make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]));
                        }
                    }
                }
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
            if (p.epi_mode != EPI_FUSED || u.role == ROLE_WHOLE) continue;

            // ---- split group: publish (contributor) or merge (owner)
            // named barrier over the 256 epilogue threads
            if (u.role == ROLE_CONTRIB) {
                __threadfence();
                asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
                if (ew == 0 && lane == 0) {
                    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p.flags + w), "r"(1)
                                 : "memory");
                }
                continue;
            }
            // owner: segments live on CTAs w+1 .. last
            const long long Tt_base = (long long)(u.g - p.q * p.W) * p.R;   // tail-local first tile
            const int last_cta = (int)((Tt_base + p.R - 1) / p.tail_c);
            if (ew == 0 && lane == 0) {
                for (int v = w + 1; v <= last_cta; ++v) {
                    int f = 0;
                    do {
                        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(p.flags + v)
                                     : "memory");
                    } while (f == 0);
                }
            }
            asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
            for (int ij = 0; ij < mn; ++ij) {
                const int i = ij / p.n, j = ij - (ij / p.n) * p.n;
#pragma unroll 1
                for (int ch = 0; ch < (kBN / 2) / 32; ++ch) {
                    const int col0 = half * (kBN / 2) + ch * 32;
                    float v[32];
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = 0.f;
                    if (first_r[ij] >= 0) {
                        const float* pt = partial_tile(p, w, ij);
#pragma unroll
                        for (int e = 0; e < 32; e += 4) {
                            float4 o = ld_cg_f4(pt + partial_off(row, (col0 + e) >> 2));
                            v[e] += o.x; v[e + 1] += o.y; v[e + 2] += o.z; v[e + 3] += o.w;
                        }
                    }
                    for (int vcta = w + 1; vcta <= last_cta; ++vcta) {
                        // does CTA vcta's segment contribute to C_ij?
                        long long lo = (long long)vcta * p.tail_c - Tt_base;
                        long long hi = lo + p.tail_c;
                        if (lo < 0) lo = 0;
                        if (hi > p.R) hi = p.R;
                        bool contributes = false;
                        for (long long r = lo; r < hi; ++r)
                            if (p.Wc[r * mn + ij]) { contributes = true; break; }
                        if (!contributes) continue;
                        const float* pt = partial_tile(p, p.W + vcta, ij);
#pragma unroll
                        for (int e = 0; e < 32; e += 4) {
                            float4 o = ld_cg_f4(pt + partial_off(row, (col0 + e) >> 2));
                            v[e] += o.x; v[e + 1] += o.y; v[e + 2] += o.z; v[e + 3] += o.w;
                        }
                    }
                    const long long crow = (long long)i * p.Mb + (long long)x * kBM + row;
                    const long long ccol = (long long)j * p.Nb + (long long)z * kBN + col0;
                    if ((long long)x * kBM + row < p.Mb && ccol < (long long)(j + 1) * p.Nb)
                        store_c_row(p, crow, ccol, v);
                }
            }
            // all reads done -> reset the flags for the next launch
            asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
            if (ew == 0 && lane == 0)
                for (int v = w + 1; v <= last_cta; ++v) p.flags[v] = 0;
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, 512);
    }
}

}  // namespace lcma
