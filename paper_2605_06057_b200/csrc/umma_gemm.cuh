// umma_gemm.cuh -- persistent, warp-specialised tcgen05 GEMM for sm_100a that
// runs the GEMM stage of the LCMA workflow (Eq. 5) and, in the
// fused mode, Combine H (Eq. 6) as its epilogue (Algorithm 2,
// stage 3/4).  The classical GEMM ("standard GEMM") is
// the same kernel with the trivial scheme <1,1,1;1>.
//
// CG = 1: one CTA per SM computes 128 x 256 tiles (tcgen05.mma cta_group::1).
// CG = 2: a CTA pair (cluster of 2 on one TPC) computes 256 x 256 tiles with
//         tcgen05.mma.cta_group::2 issued by the leader CTA; each CTA stages
//         its 128 rows of A and its 128 columns of B, so per-SM shared-memory
//         and L2 operand traffic per MMA flop are halved for B.
//
// Roles per CTA (384 threads; setmaxnreg moves registers from warpgroup 0,
// 40 per thread, to the two epilogue warpgroups, 232 per thread):
//   warp 0      TMA producer: At_r[x, y] and Bt_r[y, z] tiles -> smem ring
//   warp 1      MMA issuer (leader CTA only): one thread issues tcgen05.mma
//   warp 2      TMEM allocator (512 columns = 2 fp32 accumulators of 256)
//   warps 4-11  epilogue: TMEM -> registers -> (Combine H) -> global; each
//               thread owns one row x 128 columns of the CTA's 128 x 256 slab
//
// Fused Combine H keeps the live C_ij partials of a whole group on chip where
// it can (GemmParams::home): the most-updated slot in the epilogue threads'
// registers (REGH instantiation), the next in shared memory (column half 0)
// with column half 1 in an L2 workspace tile, further slots in L2 tiles.
//
// Work decomposition (Group-Parallel Optimization): a *group* is
// the set {H_r[x,z]}_{r=1..R} of one output tile position (x,z); the CTA (pair)
// that owns a group accumulates every C_{ij}[x,z] with W[r,i,j] != 0 and
// writes C once.  Scheduling: lockstep rounds of whole groups
// (all CTAs on the same r at the same time: cache-aware), then the tail of
// G mod W groups split at tile granularity over all CTAs (split-group); the
// segment holding r = 0 owns the group and merges the other segments'
// partials in a fixed order (deterministic, no atomics).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <type_traits>

#include "ptx.cuh"

namespace lcma {

#ifndef LCMA_MAX_STAGES
#define LCMA_MAX_STAGES 5         // smem ring depth (on-chip partial homes: 5 >= 4; earlier kernel: 4 > 5 > 6 > 7 > 3)
#endif
constexpr int kBM = 128;          // rows per CTA (TMEM lanes)
constexpr int kBN = 256;          // UMMA N = accumulator columns
constexpr int kThreads = 384;     // 12 warps
constexpr int kEpiWarp0 = 4;      // first epilogue warp
constexpr int kEpiWarps = 8;
constexpr int kMaxR = 128;
constexpr int kMaxMN = 32;
constexpr int kTlMax = 512;       // timeline entries per CTA
constexpr int kStatsPerCta = 16;  // diagnostics: wait counters per CTA (LCMA_STATS)
constexpr int kSchedDepth = 8;    // dynamic schedule: units published ahead of their consumers
constexpr int kBarBytes = 512;    // mbarriers, TMEM slot and schedule ring
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// QF = 1: the shared-memory C_ij partial covers the whole 128 x BN slab of
// the CTA (128 KB for BN = 256, leaving room for 3 operand stages); QF = 0:
// only column half 0 (64 KB, 4 stages), half 1 of that partial goes to L2.
#ifndef LCMA_MAX_STAGES_NP
#define LCMA_MAX_STAGES_NP 5      // ring depth of the instantiation without a partial area (classical)
#endif
// NP: no shared-memory partial area (the classical / unfused instantiation of
// the 256-column pair kernel), so the ring may use that space.
// PF: producer-fused combines (variant 3): 1 = Combine A, 2 = Combine A and B;
// a staging slot per stage for the second source block of each, and
// second A source block, no shared-memory partial area.
// F8: FP8 E4M3 operands (128 elements per 128-byte row) plus, per stage, the
// 512-byte UE8M0 scale chunks of the A rows and of the B columns (1 x 128
// block scaling, reading 23).
// CST: C staging area for TMA stores (costs one operand stage in the
// register-home instantiation; the long-K variant keeps the stage instead)
template <int CG, int BN = kBN, int QF = 0, bool NP = false, int PF = 0, bool F8 = false, bool CST = true>
struct Cfg {
    static constexpr int kTileM = kBM * CG;                  // rows per group tile
    static constexpr int kBNc = BN / CG;                     // B columns staged per CTA
    static constexpr int kABytes = kBM * 128;                // 128 rows x 128 bytes
    static constexpr int kBBytes = kBNc * 128;               // kBNc x 128 B (K-major) or chunks (MN-major)
    static constexpr int kSfBytes = F8 ? 1024 : 0;              // scale chunks: A rows, B columns
    static constexpr int kStageBytes =
        kABytes + kBBytes + (PF ? kABytes : 0) + (PF == 2 ? kBBytes : 0) + kSfBytes;   // PF: + staging
    // one C_ij partial kept in shared memory (fused Combine H, whole groups):
    // 128 rows x BN (QF) or BN/2 (column half 0) fp32
    // QF = 2: no shared-memory partial home (all but the register slot in L2),
    // the space goes to operand stages (long products)
    static constexpr int kPartialSmem = (NP || PF || QF == 2) ? 0 : kBM * (QF ? BN : BN / 2) * 4;
    // F8: a 128-deep E4M3 k-block is half the MMA time of a 64-deep 16-bit one,
    // so the ring needs more stages to cover the same load latency
    static constexpr int kMaxStages = F8 ? 8 : (QF == 2 ? 7 : (NP ? LCMA_MAX_STAGES_NP : LCMA_MAX_STAGES));
    // as many stages as fit in 227 KB (minus the partial, alignment slack and
    // barriers), <= LCMA_MAX_STAGES
    // C staging for TMA stores of 16-bit C (GemmParams::c_tma): two 32 x 32
    // 16-bit boxes (2 KB each) per epilogue warp
    static constexpr int kCStage = (CST && CG == 2 && PF == 0 && QF == 0) ? kEpiWarps * 2 * 2048 : 0;
    static constexpr int kFree = 232448 - 1024 - kBarBytes - kPartialSmem - kCStage;
    static constexpr int kStages = (kFree / kStageBytes) > kMaxStages ? kMaxStages : (kFree / kStageBytes);
    static constexpr int kSmemBytes = kStages * kStageBytes + kPartialSmem + kCStage + 1024 /*align*/ + kBarBytes;
};

// The 256-column pair kernel without a register home is only launched for
// classical / unfused GEMMs (no partial homes): no shared-memory partial area.
// Same for the FP8 instantiation without a register home (classical FP8).
template <int CG, int BN, int QF, bool REGH, bool F8 = false>
struct KernelNP {
    static constexpr bool value = CG == 2 && (BN == 256 || F8) && QF == 0 && !REGH;
};
// the shared-memory configuration of umma_gemm_kernel<CG, BN, QF, REGH, PF, DYN, F8>
template <int CG, int BN, int QF, bool REGH, int PF, bool F8, bool CST = true>
using KernelCfg = Cfg<CG, BN, QF, KernelNP<CG, BN, QF, REGH, F8>::value, PF, F8, CST>;

enum EpiMode : int { EPI_FUSED = 0, EPI_STORE_H = 1 };
enum OutType : int { OUT_BF16 = 0, OUT_FP16 = 1, OUT_FP32 = 2 };
enum UnitRole : int { ROLE_WHOLE = 0, ROLE_OWNER = 1, ROLE_CONTRIB = 2 };
// Where a whole group keeps a live C_ij partial (fp32, the CTA's 128 x BN
// slab): epilogue-thread registers, shared memory, or an L2 workspace slot.
enum PartialHome : int { HOME_REG = -1, HOME_SMEM = -2 };

struct GemmParams {
    // F8: the UE8M0 scale chunks of A~ and B~ as 2-D byte maps [2 * chunks][256]
    // (one 512-byte chunk per 128 rows x 128 K of an operand); chunk index =
    // (operand row / 128) * sf_nkb + k-block
    alignas(64) CUtensorMap sfa_map;
    alignas(64) CUtensorMap sfb_map;
    int sf_nkb;            // k-blocks per operand row (Kb / 128)
    int pf_kb;             // k-blocks of the next product prefetched to L2 at a product start (0: off)
    // single-term combined operands read in place (A~_r = A_il, B~_r = B_lj with
    // a +1 coefficient, exactly tiled extents): a_dir[r] = i * k + l (-1: the
    // materialised A~_r), b_dir[r] = j * k + l; a_raw / b_raw map A (M x K) and
    // B (N x K).  The combine kernels skip those outputs (2/7 of Strassen's).
    alignas(64) CUtensorMap a_raw;
    alignas(64) CUtensorMap b_raw;
    int8_t a_dir[kMaxR], b_dir[kMaxR];
    int use_dir;
    // 16-bit C written by TMA stores of 32 x 32 boxes staged in shared memory
    // (c_tma = 1): the epilogue threads' row-per-lane stores become one
    // asynchronous bulk store per warp and chunk; rows >= M / columns >= N
    // are clipped by the map ({N, M * nbatch})
    alignas(64) CUtensorMap c_map;
    int c_tma;
    // problem / blocking
    int nX, nZ;            // group tiles along M, N: Mb/kTileM, Nb/kBN
    int G;                 // groups = nX * nZ
    int R;                 // products per group
    int nK;                // k-blocks per product: Kb / BK
    int BK;                // elements per 128-byte row
    int a_rows_per_r;      // row offset of At_r in the A tensor map (Mb), 0 for R == 1
    int b_rows_per_r;      // row offset of Bt_r in the B map (Nb if K-major else Kb)
    int b_mn_major;        // B operand MN-major (B stored K x N)
    int b_3d;              // MN-major B via one 3-D TMA box per stage
    int tf32;              // kind::tf32 (else kind::f16)
    uint32_t idesc;        // instruction descriptor
    // schedule
    int W;                 // work units run in parallel (CTAs for CG=1, pairs for CG=2)
    int q;                 // lockstep rounds of whole groups
    int tail_c;            // tile capacity per unit in the split tail
    int swz;               // raster band height (tiles) for group -> (x, z)
    int n_whole;           // groups processed whole before the split tail (static: q * W, <= G)
    int dyn;               // 1: whole groups handed out at run time in raster order (ticket
                           //    counter `sched`, broadcast to every role of the pair via a shared ring)
    int* sched;            // dyn / dyn_tail: ticket counters [2] (workspace, zero between launches);
                           // [2] lockstep progress (pairs x products started), [3] exit count
    int drift;             // > 0: a pair starts product step s of the lockstep rounds only after
                           // every pair started step s - drift (bounded drift: the round's operand
                           // panels stay within the L2 window); 0: free-running
    int dyn_tail;          // 1: tail segments handed out at run time (DYN instantiation)
    int n_own;             // split groups of the tail (= owner segments)
    // batched GEMMs (two-level schemes: the R0 inner fused GEMMs of the outer
    // products in one launch): group g -> batch q = g / Gb, in-batch group
    // g % Gb; batch q's products are operand-map products r + q * R (the
    // composed index 7q + r2 of reading 3) and it writes C rows + q * M
    // (C = [nbatch][M][ldc])
    int nbatch, Gb;
    // epilogue
    int epi_mode;
    int out_type;
    int debug;             // bit0: skip epilogue global traffic (mainloop timing only)
    int partial_hint;      // 1: L2 evict_last policy on partial tiles
    int operand_hint;      // 1: L2 evict_first on operand TMA loads, 2: evict_last
    int b_layout_type;     // UMMA smem layout of B (2 = SWIZZLE_128B, 1 = 128B_BASE32B)
    int b_sbo;             // B stride byte offset (8-row (or 4-row) K group stride)
    unsigned long long* stats;   // optional per-CTA wait-cycle counters (diagnostics)
    unsigned long long* tl;      // optional per-product timeline (diagnostics): [cta][kTlMax][4] globaltimer ns:
                                 // 0 MMA slot acquired, 1 MMA issue done, 2 epilogue (half 0) has the
                                 // accumulator, 3 epilogue (half 1) released it
    int m, n;              // scheme grid (C blocks)
    long long M, N;        // true C extents (crop)
    long long Mb, Nb;      // block extents: C_ij origin = (i*Mb, j*Nb)
    long long ldc;
    int c_v8;              // C rows 32-byte aligned: 256-bit stores
    int c_cs;              // streaming (evict-first) C stores
    void* C;
    float* P;              // partial tiles (see partial_tile), each [kBN/4][kBM][4] fp32
    int* flags;            // [2 ctas] split-segment ready flags (contributor units, owner units)
    float* H;              // EPI_STORE_H: H [R][Mb][Nb] fp32
    int discard;           // 1: discard.global.L2 partial lines after their last read
    int pace_ns;           // >0: sleep between C_ij updates (spreads epilogue traffic)
    int nslot;             // partial tiles live at once for whole groups (<= m*n)
    int serpentine;        // odd lockstep rounds process their products in reverse order
    // producer-fused Combine A (PF kernel): At_r = s0 * A_blk0 + s1 * A_blk1,
    // blocks i*k + l of the raw A map (blk1 = -1: one block)
    int kgrid;             // scheme k
    int pf_Kb;             // block extent along K (columns of a source block)
    int8_t pf_blk0[kMaxR], pf_blk1[kMaxR], pf_s0[kMaxR], pf_s1[kMaxR];
    // PF = 2: Bt_r = s0 * B_blk0 + s1 * B_blk1, blocks l*n + j of the raw B
    // (stored N x K: block (l, j) at rows j*Nb, columns l*Kb)
    int ngrid, pf_Nb;
    int8_t pfb_blk0[kMaxR], pfb_blk1[kMaxR], pfb_s0[kMaxR], pfb_s1[kMaxR];
    int qslot;             // QF = 0: L2 slot of the column half 1 of the HOME_SMEM partial
    int8_t home[kMaxMN];   // whole groups: C_ij partial home (HOME_REG, HOME_SMEM, or L2 slot >= 0)
    int8_t rperm[kMaxR];   // product processing order inside a group (t -> r)
    int8_t Wc[kMaxR * kMaxMN];   // W[r][i*n + j]
    uint32_t nzmask[kMaxR];      // bit ij set iff W[r][ij] != 0
    uint8_t dbg_extra[kMaxR];    // diagnostics: (nnz(V_r)-1) << 4 | (nnz(U_r)-1)
};

// ------------------------------------------------------------ scheduling
struct Unit {
    int g, r0, r1, role;
    int rev;             // whole group of an odd lockstep round: products in reverse order
    int seg;             // split tail: segment index (its partial slot / flag); static: the unit slot w
};

// Shared-memory ring through which the pair leader's producer (the
// scheduler) hands run-time scheduling decisions to every other role of the
// pair.  One 32-bit shared address `ring` locates it (kept small: the
// producer / MMA warps run with few registers): full[d] mbarriers at
// ring + 8d (armed by the scheduler, locally and in the peer CTA), empty[d]
// at ring + 8D + 8d (leader only: the consumers that have read slot d), and
// slot[d] (int value of the k-th decision with k % D == d) at ring + 16D + 4d.
// Values: g >= 0 a whole group, -2 - s tail segment s, -1 the end.
constexpr uint32_t kRingFull = 0, kRingEmpty = 8 * kSchedDepth, kRingSlot = 16 * kSchedDepth;
constexpr int kRingBytes = 20 * kSchedDepth;
enum SchedRole : int { SR_SCHED = 0, SR_LOCAL = 1, SR_PEER = 2 };

// Enumerates the units of work-unit slot `w` in processing order.  Every role
// of the CTA (producer, MMA, epilogue) and both CTAs of a pair walk the same
// sequence.
//  DYN = false: lockstep rounds, group idx*W + w (P:391-396 cache-aware
//    reading 11), then unit w's segment of the split tail.
//  DYN = true: the pair leader's producer decides and broadcasts through the
//    ring: whole groups either in the same static rounds (dyn = 0) or drawn
//    from a ticket counter in raster order (dyn = 1, the groups in flight
//    stay a compact window of the raster), then tail segments drawn from a
//    second counter (dyn_tail), so the pairs that finish their whole groups
//    first take the tail: the owner of a split group waits only for pairs
//    that were free, not for the slowest ones.
template <bool DYN>
struct UnitIter {
    const GemmParams& p;
    int idx;             // lockstep round index
    int t;               // tail tile cursor (G * R < 2^31)
    int seg;             // tail segment being enumerated ([t, end of seg))
    int k;               // ring decisions consumed so far
    uint32_t ring;       // shared address of the ring (DYN)
    int pend;            // SR_SCHED: whole-group ticket drawn ahead (-1: none)
    int st;              // bits 0-1 SchedRole, 2 pair, 3-4 phase (SR_SCHED: 0 whole groups,
                         // 1 tail segments, 2 decided the end, 3 published it), 5 published
                         // one decision ahead of k
    __device__ UnitIter(const GemmParams& p_, int w_, uint32_t ring_ = 0u, int role_ = SR_LOCAL, int cg = 1)
        : p(p_), idx(0), t(0), seg(DYN ? -1 : w_), k(0), ring(ring_), pend(-1), st(role_ | (cg == 2 ? 4 : 0)) {
        if constexpr (!DYN) t = seg_begin(w_);
    }
    __device__ int unit_w() const { return (int)blockIdx.x / ((st & 4) ? 2 : 1); }
    __device__ int tail_tiles() const {
        const int Tt = (p.G - p.n_whole) * p.R;
        return Tt < 0 ? 0 : Tt;
    }
    __device__ int seg_begin(int s) const {
        const int b = s * p.tail_c, Tt = tail_tiles();
        return b < Tt ? b : Tt;
    }
    __device__ int seg_end() const {
        const int e = (seg + 1) * p.tail_c, Tt = tail_tiles();
        return e < Tt ? e : Tt;
    }
    __device__ int phase() const { return (st >> 3) & 3; }
    __device__ void set_phase(int ph) { st = (st & ~(3 << 3)) | (ph << 3); }
    // ---- SR_SCHED: the next decision, in order (whole groups, tail, end)
    __device__ int decide() {
        const int W = (int)gridDim.x / ((st & 4) ? 2 : 1);
        if (phase() == 0) {
            if (p.dyn) {
                const int tk = pend >= 0 ? pend : atomicAdd(p.sched, 1);
                pend = -1;
                // every unit draws exactly one failing ticket; the last one
                // drawn (n_whole + W - 1) resets the counter for the next launch
                if (tk == p.n_whole + W - 1) atomicExch(p.sched, 0);
                if (tk < p.n_whole) return tk;
            } else if (idx < p.q && idx * p.W + unit_w() < p.G) {
                return (idx++) * p.W + unit_w();
            }
            set_phase(1);
        }
        if (phase() == 1) {
            const int Tt = tail_tiles();
            const int nseg = Tt > 0 ? (Tt + p.tail_c - 1) / p.tail_c : 0;
            if (p.dyn_tail) {
                // A pair that draws an owner segment (the start of a split group)
                // draws nothing after it: its epilogue will wait there for the
                // group's other segments, which must then belong to other pairs
                // (a later segment of its own would deadlock).  Every other pair
                // ends with one failing ticket; the last of those (nseg +
                // W - n_own - 1) resets the counter for the next launch.
                const int tk = atomicAdd(p.sched + 1, 1);
                if (tk < nseg) {
                    const int b = tk * p.tail_c;
                    const int e = b + p.tail_c < Tt ? b + p.tail_c : Tt;
                    const int last_start = ((e - 1) / p.R) * p.R;       // last group starting before e
                    if (last_start >= b && last_start + p.R > e) set_phase(2);
                    return -2 - tk;
                }
                if (tk == nseg + W - p.n_own - 1) atomicExch(p.sched + 1, 0);
            } else if (idx >= 0 && unit_w() < nseg) {
                idx = -1;                           // this unit's own segment, once
                return -2 - unit_w();
            }
            set_phase(2);
        }
        return -1;
    }
    // SR_SCHED: publish ring slot `pub` (= k + ahead) with decision v
    __device__ void publish(int v) {
        const int pub = k + ((st >> 5) & 1);
        const uint32_t s = (uint32_t)(pub % kSchedDepth);
        const uint32_t ph = (uint32_t)(pub / kSchedDepth) & 1u;
        ptx::mbar_wait_u32(ring + kRingEmpty + 8u * s, ph ^ 1u);
        ptx::st_shared_u32(ring + kRingSlot + 4u * s, (uint32_t)v);
        if (st & 4) {
            // the peer's copy: an asynchronous remote store completing 4 bytes
            // of transaction on the peer's full[s] (armed by the relaxed
            // expect_tx arrival): the scheduler never waits on the DSMEM trip
            const uint32_t pbar = ptx::mapa_shared(ring + kRingFull + 8u * s, 1);
            ptx::mbar_arrive_expect_tx_cluster_relaxed(pbar, 4u);
            ptx::st_async_u32(ptx::mapa_shared(ring + kRingSlot + 4u * s, 1), (uint32_t)v, pbar);
        }
        ptx::mbar_arrive_u32(ring + kRingFull + 8u * s);
        st |= 1 << 5;                               // one ahead of k (or at k, filled)
        if (v == -1) set_phase(3);                  // the end is published
    }
    // SR_SCHED: publish the ring one decision ahead of its own position (the
    // peer CTA and the consumers learn the next group early) and, for drawn
    // whole groups, keep the ticket after that drawn (its L2 round trip
    // overlaps a unit of loads).  Called by the producer once the current
    // unit's first loads are issued, so the handshake stays off the critical
    // path.
    __device__ void advance() {
        if (!DYN || (st & 3) != SR_SCHED) return;
        if (!((st >> 5) & 1) && phase() != 3) publish(decide());
        if (phase() == 0 && p.dyn && pend == -1) pend = atomicAdd(p.sched, 1);
    }
    // the k-th decision.  Warps call this with all lanes; lane 0 (or the
    // single producer lane) does the arrivals, relaxed: the slot value is
    // already in a register.
    __device__ int ring_next(bool single_thread) {
        const uint32_t s = (uint32_t)(k % kSchedDepth);
        const uint32_t ph = (uint32_t)(k / kSchedDepth) & 1u;
        int v;
        if ((st & 3) == SR_SCHED) {
            if (!((st >> 5) & 1)) {                 // slot k not published yet
                st &= ~(1 << 5);
                publish(decide());
            }
            st &= ~(1 << 5);                        // after ++k: slot k+1 not yet published
            v = (int)ptx::ld_shared_u32(ring + kRingSlot + 4u * s);
        } else {
            const bool peer = (st & 3) == SR_PEER;
            if (peer) ptx::mbar_wait_cluster_u32(ring + kRingFull + 8u * s, ph);
            else ptx::mbar_wait_u32(ring + kRingFull + 8u * s, ph);
            v = (int)ptx::ld_shared_u32(ring + kRingSlot + 4u * s);
            if (!single_thread) __syncwarp();
            if (single_thread || ptx::lane_id() == 0) {
                if (peer) ptx::mbar_arrive_cluster_relaxed(ptx::mapa_shared(ring + kRingEmpty + 8u * s, 0));
                else ptx::mbar_arrive_relaxed_u32(ring + kRingEmpty + 8u * s);
            }
        }
        ++k;
        return v;
    }
    __device__ bool next(Unit& u, bool single_thread = false) {
        for (;;) {
            const int t_end = seg >= 0 ? seg_end() : 0;
            if (t < t_end) {                       // units of the current tail segment
                int gl = t / p.R;                  // tail-local group
                int r0 = (int)(t - gl * p.R);
                int stop = (gl + 1) * p.R;
                if (stop > t_end) stop = t_end;
                int r1 = (int)(stop - gl * p.R);
                u.g = p.n_whole + (int)gl;
                u.r0 = r0;
                u.r1 = r1;
                u.role = (r0 == 0 && r1 == p.R) ? ROLE_WHOLE : (r0 == 0 ? ROLE_OWNER : ROLE_CONTRIB);
                u.rev = 0;
                u.seg = seg;
                t = stop;
                return true;
            }
            if constexpr (DYN) {
                const int v = ring_next(single_thread);
                if (v >= 0) {
                    u.g = v;
                    u.r0 = 0;
                    u.r1 = p.R;
                    u.role = ROLE_WHOLE;
                    u.rev = 0;
                    u.seg = -1;
                    return true;
                }
                if (v == -1) return false;
                seg = -2 - v;
                t = seg_begin(seg);
                continue;
            } else {
                if (idx < p.q) {
                    const int w = unit_w();
                    u.g = idx * p.W + w;
                    if (u.g >= p.G) return false;  // schedule 3: last round of whole groups
                    u.r0 = 0;
                    u.r1 = p.R;
                    u.role = ROLE_WHOLE;
                    // serpentine product order over rounds: a round starts with the
                    // product the previous round ended with
                    u.rev = p.serpentine ? (idx & 1) : 0;
                    u.seg = -1;
                    ++idx;
                    return true;
                }
                return false;
            }
        }
    }
};

// Product processed at position t of unit u.
__device__ __forceinline__ int product_at(const GemmParams& p, const Unit& u, int t) {
    return p.rperm[u.rev ? p.R - 1 - t : t];
}

// Group index -> tile coordinates: bands of `swz` tile-rows traversed
// column by column so that the W groups of a lockstep round cover a compact
// (x, z) region (operand reuse in L2).
__device__ __forceinline__ void group_xz(const GemmParams& p, int g, int& x, int& z) {
    if (p.nbatch > 1) g %= p.Gb;
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
// 16-byte fp32 reduction performed in L2 (REDG.E.ADD.F32x4): no data returns
// to the SM, and operations of one thread on one address apply in order.
__device__ __forceinline__ void red_add_f4(float* p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}
__device__ __forceinline__ void red_add_pol_f4(float* p, float a, float b, float c, float d, uint64_t pol) {
    asm volatile("red.global.add.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(a), "f"(b), "f"(c),
                 "f"(d), "l"(pol)
                 : "memory");
}
struct GemmParams;
// partial-tile accesses with an L2 cache policy (evict_last keeps the
// group's C_ij partials resident while operand tiles stream through L2)
__device__ __forceinline__ float4 ld_pol_f4(const float* p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.cg.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_pol_f4(float* p, float4 v, uint64_t pol) {
    asm volatile("st.global.cg.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
                 :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}

// Store 32 consecutive fp32 values of one C row segment (cols c0..c0+31),
// cropping to N.  N is a multiple of 8 (TMA rule) so 8-element vectors are
// either fully inside or fully outside.
__device__ __forceinline__ void st_v8(void* dst, const uint32_t* w, bool cs) {
    if (cs)   // streaming (evict-first): C is written once and never re-read here
        asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst), "r"(w[0]), "r"(w[1]),
                     "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                     : "memory");
    else
        asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst), "r"(w[0]), "r"(w[1]), "r"(w[2]),
                     "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                     : "memory");
}
__device__ __forceinline__ uint32_t pack2(const GemmParams& p, float a, float b);

// Store 32 consecutive fp32 values of one C row segment (cols c0..c0+31),
// cropping to N.  N is a multiple of 8 (TMA rule) so 8-element vectors are
// either fully inside or fully outside.  With 32-byte aligned rows (c_v8) a
// thread writes whole 32-byte sectors (256-bit STG).
__device__ __forceinline__ void store_c_row(const GemmParams& p, long long row, long long c0,
                                            const float* v) {
    if (row >= p.M) return;
    if (p.out_type == OUT_FP32) {
        float* dst = reinterpret_cast<float*>(p.C) + row * p.ldc + c0;
        if (p.c_v8 && c0 + 32 <= p.N) {
#pragma unroll
            for (int e = 0; e < 32; e += 8) st_v8(dst + e, reinterpret_cast<const uint32_t*>(v + e), p.c_cs);
            return;
        }
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
            if (c0 + e < p.N)
                *reinterpret_cast<float4*>(dst + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
        }
    } else {
        uint16_t* dst = reinterpret_cast<uint16_t*>(p.C) + row * p.ldc + c0;
        uint32_t w[16];
#pragma unroll
        for (int h = 0; h < 16; ++h) w[h] = pack2(p, v[2 * h], v[2 * h + 1]);
        if (p.c_v8 && c0 + 32 <= p.N) {
            st_v8(dst, w, p.c_cs);
            st_v8(dst + 16, w + 8, p.c_cs);
            return;
        }
#pragma unroll
        for (int e = 0; e < 32; e += 8) {
            if (c0 + e < p.N)
                *reinterpret_cast<uint4*>(dst + e) = make_uint4(w[e / 2], w[e / 2 + 1], w[e / 2 + 2], w[e / 2 + 3]);
        }
    }
}

// Store 16 consecutive fp32 values of one C row segment (cols c0..c0+15),
// cropped like store_c_row: the final-contribution paths of the fused
// epilogue work in 16-column halves so that only 16 temporaries are live
// next to the register partial (fewer spills).
__device__ __forceinline__ void store_c_row16(const GemmParams& p, long long row, long long c0,
                                              const float* v, long long radd = 0) {
    if (row >= p.M) return;
    row += radd;                                   // batched GEMMs: batch q's rows start at q * M
    if (p.debug & 2048) {
        // diagnostics (results WRONG): the same bytes, fully coalesced -- the
        // 32 lanes of a warp write 1 KB contiguous of one row band
        uint32_t w[8];
#pragma unroll
        for (int h = 0; h < 8; ++h) w[h] = pack2(p, v[2 * h], v[2 * h + 1]);
        uint16_t* dst = reinterpret_cast<uint16_t*>(p.C) + (row & ~31ll) * p.ldc + ((c0 * 32) % (p.ldc - 512)) +
                        (threadIdx.x & 31) * 16;
        st_v8(dst, w, p.c_cs);
        return;
    }
    if (p.out_type == OUT_FP32) {
        float* dst = reinterpret_cast<float*>(p.C) + row * p.ldc + c0;
        if (p.c_v8 && c0 + 16 <= p.N) {
            st_v8(dst, reinterpret_cast<const uint32_t*>(v), p.c_cs);
            st_v8(dst + 8, reinterpret_cast<const uint32_t*>(v + 8), p.c_cs);
            return;
        }
#pragma unroll
        for (int e = 0; e < 16; e += 4) {
            if (c0 + e < p.N)
                *reinterpret_cast<float4*>(dst + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
        }
    } else {
        uint16_t* dst = reinterpret_cast<uint16_t*>(p.C) + row * p.ldc + c0;
        uint32_t w[8];
#pragma unroll
        for (int h = 0; h < 8; ++h) w[h] = pack2(p, v[2 * h], v[2 * h + 1]);
        if (p.c_v8 && c0 + 16 <= p.N) {
            st_v8(dst, w, p.c_cs);
            return;
        }
#pragma unroll
        for (int e = 0; e < 16; e += 8) {
            if (c0 + e < p.N)
                *reinterpret_cast<uint4*>(dst + e) = make_uint4(w[e / 2], w[e / 2 + 1], w[e / 2 + 2], w[e / 2 + 3]);
        }
    }
}

__device__ __forceinline__ uint32_t pack2(const GemmParams& p, float a, float b) {
    if (p.out_type == OUT_BF16) {
        __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
        return *reinterpret_cast<uint32_t*>(&t);
    }
    __half2 t = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&t);
}

// Store 8 consecutive fp32 values (cols c0..c0+7) of one C row, cropped.
__device__ __forceinline__ void store_c8(const GemmParams& p, long long row, long long c0, const float* v) {
    if (row >= p.M || c0 >= p.N) return;
    if (p.out_type == OUT_FP32) {
        float* dst = reinterpret_cast<float*>(p.C) + row * p.ldc + c0;
        *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4*>(dst + 4) = make_float4(v[4], v[5], v[6], v[7]);
    } else {
        uint32_t w4[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            if (p.out_type == OUT_BF16) {
                __nv_bfloat162 b = __floats2bfloat162_rn(v[2 * h], v[2 * h + 1]);
                w4[h] = *reinterpret_cast<uint32_t*>(&b);
            } else {
                __half2 b = __floats2half2_rn(v[2 * h], v[2 * h + 1]);
                w4[h] = *reinterpret_cast<uint32_t*>(&b);
            }
        }
        *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p.C) + row * p.ldc + c0) =
            make_uint4(w4[0], w4[1], w4[2], w4[3]);
    }
}

// Partial tile layout: [kBN/4][kBM][4] floats, so that the 32 threads of a
// warp (32 consecutive rows) touch 512 contiguous bytes per float4 access.
// Whole groups keep a C_ij partial in registers, shared memory or an L2 slot
// (GemmParams::home; C blocks whose live ranges in the product order do not
// overlap share a home); split segments keep one L2 tile per C block (they
// stay live until the owner merges them).
// Layout: whole-group slots first, slot-major ([nslot][ctas] tiles, one
// contiguous L2-persistable region), then the split-segment tiles
// ([2*ctas][m*n]).
template <int BN = kBN>
__device__ __forceinline__ float* partial_tile(const GemmParams& p, int slot, int idx, bool whole) {
    const size_t T = (size_t)(kBM * BN);
    if (whole) return p.P + ((size_t)idx * gridDim.x + slot) * T;     // idx = L2 home slot
    return p.P + ((size_t)p.m * p.n * gridDim.x + (size_t)slot * p.m * p.n + idx) * T;   // idx = ij
}
// Drop the 128-byte L2 lines of a partial tile column range after their last
// read: dead data is neither written back to DRAM nor occupies L2.  Called by
// lanes whose row is a multiple of 8 (one line = 8 rows x 16 bytes).
__device__ __forceinline__ void discard_lines(const float* pt, int row, int col4_0, int n_col4) {
    for (int c = 0; c < n_col4; ++c)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(pt + ((size_t)(col4_0 + c) * kBM + row) * 4)
                     : "memory");
}
__device__ __forceinline__ size_t partial_off(int row, int col4) {
    return ((size_t)col4 * kBM + row) * 4;
}

// mbarrier wait that accumulates the cycles spent waiting (diagnostics only)
__device__ __forceinline__ void timed_wait(uint64_t* bar, uint32_t parity, unsigned long long* acc) {
    if (acc) {
        long long t0 = clock64();
        ptx::mbar_wait(bar, parity);
        *acc += (unsigned long long)(clock64() - t0);
    } else {
        ptx::mbar_wait(bar, parity);
    }
}

// ------------------------------------------------------------ the kernel
template <int CG, int BN, int QF = 0, bool REGH = false, int PF = 0, bool DYN = false, bool F8 = false,
          bool CST = true>
__global__ void __launch_bounds__(kThreads, 1)
    umma_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a,
                     const __grid_constant__ CUtensorMap tmap_b,
                     const __grid_constant__ GemmParams p) {
    using C_ = KernelCfg<CG, BN, QF, REGH, PF, F8, CST>;
    static_assert(!F8 || (BN == 128 && PF == 0), "FP8: 128-column tiles (2 x 128 accumulator columns + scales in TMEM)");
    constexpr int kStages = C_::kStages;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    float* psmem = reinterpret_cast<float*>(smem + kStages * C_::kStageBytes);   // [QF?BN/4:BN/8][kBM][4]
    // C staging boxes [kEpiWarps][2][32 rows][64 B] (TMA stores)
    uint8_t* cstage = smem + kStages * C_::kStageBytes + C_::kPartialSmem;
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kStages * C_::kStageBytes + C_::kPartialSmem + C_::kCStage);
    uint64_t* empty_bar = full_bar + kStages;
    uint64_t* tfull_bar = empty_bar + kStages;   // [2]
    uint64_t* tempty_bar = tfull_bar + 2;        // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
    uint64_t* ld_bar = tempty_bar + 4;           // PF: [kStages] own A tiles landed (local)
    uint64_t* sched_full = ld_bar + kStages;     // dynamic schedule ring (UnitIter)
    uint64_t* sched_empty = sched_full + kSchedDepth;
    const uint32_t ring = ptx::smem_u32(sched_full);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    long long clk_entry = clock64();
    if (p.stats && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.stats[blockIdx.x * kStatsPerCta + 6] = t;
    }
    const uint32_t rank = CG == 1 ? 0u : ptx::cluster_ctarank();
    const bool leader = rank == 0;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmap_a);
        ptx::tma_prefetch_desc(&tmap_b);
        for (int s = 0; s < kStages; ++s) {
            // the leader's expect_tx arrival (+ PF: one arrival per combine warp
            // of both CTAs once the combined A tile is in place)
            ptx::mbar_init(&full_bar[s], PF ? 1 + 2 * CG : 1);
            ptx::mbar_init(&empty_bar[s], 1);       // one commit per stage
            if constexpr (PF) ptx::mbar_init(&ld_bar[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull_bar[a], 1);
            ptx::mbar_init(&tempty_bar[a], kEpiWarps * CG);
        }
        // schedule ring consumers of the leader's empty[]: MMA warp + epilogue
        // warps (+ the peer's producer and epilogue warps)
        for (int d = 0; d < kSchedDepth; ++d) {
            ptx::mbar_init(&sched_full[d], 1);
            ptx::mbar_init(&sched_empty[d], CG == 2 ? 2 + 2 * kEpiWarps : 1 + kEpiWarps);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 2) {
        ptx::tmem_alloc<CG>(tmem_slot, 512);
        ptx::tmem_relinquish<CG>();
    }
    ptx::tc_fence_before();
    if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // registers: the TMA / MMA / allocator warpgroup needs few, the two
    // epilogue warpgroups keep a 128 x BN fp32 partial (BN/2 per thread)
    // in registers on top of the H chunk (128*56 + 256*224 = 384*168).
    // Each role branch starts with its setmaxnreg so that ptxas allocates
    // the branch with that budget.

    const int w = blockIdx.x / CG;           // work-unit slot (pair index for CG = 2)
    // register split (128 * lo + 256 * hi <= 64 K): the register C_ij partial
    // (REGH) needs 128 more registers per epilogue thread; without it the
    // producer / MMA warps get room for the schedule state (no spills)
    constexpr int kRegLo = REGH ? 40 : 88;
    constexpr int kRegHi = REGH ? 232 : 208;

    if (warp == 0) {
        // ================================ TMA producer (both CTAs of a pair)
        ptx::setmaxnreg_dec<kRegLo>();
        if (ptx::elect_one()) {
            const int b_bytes_chunk = p.BK * 128;   // MN-major chunk: BK rows x 128 B
            const int n_chunks = C_::kBNc / p.BK;   // MN-major: 128-byte column chunks per CTA
            int stage = 0;
            uint32_t phase = 0;
            unsigned long long w_empty = 0;
            unsigned long long* st_empty = p.stats ? &w_empty : nullptr;
            // L2 policies of the operand loads: 1 both evict_first, 2 both
            // evict_last, 3 A evict_last / B evict_first (A panels are reused by
            // the rounds of a band, B panels stream), 4 the reverse
            const int oh = p.operand_hint;
            const uint64_t opol = oh == 2 || oh == 3 ? ptx::policy_evict_last() : ptx::policy_evict_first();
            const uint64_t opol_b = oh == 2 || oh == 4 ? ptx::policy_evict_last() : ptx::policy_evict_first();
            const bool ohint = oh != 0;
            UnitIter<DYN> it(p, w, ring, leader ? SR_SCHED : SR_PEER, CG);
            Unit u;
            int s_step = 0;          // lockstep product steps started (bounded-drift throttle)
            while (it.next(u, true)) {
                int x, z;
                group_xz(p, u.g, x, z);
                const int qb = p.nbatch > 1 ? u.g / p.Gb : 0;
                for (int t = u.r0; t < u.r1; ++t) {
                    // (batched: the batch's products are rows r + qb * R of the maps)
                    const int r = product_at(p, u, t) + qb * p.R;
                    const int a_row = r * p.a_rows_per_r + x * C_::kTileM + (int)rank * kBM;
                    const int b_col0 = z * BN + (int)rank * C_::kBNc;
                    if constexpr (CG == 2 && PF == 0) {
#ifdef LCMA_DIAG
                        // diagnostics build: the general loop below whenever a knob
                        // changes what the producer issues
                        const bool lean = !(p.debug & (16 | 32 | 64 | 4096));
#else
                        constexpr bool lean = true;
#endif
                        if (lean && (!p.b_mn_major || p.b_3d)) {
                            // lean issue loop (K-major A and B, the product build): per
                            // stage one wait, one expect_tx and the TMA issues with
                            // every per-product term hoisted -- at 128-deep E4M3
                            // k-blocks the stage lasts ~270 cycles, so the producer's
                            // instruction latency, not L2, would otherwise set the pace
                            const uint32_t lbar0 = ptx::mapa_shared(ptx::smem_u32(&full_bar[0]), 0);
                            const int b_row = r * p.b_rows_per_r + b_col0;
                            const int nk = p.nK;
                            [[maybe_unused]] const int ca0 = (a_row >> 7) * p.sf_nkb;
                            [[maybe_unused]] const int cb0 = ((r * p.b_rows_per_r + z * BN) >> 7) * p.sf_nkb;
                            if (p.drift > 0 && leader && u.role == ROLE_WHOLE && p.sched) {
                                // bounded drift: wait until every pair has started step
                                // s - drift, then count this pair's start of step s
                                const int target = (s_step - p.drift) * p.W;
                                if (target > 0) {
                                    int v;
                                    do {
                                        asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p.sched + 2) : "memory");
                                    } while (v < target);
                                }
                                atomicAdd(p.sched + 2, 1);
                                ++s_step;
                            }
                            if (p.pf_kb > 0 && t + 1 < u.r1) {
                                // product boundary: the next product's first k-blocks to L2
                                // while this one streams (its panels are new to the round)
                                const int rn = product_at(p, u, t + 1) + qb * p.R;
                                const int an = rn * p.a_rows_per_r + x * C_::kTileM + (int)rank * kBM;
                                const int bn = rn * p.b_rows_per_r + b_col0;
                                const int np = p.pf_kb < nk ? p.pf_kb : nk;
                                for (int q = 0; q < np; ++q) {
                                    ptx::tma_prefetch_2d(&tmap_a, q * (F8 ? 128 : p.BK), an);
                                    ptx::tma_prefetch_2d(&tmap_b, q * (F8 ? 128 : p.BK), bn);
                                }
                            }
                            // in-place operands (p.a_dir / p.b_dir): the source block's rows
                            // and column offset inside A (B)
                            const CUtensorMap* ma = &tmap_a;
                            const CUtensorMap* mb = &tmap_b;
                            int ar = a_row, br = b_row, ak0 = 0, bk0 = 0;
                            if (!F8 && p.use_dir) {
                                const int da = p.a_dir[r], db = p.b_dir[r];
                                if (da >= 0) {
                                    ma = &p.a_raw;
                                    ar = (da / p.kgrid) * (int)p.Mb + x * C_::kTileM + (int)rank * kBM;
                                    ak0 = (da % p.kgrid) * p.pf_Kb;
                                }
                                if (db >= 0) {
                                    mb = &p.b_raw;
                                    br = (db / p.kgrid) * (int)p.Nb + b_col0;
                                    bk0 = (db % p.kgrid) * p.pf_Kb;
                                }
                            }
                            for (int kb = 0; kb < nk; ++kb) {
                                ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
                                uint8_t* sa = smem + stage * C_::kStageBytes;
                                const uint32_t lbar = lbar0 + 8u * (uint32_t)stage;
                                if (leader) ptx::mbar_arrive_expect_tx(&full_bar[stage], C_::kStageBytes * CG);
                                const int kcol = kb * (F8 ? 128 : p.BK);
                                ptx::tma_load_2d_cg2(sa, ma, lbar, ak0 + kcol, ar, ohint, opol);
                                if (!p.b_mn_major)
                                    ptx::tma_load_2d_cg2(sa + C_::kABytes, mb, lbar, bk0 + kcol, br, ohint, opol_b);
                                else   // B stored K x N: one 3-D box {128 B, BK rows, BN/CG/BK chunks}
                                    ptx::tma_load_3d_cg2(sa + C_::kABytes, &tmap_b, lbar, 0, r * p.b_rows_per_r + kcol,
                                                         b_col0 / p.BK);
                                if constexpr (F8) {
                                    ptx::tma_load_2d_cg2(sa + C_::kABytes + C_::kBBytes, &p.sfa_map, lbar, 0,
                                                         2 * (ca0 + kb));
                                    ptx::tma_load_2d_cg2(sa + C_::kABytes + C_::kBBytes + 512, &p.sfb_map, lbar, 0,
                                                         2 * (cb0 + kb));
                                }
                                if (++stage == kStages) { stage = 0; phase ^= 1; }
                                if constexpr (DYN) {
                                    if (kb == 0 && t == u.r0) it.advance();
                                }
                            }
                            continue;
                        }
                    }
                    for (int kb = 0; kb < p.nK; ++kb) {
                        timed_wait(&empty_bar[stage], phase ^ 1, st_empty);
                        uint8_t* sa = smem + stage * C_::kStageBytes;
                        uint8_t* sb = sa + C_::kABytes;
                        const int kcol = kb * p.BK;
                        if constexpr (CG == 1) {
                            ptx::mbar_arrive_expect_tx(&full_bar[stage], C_::kStageBytes);
                            ptx::tma_load_2d(sa, &tmap_a, &full_bar[stage], kcol, a_row);
                            if (!p.b_mn_major) {
                                ptx::tma_load_2d(sb, &tmap_b, &full_bar[stage], kcol, r * p.b_rows_per_r + b_col0);
                            } else if (p.b_3d) {
                                ptx::tma_load_3d(sb, &tmap_b, &full_bar[stage], 0, r * p.b_rows_per_r + kcol,
                                                 b_col0 / p.BK);
                            } else {
                                for (int c = 0; c < n_chunks; ++c)
                                    ptx::tma_load_2d(sb + c * b_bytes_chunk, &tmap_b, &full_bar[stage],
                                                     b_col0 + c * p.BK, r * p.b_rows_per_r + kcol);
                            }
                            if constexpr (F8) {
                                const int ca = ((r * p.a_rows_per_r + x * C_::kTileM) >> 7) * p.sf_nkb + kb;
                                const int cb = ((r * p.b_rows_per_r + z * BN) >> 7) * p.sf_nkb + kb;
                                ptx::tma_load_2d(sb + C_::kBBytes, &p.sfa_map, &full_bar[stage], 0, 2 * ca);
                                ptx::tma_load_2d(sb + C_::kBBytes + 512, &p.sfb_map, &full_bar[stage], 0, 2 * cb);
                            }
                        } else {
                            // only the leader arms its barrier (with both CTAs' bytes);
                            // the peer's TMA completes bytes on the leader's barrier
                            const uint32_t lbar = ptx::mapa_shared(ptx::smem_u32(&full_bar[stage]), 0);
                            if (p.debug & 16) {   // diagnostics: MMA on stale smem, no operand traffic
                                if (leader) ptx::mbar_arrive(&full_bar[stage]);
                                if (++stage == kStages) { stage = 0; phase ^= 1; }
                                continue;
                            }
                            // diagnostics (debug bit 5): extra operand tile loads per product,
                            // the L2 traffic of Combine A/B done in the producer (nnz(U_r)
                            // resp. nnz(V_r) source tiles instead of one combined tile)
                            const int ea = (p.debug & 32) ? (p.dbg_extra[r] & 15) : 0;
                            const int eb = (p.debug & 32) ? (p.dbg_extra[r] >> 4) : 0;
                            // diagnostics (debug bit 6): A tile loaded only on even k-blocks,
                            // i.e. the L2 operand traffic of an A-multicast cluster of 2 pairs
                            const bool skip_a = (p.debug & 64) && (kb & 1);
                            // diagnostics (debug bit 12, F8): no scale-chunk loads (stale scales)
                            const bool skip_sf = F8 && (p.debug & 4096);
                            if (leader) {
                                if constexpr (PF == 2) ptx::mbar_arrive(&full_bar[stage]);   // all bytes on ld_bar
                                else if constexpr (PF == 1) ptx::mbar_arrive_expect_tx(&full_bar[stage], C_::kBBytes * CG);
                                else
                                    ptx::mbar_arrive_expect_tx(&full_bar[stage],
                                                               (C_::kStageBytes - (skip_a ? C_::kABytes : 0) -
                                                                (skip_sf ? C_::kSfBytes : 0) +
                                                                ea * C_::kABytes + eb * C_::kBBytes) * CG);
                            }
                            for (int e = 1; e <= ea; ++e)
                                ptx::tma_load_2d_cg2(sa, &tmap_a, lbar, kcol,
                                                     ((r + e) % p.R) * p.a_rows_per_r + x * C_::kTileM + (int)rank * kBM,
                                                     ohint, opol);
                            for (int e = 1; e <= eb && !p.b_mn_major; ++e)
                                ptx::tma_load_2d_cg2(sb, &tmap_b, lbar, kcol,
                                                     ((r + e) % p.R) * p.b_rows_per_r + b_col0, ohint, opol);
                            if constexpr (PF) {
                                // Combine A in the producer path: the (one or two) nonzero
                                // A blocks land in this CTA's A slot and staging slot on
                                // the local ld_bar; the combine warps sum them
                                const int b0 = p.pf_blk0[r], b1 = p.pf_blk1[r];
                                const int xr = x * C_::kTileM + (int)rank * kBM;
                                int ld_bytes = (b1 >= 0 ? 2 : 1) * C_::kABytes;
                                if constexpr (PF == 2) ld_bytes += (p.pfb_blk1[r] >= 0 ? 2 : 1) * C_::kBBytes;
                                ptx::mbar_arrive_expect_tx(&ld_bar[stage], ld_bytes);
                                ptx::tma_load_2d(sa, &tmap_a, &ld_bar[stage], (b0 % p.kgrid) * p.pf_Kb + kcol,
                                                 (b0 / p.kgrid) * (int)p.Mb + xr);
                                if (b1 >= 0)
                                    ptx::tma_load_2d(sa + C_::kABytes + C_::kBBytes, &tmap_a, &ld_bar[stage],
                                                     (b1 % p.kgrid) * p.pf_Kb + kcol, (b1 / p.kgrid) * (int)p.Mb + xr);
                            } else if (!skip_a) {
                                ptx::tma_load_2d_cg2(sa, &tmap_a, lbar, kcol, a_row, ohint, opol);
                            }
                            if constexpr (PF == 2) {
                                // Combine B in the producer path: this CTA's B-half of the
                                // one or two nonzero B blocks, on the local ld_bar
                                const int c0 = p.pfb_blk0[r], c1 = p.pfb_blk1[r];
                                ptx::tma_load_2d(sb, &tmap_b, &ld_bar[stage], (c0 / p.ngrid) * p.pf_Kb + kcol,
                                                 (c0 % p.ngrid) * p.pf_Nb + b_col0);
                                if (c1 >= 0)
                                    ptx::tma_load_2d(sa + 2 * C_::kABytes + C_::kBBytes, &tmap_b, &ld_bar[stage],
                                                     (c1 / p.ngrid) * p.pf_Kb + kcol, (c1 % p.ngrid) * p.pf_Nb + b_col0);
                            } else if (!p.b_mn_major) {
                                ptx::tma_load_2d_cg2(sb, &tmap_b, lbar, kcol, r * p.b_rows_per_r + b_col0, ohint, opol_b);
                                if (F8 && !skip_sf) {
                                    // scale chunks: this CTA's 128 A rows; the pair tile's B columns
                                    // (both CTAs hold the same chunk: the MMA of each CTA scales
                                    // all BN columns of its accumulator rows)
                                    const int ca = (a_row >> 7) * p.sf_nkb + kb;
                                    const int cb = ((r * p.b_rows_per_r + z * BN) >> 7) * p.sf_nkb + kb;
                                    ptx::tma_load_2d_cg2(sb + C_::kBBytes, &p.sfa_map, lbar, 0, 2 * ca);
                                    ptx::tma_load_2d_cg2(sb + C_::kBBytes + 512, &p.sfb_map, lbar, 0, 2 * cb);
                                }
                            } else if (p.b_3d) {
                                ptx::tma_load_3d_cg2(sb, &tmap_b, lbar, 0, r * p.b_rows_per_r + kcol,
                                                     b_col0 / p.BK);
                            } else {
                                for (int c = 0; c < n_chunks; ++c)
                                    ptx::tma_load_2d_cg2(sb + c * b_bytes_chunk, &tmap_b, lbar,
                                                         b_col0 + c * p.BK, r * p.b_rows_per_r + kcol, ohint, opol_b);
                            }
                        }
                        if (++stage == kStages) { stage = 0; phase ^= 1; }
                        if constexpr (DYN) {
                            if (kb == 0 && t == u.r0) it.advance();
                        }
                    }
                }
            }
            if (p.stats) p.stats[blockIdx.x * kStatsPerCta + 0] = w_empty;
        }
    } else if (warp == 1) {
        // ================================ MMA issuer (leader CTA)
        // The whole warp walks the schedule so that stage / descriptor
        // arithmetic stays in uniform registers; one lane issues the MMAs and
        // the commits (a commit tracks the MMAs of the issuing thread).
        ptx::setmaxnreg_dec<kRegLo>();
        if (leader) {
            const uint32_t b_lbo = p.BK * 128;            // MN-major: chunk stride
            const uint32_t b_kstep = p.b_mn_major ? (uint32_t)(32 / (p.tf32 ? 4 : 2)) * 128u : 32u;
            const uint32_t smem0 = ptx::smem_u32(smem);
            // descriptors of stage 0, k-step 0; the start-address field (addr >> 4,
            // bits [0,14)) of later stages / k-steps is reached by plain addition
            const uint64_t a_desc0 = ptx::smem_desc_sw128(smem0, 16, 1024);
            const uint64_t b_desc0 = p.b_mn_major
                                         ? ptx::smem_desc(smem0 + C_::kABytes, b_lbo, p.b_sbo, p.b_layout_type)
                                         : ptx::smem_desc_sw128(smem0 + C_::kABytes, 16, 1024);
            const uint32_t b_step = b_kstep >> 4;
            constexpr uint32_t kStageStep = C_::kStageBytes >> 4;
            const bool tf32 = p.tf32 != 0;
            const uint32_t idesc = p.idesc;
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            unsigned long long w_tempty = 0, w_full = 0;
            unsigned long long w_kb[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            const long long t_start = clock64();
            UnitIter<DYN> it(p, w, ring, SR_LOCAL, CG);
            Unit u;
            int tli = 0;
            while (it.next(u)) {
                for (int r = u.r0; r < u.r1; ++r) {
                    timed_wait(&tempty_bar[acc], acc_phase ^ 1, (p.stats && lane == 0) ? &w_tempty : nullptr);
                    ptx::tc_fence_after();
                    if (p.tl && lane == 0 && tli < kTlMax) p.tl[((size_t)blockIdx.x * kTlMax + tli) * 4 + 0] = gtimer();
                    const uint32_t d_tmem = tmem_base + acc * BN;
                    for (int kb = 0; kb < p.nK; ++kb) {
                        if (p.stats && lane == 0) {
                            // operand wait by k-block position inside the product
                            // (0, 1, 2, 3, 4-7, 8-15, 16-31, 32+): stats slots 8..15
                            const long long t0w = clock64();
                            ptx::mbar_wait(&full_bar[stage], phase);
                            const unsigned long long dw = (unsigned long long)(clock64() - t0w);
                            w_full += dw;
                            const int bkt = kb < 4 ? kb : kb < 8 ? 4 : kb < 16 ? 5 : kb < 32 ? 6 : 7;
                            w_kb[bkt] += dw;
                        } else {
                            ptx::mbar_wait(&full_bar[stage], phase);
                        }
                        ptx::tc_fence_after();
                        const uint64_t ad = a_desc0 + (uint64_t)(stage * kStageStep);
                        const uint64_t bd = b_desc0 + (uint64_t)(stage * kStageStep);
                        if (ptx::elect_one()) {
                            if constexpr (F8) {
                                // scales of this stage -> TMEM (columns 2*BN + 8*stage: A rows,
                                // + 4: B columns), then the four K = 32 block-scaled MMAs; the
                                // copy and the MMAs execute in issue order
                                const uint32_t sf_t = tmem_base + 2 * BN + 8 * stage;
                                const uint32_t sf_s = smem0 + stage * C_::kStageBytes + C_::kABytes + C_::kBBytes;
                                if (!(p.debug & 8192)) {     // diagnostics (bit 13): stale TMEM scales
                                    ptx::tmem_cp_32x128b_x4<CG>(sf_t, ptx::smem_desc(sf_s, 0, 128, 0));
                                    ptx::tmem_cp_32x128b_x4<CG>(sf_t + 4, ptx::smem_desc(sf_s + 512, 0, 128, 0));
                                }
#pragma unroll
                                for (int ks = 0; ks < 4; ++ks) {
                                    const uint32_t accum = (kb | ks) ? 1u : 0u;
                                    ptx::mma_mxf8_ss<CG>(d_tmem, ad + 2 * ks, bd + b_step * ks,
                                                         ptx::idesc_sf_ids(idesc, ks, ks), sf_t, sf_t + 4, accum);
                                }
                            } else if (tf32) {
#pragma unroll
                                for (int ks = 0; ks < 4; ++ks) {
                                    const uint32_t accum = (kb | ks) ? 1u : 0u;
                                    if constexpr (CG == 1)
                                        ptx::mma_tf32_ss(d_tmem, ad + 2 * ks, bd + b_step * ks, idesc, accum);
                                    else
                                        ptx::mma_tf32_ss_cg2(d_tmem, ad + 2 * ks, bd + b_step * ks, idesc, accum);
                                }
                            } else {
#pragma unroll
                                for (int ks = 0; ks < 4; ++ks) {
                                    const uint32_t accum = (kb | ks) ? 1u : 0u;
                                    if constexpr (CG == 1)
                                        ptx::mma_f16_ss(d_tmem, ad + 2 * ks, bd + b_step * ks, idesc, accum);
                                    else
                                        ptx::mma_f16_ss_cg2(d_tmem, ad + 2 * ks, bd + b_step * ks, idesc, accum);
                                }
                            }
                            // smem slot free (in both CTAs) once these MMAs completed
                            if constexpr (CG == 1) ptx::mma_commit(&empty_bar[stage]);
                            else ptx::mma_commit_cg2_mc(&empty_bar[stage], 0x3);
                        }
                        __syncwarp();
                        if (++stage == kStages) { stage = 0; phase ^= 1; }
                    }
                    // accumulator ready (in both CTAs)
                    if (ptx::elect_one()) {
                        if constexpr (CG == 1) ptx::mma_commit(&tfull_bar[acc]);
                        else ptx::mma_commit_cg2_mc(&tfull_bar[acc], 0x3);
                    }
                    __syncwarp();
                    if (p.tl && lane == 0 && tli < kTlMax) p.tl[((size_t)blockIdx.x * kTlMax + tli) * 4 + 1] = gtimer();
                    ++tli;
                    if (++acc == 2) { acc = 0; acc_phase ^= 1; }
                }
            }
            if (p.stats && lane == 0) {
                p.stats[blockIdx.x * kStatsPerCta + 1] = w_tempty;
                p.stats[blockIdx.x * kStatsPerCta + 2] = w_full;
                p.stats[blockIdx.x * kStatsPerCta + 3] = (unsigned long long)(clock64() - t_start);
                for (int b = 0; b < 8; ++b) p.stats[blockIdx.x * kStatsPerCta + 8 + b] = w_kb[b];
            }
        }
    } else if (warp < kEpiWarp0) {
        ptx::setmaxnreg_dec<kRegLo>();   // allocator / idle warps
        if constexpr (PF && CG == 2) {
            // ================================ Combine A (PF): warps 2-3 of both CTAs
            // At_r tile = s0 * A_blk0 + s1 * A_blk1 in fp32, one RN rounding to
            // the 16-bit type, written over the A slot (both source tiles carry
            // the same 128B swizzle, so the sum is element-wise on raw bytes)
            const int ct = (warp - 2) * 32 + lane;            // 0..63
            const uint32_t full_leader0 = ptx::mapa_shared(ptx::smem_u32(&full_bar[0]), 0);
            const bool bf16 = ((p.idesc >> 7) & 7u) == 1u;   // kind::f16 a_format: 1 = bf16, 0 = fp16
            int stage = 0;
            uint32_t phase = 0;
            UnitIter<false> it(p, w, 0u, SR_LOCAL, CG);
            Unit u;
            while (it.next(u)) {
                for (int t = u.r0; t < u.r1; ++t) {
                    const int r = product_at(p, u, t);
                    const float s0 = (float)p.pf_s0[r], s1 = (float)p.pf_s1[r];
                    const bool two = p.pf_blk1[r] >= 0;
                    const float t0 = PF == 2 ? (float)p.pfb_s0[r] : 1.f, t1 = PF == 2 ? (float)p.pfb_s1[r] : 0.f;
                    const bool twob = PF == 2 && p.pfb_blk1[r] >= 0;
                    for (int kb = 0; kb < p.nK; ++kb) {
                        ptx::mbar_wait(&ld_bar[stage], phase);
                        uint8_t* sa = smem + stage * C_::kStageBytes;
                        bool wrote = false;
                        // A: slot = s0 * slot + s1 * staging; B (PF 2): the same on the B slot
                        for (int op = 0; op < (PF == 2 ? 2 : 1); ++op) {
                            const bool pair = op == 0 ? two : twob;
                            const float w0 = op == 0 ? s0 : t0, w1 = op == 0 ? s1 : t1;
                            if (!pair && w0 > 0.f) continue;
                            uint8_t* dst = op == 0 ? sa : sa + C_::kABytes;
                            const uint8_t* sx = op == 0 ? sa + C_::kABytes + C_::kBBytes
                                                        : sa + 2 * C_::kABytes + C_::kBBytes;
                            const int nq = (op == 0 ? C_::kABytes : C_::kBBytes) / 16;
                            for (int q = ct; q < nq; q += 64) {
                                uint4 a = *reinterpret_cast<const uint4*>(dst + q * 16);
                                uint4 b = pair ? *reinterpret_cast<const uint4*>(sx + q * 16) : make_uint4(0, 0, 0, 0);
                                uint32_t* pa = reinterpret_cast<uint32_t*>(&a);
                                const uint32_t* pb = reinterpret_cast<const uint32_t*>(&b);
#pragma unroll
                                for (int h = 0; h < 4; ++h) {
                                    float2 fa, fb;
                                    if (bf16) {
                                        fa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pa[h]));
                                        fb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pb[h]));
                                        __nv_bfloat162 o = __floats2bfloat162_rn(w0 * fa.x + w1 * fb.x, w0 * fa.y + w1 * fb.y);
                                        pa[h] = *reinterpret_cast<uint32_t*>(&o);
                                    } else {
                                        fa = __half22float2(*reinterpret_cast<const __half2*>(&pa[h]));
                                        fb = __half22float2(*reinterpret_cast<const __half2*>(&pb[h]));
                                        __half2 o = __floats2half2_rn(w0 * fa.x + w1 * fb.x, w0 * fa.y + w1 * fb.y);
                                        pa[h] = *reinterpret_cast<uint32_t*>(&o);
                                    }
                                }
                                *reinterpret_cast<uint4*>(dst + q * 16) = a;
                            }
                            wrote = true;
                        }
                        // generic-proxy writes -> visible to the tensor core (async proxy)
                        if (wrote) ptx::fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive_cluster(full_leader0 + stage * 8);
                        if (++stage == kStages) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else {
        // ================================ epilogue (both CTAs: own 128 rows)
        ptx::setmaxnreg_inc<kRegHi>();
        const int ew = warp - kEpiWarp0;           // 0..7
        const int quarter = warp & 3;              // TMEM lane quarter
        const int half = ew >> 2;                  // column half
        const int row = quarter * 32 + lane;       // row of this CTA's 128-row slab
        const int mn = p.m * p.n;
        const uint64_t pol = ptx::policy_evict_last();
        unsigned long long w_tfull = 0;
        const long long t_epi0 = clock64();
        const uint32_t tempty_leader0 =
            CG == 2 ? ptx::mapa_shared(ptx::smem_u32(&tempty_bar[0]), 0) : 0u;
        int acc = 0;
        uint32_t acc_phase = 0;
        // HOME_REG partial: (row, this thread's column half); one dummy
        // register when the instantiation has no register home (REGH false:
        // classical and unfused GEMMs keep the register budget)
        constexpr int kPregCols = REGH ? BN / 2 : 1;
        float preg[kPregCols];
        const uint32_t cst = ptx::smem_u32(cstage) + ew * 2 * 2048;   // this warp's two C staging boxes
        int cbuf = 0;
        int tl_i = 0;             // timeline product index (diagnostics)
        // the static tail's merges, after the segment: wait for the group's
        // other units, merge this unit's share of the (C_ij, 16-column slice)
        // items in segment order, store C, count the read flags down
        auto merge_split = [&](const int g_m, const int seg_m) {
            int x, z;
            group_xz(p, g_m, x, z);
            const long long radd = p.nbatch > 1 ? (long long)(g_m / p.Gb) * p.M : 0;
            const long long brow = (long long)x * C_::kTileM + (long long)rank * kBM + row;
            const long long Tb = (long long)(g_m - p.n_whole) * p.R;      // tail-local first tile
            const int s0 = (int)(Tb / p.tail_c), s1 = (int)((Tb + p.R - 1) / p.tail_c);
            const int nseg = s1 - s0 + 1;
            const int me = seg_m - s0;
            auto fidx = [&](int v) { return (v == s0 ? (int)gridDim.x : 0) + v * CG + (int)rank; };
            if (ew == 0 && lane == 0) {
                for (int v = s0; v <= s1; ++v) {
                    if (v == seg_m) continue;
                    int f = 0;
                    do {
                        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(p.flags + fidx(v)) : "memory");
                    } while (f <= 0);
                }
            }
            asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
            constexpr int kSl = (BN / 2) / 16;                              // 16-column slices per thread
            for (int ij = 0; ij < mn; ++ij) {
                const int i = ij / p.n, j = ij - (ij / p.n) * p.n;
                for (int ch = 0; ch < kSl; ++ch) {
                    if ((ij * kSl + ch) % nseg != me) continue;
                    const int col0 = half * (BN / 2) + ch * 16;
                    float v[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) v[e] = 0.f;
                    int vs = s0;
                    for (;;) {
                        // next batch of up to 4 units that touch C_ij, in order
                        int src[4];
                        int ns = 0;
                        for (; vs <= s1 && ns < 4; ++vs) {
                            const long long lo_t = (long long)vs * p.tail_c > Tb ? (long long)vs * p.tail_c : Tb;
                            const long long hi_t = (long long)(vs + 1) * p.tail_c < Tb + p.R ? (long long)(vs + 1) * p.tail_c
                                                                                            : Tb + p.R;
                            bool touch = false;
                            for (long long t = lo_t; t < hi_t && !touch; ++t)
                                touch = p.Wc[p.rperm[(int)(t - Tb)] * mn + ij] != 0;
                            if (touch) src[ns++] = (vs == s0 ? 0 : (int)gridDim.x) + vs * CG + (int)rank;
                        }
                        if (ns == 0) break;
                        float4 o[4][4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const float* pt = partial_tile<BN>(p, q < ns ? src[q] : src[0], ij, false);
#pragma unroll
                            for (int e = 0; e < 4; ++e) o[q][e] = ld_cg_f4(pt + partial_off(row, (col0 >> 2) + e));
                        }
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            if (q < ns) {
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    v[4 * e] += o[q][e].x; v[4 * e + 1] += o[q][e].y;
                                    v[4 * e + 2] += o[q][e].z; v[4 * e + 3] += o[q][e].w;
                                }
                            }
                        }
                        if (ns < 4) break;
                    }
                    const long long ccol = (long long)j * p.Nb + (long long)z * BN + col0;
                    if (brow < p.Mb && ccol < (long long)(j + 1) * p.Nb)
                        store_c_row16(p, (long long)i * p.Mb + brow, ccol, v, radd);
                }
            }
            asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
            if (ew == 0 && lane == 0)
                for (int v = s0; v <= s1; ++v)
                    if (v != seg_m) atomicSub(p.flags + fidx(v), 1);
        };
        int pend_g[2] = {-1, -1};
        int npend = 0;
        UnitIter<DYN> it(p, w, ring, leader ? SR_LOCAL : SR_PEER, CG);
        Unit u;
        while (it.next(u)) {
            int x, z;
            group_xz(p, u.g, x, z);
            const long long radd = p.nbatch > 1 ? (long long)(u.g / p.Gb) * p.M : 0;   // batch's C rows
            // rows of this CTA inside the block grid
            const long long brow = (long long)x * C_::kTileM + (long long)rank * kBM + row;
            // C_ij already touched inside this unit (bit ij): first contribution test
            uint32_t seen = 0;
            // split segments: a contributor's partials live in its segment's slot
            // (the owner reads them after this pair may have moved on)
            const int slot = (u.role == ROLE_CONTRIB) ? (int)gridDim.x + u.seg * CG + (int)rank : (int)blockIdx.x;
            const bool whole = u.role == ROLE_WHOLE;
            for (int t = u.r0; t < u.r1; ++t) {
                const int r = product_at(p, u, t);
                // C_ij that later products of this unit still update
                uint32_t later = 0;
                for (int t2 = t + 1; t2 < u.r1; ++t2) later |= p.nzmask[product_at(p, u, t2)];
                if (p.debug & 8) ptx::mbar_wait_sleep(&tfull_bar[acc], acc_phase, 256);
                else timed_wait(&tfull_bar[acc], acc_phase, (p.stats && ew == 0 && lane == 0) ? &w_tfull : nullptr);
                ptx::tc_fence_after();
                if (p.tl && ew == 0 && lane == 0 && tl_i < kTlMax) p.tl[((size_t)blockIdx.x * kTlMax + tl_i) * 4 + 2] = gtimer();
                const uint32_t t_addr = tmem_base + ((uint32_t)(quarter * 32) << 16) +
                                        (uint32_t)(acc * BN + half * (BN / 2));
                const uint32_t nz = p.nzmask[r];
                // destinations whose last contribution this is come first: a
                // home they free may be taken by a first contribution of the
                // same product (each thread touches only its own elements)
                const uint32_t fin = whole ? (nz & ~later) : 0u;
                const int col_base = half * (BN / 2);
                // first C row of this warp's 32-row box (TMA-store path)
                // the accumulator is consumed in chunks of 32 columns; it is
                // released to the MMA warp right after the last chunk's load.
                // The chunk index is a template constant so that the register
                // partial preg is indexed statically (stays in registers).
                auto chunk = [=, &preg, &p, &cbuf](auto ch_c) {
                    // 16-bit C through shared memory and a TMA store: this lane's 16
                    // values at column half hh of the warp's current 32 x 32 box
                    auto c_stage16 = [&](int hh, const float* v) {
                        if (p.c_tma == 2) {   // fp32 C: one 4 KB box (128-byte rows)
                            const uint32_t dst = cst + lane * 128 + hh * 64;
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                ptx::st_shared_v4(dst + 16 * q, __float_as_uint(v[4 * q]), __float_as_uint(v[4 * q + 1]),
                                                  __float_as_uint(v[4 * q + 2]), __float_as_uint(v[4 * q + 3]));
                            return;
                        }
                        uint32_t wv[8];
#pragma unroll
                        for (int h = 0; h < 8; ++h) wv[h] = pack2(p, v[2 * h], v[2 * h + 1]);
                        const uint32_t dst = cst + cbuf * 2048 + lane * 64 + hh * 32;
                        ptx::st_shared_v4(dst, wv[0], wv[1], wv[2], wv[3]);
                        ptx::st_shared_v4(dst + 16, wv[4], wv[5], wv[6], wv[7]);
                    };
                    // the warp's box is complete: one bulk store (rows >= M, columns
                    // >= N clipped by the map), then the other box; it is reused once
                    // the store issued before this one has read it
                    auto c_flush = [&](int i_blk, long long ccol) {
                        ptx::fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            const int brow0 = x * C_::kTileM + (int)rank * kBM + quarter * 32;
                            if (p.c_cs && p.c_tma != 2)   // C is never re-read here: evict-first in L2
                                ptx::tma_store_2d_hint(&p.c_map, cst + cbuf * 2048, (int)ccol,
                                                       (int)((long long)i_blk * p.Mb + brow0 + radd),
                                                       ptx::policy_evict_first());
                            else
                                ptx::tma_store_2d(&p.c_map, cst + cbuf * 2048, (int)ccol,
                                                  (int)((long long)i_blk * p.Mb + brow0 + radd));
                            ptx::bulk_commit_group();
                            // 16-bit: two boxes, the older store must have read its box;
                            // fp32: one box, this store must have read it
                            if (p.c_tma == 2) ptx::bulk_wait_group_read<0>();
                            else ptx::bulk_wait_group_read<1>();
                        }
                        if (p.c_tma != 2) cbuf ^= 1;
                        __syncwarp();
                    };
                    constexpr int ch = decltype(ch_c)::value;
                    uint32_t raw[32];
                    if (!(p.debug & 2)) {
                        ptx::tmem_ld_32x32b_x32(t_addr + ch * 32, raw);
                        ptx::tmem_wait_ld();
                    } else {
#pragma unroll
                        for (int e = 0; e < 32; ++e) raw[e] = 0u;
                    }
                    if (ch == (BN / 2) / 32 - 1) {
                        // relaxed: the arrival must not wait for this product's
                        // earlier C / partial stores to complete
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) {
                            if constexpr (CG == 1) ptx::mbar_arrive_relaxed(&tempty_bar[acc]);
                            else ptx::mbar_arrive_cluster_relaxed(tempty_leader0 + acc * 8);
                        }
                        if (p.tl && ew == 4 && lane == 0 && tl_i < kTlMax) p.tl[((size_t)blockIdx.x * kTlMax + tl_i) * 4 + 3] = gtimer();
                    }
                    if (p.debug & 1) return;
                    const int c4 = (col_base + ch * 32) >> 2;     // first float4 column of the chunk
                    if (p.epi_mode == EPI_STORE_H) {
                        // Algorithm 1 stage 3: H_r to main memory
                        float* dst = p.H + ((long long)r * p.Mb + brow) * p.Nb + (long long)z * BN + col_base + ch * 32;
#pragma unroll
                        for (int e = 0; e < 32; e += 4)
                            st_cg_f4(dst + e, make_float4(__uint_as_float(raw[e]), __uint_as_float(raw[e + 1]),
                                                          __uint_as_float(raw[e + 2]), __uint_as_float(raw[e + 3])));
                        return;
                    }
                    // Combine H (Eq. 6): C_ij += W[r,i,j] * H_r for every nonzero W
                    for (int pass = 0; pass < 2; ++pass) {
                        uint32_t todo = pass == 0 ? fin : (nz & ~fin);
                        while (todo) {
                            const int ij = __ffs(todo) - 1;
                            todo &= todo - 1;
                            const float sw = (float)p.Wc[r * mn + ij];
                            const bool first = !((seen >> ij) & 1u);
                            const bool final_here = pass == 0;
                            int home = whole ? (int)p.home[ij] : 0;
                            if (QF == 0 && home == HOME_SMEM && half == 1) home = p.qslot;
                            const int i = ij / p.n, j = ij - (ij / p.n) * p.n;
                            const long long ccol = (long long)j * p.Nb + (long long)z * BN + col_base + ch * 32;
                            const bool in_range = brow < p.Mb && ccol < (long long)(j + 1) * p.Nb;
                            if (!REGH && home == HOME_REG) home = 0;   // (the host never assigns it here)
                            if (REGH && whole && home == HOME_REG) {
                                if (p.debug & 1024) continue;
                                float* pr = &preg[(ch * 32) % kPregCols];
                                if (final_here) {
                                    // the partial dies here: finish C in place (no extra
                                    // 32-register buffer; a first contribution of this
                                    // product into the same home comes after)
#pragma unroll
                                    for (int e = 0; e < 32; ++e)
                                        pr[e] = (first ? 0.f : pr[e]) + sw * __uint_as_float(raw[e]);
                                    if (in_range && !(p.debug & 128)) {
                                        if (p.c_tma) {
                                            c_stage16(0, pr);
                                            c_stage16(1, pr + 16);
                                            c_flush(i, ccol);
                                        } else {
                                            store_c_row16(p, (long long)i * p.Mb + brow, ccol, pr, radd);
                                            store_c_row16(p, (long long)i * p.Mb + brow, ccol + 16, pr + 16, radd);
                                        }
                                    }
                                } else if (first) {
#pragma unroll
                                    for (int e = 0; e < 32; ++e) pr[e] = sw * __uint_as_float(raw[e]);
                                } else {
#pragma unroll
                                    for (int e = 0; e < 32; ++e) pr[e] += sw * __uint_as_float(raw[e]);
                                }
                            } else if (whole && home == HOME_SMEM) {
                                if (p.debug & 512) continue;
                                // this thread alone owns (row, its column half) of the
                                // shared partial: plain loads / stores in program order
                                float* sp = psmem;
                                if (final_here) {
#pragma unroll
                                    for (int hh = 0; hh < 32; hh += 16) {
                                        float v[16];
#pragma unroll
                                        for (int e = 0; e < 16; e += 4) {
                                            float4 o = first ? make_float4(0.f, 0.f, 0.f, 0.f)
                                                             : *reinterpret_cast<const float4*>(sp + partial_off(row, c4 + ((hh + e) >> 2)));
                                            v[e] = o.x + sw * __uint_as_float(raw[hh + e]);
                                            v[e + 1] = o.y + sw * __uint_as_float(raw[hh + e + 1]);
                                            v[e + 2] = o.z + sw * __uint_as_float(raw[hh + e + 2]);
                                            v[e + 3] = o.w + sw * __uint_as_float(raw[hh + e + 3]);
                                        }
                                        if (in_range && !(p.debug & 128)) {
                                            if (p.c_tma) c_stage16(hh >> 4, v);
                                            else store_c_row16(p, (long long)i * p.Mb + brow, ccol + hh, v, radd);
                                        }
                                    }
                                    if (p.c_tma && in_range && !(p.debug & 128)) c_flush(i, ccol);
                                } else {
#pragma unroll
                                    for (int e = 0; e < 32; e += 4) {
                                        float4* q = reinterpret_cast<float4*>(sp + partial_off(row, c4 + (e >> 2)));
                                        float4 o = first ? make_float4(0.f, 0.f, 0.f, 0.f) : *q;
                                        o.x += sw * __uint_as_float(raw[e]);
                                        o.y += sw * __uint_as_float(raw[e + 1]);
                                        o.z += sw * __uint_as_float(raw[e + 2]);
                                        o.w += sw * __uint_as_float(raw[e + 3]);
                                        *q = o;
                                    }
                                }
                            } else if (!(p.debug & 256)) {
                                // L2 workspace slot
                                float* pt = whole ? partial_tile<BN>(p, slot, home, true)
                                                  : partial_tile<BN>(p, slot, ij, false);
                                if (final_here) {
                                    // last contribution: C_ij = partial + w*H_r, rounded once,
                                    // in two 16-column halves (4 partial loads issued together;
                                    // only 16 temporaries live next to the register partial)
#pragma unroll
                                    for (int hh = 0; hh < 32; hh += 16) {
                                        float v[16];
#pragma unroll
                                        for (int e = 0; e < 16; ++e) v[e] = sw * __uint_as_float(raw[hh + e]);
                                        if (!first) {
                                            float4 o[4];
#pragma unroll
                                            for (int q = 0; q < 4; ++q) o[q] = ld_cg_f4(pt + partial_off(row, c4 + (hh >> 2) + q));
#pragma unroll
                                            for (int q = 0; q < 4; ++q) {
                                                v[4 * q] += o[q].x; v[4 * q + 1] += o[q].y;
                                                v[4 * q + 2] += o[q].z; v[4 * q + 3] += o[q].w;
                                            }
                                        }
                                        if (in_range && !(p.debug & 128)) {
                                            if (p.c_tma) c_stage16(hh >> 4, v);
                                            else store_c_row16(p, (long long)i * p.Mb + brow, ccol + hh, v, radd);
                                        }
                                    }
                                    if (p.c_tma && in_range && !(p.debug & 128)) c_flush(i, ccol);
                                    if (!first && p.discard) {
                                        __syncwarp();      // the 8 lanes sharing a line have read it
                                        if ((row & 7) == 0) discard_lines(pt, row, c4, 8);
                                        // a discard is a weak write of the whole line: order it
                                        // before any lane's next store to the same home (a first
                                        // contribution of this product may take it over)
                                        __syncwarp();
                                    }
                                } else if (first) {
#pragma unroll
                                    for (int e = 0; e < 32; e += 4) {
                                        const float4 hv = make_float4(sw * __uint_as_float(raw[e]), sw * __uint_as_float(raw[e + 1]),
                                                                      sw * __uint_as_float(raw[e + 2]), sw * __uint_as_float(raw[e + 3]));
                                        if (p.partial_hint) st_pol_f4(pt + partial_off(row, c4 + (e >> 2)), hv, pol);
                                        else st_cg_f4(pt + partial_off(row, c4 + (e >> 2)), hv);
                                    }
                                } else {
                                    // middle contribution: fire-and-forget L2 reduction (same
                                    // thread, same address => applied in program order)
#pragma unroll
                                    for (int e = 0; e < 32; e += 4) {
                                        float* a = pt + partial_off(row, c4 + (e >> 2));
                                        if (p.partial_hint)
                                            red_add_pol_f4(a, sw * __uint_as_float(raw[e]), sw * __uint_as_float(raw[e + 1]),
                                                           sw * __uint_as_float(raw[e + 2]), sw * __uint_as_float(raw[e + 3]), pol);
                                        else
                                            red_add_f4(a, sw * __uint_as_float(raw[e]), sw * __uint_as_float(raw[e + 1]),
                                                       sw * __uint_as_float(raw[e + 2]), sw * __uint_as_float(raw[e + 3]));
                                    }
                                }
                            }
                        }
                    }
                    if (p.pace_ns) __nanosleep(p.pace_ns);   // spread the epilogue's L2 traffic
                };
                static_assert((BN / 2) / 32 == 4 || (BN / 2) / 32 == 2, "chunks per column half");
                chunk(std::integral_constant<int, 0>{});
                chunk(std::integral_constant<int, 1>{});
                if constexpr ((BN / 2) / 32 == 4) {
                    chunk(std::integral_constant<int, 2>{});
                    chunk(std::integral_constant<int, 3>{});
                }
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
                ++tl_i;
                seen |= nz;
            }
            if (p.epi_mode != EPI_FUSED || u.role == ROLE_WHOLE || (p.debug & 1)) continue;

            if (!DYN || !p.dyn_tail) {
                // ---- split group, static tail (segment v runs on pair v): every
                // unit of a split group publishes its partials right after its
                // products (no wait here: a wait inside the segment would chain
                // the pairs), the merges run once the whole segment is done
                // (merge_split below).  Flags count down: a unit sets nseg - 1,
                // every reader decrements once after its reads, so they are zero
                // again at the end of the launch.  flags: [0, ctas) contributor
                // units, [ctas, 2 ctas) owner units.
                const long long Tb = (long long)(u.g - p.n_whole) * p.R;
                const int s0 = (int)(Tb / p.tail_c), s1 = (int)((Tb + p.R - 1) / p.tail_c);
                __threadfence();
                asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
                if (ew == 0 && lane == 0)
                    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p.flags + (u.seg == s0 ? (int)gridDim.x : 0) +
                                                                             u.seg * CG + (int)rank),
                                 "r"(s1 - s0) : "memory");
                if (npend < 2) pend_g[npend++] = u.g;
                continue;
            }

            // ---- split group: publish (contributor) or merge (owner)
            if (u.role == ROLE_CONTRIB) {
                __threadfence();
                asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
                if (ew == 0 && lane == 0) {
                    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p.flags + u.seg * CG + (int)rank), "r"(1)
                                 : "memory");
                }
                continue;
            }
            // owner: the other segments of the group are segments seg+1 .. last
            // (same rank); static tail: segment == work unit
            const long long Tt_base = (long long)(u.g - p.n_whole) * p.R;   // tail-local first tile
            const int last_w = (int)((Tt_base + p.R - 1) / p.tail_c);
            if (ew == 0 && lane == 0) {
                for (int v = u.seg + 1; v <= last_w; ++v) {
                    int f = 0;
                    do {
                        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(p.flags + v * CG + rank)
                                     : "memory");
                    } while (f == 0);
                }
            }
            asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
            // merge: C_ij = own partial + the contributing segments' partials in
            // unit order (fixed: bitwise deterministic).  The source tiles of a
            // 16-column slice are loaded in batches of 4 before any add, so one
            // L2 round trip serves up to four partials (the tail used to
            // serialise ~100 dependent round trips per thread)
            for (int ij = 0; ij < mn; ++ij) {
                const int i = ij / p.n, j = ij - (ij / p.n) * p.n;
                // sources in merge order: own (if this segment touched C_ij), then
                // units w+1 .. last_w whose positions contribute to C_ij (bit d of
                // cm[] = unit w+1+d; last_w - w < R <= kMaxR = 128)
                uint64_t cm[2] = {0ull, 0ull};
                for (int vw = u.seg + 1; vw <= last_w; ++vw) {
                    int lo = (int)((long long)vw * p.tail_c - Tt_base);
                    int hi = lo + p.tail_c;
                    if (lo < 0) lo = 0;
                    if (hi > p.R) hi = p.R;
                    bool contributes = false;
                    for (int t = lo; t < hi; ++t)
                        if (p.Wc[p.rperm[t] * mn + ij]) { contributes = true; break; }
                    const int d = vw - u.seg - 1;
                    if (contributes) cm[d >> 6] |= 1ull << (d & 63);
                }
                const bool own = (seen >> ij) & 1u;
#pragma unroll 1
                for (int ch = 0; ch < (BN / 2) / 16; ++ch) {
                    const int col0 = half * (BN / 2) + ch * 16;
                    float v[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) v[e] = 0.f;
                    uint64_t m0 = cm[0], m1 = cm[1];
                    bool take_own = own;
                    for (;;) {
                        // next batch of up to 4 source slots, in merge order
                        int src[4];
                        int ns = 0;
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            int sl = -1;
                            if (take_own) {
                                sl = (int)blockIdx.x;
                                take_own = false;
                            } else if (m0 | m1) {
                                const int d = m0 ? __ffsll((long long)m0) - 1 : 64 + __ffsll((long long)m1) - 1;
                                if (d < 64) m0 &= m0 - 1; else m1 &= m1 - 1;
                                sl = (int)gridDim.x + (u.seg + 1 + d) * CG + (int)rank;
                            }
                            src[q] = sl;
                            ns += sl >= 0;
                        }
                        if (ns == 0) break;
                        float4 o[4][4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            // (a valid address for every q: empty entries re-read the
                            // first source and are discarded)
                            const float* pt = partial_tile<BN>(p, src[q] >= 0 ? src[q] : src[0], ij, false);
#pragma unroll
                            for (int e = 0; e < 4; ++e) o[q][e] = ld_cg_f4(pt + partial_off(row, (col0 >> 2) + e));
                        }
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            if (src[q] >= 0) {
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    v[4 * e] += o[q][e].x; v[4 * e + 1] += o[q][e].y;
                                    v[4 * e + 2] += o[q][e].z; v[4 * e + 3] += o[q][e].w;
                                }
                            }
                        }
                        if (ns < 4) break;
                    }
                    const long long ccol = (long long)j * p.Nb + (long long)z * BN + col0;
                    if (brow < p.Mb && ccol < (long long)(j + 1) * p.Nb)
                        store_c_row16(p, (long long)i * p.Mb + brow, ccol, v, radd);
                }
            }
            // all reads done -> reset the flags for the next launch
            asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
            if (ew == 0 && lane == 0)
                for (int v = u.seg + 1; v <= last_w; ++v) p.flags[v * CG + rank] = 0;
        }
        if (!DYN || !p.dyn_tail) {
            // static tail: the segment's split units are merged after all of them
            // published (segment v = unit v, the pair's last work)
            for (int q = 0; q < npend; ++q) merge_split(pend_g[q], w);
        }
        if (p.stats && ew == 0 && lane == 0) {
            p.stats[blockIdx.x * kStatsPerCta + 4] = w_tfull;
            (void)t_epi0;
        }
        if (p.c_tma && lane == 0) ptx::bulk_wait_group_all();   // staging stays valid until read
    }

    ptx::tc_fence_before();
    if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
    if (p.drift > 0 && p.sched && threadIdx.x == 0) {
        // the last CTA out resets the progress counter for the next launch
        // (every producer of the grid has finished by then)
        if (atomicAdd(p.sched + 3, 1) == (int)gridDim.x - 1) {
            atomicExch(p.sched + 2, 0);
            atomicExch(p.sched + 3, 0);
        }
    }
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<CG>(tmem_base, 512);
    }
    if (p.stats && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.stats[blockIdx.x * kStatsPerCta + 7] = t;
        p.stats[blockIdx.x * kStatsPerCta + 5] = (unsigned long long)(clock64() - clk_entry);
    }
}

}  // namespace lcma
