// lcma_api.cu -- C ABI of liblcma.so (see include/lcma.h): plan creation
// (Decision Module, block extents, split-group schedule, workspace layout),
// TMA descriptor encoding and kernel launches.  No CPU fallback: every step
// of C = A*B runs in the kernels of umma_gemm.cuh / combine.cuh.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <mutex>
#include <sstream>
#include <string>

#include "../../include/lcma.h"
#include "combine.cuh"
#include "decision.h"
#include "diag.h"
#include "schemes.h"
#include "umma_gemm.cuh"

using namespace lcma;

namespace {

thread_local std::string t_err;
thread_local int t_launches = 0;
// optional CUDA events recorded around the tcgen05 GEMM launch (lcma_set_kernel_events)
thread_local cudaEvent_t t_ev_start = nullptr, t_ev_end = nullptr;

lcma_status fail(lcma_status st, const std::string& msg) {
    t_err = msg;
    return st;
}

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

int64_t roundup(int64_t a, int64_t b) { return cdiv(a, b) * b; }
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// input element bytes (FP8 plans take bf16 A and B and quantize them)
int elem_bytes(lcma_dtype d) { return (d == LCMA_BF16 || d == LCMA_FP16 || d == LCMA_FP8_E4M3) ? 2 : 4; }
// FP8 operand bytes of the quantized A~ / B~ (E4M3) and their UE8M0 scale
// chunks: 4 bytes per operand row and 128-element k-block (512-byte chunks)
size_t fp8_operand_bytes(int64_t R, int64_t rows, int64_t Kb) {
    return (size_t)R * rows * Kb + (size_t)R * rows * (Kb / 128) * 4;
}

int device_sm_count() {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return 148; }
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) {
        cudaGetLastError();
        return 148;
    }
    return sms;
}

constexpr int kMaxDev = 64;
// register-home fused kernel: products of at most this many k-blocks take the
// C-staging (TMA store) instantiation
constexpr int kCstMaxNK = 48;
int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return -1; }
    return (dev >= 0 && dev < kMaxDev) ? dev : -1;
}

// Co-resident clusters of 2 for umma_gemm_kernel<2> on the current device
// (0 if unknown / no GPU).
int max_active_pairs() {
    static int cached[kMaxDev];
    static std::once_flag once[kMaxDev];
    const int dv = current_device();
    if (dv < 0) return 0;
    std::call_once(once[dv], [dv] {
        int& c = cached[dv];
        c = 0;
        if (cudaFuncSetAttribute(umma_gemm_kernel<2, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Cfg<2, 256, 0, true>::kSmemBytes) != cudaSuccess) { cudaGetLastError(); return; }
        cudaLaunchConfig_t cfg;
        std::memset(&cfg, 0, sizeof(cfg));
        cfg.gridDim = dim3(2);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = Cfg<2, 256, 0, true>::kSmemBytes;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, umma_gemm_kernel<2, 256>, &cfg) == cudaSuccess) c = n;
        else cudaGetLastError();
    });
    return cached[dv];
}

}  // namespace

struct lcma_plan_s {
    lcma_plan_desc d;
    Profile hw;
    int scheme_id;
    Scheme sch;
    lcma_algo algo;
    int variant;
    int64_t Mb, Nb, Kb;
    int BK, e;
    int oe = 0;                    // operand element bytes in the GEMM (FP8: 1)
    int nX, nZ, G, nK;
    int ctas, cg, bn, q, tail_c, swz;
    int n_whole, dyn, dyn_tail;
    int nbatch = 1;                // batched inner GEMMs of a two-level plan (groups = nbatch x nX x nZ)
    size_t off_sched, off_P, off_flags, off_At, off_Bt, off_H, ws_bytes, bt_bytes;
    size_t off_inner = 0;          // two-level: the inner plan's partial slots + flags
    int8_t a_dir[kMaxR], b_dir[kMaxR];   // single-term operands read in place (-1: materialised)
    bool any_a_dir = false, any_b_dir = false;
    lcma_plan_s* inner = nullptr;  // two-level: fused GEMM plan of the base scheme
    lcma_plan_info info;
    ~lcma_plan_s() { delete inner; }
};

// ---------------------------------------------------------------- schedule
namespace {

struct HostUnit { int g, r0, r1, role; };

// Mirror of the device UnitIter (umma_gemm.cuh).
std::vector<HostUnit> host_units(const lcma_plan_s* p, int w) {
    std::vector<HostUnit> out;
    const int R = p->sch.R;
    const int W = p->ctas / p->cg;
    // (dynamic schedules hand the n_whole whole groups out at run time; the
    // static view below assigns them round by round)
    for (int i = 0; i * W + w < p->n_whole; ++i) out.push_back({i * W + w, 0, R, ROLE_WHOLE});
    const long long Tt = std::max<long long>(0, (long long)(p->G - (long long)p->n_whole) * R);
    long long t = std::min<long long>((long long)w * p->tail_c, Tt);
    long long t_end = std::min<long long>(t + p->tail_c, Tt);
    while (t < t_end) {
        long long gl = t / R;
        int r0 = (int)(t - gl * R);
        long long stop = std::min<long long>((gl + 1) * R, t_end);
        int r1 = (int)(stop - gl * R);
        int role = (r0 == 0 && r1 == R) ? ROLE_WHOLE : (r0 == 0 ? ROLE_OWNER : ROLE_CONTRIB);
        out.push_back({p->n_whole + (int)gl, r0, r1, role});
        t = stop;
    }
    return out;
}

void make_schedule(lcma_plan_s* p, int mode) {
    const int R = p->sch.R;
    const int W = p->ctas / p->cg;
    p->dyn = 0;
    p->dyn_tail = 0;
    if (mode == 2) {
        p->q = 0;                              // paper: contiguous split-group chunks
    } else if (mode == 3) {
        p->q = (int)cdiv(p->G, W);             // group-parallel only: whole groups, no split
    } else {
        p->q = p->G / W;                       // lockstep rounds (cache-aware)
        // mode 5: the whole groups are handed out at run time in raster order
        // (the pairs of the static assignment drift apart by about one round
        // every 50 rounds, tools/r02/drift.py; the dynamic order keeps the
        // groups in flight a compact window of the raster and halves the DRAM
        // reads at the cfg5 shape, but measured no faster: within +-1 % at
        // cfg2, -8..-16 % (classical) / -2..+9 % (Strassen) at cfg5,
        // profiles/r02_schedule.txt), so the default (1 = 4) stays static
        p->dyn = (mode == 5 || mode == 7) ? 1 : 0;
        // modes 5 and 6: the split tail's segments are handed out at run time
        // to the pairs that finish their whole groups first; mode 7: whole
        // groups at run time, the static tail (segment w on pair w, merged by
        // all of a group's pairs)
        p->dyn_tail = (mode == 5 || mode == 6) ? 1 : 0;
    }
    p->n_whole = (int)std::min<long long>((long long)p->q * W, p->G);
    // R == 1 (classical): nothing to split, every group is handed out whole
    if (p->dyn && R == 1) p->n_whole = p->G;
    const long long Tt = std::max<long long>(0, (long long)(p->G - (long long)p->n_whole) * R);
    p->tail_c = Tt > 0 ? (int)cdiv(Tt, W) : 1;
    // raster band height (tile rows): LCMA rounds touch R operand panels per
    // tile, so a lower band keeps the round's A panels L2-resident (measured
    // cfg2 Strassen -1..2 %, classical best at 16; tools/swz_exp*.sh)
    p->swz = p->d.raster_rows > 0 ? p->d.raster_rows : (R > 1 ? 8 : 16);
    p->info.groups = p->G;
    p->info.tiles = (int)std::min<long long>((long long)p->G * R, INT32_MAX);
    p->info.ctas = p->ctas;
    p->info.waves = (int)(p->dyn ? cdiv(p->n_whole, W) : p->q) * R + (Tt > 0 ? p->tail_c : 0);
    p->info.group_waves = (int)cdiv(p->G, W) * R;
    int splits = 0;
    for (long long gl = 0; gl < p->G - p->n_whole; ++gl) {
        long long a = gl * R, b = gl * R + R - 1;
        if (a / p->tail_c != b / p->tail_c) ++splits;
    }
    p->info.split_groups = splits;
}

}  // namespace

// ---------------------------------------------------------------- planning
extern "C" lcma_status lcma_plan_ex(const lcma_plan_desc* desc, lcma_plan_t* out) {
    t_err.clear();
    if (!desc || !out) return fail(LCMA_ERR_INVALID_VALUE, "null argument");
    *out = nullptr;
    const lcma_plan_desc& d = *desc;
    if (d.M < 1 || d.N < 1 || d.K < 1) return fail(LCMA_ERR_INVALID_VALUE, "M, N, K must be >= 1");
    if (d.dtype < LCMA_BF16 || d.dtype > LCMA_FP8_E4M3) return fail(LCMA_ERR_INVALID_VALUE, "bad dtype");
    const bool fp8 = d.dtype == LCMA_FP8_E4M3;
    lcma_dtype od = d.out_dtype;
    if (fp8) {
        // C of the FP8 path is bf16 (or fp32); B is N x K (K-major E4M3 operand)
        if (od == LCMA_FP8_E4M3) od = LCMA_BF16;
        if (od != LCMA_BF16 && od != LCMA_FP32) return fail(LCMA_ERR_NOT_SUPPORTED, "FP8 output is bf16 or fp32");
        if (d.b_layout != 1) return fail(LCMA_ERR_NOT_SUPPORTED, "FP8 needs B stored N x K (b_layout 1)");
    }
    if (!fp8 && od != d.dtype && od != LCMA_FP32)
        return fail(LCMA_ERR_NOT_SUPPORTED, "out_dtype must equal dtype or be FP32");
    if (d.dtype == LCMA_TF32 && od != LCMA_FP32 && od != LCMA_TF32)
        return fail(LCMA_ERR_NOT_SUPPORTED, "tf32 output is fp32");
    if (d.b_layout != 0 && d.b_layout != 1) return fail(LCMA_ERR_INVALID_VALUE, "b_layout must be 0 or 1");
    if (d.algo < LCMA_ALGO_AUTO || d.algo > LCMA_ALGO_SCHEME) return fail(LCMA_ERR_INVALID_VALUE, "bad algo");
    if (d.variant < 0 || d.variant > 4) return fail(LCMA_ERR_INVALID_VALUE, "bad variant");
    const int e = elem_bytes(d.dtype);
    if ((d.K * e) % 16 != 0 || (d.N * e) % 16 != 0)
        return fail(LCMA_ERR_MISALIGNED, "K and N row lengths must be multiples of 16 bytes (TMA)");

    auto* p = new lcma_plan_s();
    p->d = d;
    p->d.out_dtype = od;
    p->e = e;
    p->oe = fp8 ? 1 : e;
    p->hw = d.hw ? Profile{d.hw->flops_mul, d.hw->flops_add, d.hw->beta_elems}
                 : default_profile((int)d.dtype);
    if (!(p->hw.flops_mul > 0 && p->hw.flops_add > 0 && p->hw.beta > 0)) {
        delete p;
        return fail(LCMA_ERR_INVALID_VALUE, "hardware profile entries must be > 0");
    }
    std::memset(&p->info, 0, sizeof(p->info));

    // ---- Decision Module; reported even when algo is forced
    const bool fused_model = d.variant != LCMA_VARIANT_UNFUSED && d.dtype != LCMA_FP32;
    std::vector<int> cands = {SCHEME_STRASSEN, SCHEME_STRASSEN2, SCHEME_LADERMAN};
    // decision_model 0: this build's calibrated B200 model; 1: the paper's model verbatim
    const bool paper_model = d.decision_model == 1;
    if (!paper_model && !d.hw) {
        if (p->hw.beta_combine <= 0) p->hw.beta_combine = p->hw.beta;
    } else if (!paper_model) {
        Profile def = default_profile((int)d.dtype);
        p->hw.beta_combine = def.beta_combine * (p->hw.beta / def.beta);
        p->hw.alpha_partial = def.alpha_partial;
        p->hw.epi_overhead = def.epi_overhead;
    }
    DecisionResult dec = paper_model
        ? decide(cands, (double)d.M, (double)d.N, (double)d.K, p->hw, fused_model, d.b_static != 0)
        : decide_b200(cands, (double)d.M, (double)d.N, (double)d.K, p->hw, fused_model, d.b_static != 0,
                      (double)e);
    switch (d.algo) {
        case LCMA_ALGO_AUTO: p->scheme_id = dec.scheme_id; break;
        case LCMA_ALGO_CLASSICAL: p->scheme_id = SCHEME_CLASSICAL; break;
        case LCMA_ALGO_STRASSEN: p->scheme_id = SCHEME_STRASSEN; break;
        case LCMA_ALGO_STRASSEN2: p->scheme_id = SCHEME_STRASSEN2; break;
        case LCMA_ALGO_LADERMAN: p->scheme_id = SCHEME_LADERMAN; break;
        case LCMA_ALGO_SCHEME: p->scheme_id = d.scheme_id; break;
    }
    const Scheme* s = scheme_get(p->scheme_id);
    if (!s) {
        delete p;
        return fail(LCMA_ERR_INVALID_VALUE, "unknown scheme id");
    }
    p->sch = *s;
    const bool classical = (p->scheme_id == SCHEME_CLASSICAL);
    p->algo = classical ? LCMA_ALGO_CLASSICAL
                        : (p->scheme_id == SCHEME_STRASSEN ? LCMA_ALGO_STRASSEN
                           : p->scheme_id == SCHEME_STRASSEN2 ? LCMA_ALGO_STRASSEN2
                           : p->scheme_id == SCHEME_LADERMAN ? LCMA_ALGO_LADERMAN
                                                             : LCMA_ALGO_SCHEME);
    // ---- variant
    int variant = d.variant;
    if (classical) variant = 0;
    else if (d.dtype == LCMA_FP32) {
        if (variant == LCMA_VARIANT_AUTO) variant = LCMA_VARIANT_UNFUSED;
        if (variant != LCMA_VARIANT_UNFUSED) {
            delete p;
            return fail(LCMA_ERR_NOT_SUPPORTED, "fp32 (SIMT) LCMA runs the unfused variant only");
        }
    } else if (fp8) {
        // FP8: the quantizing combines + the block-scaled fused-Combine-H GEMM
        if (variant == LCMA_VARIANT_AUTO) variant = LCMA_VARIANT_FUSED_H;
        if (variant != LCMA_VARIANT_FUSED_H) {
            delete p;
            return fail(LCMA_ERR_NOT_SUPPORTED, "FP8 LCMA runs the fused Combine H variant only");
        }
    } else {
        // composed schemes run two-level (measured 1.06-1.34x faster than the
        // flat 49-product fused kernel: its 11 live partials per CTA spill L2)
        if (variant == LCMA_VARIANT_AUTO)
            variant = p->sch.base_id >= 0 ? LCMA_VARIANT_TWO_LEVEL : LCMA_VARIANT_FUSED_H;
        if (variant == LCMA_VARIANT_PRODUCER) {
            // Combine A in the GEMM producer path (two A source blocks at most
            // per product, summed in shared memory by warps 2-3): measured
            // variant, not the default
            bool ok = p->sch.R <= kMaxR;
            for (int r = 0; r < p->sch.R && ok; ++r) {
                int nz = 0;
                for (int a = 0; a < p->sch.m; ++a)
                    for (int b = 0; b < p->sch.k; ++b) nz += p->sch.u(r, a, b) != 0;
                ok = nz >= 1 && nz <= 2;
            }
            if (!ok) {
                delete p;
                return fail(LCMA_ERR_NOT_SUPPORTED, "producer-fused variant: at most two A blocks per product");
            }
        }
        if (variant == LCMA_VARIANT_TWO_LEVEL && p->sch.base_id < 0) {
            delete p;
            return fail(LCMA_ERR_NOT_SUPPORTED, "two-level variant needs a composed scheme (Strassen^2)");
        }
    }
    p->variant = variant;

    // ---- blocking (P:612 ceil extents, tile-rounded: DESIGN.md reading 6)
    const Scheme& S = p->sch;
    if (d.dtype == LCMA_FP32) {
        p->BK = 8;
        p->Mb = classical ? d.M : roundup(cdiv(d.M, S.m), 8);
        p->Nb = classical ? d.N : roundup(cdiv(d.N, S.n), 8);
        p->Kb = classical ? d.K : roundup(cdiv(d.K, S.k), 8);
        p->nX = p->nZ = p->nK = 0;
        p->G = 0;
        p->ctas = 0;
        p->cg = 1;
    } else {
        p->BK = 128 / p->oe;
        const int sms = device_sm_count();
        p->ctas = d.num_ctas > 0 ? std::min(d.num_ctas, sms) : sms;
        p->cg = 2;
        if (const char* e_cg = diag_env("LCMA_CG")) p->cg = std::atoi(e_cg) == 1 ? 1 : 2;
        if (p->ctas < 2) p->cg = 1;
        p->ctas -= p->ctas % p->cg;
        if (p->cg == 2) {
            // a persistent grid must be fully co-resident (split groups wait on
            // each other): use the number of CTA pairs the device can host
            const int pairs = max_active_pairs();
            if (pairs > 0) p->ctas = std::min(p->ctas, 2 * pairs);
        }
        const int tileM = kBM * p->cg;
        p->bn = kBN;
        if (const char* e_bn = diag_env("LCMA_BN")) p->bn = std::atoi(e_bn) == 128 ? 128 : 256;
        // FP8: 2 x 128 accumulator columns leave TMEM room for the scale factors
        if (fp8) { p->bn = 128; p->cg = 2; }
        const int BNp = p->bn;
        if (classical) {
            p->nX = (int)cdiv(d.M, tileM);
            p->nZ = (int)cdiv(d.N, BNp);
            p->nK = (int)cdiv(d.K, p->BK);
            p->Mb = (int64_t)p->nX * tileM;
            p->Nb = (int64_t)p->nZ * BNp;
            p->Kb = (int64_t)p->nK * p->BK;
        } else {
            p->Mb = roundup(cdiv(d.M, S.m), tileM);
            p->Nb = roundup(cdiv(d.N, S.n), BNp);
            p->Kb = roundup(cdiv(d.K, S.k), p->BK);
            p->nX = (int)(p->Mb / tileM);
            p->nZ = (int)(p->Nb / BNp);
            p->nK = (int)(p->Kb / p->BK);
        }
        if ((long long)p->nX * p->nZ > INT32_MAX / 2 || S.R * p->Mb > INT32_MAX ||
            S.R * p->Kb > INT32_MAX || S.R * p->Nb > INT32_MAX) {
            delete p;
            return fail(LCMA_ERR_NOT_SUPPORTED, "problem too large for 32-bit tile coordinates");
        }
        p->G = p->nX * p->nZ;
        // default (0): the classical kernel hands its groups out at run time
        // (schedule 5: the lockstep pairs drift apart; measured +2.6..5.4 %
        // over the static rounds at cfg2 / cfg4 / cfg5 with the lean producer,
        // tools/r02/sched7.sh), LCMA plans keep the static lockstep rounds
        // (r-aligned products; the run-time hand-out measured 2-13 % slower)
        make_schedule(p, (d.schedule >= 1 && d.schedule <= 7) ? d.schedule : (classical ? 5 : 1));
        // the dynamic schedule is instantiated for the 256-column pair kernels
        // (classical and fused Combine H); the producer-fused variant's
        // combine warps walk the static schedule
        if ((p->dyn || p->dyn_tail) && (p->cg != 2 || p->bn != 256 || variant == LCMA_VARIANT_PRODUCER))
            make_schedule(p, 1);

        if (variant == LCMA_VARIANT_PRODUCER &&
            (p->cg != 2 || p->bn != 256 || d.M != (int64_t)S.m * p->Mb || d.K != (int64_t)S.k * p->Kb)) {
            delete p;
            return fail(LCMA_ERR_NOT_SUPPORTED,
                        "producer-fused variant: needs 256-column CTA-pair tiles and M, K that the m x k "
                        "block grid tiles exactly (the source blocks are read in place)");
        }
    }

    // ---- two-level: the inner (base-scheme) fused GEMM over the composed
    // scheme's block extents; its C is the outer H_q (fp32)
    if (variant == LCMA_VARIANT_TWO_LEVEL) {
        const Scheme& B0 = *scheme_get(S.base_id);
        lcma_plan_desc di = d;
        di.M = (int64_t)B0.m * p->Mb;
        di.N = (int64_t)B0.n * p->Nb;
        di.K = (int64_t)B0.k * p->Kb;
        di.out_dtype = LCMA_FP32;
        di.algo = LCMA_ALGO_SCHEME;
        di.scheme_id = S.base_id;
        di.variant = LCMA_VARIANT_FUSED_H;
        di.b_static = 0;
        lcma_plan_t in = nullptr;
        lcma_status st_in = lcma_plan_ex(&di, &in);
        if (st_in != LCMA_OK) {
            delete p;
            return st_in;
        }
        if (in->Mb != p->Mb || in->Nb != p->Nb || in->Kb != p->Kb) {
            delete in;
            delete p;
            return fail(LCMA_ERR_NOT_SUPPORTED, "two-level: inner block extents differ");
        }
        // the R0 inner GEMMs (one per outer product q) run as ONE batched
        // launch over R0 x nX x nZ groups: one split tail instead of R0, and
        // enough groups per launch for the persistent grid
        in->nbatch = B0.R;
        in->G = in->nX * in->nZ * in->nbatch;
        make_schedule(in, (d.schedule >= 2 && d.schedule <= 7) ? d.schedule : 1);
        if ((in->dyn || in->dyn_tail) && (in->cg != 2 || in->bn != 256)) make_schedule(in, 1);
        p->inner = in;
    }

    // ---- workspace layout
    size_t off = 0;
    p->off_sched = p->off_P = p->off_flags = p->off_At = p->off_Bt = p->off_H = 0;
    const int mn = S.m * S.n;
    if (d.dtype != LCMA_FP32 && variant != LCMA_VARIANT_TWO_LEVEL) {
        p->off_sched = off;                    // dynamic-schedule ticket counter
        off = align256(off + 256);
    }
    if (fp8) {
        // quantized operands (+ scale chunks), per call for classical too
        if (!classical) {
            p->off_P = off;
            off = align256(off + (size_t)3 * p->ctas * mn * kBM * p->bn * sizeof(float));
            p->off_flags = off;
            off = align256(off + (size_t)2 * p->ctas * sizeof(int));   // split flags: contributor + owner units
        }
        p->off_At = off;
        off = align256(off + fp8_operand_bytes(S.R, p->Mb, p->Kb));
        p->off_Bt = off;
        off = align256(off + fp8_operand_bytes(S.R, p->Nb, p->Kb));
    } else if (!classical) {
        if (d.dtype != LCMA_FP32 && (variant == LCMA_VARIANT_FUSED_H || variant == LCMA_VARIANT_PRODUCER)) {
            p->off_P = off;
            off = align256(off + (size_t)3 * p->ctas * mn * kBM * p->bn * sizeof(float));
            p->off_flags = off;
            off = align256(off + (size_t)2 * p->ctas * sizeof(int));   // split flags: contributor + owner units
        }
        p->off_At = off;
        off = align256(off + (size_t)S.R * p->Mb * p->Kb * e);
        p->off_Bt = off;
        off = align256(off + (size_t)S.R * p->Kb * p->Nb * e);
        if (variant == LCMA_VARIANT_UNFUSED) {
            p->off_H = off;
            off = align256(off + (size_t)S.R * p->Mb * p->Nb * sizeof(float));
        }
        if (variant == LCMA_VARIANT_TWO_LEVEL) {
            const Scheme& B0 = *scheme_get(S.base_id);
            p->off_H = off;    // outer H_q, q < R_base: [R_base][m0*Mb][n0*Nb] fp32
            off = align256(off + (size_t)B0.R * (B0.m * p->Mb) * (B0.n * p->Nb) * sizeof(float));
            p->off_inner = off;
            off = align256(off + p->inner->off_At);   // the inner plan's partials + flags
        }
    }
    p->ws_bytes = off;
    // single +1-term combined operands read in place by the fused GEMM (16-bit
    // data, block grid tiling M, K (and N for B, stored N x K) exactly)
    for (int r = 0; r < kMaxR; ++r) p->a_dir[r] = p->b_dir[r] = -1;
    if (!classical && variant == LCMA_VARIANT_FUSED_H && (d.dtype == LCMA_BF16 || d.dtype == LCMA_FP16) &&
        S.R <= kMaxR && p->cg == 2 && p->bn == 256) {
        const bool a_ok = d.M == (int64_t)S.m * p->Mb && d.K == (int64_t)S.k * p->Kb;
        const bool b_ok = d.b_layout == 1 && d.N == (int64_t)S.n * p->Nb && d.K == (int64_t)S.k * p->Kb;
        for (int r = 0; r < S.R; ++r) {
            int nz = 0, blk = -1, val = 0;
            for (int a = 0; a < S.m; ++a)
                for (int b = 0; b < S.k; ++b)
                    if (S.u(r, a, b)) { ++nz; blk = a * S.k + b; val = S.u(r, a, b); }
            if (a_ok && nz == 1 && val == 1) { p->a_dir[r] = (int8_t)blk; p->any_a_dir = true; }
            nz = 0; blk = -1; val = 0;
            for (int l = 0; l < S.k; ++l)
                for (int j = 0; j < S.n; ++j)
                    if (S.v(r, l, j)) { ++nz; blk = j * S.k + l; val = S.v(r, l, j); }
            if (b_ok && nz == 1 && val == 1) { p->b_dir[r] = (int8_t)blk; p->any_b_dir = true; }
        }
    }
    p->bt_bytes = fp8 ? fp8_operand_bytes(S.R, p->Nb, p->Kb) : classical ? 0 : (size_t)S.R * p->Kb * p->Nb * e;

    // ---- info
    lcma_plan_info& I = p->info;
    I.algo = p->algo;
    I.variant = variant;
    I.m = S.m; I.k = S.k; I.n = S.n; I.R = S.R;
    I.depth = p->scheme_id == SCHEME_STRASSEN ? 1 : p->scheme_id == SCHEME_STRASSEN2 ? 2 : (classical ? 0 : 1);
    std::snprintf(I.scheme, sizeof(I.scheme), "%s", S.name.c_str());
    I.Mb = p->Mb; I.Nb = p->Nb; I.Kb = p->Kb;
    I.BM = d.dtype == LCMA_FP32 ? 128 : kBM * p->cg;
    I.BN = d.dtype == LCMA_FP32 ? 128 : p->bn;
    I.BK = p->BK;
    I.cta_group = p->cg;
    I.t_pred_classical = dec.t_std;
    if (classical) {
        I.t_pred_choice = dec.t_std;
    } else {
        I.t_pred_choice = paper_model
            ? estimate_time(S, (double)d.M, (double)d.N, (double)d.K, p->hw, variant != LCMA_VARIANT_UNFUSED,
                            d.b_static != 0)
            : estimate_time_b200(S, (double)d.M, (double)d.N, (double)d.K, p->hw,
                                 variant != LCMA_VARIANT_UNFUSED, d.b_static != 0, (double)e);
    }
    I.speedup_pred = I.t_pred_classical / I.t_pred_choice;
    I.memory_bound = dec.memory_bound;
    const double ratio = p->hw.flops_mul / p->hw.beta;
    I.lcma_condition = !classical && condition_lhs(S, (double)d.M, (double)d.N, (double)d.K, false) > ratio;
    I.fused_condition = !classical && condition_lhs(S, (double)d.M, (double)d.N, (double)d.K, true) > ratio;
    I.workspace_bytes = p->ws_bytes;
    I.btilde_bytes = p->bt_bytes;
    I.partial_slots = 0;
    if (!classical && d.dtype != LCMA_FP32 && (variant == LCMA_VARIANT_FUSED_H || variant == LCMA_VARIANT_PRODUCER)) {
        const bool use_order = !diag_env("LCMA_ORDER") || std::atoi(diag_env("LCMA_ORDER")) != 0;
        I.partial_slots = use_order ? scheme_product_order(p->scheme_id).nslot : S.m * S.n;
    }
    if (variant == LCMA_VARIANT_TWO_LEVEL) I.partial_slots = p->inner->info.partial_slots;
    *out = p;
    return LCMA_OK;
}

extern "C" lcma_status lcma_plan(int64_t M, int64_t N, int64_t K, lcma_dtype dtype, lcma_algo algo,
                                 lcma_plan_t* out) {
    lcma_plan_desc d;
    std::memset(&d, 0, sizeof(d));
    d.M = M; d.N = N; d.K = K;
    d.dtype = dtype;
    d.out_dtype = (dtype == LCMA_TF32) ? LCMA_FP32 : dtype;
    d.algo = algo;
    return lcma_plan_ex(&d, out);
}

extern "C" void lcma_free(lcma_plan_t p) { delete p; }

extern "C" lcma_status lcma_plan_get_info(lcma_plan_t p, lcma_plan_info* out) {
    if (!p || !out) return fail(LCMA_ERR_INVALID_VALUE, "null argument");
    *out = p->info;
    return LCMA_OK;
}
extern "C" lcma_status lcma_workspace_size(lcma_plan_t p, size_t* bytes) {
    if (!p || !bytes) return fail(LCMA_ERR_INVALID_VALUE, "null argument");
    *bytes = p->ws_bytes;
    return LCMA_OK;
}
extern "C" lcma_status lcma_btilde_size(lcma_plan_t p, size_t* bytes) {
    if (!p || !bytes) return fail(LCMA_ERR_INVALID_VALUE, "null argument");
    *bytes = p->bt_bytes;
    return LCMA_OK;
}

extern "C" lcma_status lcma_plan_schedule(lcma_plan_t p, int32_t cta, int32_t* units, int32_t cap,
                                          int32_t* n) {
    if (!p || !n) return fail(LCMA_ERR_INVALID_VALUE, "null argument");
    if (p->ctas <= 0 || cta < 0 || cta >= p->ctas) return fail(LCMA_ERR_INVALID_VALUE, "bad cta");
    auto us = host_units(p, cta);
    *n = (int32_t)us.size();
    for (int i = 0; i < (int)us.size() && i < cap && units; ++i) {
        units[4 * i] = us[i].g;
        units[4 * i + 1] = us[i].r0;
        units[4 * i + 2] = us[i].r1;
        units[4 * i + 3] = us[i].role;
    }
    return LCMA_OK;
}

extern "C" lcma_status lcma_decide(int64_t M, int64_t N, int64_t K, lcma_dtype dtype,
                                   const lcma_hw_profile* hw, int32_t fused, lcma_plan_info* out) {
    if (!out) return fail(LCMA_ERR_INVALID_VALUE, "null argument");
    if (M < 1 || N < 1 || K < 1) return fail(LCMA_ERR_INVALID_VALUE, "M, N, K must be >= 1");
    Profile P = hw ? Profile{hw->flops_mul, hw->flops_add, hw->beta_elems} : default_profile((int)dtype);
    if (!(P.flops_mul > 0 && P.flops_add > 0 && P.beta > 0))
        return fail(LCMA_ERR_INVALID_VALUE, "hardware profile entries must be > 0");
    std::vector<int> cands = {SCHEME_STRASSEN, SCHEME_STRASSEN2, SCHEME_LADERMAN};
    DecisionResult dec = decide(cands, (double)M, (double)N, (double)K, P, fused != 0, false);
    std::memset(out, 0, sizeof(*out));
    const Scheme* s = scheme_get(dec.scheme_id);
    out->algo = dec.scheme_id == SCHEME_CLASSICAL ? LCMA_ALGO_CLASSICAL
                : dec.scheme_id == SCHEME_STRASSEN ? LCMA_ALGO_STRASSEN
                : dec.scheme_id == SCHEME_STRASSEN2 ? LCMA_ALGO_STRASSEN2
                                                     : LCMA_ALGO_LADERMAN;
    out->m = s->m; out->k = s->k; out->n = s->n; out->R = s->R;
    std::snprintf(out->scheme, sizeof(out->scheme), "%s", s->name.c_str());
    out->t_pred_classical = dec.t_std;
    out->t_pred_choice = dec.t_choice;
    out->speedup_pred = dec.t_std / dec.t_choice;
    out->memory_bound = dec.memory_bound;
    const double ratio = P.flops_mul / P.beta;
    const Scheme* st = scheme_get(SCHEME_STRASSEN);
    const Scheme* ref = dec.scheme_id == SCHEME_CLASSICAL ? st : s;
    out->lcma_condition = condition_lhs(*ref, (double)M, (double)N, (double)K, false) > ratio;
    out->fused_condition = condition_lhs(*ref, (double)M, (double)N, (double)K, true) > ratio;
    return LCMA_OK;
}

// ---------------------------------------------------------------- schemes
extern "C" lcma_status lcma_scheme_register(int32_t m, int32_t k, int32_t n, int32_t R,
                                            const int8_t* U, const int8_t* V, const int8_t* W,
                                            const char* name, int32_t* scheme_id) {
    if (!U || !V || !W || !scheme_id) return fail(LCMA_ERR_INVALID_VALUE, "null argument");
    if (m < 1 || k < 1 || n < 1 || R < 1 || m > 16 || k > 16 || n > 16 || R > 4096)
        return fail(LCMA_ERR_INVALID_VALUE, "bad scheme dimensions");
    Scheme s;
    s.name = name ? name : "registered";
    s.m = m; s.k = k; s.n = n; s.R = R;
    s.U.assign(U, U + (size_t)R * m * k);
    s.V.assign(V, V + (size_t)R * k * n);
    s.W.assign(W, W + (size_t)R * m * n);
    std::string err;
    int id = scheme_register(s, err);
    if (id < 0) return fail((lcma_status)(-id), err);
    *scheme_id = id;
    return LCMA_OK;
}

extern "C" lcma_status lcma_scheme_register_file(const char* path, int32_t* scheme_id) {
    if (!path || !scheme_id) return fail(LCMA_ERR_INVALID_VALUE, "null argument");
    std::ifstream f(path);
    if (!f) return fail(LCMA_ERR_INVALID_VALUE, std::string("cannot open ") + path);
    std::stringstream ss;
    ss << f.rdbuf();
    Scheme s;
    std::string err;
    int rc = scheme_parse(ss.str(), s, err);
    if (rc < 0) return fail((lcma_status)(-rc), err);
    s.name = path;
    int id = scheme_register(s, err);
    if (id < 0) return fail((lcma_status)(-id), err);
    *scheme_id = id;
    return LCMA_OK;
}

extern "C" lcma_status lcma_scheme_get(int32_t id, int32_t* mknR, int8_t* U, int8_t* V, int8_t* W) {
    const Scheme* s = scheme_get(id);
    if (!s) return fail(LCMA_ERR_INVALID_VALUE, "unknown scheme id");
    if (mknR) { mknR[0] = s->m; mknR[1] = s->k; mknR[2] = s->n; mknR[3] = s->R; }
    if (U) std::memcpy(U, s->U.data(), s->U.size());
    if (V) std::memcpy(V, s->V.data(), s->V.size());
    if (W) std::memcpy(W, s->W.data(), s->W.size());
    return LCMA_OK;
}

extern "C" const char* lcma_last_error(void) { return t_err.c_str(); }
extern "C" int32_t lcma_last_launch_count(void) { return t_launches; }

// ---------------------------------------------------------------- launching
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
        cudaGetLastError();
    });
    return fn;
}

lcma_status make_map_t(CUtensorMap* m, const void* ptr, CUtensorMapDataType t, int e, uint64_t cols,
                       uint64_t rows, uint32_t box_c, uint32_t box_r,
                       CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    auto fn = encode_fn();
    if (!fn) return fail(LCMA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * (cuuint64_t)e};
    cuuint32_t box[2] = {box_c, box_r};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(m, t, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        char buf[160];
        std::snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled failed (%d) dims %llu x %llu box %u x %u",
                      (int)r, (unsigned long long)cols, (unsigned long long)rows, box_c, box_r);
        return fail(LCMA_ERR_CUDA, buf);
    }
    return LCMA_OK;
}

lcma_status make_map(CUtensorMap* m, const void* ptr, lcma_dtype dt, uint64_t cols, uint64_t rows,
                     uint32_t box_c, uint32_t box_r,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    const CUtensorMapDataType t = dt == LCMA_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                  : dt == LCMA_FP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                    : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    return make_map_t(m, ptr, t, elem_bytes(dt), cols, rows, box_c, box_r, swz);
}

// MN-major B (rows x cols row-major, cols % epr == 0) as a 3-D map
// {epr elements (128 B), row, cols/epr chunks}: one box of {epr, box_r, n_chunks}
// lands as [chunk][row][128 B], the layout the UMMA MN-major descriptor reads.
lcma_status make_map_mn3d(CUtensorMap* m, const void* ptr, lcma_dtype dt, uint64_t cols, uint64_t rows,
                          uint32_t epr, uint32_t box_r, uint32_t n_chunks, CUtensorMapSwizzle swz) {
    auto fn = encode_fn();
    if (!fn) return fail(LCMA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    CUtensorMapDataType t = dt == LCMA_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                            : dt == LCMA_FP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                              : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    const int e = elem_bytes(dt);
    cuuint64_t dims[3] = {epr, rows, cols / epr};
    cuuint64_t strides[2] = {cols * (cuuint64_t)e, (cuuint64_t)epr * e};
    cuuint32_t box[3] = {epr, box_r, n_chunks};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(m, t, 3, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? LCMA_OK : LCMA_ERR_NOT_SUPPORTED;
}

// Diagnostics only (LCMA_STATS set): a process-lifetime device buffer for the
// per-CTA wait-cycle counters; read back with lcma_debug_stats().
unsigned long long* g_stats = nullptr;
unsigned long long* lcma_debug_stats_buffer() {
    if (!g_stats) {
        if (cudaMalloc(&g_stats, 1024 * kStatsPerCta * sizeof(unsigned long long)) != cudaSuccess) {
            cudaGetLastError();
            g_stats = nullptr;
        } else {
            cudaMemset(g_stats, 0, 1024 * kStatsPerCta * sizeof(unsigned long long));
        }
    }
    return g_stats;
}

// per-product timeline (LCMA_TIMELINE=1); read back with lcma_debug_timeline().
unsigned long long* g_tl = nullptr;
unsigned long long* lcma_debug_timeline_buffer() {
    if (!g_tl) {
        const size_t bytes = (size_t)1024 * kTlMax * 4 * sizeof(unsigned long long);
        if (cudaMalloc(&g_tl, bytes) != cudaSuccess) { cudaGetLastError(); g_tl = nullptr; }
        else cudaMemset(g_tl, 0, bytes);
    }
    return g_tl;
}

lcma_status check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(LCMA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    ++t_launches;
    return LCMA_OK;
}

// The dynamic shared-memory limit is a per-device function attribute: set it
// once per (instantiation, device).
template <int CG, int BN, int QF = 0, bool REGH = false, int PF = 0, bool DYN = false, bool F8 = false,
          bool CST = true>
lcma_status ensure_smem_attr() {
    static std::once_flag once[kMaxDev];
    static cudaError_t err[kMaxDev];
    const int dv = current_device();
    if (dv < 0) return fail(LCMA_ERR_CUDA, "no current CUDA device (or ordinal >= 64)");
    std::call_once(once[dv], [dv] {
        err[dv] = cudaFuncSetAttribute(umma_gemm_kernel<CG, BN, QF, REGH, PF, DYN, F8, CST>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       KernelCfg<CG, BN, QF, REGH, PF, F8, CST>::kSmemBytes);
    });
    if (err[dv] != cudaSuccess)
        return fail(LCMA_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(err[dv]));
    return LCMA_OK;
}

int grid_for(long long work, int per_block) {
    long long b = (work + per_block - 1) / per_block;
    if (b < 1) b = 1;
    static const long long cap = diag_env("LCMA_COMB_BLOCKS") ? std::atoll(diag_env("LCMA_COMB_BLOCKS"))
                                                                 : 148 * 16;
    if (b > cap) b = cap;
    return (int)b;
}

// Group combine of one operand into dst[R][E0][E1] (Alg. 2 stage 1 or 2).
// Parameters of the group combine of one operand into dst[R][E0][E1]; inst =
// the kernels' coefficient-table width (PQ instantiation).
lcma_status make_combine_params(const lcma_plan_s* p, const void* src, void* dst, bool is_b, bool direct,
                                CombineParams& c, int& inst) {
    const Scheme& S = p->sch;
    std::memset(&c, 0, sizeof(c));
    c.src = src;
    c.dst = dst;
    c.R = S.R;
    c.elem = p->d.dtype == LCMA_BF16 ? ELEM_BF16 : p->d.dtype == LCMA_FP16 ? ELEM_FP16 : ELEM_FP32;
    c.round_tf32 = p->d.dtype == LCMA_TF32;
    if (direct)   // outputs the GEMM reads in place (single +1 source block)
        for (int r = 0; r < S.R && r < kCombMaxR; ++r) c.skip[r] = (is_b ? p->b_dir[r] : p->a_dir[r]) >= 0;
    int P, Q;
    if (!is_b) {                      // A (M x K): blocks (i, l), coef U[r][i][l]
        c.rows = p->d.M; c.cols = p->d.K; c.E0 = p->Mb; c.E1 = p->Kb; P = S.m; Q = S.k;
    } else if (p->d.b_layout == 0) {  // B (K x N): blocks (l, j), coef V[r][l][j]
        c.rows = p->d.K; c.cols = p->d.N; c.E0 = p->Kb; c.E1 = p->Nb; P = S.k; Q = S.n;
    } else {                          // B (N x K): blocks (j, l), coef V[r][l][j]
        c.rows = p->d.N; c.cols = p->d.K; c.E0 = p->Nb; c.E1 = p->Kb; P = S.n; Q = S.k;
    }
    c.P = P;
    c.Q = Q;
    const int pq = P * Q;
    inst = pq <= 4 ? 4 : pq <= 9 ? 9 : pq <= 16 ? 16 : pq <= 25 ? 25 : 32;
    if (S.R > kCombMaxR || pq > kCombMaxPQ) return fail(LCMA_ERR_NOT_SUPPORTED, "scheme too large");
    for (int r = 0; r < S.R; ++r)
        for (int a = 0; a < P; ++a)
            for (int b = 0; b < Q; ++b) {
                int8_t v;
                if (!is_b) v = S.u(r, a, b);
                else if (p->d.b_layout == 0) v = S.v(r, a, b);
                else v = S.v(r, b, a);
                c.coef[r * inst + a * Q + b] = v;
            }
    return LCMA_OK;
}

// Combine A and Combine B of one call (16-bit, packed kernels of the same
// width) as one launch; otherwise two.
lcma_status launch_combine(const lcma_plan_s* p, const void* src, void* dst, bool is_b, cudaStream_t st,
                           bool direct = false);
lcma_status launch_combine_ab(const lcma_plan_s* p, const void* A, void* At, const void* B, void* Bt,
                              cudaStream_t st, bool dirA, bool dirB) {
    CombineParams ca, cb;
    int ia = 0, ib = 0;
    lcma_status rs = make_combine_params(p, A, At, false, dirA, ca, ia);
    if (rs == LCMA_OK) rs = make_combine_params(p, B, Bt, true, dirB, cb, ib);
    if (rs != LCMA_OK) return rs;
    if (ca.elem != ELEM_FP32 && ia == ib && (ia == 4 || ia == 9 || ia == 16) && !diag_env("LCMA_OLD_COMBINE") &&
        !diag_env("LCMA_COMB_SPLIT")) {
        const int ga = grid_for(ca.E0 * (ca.E1 / 8), 256), gb = grid_for(cb.E0 * (cb.E1 / 8), 256);
        if (ia == 4) group_combine16_dual_kernel<4, 4><<<ga + gb, 256, 0, st>>>(ca, cb, ga);
        else if (ia == 9) group_combine16_dual_kernel<9, 9><<<ga + gb, 256, 0, st>>>(ca, cb, ga);
        else group_combine16_dual_kernel<16, 16><<<ga + gb, 256, 0, st>>>(ca, cb, ga);
        return check_launch("group_combine16_dual_kernel");
    }
    rs = launch_combine(p, A, At, false, st, dirA);
    if (rs != LCMA_OK) return rs;
    return launch_combine(p, B, Bt, true, st, dirB);
}

lcma_status launch_combine(const lcma_plan_s* p, const void* src, void* dst, bool is_b,
                           cudaStream_t st, bool direct) {   // (default: declaration above)
    CombineParams c;
    int inst = 0;
    lcma_status rc = make_combine_params(p, src, dst, is_b, direct, c, inst);
    if (rc != LCMA_OK) return rc;
    const bool fp32 = c.elem == ELEM_FP32;
    if (!fp32 && (inst == 4 || inst == 9 || inst == 16) && !diag_env("LCMA_OLD_COMBINE")) {
        // 16-bit sources with 9 or 16 blocks: packed sources keep more loads in
        // flight (measured 1.4x / 2.3x faster than the unpacked kernel below)
        const long long nv = c.E0 * (c.E1 / 8);
        const int g = grid_for(nv, 256);
        if (inst == 9) group_combine16_kernel<9, 1><<<g, 256, 0, st>>>(c);
        else if (inst == 4) group_combine16_kernel<4, 1><<<g, 256, 0, st>>>(c);
        else group_combine16_kernel<16, 1><<<g, 256, 0, st>>>(c);
        return check_launch("group_combine16_kernel");
    }
    const int vec = (fp32 || inst > 9) ? 4 : 8;
    const long long nvec = c.E0 * (c.E1 / vec);
    const int grid = grid_for(nvec, 256);
#define LCMA_COMB(V, PQ) group_combine_kernel<V, PQ><<<grid, 256, 0, st>>>(c)
    if (vec == 8) {
        if (inst == 4) LCMA_COMB(8, 4); else LCMA_COMB(8, 9);
    } else {
        if (inst == 4) LCMA_COMB(4, 4);
        else if (inst == 9) LCMA_COMB(4, 9);
        else if (inst == 16) LCMA_COMB(4, 16);
        else if (inst == 25) LCMA_COMB(4, 25);
        else LCMA_COMB(4, 32);
    }
#undef LCMA_COMB
    return check_launch("group_combine_kernel");
}

// FP8: group combine of one bf16 operand with the 1 x 128 quantization fused
// in: dst = E4M3 [R][E0][Kb] followed by the UE8M0 scale chunks.
// A: M x K, blocks (i, l), coef U[r][i][l]; B: N x K, blocks (j, l), coef V[r][l][j].
lcma_status launch_combine_q8(const lcma_plan_s* p, const void* src, void* dst, bool is_b, cudaStream_t st) {
    const Scheme& S = p->sch;
    CombineQ8Params c;
    std::memset(&c, 0, sizeof(c));
    c.src = reinterpret_cast<const uint16_t*>(src);
    c.dst = reinterpret_cast<uint8_t*>(dst);
    c.R = S.R;
    if (!is_b) {
        c.rows = p->d.M; c.cols = p->d.K; c.E0 = p->Mb; c.E1 = p->Kb; c.P = S.m; c.Q = S.k;
    } else {
        c.rows = p->d.N; c.cols = p->d.K; c.E0 = p->Nb; c.E1 = p->Kb; c.P = S.n; c.Q = S.k;
    }
    c.sf = reinterpret_cast<uint32_t*>(c.dst + (size_t)S.R * c.E0 * c.E1);
    const int pq = c.P * c.Q;
    const int inst = pq <= 1 ? 1 : pq <= 4 ? 4 : pq <= 9 ? 9 : 16;
    if (S.R > kCombMaxR || pq > 16) return fail(LCMA_ERR_NOT_SUPPORTED, "scheme too large for the FP8 combine");
    for (int r = 0; r < S.R; ++r)
        for (int a = 0; a < c.P; ++a)
            for (int b = 0; b < c.Q; ++b)
                c.coef[r * inst + a * c.Q + b] = !is_b ? S.u(r, a, b) : S.v(r, b, a);
    // the plain quantization (one source block): two 8-element vectors per
    // thread with every load issued up front (measured 41 -> 35 us for A at
    // cfg2); the multi-source combines keep one vector per thread (two cost
    // registers and occupancy: 44 -> 52 us)
    const long long nv = c.E0 * (c.E1 / 8);
    const int g1 = (int)std::min<long long>((nv + 255) / 256, 1 << 30);
    const int g2 = (int)std::min<long long>((nv + 511) / 512, 1 << 30);
    if (inst == 1) group_combine_q8_kernel<1, 2><<<g2, 256, 0, st>>>(c);
    else if (inst == 4) group_combine_q8_kernel<4, 1><<<g1, 256, 0, st>>>(c);
    else if (inst == 9) group_combine_q8_kernel<9, 1><<<g1, 256, 0, st>>>(c);
    else group_combine_q8_kernel<16, 1><<<g1, 256, 0, st>>>(c);
    return check_launch("group_combine_q8_kernel");
}

// Combine H (Eq. 6) of scheme S over H [R][Mb][Nb] fp32 into C (M x N, crop).
lcma_status launch_combine_h_ex(const lcma_plan_s* p, const Scheme& S, long long Mb, long long Nb, const float* H,
                                void* C, cudaStream_t st) {
    CombineHParams c;
    std::memset(&c, 0, sizeof(c));
    c.H = H; c.C = C;
    c.M = p->d.M; c.N = p->d.N; c.Mb = Mb; c.Nb = Nb; c.ldc = p->d.N;
    c.m = S.m; c.n = S.n; c.R = S.R;
    c.out_type = p->d.out_dtype == LCMA_FP32 || p->d.out_dtype == LCMA_TF32 ? 2
                 : p->d.out_dtype == LCMA_BF16 ? 0 : 1;
    const int mn = S.m * S.n;
    const int inst = mn <= 1 ? 1 : mn <= 4 ? 4 : mn <= 9 ? 9 : mn <= 16 ? 16 : mn <= 25 ? 25 : 32;
    for (int r = 0; r < S.R; ++r)
        for (int ij = 0; ij < mn; ++ij) c.Wc[r * inst + ij] = S.W[(size_t)r * mn + ij];
    const long long nvec = c.Mb * (c.Nb / 4);
    const int grid = grid_for(nvec, 256);
    switch (inst) {
        case 1: group_combine_h_kernel<1><<<grid, 256, 0, st>>>(c); break;
        case 4: group_combine_h_kernel<4><<<grid, 256, 0, st>>>(c); break;
        case 9: group_combine_h_kernel<9><<<grid, 256, 0, st>>>(c); break;
        case 16: group_combine_h_kernel<16><<<grid, 256, 0, st>>>(c); break;
        case 25: group_combine_h_kernel<25><<<grid, 256, 0, st>>>(c); break;
        default: group_combine_h_kernel<32><<<grid, 256, 0, st>>>(c); break;
    }
    return check_launch("group_combine_h_kernel");
}
lcma_status launch_combine_h(const lcma_plan_s* p, const float* H, void* C, cudaStream_t st) {
    return launch_combine_h_ex(p, p->sch, p->Mb, p->Nb, H, C, st);
}

// tcgen05 GEMM: classical (R == 1 over A, B) or the LCMA GEMM stage over the
// materialised At / Bt with the fused Combine H (or H store) epilogue.
lcma_status launch_umma(const lcma_plan_s* p, const void* Aop, const void* Bop, void* C, float* P,
                        int* flags, int* sched, float* H, cudaStream_t st, int pf = 0,
                        const void* Araw = nullptr, const void* Braw = nullptr) {
    const Scheme& S = p->sch;
    const bool classical = p->scheme_id == SCHEME_CLASSICAL;
    // QF: the shared-memory partial home covers both column halves (3 operand
    // stages; measured slower than 4 stages with column half 1 in L2: cfg2
    // 910 vs 824 us, so opt-in only)
    int qf = 0;
    if (const char* v = diag_env("LCMA_QFULL"))
        qf = (!classical && !H && p->cg == 2 && p->bn == 256 && S.m * S.n > 1 && std::atoi(v) != 0) ? 1 : 0;
    // diagnostics: the long-product register-home kernel without the shared
    // partial home and with 7 operand stages
    if (const char* v = diag_env("LCMA_NOSMEMP"))
        if (std::atoi(v) != 0 && !classical && !H && p->cg == 2 && p->bn == 256 && p->nK > kCstMaxNK) qf = 2;
    // REGH: the instantiation with a register partial home (fused Combine H of
    // an LCMA scheme on 256-column pair tiles); classical / unfused GEMMs use
    // the one without (no 128 live registers reserved in the epilogue)
    const bool f8 = p->d.dtype == LCMA_FP8_E4M3;
    // register-home kernel: C through shared memory + TMA stores (one operand
    // stage fewer) when a product is short (the fused epilogue then paces the
    // MMA); long products keep 5 stages and store C from registers
    bool cst_regh = p->nK <= kCstMaxNK;
    if (const char* v = diag_env("LCMA_CST")) cst_regh = std::atoi(v) != 0;
    const bool regh = f8 ? (!classical && !H) : (!classical && !H && p->cg == 2 && p->bn == 256);
    // the plan only sets dyn / dyn_tail for 256-column pair kernels
    const bool dyn = (p->dyn || p->dyn_tail) && sched && !pf;
    if (pf || dyn || f8) qf = 0;
    lcma_status rs = f8 ? (regh ? ensure_smem_attr<2, 128, 0, true, 0, false, true>()
                                : ensure_smem_attr<2, 128, 0, false, 0, false, true>())
                   : pf == 2 ? ensure_smem_attr<2, 256, 0, true, 2>()
                   : pf == 1 ? ensure_smem_attr<2, 256, 0, true, 1>()
                   : p->cg == 2 ? (p->bn == 128 ? ensure_smem_attr<2, 128>()
                                                : (qf == 2 ? ensure_smem_attr<2, 256, 2, true>()
                                                   : qf ? ensure_smem_attr<2, 256, 1, true>()
                                                      : regh ? (dyn ? (cst_regh ? ensure_smem_attr<2, 256, 0, true, 0, true>()
                                                                          : ensure_smem_attr<2, 256, 0, true, 0, true, false, false>())
                                                                    : cst_regh ? ensure_smem_attr<2, 256, 0, true>()
                                                                    : ensure_smem_attr<2, 256, 0, true, 0, false, false, false>())
                                                             : (dyn ? ensure_smem_attr<2, 256, 0, false, 0, true>()
                                                                    : ensure_smem_attr<2, 256>())))
                                : (p->bn == 128 ? ensure_smem_attr<1, 128>() : ensure_smem_attr<1, 256>());
    if (rs != LCMA_OK) return rs;
    const lcma_dtype dt = p->d.dtype;
    const int epr = 128 / p->e;           // elements per 128-byte row
    CUtensorMap ta, tb;
    const bool b_mn = p->d.b_layout == 0;
    bool b3d = false;
    if (f8) {
        // quantized operands: A~ [R][Mb][Kb], B~ [R][Nb][Kb] E4M3 (K-major, 128
        // elements per 128-byte row), each followed by its scale chunks
        rs = make_map_t(&ta, Aop, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, p->Kb, (uint64_t)S.R * p->Mb, 128, kBM);
        if (rs != LCMA_OK) return rs;
        rs = make_map_t(&tb, Bop, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, p->Kb, (uint64_t)S.R * p->Nb, 128,
                        p->bn / p->cg);
        if (rs != LCMA_OK) return rs;
    } else {
    // A operand: K-major rows (PF: the raw A, its blocks are combined in the kernel)
    const uint64_t a_cols = (classical || pf) ? p->d.K : p->Kb;
    const uint64_t a_rows = (classical || pf) ? p->d.M : (uint64_t)S.R * p->Mb * p->nbatch;
    rs = make_map(&ta, Aop, dt, a_cols, a_rows, epr, kBM);
    if (rs != LCMA_OK) return rs;
    if (!b_mn) {   // N x K (K-major); PF 2: the raw B, its blocks are combined in the kernel
        const uint64_t cols = (classical || pf == 2) ? p->d.K : p->Kb;
        const uint64_t rows = (classical || pf == 2) ? p->d.N : (uint64_t)S.R * p->Nb * p->nbatch;
        rs = make_map(&tb, Bop, dt, cols, rows, epr, p->bn / p->cg);
    } else {       // K x N (MN-major): boxes of 128 bytes of N x BK rows
        const uint64_t cols = classical ? p->d.N : p->Nb;
        const uint64_t rows = classical ? p->d.K : (uint64_t)S.R * p->Kb * p->nbatch;
        CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B;
        if (dt == LCMA_TF32 || dt == LCMA_FP32) {
            if (const char* v = diag_env("LCMA_TF32_MN_SWZ")) swz = (CUtensorMapSwizzle)std::atoi(v);
            else swz = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
        }
        b3d = cols % (uint64_t)epr == 0 && !diag_env("LCMA_B2D") &&
              make_map_mn3d(&tb, Bop, dt, cols, rows, epr, p->BK, (uint32_t)((p->bn / p->cg) / p->BK), swz) ==
                  LCMA_OK;
        if (!b3d) rs = make_map(&tb, Bop, dt, cols, rows, epr, p->BK, swz);
    }
    if (rs != LCMA_OK) return rs;
    }

    GemmParams g;
    std::memset(&g, 0, sizeof(g));
    g.nX = p->nX; g.nZ = p->nZ; g.G = p->G; g.R = S.R; g.nK = p->nK; g.BK = p->BK;
    g.nbatch = p->nbatch;
    g.Gb = p->nX * p->nZ;
    g.a_rows_per_r = classical ? 0 : (int)p->Mb;
    g.b_rows_per_r = classical ? 0 : (int)(b_mn ? p->Kb : p->Nb);
    g.b_mn_major = b_mn;
    g.b_3d = b3d ? 1 : 0;
    // MN-major 32-bit operands use the 128B_BASE32B layout (4-row swizzle atoms)
    g.b_layout_type = (dt == LCMA_TF32) ? 1 : 2;
    g.b_sbo = (dt == LCMA_TF32) ? 512 : 1024;
    if (const char* v = diag_env("LCMA_TF32_MN_LT")) g.b_layout_type = std::atoi(v);
    if (const char* v = diag_env("LCMA_TF32_MN_SBO")) g.b_sbo = std::atoi(v);
    g.tf32 = dt == LCMA_TF32;
    g.idesc = f8 ? ptx::make_idesc_mxf8(kBM * p->cg, p->bn)
                 : ptx::make_idesc(dt == LCMA_BF16 ? 1u : dt == LCMA_FP16 ? 0u : 2u, kBM * p->cg, p->bn,
                                   b_mn ? 1u : 0u, 0u);
    if (f8) {
        // UE8M0 scale chunks behind the operands, as [2 * chunks][256] byte maps
        g.a_rows_per_r = (int)p->Mb;
        g.b_rows_per_r = (int)p->Nb;
        g.sf_nkb = (int)(p->Kb / 128);
        const uint64_t ca = (uint64_t)S.R * (p->Mb / 128) * (p->Kb / 128);
        const uint64_t cb = (uint64_t)S.R * (p->Nb / 128) * (p->Kb / 128);
        const uint8_t* sa = reinterpret_cast<const uint8_t*>(Aop) + (size_t)S.R * p->Mb * p->Kb;
        const uint8_t* sb = reinterpret_cast<const uint8_t*>(Bop) + (size_t)S.R * p->Nb * p->Kb;
        rs = make_map_t(&g.sfa_map, sa, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, 256, 2 * ca, 256, 2,
                        CU_TENSOR_MAP_SWIZZLE_NONE);
        if (rs != LCMA_OK) return rs;
        rs = make_map_t(&g.sfb_map, sb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, 256, 2 * cb, 256, 2,
                        CU_TENSOR_MAP_SWIZZLE_NONE);
        if (rs != LCMA_OK) return rs;
    }
    g.W = p->ctas / p->cg; g.q = p->q; g.tail_c = p->tail_c; g.swz = p->swz;
    g.n_whole = p->n_whole;
    g.dyn = dyn && p->dyn ? 1 : 0;
    g.dyn_tail = dyn && p->dyn_tail ? 1 : 0;
    g.n_own = p->info.split_groups;
    g.sched = sched;

    g.epi_mode = H ? EPI_STORE_H : EPI_FUSED;
    g.out_type = (p->d.out_dtype == LCMA_FP32 || p->d.out_dtype == LCMA_TF32) ? OUT_FP32
                 : p->d.out_dtype == LCMA_BF16 ? OUT_BF16 : OUT_FP16;
    g.m = S.m; g.n = S.n;
    g.M = p->d.M; g.N = p->d.N; g.Mb = p->Mb; g.Nb = p->Nb; g.ldc = p->d.N;
    g.C = C; g.P = P; g.flags = flags; g.H = H;
    {
        const int ce = g.out_type == OUT_FP32 ? 4 : 2;
        g.c_v8 = ((reinterpret_cast<uintptr_t>(C) & 31) == 0 && (g.ldc * ce) % 32 == 0) ? 1 : 0;
        if (diag_env("LCMA_NO_V8")) g.c_v8 = 0;
        g.c_cs = diag_env("LCMA_C_CS") ? std::atoi(diag_env("LCMA_C_CS")) : 0;
    }
    // 16-bit C by TMA stores from shared-memory staging (the instantiations
    // with a staging area: CTA pairs, no producer-fused combine, QF 0)
    g.c_tma = 0;
    const bool has_stage = f8 || !regh || cst_regh;
    const int ce = g.out_type == OUT_FP32 ? 4 : 2;
    if (has_stage && p->cg == 2 && !pf && !qf && !H && (reinterpret_cast<uintptr_t>(C) & 15) == 0 &&
        (g.ldc * ce) % 16 == 0 && !(diag_env("LCMA_C_TMA") && std::atoi(diag_env("LCMA_C_TMA")) == 0)) {
        // 16-bit C: two 32 x 32 boxes per warp; fp32 C (e.g. the two-level
        // inner GEMMs' H_q): one 32 x 32 box of 4 KB
        const CUtensorMapDataType ct = g.out_type == OUT_BF16   ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                       : g.out_type == OUT_FP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                                : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
        if (make_map_t(&g.c_map, C, ct, ce, (uint64_t)p->d.N, (uint64_t)p->d.M * p->nbatch, 32, 32,
                       CU_TENSOR_MAP_SWIZZLE_NONE) == LCMA_OK)
            g.c_tma = g.out_type == OUT_FP32 ? 2 : 1;
        else
            t_err.clear();
    }
    g.pf_kb = 0;
    g.drift = 0;
    if (const char* v = diag_env("LCMA_DRIFT")) g.drift = std::atoi(v);
    // in-place single-term operands (lean producer path only; the diagnostics
    // build takes the general loop when a producer knob is set)
    g.use_dir = 0;
    for (int r = 0; r < kMaxR; ++r) g.a_dir[r] = g.b_dir[r] = -1;
    if (Araw || Braw) {   // run() decided (direct_ok): the combines skipped these outputs
        if (Araw) {
            rs = make_map(&g.a_raw, Araw, dt, p->d.K, p->d.M, epr, kBM);
            if (rs != LCMA_OK) return rs;
            for (int r = 0; r < S.R; ++r) g.a_dir[r] = p->a_dir[r];
        }
        if (Braw) {
            rs = make_map(&g.b_raw, Braw, dt, p->d.K, p->d.N, epr, p->bn / p->cg);
            if (rs != LCMA_OK) return rs;
            for (int r = 0; r < S.R; ++r) g.b_dir[r] = p->b_dir[r];
        }
        g.use_dir = 1;
        g.kgrid = S.k;
        g.pf_Kb = (int)p->Kb;
    }
    if (const char* v = diag_env("LCMA_PFKB")) g.pf_kb = std::atoi(v);
    if (const char* dbg = diag_env("LCMA_DEBUG")) g.debug = std::atoi(dbg);
    // fused Combine H partials carry an L2 evict_last policy (measured: -1 %
    // at cfg2, -3..7 % at the cfg5 shard; profiles/r01b_l2_residency.txt)
    g.partial_hint = 1;
    if (const char* ph = diag_env("LCMA_PARTIAL_HINT")) g.partial_hint = std::atoi(ph);
    if (const char* oh = diag_env("LCMA_OPERAND_HINT")) g.operand_hint = std::atoi(oh);
    if (const char* sw = diag_env("LCMA_SWZ")) g.swz = std::max(1, std::atoi(sw));
    if (diag_env("LCMA_STATS")) g.stats = lcma_debug_stats_buffer();
    if (diag_env("LCMA_TIMELINE")) g.tl = lcma_debug_timeline_buffer();
    const int mn = S.m * S.n;
    if (S.R > kMaxR || mn > kMaxMN) return fail(LCMA_ERR_NOT_SUPPORTED, "scheme too large for the fused kernel");
    for (int r = 0; r < S.R; ++r) {
        int nu = 0, nv = 0;
        for (int q = 0; q < S.m * S.k; ++q) nu += S.U[(size_t)r * S.m * S.k + q] != 0;
        for (int q = 0; q < S.k * S.n; ++q) nv += S.V[(size_t)r * S.k * S.n + q] != 0;
        g.dbg_extra[r] = (uint8_t)((std::min(nv, 16) - 1) << 4 | (std::min(nu, 16) - 1));
        g.nzmask[r] = 0;
        for (int ij = 0; ij < mn; ++ij) {
            g.Wc[r * mn + ij] = S.W[(size_t)r * mn + ij];
            if (S.W[(size_t)r * mn + ij]) g.nzmask[r] |= 1u << ij;
        }
    }
    // product order inside a group + partial homes (fused Combine H, whole
    // groups): the two C_ij slots with the most partial updates live on chip
    // (epilogue registers, shared memory), the others in L2 workspace slots
    const bool use_order = !diag_env("LCMA_ORDER") || std::atoi(diag_env("LCMA_ORDER")) != 0;
    for (int ij = 0; ij < kMaxMN; ++ij) g.home[ij] = 0;
    if (use_order && !classical) {
        const ProductOrder& po = scheme_product_order(p->scheme_id);
        for (int t = 0; t < S.R; ++t) g.rperm[t] = (int8_t)po.perm[t];
        // slot -> home
        const int ns = po.nslot;
        const std::vector<int>& by_use = po.by_use;
        const bool use_reg = regh && !(diag_env("LCMA_REG_PARTIAL") && std::atoi(diag_env("LCMA_REG_PARTIAL")) == 0);
        const bool use_smem = !H && !pf && qf != 2 &&
                              !(diag_env("LCMA_SMEM_PARTIAL") && std::atoi(diag_env("LCMA_SMEM_PARTIAL")) == 0);
        std::vector<int> slot_home(ns, 0);
        int nl2 = 0, k0 = 0;
        if (use_reg && k0 < ns) slot_home[by_use[k0++]] = HOME_REG;
        if (use_smem && k0 < ns) slot_home[by_use[k0++]] = HOME_SMEM;
        for (int k = k0; k < ns; ++k) slot_home[by_use[k]] = nl2++;
        g.qslot = nl2;                    // L2 tile of the shared partial's column half 1 (QF = 0)
        for (int ij = 0; ij < mn; ++ij) g.home[ij] = (int8_t)(po.slot[ij] >= 0 ? slot_home[po.slot[ij]] : 0);
        g.nslot = nl2 + (use_smem ? 1 : 0);
    } else {
        // every C_ij keeps its own L2 slot
        for (int t = 0; t < S.R; ++t) g.rperm[t] = (int8_t)t;
        for (int ij = 0; ij < mn; ++ij) g.home[ij] = (int8_t)ij;
        g.qslot = 0;
        g.nslot = mn;
    }
    g.serpentine = 0;
    if (const char* v = diag_env("LCMA_SERPENTINE")) g.serpentine = std::atoi(v);
    g.discard = 1;
    if (const char* dc = diag_env("LCMA_DISCARD")) g.discard = std::atoi(dc);
    if (const char* pn = diag_env("LCMA_PACE_NS")) g.pace_ns = std::atoi(pn);
    if (t_ev_start) cudaEventRecord(t_ev_start, st);
    cudaLaunchConfig_t cfg;
    std::memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(p->ctas);
    cfg.blockDim = dim3(kThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr[3];
    int na = 0;
    if (p->cg == 2) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = p->cg;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    // optional: keep the whole-group partial slots L2-resident (access-policy
    // window over [P, P + nslot*ctas tiles), persisting)
    if (P && g.epi_mode == EPI_FUSED && diag_env("LCMA_L2PERSIST")) {
        size_t want = (size_t)std::atoll(diag_env("LCMA_L2PERSIST")) << 20;
        int maxp = 0, dev0 = 0;
        cudaGetDevice(&dev0);
        cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev0);
        want = std::min(want, (size_t)maxp);
        size_t cur = 0;
        cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
        if (cur < want) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
        int maxw = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev);
        const size_t region = (size_t)g.nslot * p->ctas * kBM * p->bn * sizeof(float);
        const size_t nb = std::min(region, (size_t)maxw);
        attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[na].val.accessPolicyWindow.base_ptr = P;
        attr[na].val.accessPolicyWindow.num_bytes = nb;
        attr[na].val.accessPolicyWindow.hitRatio = nb ? (float)std::min(1.0, (double)want / (double)nb) : 0.f;
        attr[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        ++na;
    }
    // diagnostics: a persisting access-policy window over the A operand
    // (A~ panels are re-read by the lockstep rounds of a band)
    if (!classical && !(P && g.epi_mode == EPI_FUSED && diag_env("LCMA_L2PERSIST")) && diag_env("LCMA_L2PERSIST_A")) {
        size_t want = (size_t)std::atoll(diag_env("LCMA_L2PERSIST_A")) << 20;
        int maxp = 0, maxw = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
        cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev);
        want = std::min(want, (size_t)maxp);
        size_t cur = 0;
        cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
        if (cur < want) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
        const size_t region = (size_t)S.R * p->Mb * p->Kb * p->e;
        const size_t nb = std::min(region, (size_t)maxw);
        attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[na].val.accessPolicyWindow.base_ptr = const_cast<void*>(Aop);
        attr[na].val.accessPolicyWindow.num_bytes = nb;
        attr[na].val.accessPolicyWindow.hitRatio = nb ? (float)std::min(1.0, (double)want / (double)nb) : 0.f;
        attr[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaError_t e;
    if (f8) {
        cfg.dynamicSmemBytes = regh ? KernelCfg<2, 128, 0, true, 0, true>::kSmemBytes
                                    : KernelCfg<2, 128, 0, false, 0, true>::kSmemBytes;
        e = regh ? cudaLaunchKernelEx(&cfg, umma_gemm_kernel<2, 128, 0, true, 0, false, true>, ta, tb, g)
                 : cudaLaunchKernelEx(&cfg, umma_gemm_kernel<2, 128, 0, false, 0, false, true>, ta, tb, g);
    } else if (pf) {
        g.kgrid = S.k;
        g.pf_Kb = (int)p->Kb;
        for (int r = 0; r < S.R; ++r) {
            g.pf_blk0[r] = g.pf_blk1[r] = -1;
            g.pf_s0[r] = g.pf_s1[r] = 0;
            for (int a = 0; a < S.m; ++a)
                for (int b = 0; b < S.k; ++b) {
                    const int v = S.u(r, a, b);
                    if (!v) continue;
                    if (g.pf_blk0[r] < 0) { g.pf_blk0[r] = (int8_t)(a * S.k + b); g.pf_s0[r] = (int8_t)v; }
                    else { g.pf_blk1[r] = (int8_t)(a * S.k + b); g.pf_s1[r] = (int8_t)v; }
                }
        }
        g.ngrid = S.n;
        g.pf_Nb = (int)p->Nb;
        for (int r = 0; r < S.R; ++r) {
            g.pfb_blk0[r] = g.pfb_blk1[r] = -1;
            g.pfb_s0[r] = g.pfb_s1[r] = 0;
            for (int a = 0; a < S.k; ++a)
                for (int b = 0; b < S.n; ++b) {
                    const int v = S.v(r, a, b);
                    if (!v || pf != 2) continue;
                    if (g.pfb_blk0[r] < 0) { g.pfb_blk0[r] = (int8_t)(a * S.n + b); g.pfb_s0[r] = (int8_t)v; }
                    else { g.pfb_blk1[r] = (int8_t)(a * S.n + b); g.pfb_s1[r] = (int8_t)v; }
                }
        }
        g.debug &= ~(16 | 32 | 64);   // stale-operand / extra-load diagnostics do not apply
        if (pf == 2) {
            cfg.dynamicSmemBytes = Cfg<2, 256, 0, false, 2>::kSmemBytes;
            e = cudaLaunchKernelEx(&cfg, umma_gemm_kernel<2, 256, 0, true, 2>, ta, tb, g);
        } else {
            cfg.dynamicSmemBytes = Cfg<2, 256, 0, false, 1>::kSmemBytes;
            e = cudaLaunchKernelEx(&cfg, umma_gemm_kernel<2, 256, 0, true, 1>, ta, tb, g);
        }
    } else if (p->cg == 2 && p->bn == 256 && qf == 2) {
        cfg.dynamicSmemBytes = Cfg<2, 256, 2>::kSmemBytes;
        e = cudaLaunchKernelEx(&cfg, umma_gemm_kernel<2, 256, 2, true>, ta, tb, g);
    } else if (p->cg == 2 && p->bn == 256 && qf) {
        cfg.dynamicSmemBytes = Cfg<2, 256, 1>::kSmemBytes;
        e = cudaLaunchKernelEx(&cfg, umma_gemm_kernel<2, 256, 1, true>, ta, tb, g);
    } else if (p->cg == 2 && p->bn == 256 && regh) {
        cfg.dynamicSmemBytes = cst_regh ? Cfg<2, 256>::kSmemBytes : Cfg<2, 256, 0, false, 0, false, false>::kSmemBytes;
        e = dyn ? (cst_regh ? cudaLaunchKernelEx(&cfg, umma_gemm_kernel<2, 256, 0, true, 0, true>, ta, tb, g)
                            : cudaLaunchKernelEx(&cfg, umma_gemm_kernel<2, 256, 0, true, 0, true, false, false>, ta, tb, g))
            : cst_regh ? cudaLaunchKernelEx(&cfg, umma_gemm_kernel<2, 256, 0, true>, ta, tb, g)
                       : cudaLaunchKernelEx(&cfg, umma_gemm_kernel<2, 256, 0, true, 0, false, false, false>, ta, tb, g);
    } else if (p->cg == 2 && p->bn == 256) {
        cfg.dynamicSmemBytes = Cfg<2, 256, 0, true>::kSmemBytes;
        e = dyn ? cudaLaunchKernelEx(&cfg, umma_gemm_kernel<2, 256, 0, false, 0, true>, ta, tb, g)
                : cudaLaunchKernelEx(&cfg, umma_gemm_kernel<2, 256>, ta, tb, g);
    } else if (p->cg == 2) {
        cfg.dynamicSmemBytes = Cfg<2, 128>::kSmemBytes;
        e = cudaLaunchKernelEx(&cfg, umma_gemm_kernel<2, 128>, ta, tb, g);
    } else if (p->bn == 256) {
        cfg.dynamicSmemBytes = Cfg<1, 256>::kSmemBytes;
        e = cudaLaunchKernelEx(&cfg, umma_gemm_kernel<1, 256>, ta, tb, g);
    } else {
        cfg.dynamicSmemBytes = Cfg<1, 128>::kSmemBytes;
        e = cudaLaunchKernelEx(&cfg, umma_gemm_kernel<1, 128>, ta, tb, g);
    }
    if (e != cudaSuccess) return fail(LCMA_ERR_CUDA, std::string("cudaLaunchKernelEx: ") + cudaGetErrorString(e));
    lcma_status ls = check_launch("umma_gemm_kernel");
    if (t_ev_end) cudaEventRecord(t_ev_end, st);
    return ls;
}

lcma_status launch_simt(const lcma_plan_s* p, const float* A, const float* B, float* H,
                        cudaStream_t st) {
    const Scheme& S = p->sch;
    const bool classical = p->scheme_id == SCHEME_CLASSICAL;
    SimtParams s;
    std::memset(&s, 0, sizeof(s));
    s.A = A; s.B = B; s.H = H;
    s.b_kmajor = p->d.b_layout == 1;
    if (classical) {
        s.Mr = p->d.M; s.Nr = p->d.N; s.Kr = p->d.K;
        s.lda = p->d.K; s.ldb = s.b_kmajor ? p->d.K : p->d.N; s.ldh = p->d.N;
    } else {
        s.Mr = p->Mb; s.Nr = p->Nb; s.Kr = p->Kb;
        s.lda = p->Kb; s.ldb = s.b_kmajor ? p->Kb : p->Nb; s.ldh = p->Nb;
        s.sAr = p->Mb * p->Kb; s.sBr = p->Kb * p->Nb; s.sHr = p->Mb * p->Nb;
    }
    dim3 grid((unsigned)cdiv(s.Nr, 128), (unsigned)cdiv(s.Mr, 128), classical ? 1 : S.R);
    simt_sgemm_batched_kernel<<<grid, 256, 0, st>>>(s);
    return check_launch("simt_sgemm_batched_kernel");
}

// In-place single-term operands apply to the fused (FUSED_H) GEMM through
// its lean producer loop: not in diagnostics runs whose knobs change what the
// producer issues (the general loop does not read in place).
bool direct_ok(const lcma_plan_s* p) {
    if (p->variant != LCMA_VARIANT_FUSED_H || p->nbatch != 1 || p->d.b_layout != 1) return false;
    if (diag_env("LCMA_DEBUG") && (std::atoi(diag_env("LCMA_DEBUG")) & (16 | 32 | 64 | 4096))) return false;
    if (diag_env("LCMA_DIRECT") && std::atoi(diag_env("LCMA_DIRECT")) == 0) return false;
    return true;
}

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
    auto x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
    return na && nb && x < y + nb && y < x + na;
}

lcma_status run(lcma_plan_t p, const void* A, const void* B, const void* Bt_user, void* C, void* ws,
                size_t ws_bytes, void* stream) {
    t_err.clear();
    t_launches = 0;
    if (!p || !A || !C || (!B && !Bt_user)) return fail(LCMA_ERR_INVALID_VALUE, "null argument");
    auto mis = [](const void* x) { return (reinterpret_cast<uintptr_t>(x) & 15) != 0; };
    if (mis(A) || mis(C) || (B && mis(B)) || (Bt_user && mis(Bt_user)) || (ws && mis(ws)))
        return fail(LCMA_ERR_MISALIGNED, "device pointers must be 16-byte aligned");
    if (ws_bytes < p->ws_bytes || (p->ws_bytes && !ws))
        return fail(LCMA_ERR_WORKSPACE, "workspace smaller than lcma_workspace_size()");
    const size_t eo = (p->d.out_dtype == LCMA_FP32 || p->d.out_dtype == LCMA_TF32) ? 4 : p->e;
    const size_t cb = (size_t)p->d.M * p->d.N * eo;
    if (overlaps(C, cb, A, (size_t)p->d.M * p->d.K * p->e) ||
        (B && overlaps(C, cb, B, (size_t)p->d.K * p->d.N * p->e)) ||
        overlaps(C, cb, ws, p->ws_bytes))
        return fail(LCMA_ERR_INVALID_VALUE, "C must not overlap A, B or the workspace");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    uint8_t* w = reinterpret_cast<uint8_t*>(ws);
    const bool classical = p->scheme_id == SCHEME_CLASSICAL;
    const bool fp32 = p->d.dtype == LCMA_FP32;
    if (p->d.dtype == LCMA_FP8_E4M3) {
        // Combine A with the 1 x 128 quantization fused in, the same
        // for B unless B~ was quantized offline, then the block-scaled
        // GEMM with the fused Combine H (classical: quantization passes + GEMM)
        void* At = w + p->off_At;
        lcma_status rq = launch_combine_q8(p, A, At, false, st);
        if (rq != LCMA_OK) return rq;
        const void* Bq = Bt_user;
        if (!Bq) {
            rq = launch_combine_q8(p, B, w + p->off_Bt, true, st);
            if (rq != LCMA_OK) return rq;
            Bq = w + p->off_Bt;
        }
        return launch_umma(p, At, Bq, C, classical ? nullptr : reinterpret_cast<float*>(w + p->off_P),
                           classical ? nullptr : reinterpret_cast<int*>(w + p->off_flags),
                           reinterpret_cast<int*>(w + p->off_sched), nullptr, st);
    }
    if (classical) {
        if (fp32) {
            if (p->d.out_dtype != LCMA_FP32) return fail(LCMA_ERR_NOT_SUPPORTED, "fp32 output only");
            return launch_simt(p, (const float*)A, (const float*)B, (float*)C, st);
        }
        return launch_umma(p, A, B, C, nullptr, nullptr, reinterpret_cast<int*>(w + p->off_sched), nullptr, st);
    }
    void* At = w + p->off_At;
    const void* Bt = Bt_user;
    lcma_status rs = LCMA_OK;
    const bool dir = direct_ok(p);
    const bool dirA = dir && p->any_a_dir;
    const bool dirB = dir && p->any_b_dir && !Bt_user && B;
    if (p->variant != LCMA_VARIANT_PRODUCER && !Bt_user) {
        // Combine A (Eq. 3) and Combine B (Eq. 4) of this call in one launch
        rs = launch_combine_ab(p, A, At, B, w + p->off_Bt, st, dirA, dirB);
        if (rs != LCMA_OK) return rs;
        Bt = w + p->off_Bt;
    } else if (p->variant != LCMA_VARIANT_PRODUCER) {
        rs = launch_combine(p, A, At, false, st, dirA);            // Combine A (Eq. 3)
        if (rs != LCMA_OK) return rs;
    }
    // variant 3: Combine B joins Combine A in the producer path when B is
    // given per call, stored N x K, tiled exactly and <= 2 B blocks per product
    int pf = 0;
    if (p->variant == LCMA_VARIANT_PRODUCER) {
        pf = 1;
        const Scheme& S = p->sch;
        bool two = p->d.b_layout == 1 && !Bt_user && p->d.N == (int64_t)S.n * p->Nb &&
                   p->d.K == (int64_t)S.k * p->Kb && !diag_env("LCMA_PF_A_ONLY");
        for (int r = 0; r < S.R && two; ++r) {
            int nz = 0;
            for (int a = 0; a < S.k; ++a)
                for (int b = 0; b < S.n; ++b) nz += S.v(r, a, b) != 0;
            two = nz >= 1 && nz <= 2;
        }
        if (two) pf = 2;
    }
    if (!Bt && pf != 2) {
        rs = launch_combine(p, B, w + p->off_Bt, true, st, dirB);  // Combine B (Eq. 4)
        if (rs != LCMA_OK) return rs;
        Bt = w + p->off_Bt;
    }
    if (fp32) {
        float* H = reinterpret_cast<float*>(w + p->off_H);
        rs = launch_simt(p, (const float*)At, (const float*)Bt, H, st);   // Eq. 5
        if (rs != LCMA_OK) return rs;
        return launch_combine_h(p, H, C, st);                              // Eq. 6
    }
    if (p->variant == LCMA_VARIANT_TWO_LEVEL) {
        // inner level: one fused GEMM per outer product q over the contiguous
        // slices At[q*R0 .. q*R0+R0-1], Bt[...] (r = q*R0 + r2, reading 3),
        // writing H_q (fp32); outer level: Combine H of the base scheme
        const Scheme& B0 = *scheme_get(p->sch.base_id);
        const lcma_plan_s* in = p->inner;
        float* H = reinterpret_cast<float*>(w + p->off_H);
        const size_t a_slice = (size_t)B0.R * p->Mb * p->Kb * p->e;
        const size_t b_slice = (size_t)B0.R * p->Kb * p->Nb * p->e;
        const size_t h_slice = (size_t)(B0.m * p->Mb) * (B0.n * p->Nb);
        float* Pi = reinterpret_cast<float*>(w + p->off_inner + in->off_P);
        int* Fi = reinterpret_cast<int*>(w + p->off_inner + in->off_flags);
        int* Si = reinterpret_cast<int*>(w + p->off_inner + in->off_sched);
        // all R0 inner GEMMs in one batched launch: batch q reads the slices
        // At[q*R0 .. q*R0+R0-1], Bt[...] and writes H_q = H + q * h_slice
        (void)a_slice; (void)b_slice; (void)h_slice;
        rs = launch_umma(in, At, Bt, H, Pi, Fi, Si, nullptr, st);
        if (rs != LCMA_OK) return rs;
        return launch_combine_h_ex(p, B0, B0.m * p->Mb, B0.n * p->Nb, H, C, st);
    }
    if (p->variant == LCMA_VARIANT_UNFUSED) {
        float* H = reinterpret_cast<float*>(w + p->off_H);
        rs = launch_umma(p, At, Bt, C, nullptr, nullptr, reinterpret_cast<int*>(w + p->off_sched), H, st);
        if (rs != LCMA_OK) return rs;
        return launch_combine_h(p, H, C, st);
    }
    if (p->variant == LCMA_VARIANT_PRODUCER)   // Combine A (and B) inside the GEMM's producer path
        return launch_umma(p, A, pf == 2 ? B : Bt, C, reinterpret_cast<float*>(w + p->off_P),
                           reinterpret_cast<int*>(w + p->off_flags), nullptr, nullptr, st, pf);
    return launch_umma(p, At, Bt, C, reinterpret_cast<float*>(w + p->off_P),
                       reinterpret_cast<int*>(w + p->off_flags), reinterpret_cast<int*>(w + p->off_sched), nullptr,
                       st, 0, dirA ? A : nullptr, dirB ? B : nullptr);
}

}  // namespace

// Copies the diagnostic counters (8 per CTA) to host memory; 0 on success.
extern "C" int lcma_debug_stats(unsigned long long* host, int n) {
    if (!g_stats) return -1;
    return cudaMemcpy(host, g_stats, (size_t)n * sizeof(unsigned long long), cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : -1;
}

extern "C" lcma_status lcma_gemm(lcma_plan_t p, const void* A, const void* B, void* C, void* ws,
                                 size_t ws_bytes, void* stream) {
    if (p && !B) return fail(LCMA_ERR_INVALID_VALUE, "null B");
    return run(p, A, B, nullptr, C, ws, ws_bytes, stream);
}

extern "C" lcma_status lcma_gemm_precombined(lcma_plan_t p, const void* A, const void* Bt, void* C,
                                             void* ws, size_t ws_bytes, void* stream) {
    if (!p || !Bt) return fail(LCMA_ERR_INVALID_VALUE, "null argument");
    if (p->scheme_id == SCHEME_CLASSICAL && p->d.dtype != LCMA_FP8_E4M3)
        return run(p, A, Bt, nullptr, C, ws, ws_bytes, stream);   // classical: Bt is B itself
    return run(p, A, nullptr, Bt, C, ws, ws_bytes, stream);
}

extern "C" lcma_status lcma_precombine_b(lcma_plan_t p, const void* B, void* Bt, void* stream) {
    t_err.clear();
    t_launches = 0;
    if (!p || !B || !Bt) return fail(LCMA_ERR_INVALID_VALUE, "null argument");
    if ((reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(Bt)) & 15)
        return fail(LCMA_ERR_MISALIGNED, "device pointers must be 16-byte aligned");
    if (p->d.dtype == LCMA_FP8_E4M3)      // quantized B~ (classical: B itself, quantized)
        return launch_combine_q8(p, B, Bt, true, reinterpret_cast<cudaStream_t>(stream));
    if (p->scheme_id == SCHEME_CLASSICAL) return fail(LCMA_ERR_INVALID_VALUE, "classical plan has no Bt");
    return launch_combine(p, B, Bt, true, reinterpret_cast<cudaStream_t>(stream));
}

// Workspace layout accessor: byte offset of region `which` (0: A~ -- for
// LCMA_FP8_E4M3 the E4M3 A~ followed by its scale chunks --, 1: B~ when B is
// combined per call) inside the plan's workspace.
extern "C" lcma_status lcma_workspace_region(lcma_plan_t p, int32_t which, size_t* offset) {
    if (!p || !offset || which < 0 || which > 1) return fail(LCMA_ERR_INVALID_VALUE, "bad argument");
    const bool has = p->d.dtype == LCMA_FP8_E4M3 || p->scheme_id != SCHEME_CLASSICAL;
    if (!has) return fail(LCMA_ERR_INVALID_VALUE, "plan has no A~ / B~ region");
    *offset = which == 0 ? p->off_At : p->off_Bt;
    return LCMA_OK;
}

// Measurement hook: when set (non-NULL cudaEvent_t handles), every following
// lcma_gemm* call on this thread records `ev_start` / `ev_end` on the call's
// stream immediately before / after the tcgen05 GEMM kernel, so a caller can
// time the dominant kernel live.  Pass NULLs to disable.
extern "C" void lcma_set_kernel_events(void* ev_start, void* ev_end) {
    t_ev_start = reinterpret_cast<cudaEvent_t>(ev_start);
    t_ev_end = reinterpret_cast<cudaEvent_t>(ev_end);
}

// Diagnostics: co-resident clusters of `cluster_size` CTAs for the tcgen05
// GEMM kernel configuration (cudaOccupancyMaxActiveClusters); -1 on error.
// Diagnostics (LCMA_TIMELINE=1): copies n entries of the per-product timeline
// ([cta][512][4] globaltimer ns) to host memory; 0 on success.
extern "C" int lcma_debug_timeline(unsigned long long* host, long long n) {
    if (!g_tl) return -1;
    return cudaMemcpy(host, g_tl, (size_t)n * sizeof(unsigned long long), cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : -1;
}

// Diagnostics: fused Combine-H partial tile transfers per group that go to L2
// (the on-chip homes excluded) and live partials per CTA, for scheme_id.
extern "C" double lcma_debug_l2_partial_tiles(int32_t scheme_id, int32_t* live) {
    const ProductOrder& po = scheme_product_order(scheme_id);
    if (live) *live = po.nslot;
    return po.l2_tiles;
}

extern "C" int lcma_debug_max_clusters(int cluster_size) {
    if (cudaFuncSetAttribute(umma_gemm_kernel<2, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Cfg<2, 256, 0, true>::kSmemBytes) != cudaSuccess) { cudaGetLastError(); return -1; }
    if (cluster_size > 8)
        cudaFuncSetAttribute(umma_gemm_kernel<2, 256>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg;
    std::memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(cluster_size);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Cfg<2, 256, 0, true>::kSmemBytes;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster_size;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, umma_gemm_kernel<2, 256>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    return n;
}
