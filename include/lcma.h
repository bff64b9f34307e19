/*
 * lcma.h -- C ABI of the B200-native LCMA GEMM library (liblcma.so).
 *
 * The library computes C = A * B (Eq. 1) either with a
 * classical tcgen05 GEMM or through a Lower-Complexity Matrix Multiplication
 * Algorithm <m,k,n,R,U,V,W>: Combine A (Eq. 3),
 * Combine B (Eq. 4), R sub-GEMMs H_r = At_r * Bt_r (Eq. 5,
 * P:630-634) and Combine H (Eq. 6), organised by the paper's
 * group-parallel fusion (Alg. 2; Split-Group P:362-387;
 * Cache-Aware P:391-396) and chosen by the Decision Module.
 * "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n.
 *
 * Conventions (all entry points):
 *  - Shapes are (M, N, K); A is M x K, B is K x N (b_layout 0, the paper's
 *    layout) or N x K (b_layout 1, nn.Linear weight), C is M x N; all
 *    row-major with the leading dimension equal to the row length.
 *  - A, B, Bt, C and the workspace are DEVICE pointers owned by the caller.
 *    They must be 16-byte aligned and row lengths must be multiples of
 *    16 bytes (TMA), else LCMA_ERR_MISALIGNED.  There is no CPU fallback and
 *    no silent copy.
 *  - The plan owns host metadata only; it is immutable after creation and
 *    may be shared across threads.  lcma_free(NULL) is a no-op.
 *  - lcma_gemm* only enqueue work on `cuda_stream` (a cudaStream_t; NULL =
 *    legacy default stream): no allocation, no host synchronisation, so they
 *    are CUDA-graph capturable.  Launch failures return LCMA_ERR_CUDA with
 *    the CUDA error string in lcma_last_error(); asynchronous faults surface
 *    at the caller's next synchronisation.
 *  - The workspace must be zero-filled once before its first use (the
 *    library keeps its schedule counter and split-group flags at zero between
 *    calls).  A workspace may be used by ONE in-flight call at a time (two
 *    streams need two workspaces).  If a launch fails or is aborted mid-way
 *    (LCMA_ERR_CUDA, a device fault), zero the workspace again before reuse.
 *  - The tcgen05 GEMM is a persistent kernel sized to the device's co-resident
 *    CTA pairs; the plan is bound to the device current at lcma_plan* time.
 *  - Results are bitwise deterministic for a fixed plan: no floating-point
 *    atomics; split groups merge in a fixed order (reading 10).
 */
#ifndef LCMA_H_
#define LCMA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    LCMA_OK = 0,
    LCMA_ERR_INVALID_VALUE = 1,  /* bad shape/enum/pointer, aliasing C with inputs */
    LCMA_ERR_NOT_SUPPORTED = 2,  /* combination not built (e.g. dtype x algo)       */
    LCMA_ERR_MISALIGNED = 3,     /* TMA 16-byte rules violated                      */
    LCMA_ERR_SCHEME_INVALID = 4, /* Brent identity fails; see lcma_last_error */
    LCMA_ERR_COEFF_RANGE = 5,    /* coefficient outside {-1,0,1}      */
    LCMA_ERR_PARSE = 6,          /* scheme file syntax error, line in message */
    LCMA_ERR_WORKSPACE = 7,      /* workspace too small                             */
    LCMA_ERR_CUDA = 8            /* CUDA runtime/driver error                       */
} lcma_status;

typedef enum {
    LCMA_BF16 = 0,   /* bf16 storage, bf16 MMA, fp32 accumulation                  */
    LCMA_FP16 = 1,   /* fp16 storage, fp16 MMA, fp32 accumulation                  */
    LCMA_TF32 = 2,   /* fp32 storage, tf32 MMA (RN-away rounding of combined terms) */
    LCMA_FP32 = 3,   /* fp32 storage, true fp32 SIMT arithmetic                     */
    LCMA_FP8_E4M3 = 4 /* bf16 A and B in, FP8 E4M3 MMA: the combines quantize
                        every 1 x 128 block (one row, 128 consecutive K) of A~_r and
                        B~_r with a power-of-two UE8M0 scale (quantization fused into
                        Combine A; reading 23); block-scaled
                        tcgen05 MMA, fp32 accumulation; C bf16 (out_dtype BF16 or
                        FP8_E4M3) or fp32.  B must be N x K (b_layout 1).  The
                        classical plan quantizes A (and B) with the same pass.     */
} lcma_dtype;

typedef enum {
    LCMA_ALGO_AUTO = 0,        /* Decision Module picks               */
    LCMA_ALGO_CLASSICAL = 1,   /* single tcgen05 GEMM (the no-LCMA reference)     */
    LCMA_ALGO_STRASSEN = 2,    /* <2,2,2;7>, depth 1                      */
    LCMA_ALGO_STRASSEN2 = 3,   /* <4,4,4;49> = Strassen composed twice, depth 2 */
    LCMA_ALGO_LADERMAN = 4,    /* <3,3,3;23>                              */
    LCMA_ALGO_SCHEME = 5       /* scheme registered from a file (scheme_id)       */
} lcma_algo;

typedef enum {
    LCMA_VARIANT_AUTO = 0,
    LCMA_VARIANT_UNFUSED = 1,  /* Algorithm 1: At, Bt, H materialised     */
    LCMA_VARIANT_FUSED_H = 2,  /* Algorithm 2: At/Bt materialised by group-parallel
                                  combines, GEMM + Combine H fused       */
    LCMA_VARIANT_PRODUCER = 3, /* Combine A in the GEMM producer path (TMA loads of
                                  the nonzero A blocks of U_r, summed in shared
                                  memory before the MMAs); Combine B too when B is
                                  passed per call, stored N x K and N, K are tiled
                                  exactly (else B~ materialised / offline);
                                  Combine H fused.  Needs <= 2 blocks per product
                                  (Strassen), 16-bit data and M, K tiled exactly
                                  by the block grid, else LCMA_ERR_NOT_SUPPORTED.
                                  Measured 3-4.6x slower than FUSED_H on B200
                                  (DESIGN.md s.7); never chosen by AUTO.          */
    LCMA_VARIANT_TWO_LEVEL = 4 /* two-level scheme (Strassen^2 = Strassen o Strassen,
                                  P:663): combines of the composed scheme, then one
                                  fused-Combine-H GEMM per outer product writing the
                                  outer H_q in fp32, then the outer Combine H as an
                                  HBM pass (Eq. 6 at the outer level)               */
} lcma_variant;

typedef struct lcma_plan_s* lcma_plan_t;

/* Hardware triple of P:171-175: FLOPS_x (GEMM stage), FLOPS_+ (combine adds),
 * beta (off-chip bandwidth in ELEMENTS/s of the dtype), worker count. */
typedef struct {
    double flops_mul;
    double flops_add;
    double beta_elems;
    int32_t workers;
} lcma_hw_profile;

typedef struct {
    int64_t M, N, K;
    lcma_dtype dtype;
    lcma_dtype out_dtype;     /* C element type: same as dtype, or LCMA_FP32      */
    lcma_algo algo;
    int32_t scheme_id;        /* for LCMA_ALGO_SCHEME                              */
    int32_t b_layout;         /* 0: B is K x N (paper), 1: B is N x K              */
    int32_t b_static;         /* 1: lcma_gemm_precombined will be used     */
    int32_t variant;          /* lcma_variant                                      */
    int32_t schedule;         /* 0 auto (classical 5, LCMA 1); 1 = 4: cache-aware lockstep rounds
                                 (group w + i*W to unit w) + split tail;
                                 2 paper's contiguous split-group order;
                                 3 whole groups only (group-parallel, no split);
                                 5 whole groups handed out in raster order at run
                                   time (ticket counter in the workspace: the groups
                                   in flight stay a compact window of the raster)
                                   + the split tail's segments handed out at run
                                   time to the pairs that finish first;
                                 6 static lockstep rounds + the run-time tail;
                                 7 whole groups at run time (as 5) + the static
                                   tail, merged by all of a split group's pairs */
    int32_t num_ctas;         /* 0 = one per SM                                    */
    const lcma_hw_profile* hw;/* NULL -> built-in B200 profile                     */
    int32_t decision_model;   /* algo AUTO: 0 = this build's B200-calibrated model
                                 (reading 19), 1 = the paper's model
                                 verbatim (as lcma_decide)              */
    /* tuning (0 = the measured default for the shape; results are identical
       for every value, only the time changes) */
    int32_t raster_rows;      /* group raster: band height in tile rows            */
    int32_t reserved;         /* must be 0                                         */
} lcma_plan_desc;

typedef struct {
    lcma_algo algo;           /* resolved algorithm                               */
    int32_t variant;          /* resolved lcma_variant                            */
    int32_t m, k, n, R, depth;
    char scheme[64];
    int64_t Mb, Nb, Kb;       /* padded block extents (>= ceil(M/m) etc.)  */
    int32_t BM, BN, BK;
    int32_t cta_group;        /* 1: cta_group::1 128-row tiles, 2: CTA pairs, 256-row tiles */
    int32_t groups, tiles, ctas, waves, group_waves, split_groups;
    double t_pred_classical, t_pred_choice, speedup_pred;  /* seconds, model      */
    int32_t memory_bound;     /* Eq. stdgemm held                          */
    int32_t lcma_condition;   /* Eq. lcma_condition holds                  */
    int32_t fused_condition;  /* Eq. fused_condition holds                 */
    size_t workspace_bytes, btilde_bytes;
    int32_t partial_slots;    /* fused Combine H: live fp32 C_ij partial tiles per
                                 CTA of a whole group (product order + interval
                                 colouring); 0 for classical / unfused            */
} lcma_plan_info;

/* Create a plan for C = A*B of shape (M,N,K).  out: new plan on LCMA_OK. */
lcma_status lcma_plan(int64_t M, int64_t N, int64_t K, lcma_dtype dtype,
                      lcma_algo algo, lcma_plan_t* out);
lcma_status lcma_plan_ex(const lcma_plan_desc* desc, lcma_plan_t* out);
void lcma_free(lcma_plan_t plan);
lcma_status lcma_plan_get_info(lcma_plan_t plan, lcma_plan_info* out);
lcma_status lcma_workspace_size(lcma_plan_t plan, size_t* bytes);
lcma_status lcma_btilde_size(lcma_plan_t plan, size_t* bytes);

/* C = A*B on the device.  workspace: >= lcma_workspace_size bytes (zeroed
 * before first use).  Number of kernels launched is reported by
 * lcma_last_launch_count(). */
lcma_status lcma_gemm(lcma_plan_t plan, const void* A, const void* B, void* C,
                      void* workspace, size_t workspace_bytes, void* cuda_stream);

/* Byte offset of a workspace region (which 0: A~, 1: B~ combined per call;
 * LCMA_FP8_E4M3: the E4M3 operand followed by its UE8M0 scale chunks).  For
 * tests and tools that read the materialised combines back; INVALID_VALUE
 * for a plan without such a region (a classical bf16/fp16/tf32 plan). */
lcma_status lcma_workspace_region(lcma_plan_t plan, int32_t which, size_t* offset);

/* Offline Combine B for static weights: Bt = group-combined
 * B for this plan's scheme and extents (lcma_btilde_size bytes).  Bt is bound
 * to the plan's (N, K, dtype, scheme, extents, b_layout); lcma_gemm_precombined
 * trusts the caller to pass a matching Bt.  LCMA_FP8_E4M3: Bt holds the
 * quantized B~ (E4M3 [R][Nb][Kb]) followed by its UE8M0 scale chunks
 * ([R][Nb/128][Kb/128] x 512 bytes, the tcgen05 block-scale layout); the
 * classical FP8 plan accepts it too (B quantized once, R = 1). */
lcma_status lcma_precombine_b(lcma_plan_t plan, const void* B, void* Bt, void* cuda_stream);
lcma_status lcma_gemm_precombined(lcma_plan_t plan, const void* A, const void* Bt, void* C,
                                  void* workspace, size_t workspace_bytes, void* cuda_stream);

/* Decision Module only (host, no device): fills algo/scheme/t_pred_* and
 * the Eq. flags.  fused: 1 -> Eq. fused_condition model. */
lcma_status lcma_decide(int64_t M, int64_t N, int64_t K, lcma_dtype dtype,
                        const lcma_hw_profile* hw, int32_t fused, lcma_plan_info* out);

/* Scheme registry.  Built-in ids: 0 classical(1,1,1), 1 Strassen, 2 Strassen^2,
 * 3 Laderman.  Registration validates the Brent identity. */
lcma_status lcma_scheme_register_file(const char* path, int32_t* scheme_id);
lcma_status lcma_scheme_register(int32_t m, int32_t k, int32_t n, int32_t R,
                                 const int8_t* U, const int8_t* V, const int8_t* W,
                                 const char* name, int32_t* scheme_id);
/* mknR[4] <- (m,k,n,R); U/V/W (may be NULL) <- R*m*k, R*k*n, R*m*n int8. */
lcma_status lcma_scheme_get(int32_t scheme_id, int32_t* mknR, int8_t* U, int8_t* V, int8_t* W);

/* Split-group schedule of a plan (host view of the device enumeration):
 * for CTA `cta`, writes up to `cap` units as (group, r_begin, r_end, role)
 * int32 quadruples (role 0 whole group, 1 owner segment, 2 contributing
 * segment) and returns the count in *n. */
lcma_status lcma_plan_schedule(lcma_plan_t plan, int32_t cta, int32_t* units, int32_t cap,
                               int32_t* n);

/* Measurement hook: when non-NULL cudaEvent_t handles are set, each later
 * lcma_gemm* call on this thread records ev_start / ev_end on its stream right
 * before / after the tcgen05 GEMM kernel (the dominant kernel; for two-level
 * plans, around all inner GEMM launches), so callers can time it live with
 * CUDA events.  NULL, NULL disables. */
void lcma_set_kernel_events(void* ev_start, void* ev_end);
/* Diagnostics (LCMA_STATS=1 in the environment): copies n per-CTA wait-cycle
 * counters to host memory; returns 0 on success. */
int lcma_debug_stats(unsigned long long* host, int n);
/* Diagnostics (host only): fused Combine-H partial tile transfers per group
 * that still go through L2 once the two most-updated partial slots live on
 * chip (epilogue registers; shared memory for column half 0), for a scheme
 * id; *live (if non-NULL) receives the partials live at once per CTA. */
double lcma_debug_l2_partial_tiles(int32_t scheme_id, int32_t* live);
/* Diagnostics (LCMA_TIMELINE=1 in the environment): copies n entries of the
 * per-product timeline of the last tcgen05 GEMM launch ([cta][512][4]
 * globaltimer ns: MMA slot acquired, MMA issue done, epilogue has the
 * accumulator, epilogue released it) to host memory; returns 0 on success. */
int lcma_debug_timeline(unsigned long long* host, long long n);

/* Thread-local message for the last error on this thread ("" if none). */
const char* lcma_last_error(void);
/* Number of kernels the last lcma_gemm* call on this thread enqueued. */
int32_t lcma_last_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* LCMA_H_ */
