// decision.h -- the Decision Module of Sec. III-C, product copy.
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

#include "schemes.h"

namespace lcma {

struct Profile {
    double flops_mul;   // FLOPS_x: GEMM-stage throughput
    double flops_add;   // FLOPS_+: combine add/sub throughput
    double beta;        // off-chip bandwidth, elements/s of the dtype
    // B200-calibrated model only (decide_b200):
    double beta_combine = 0.0;    // combine kernels' element rate (elements/s)
    double alpha_partial = 0.0;   // fused Combine-H slowdown per (L2 partial / operand bytes)^2
    double epi_overhead = 0.0;    // fused GEMM time over R/mnk of the classical kernel's, on-chip part
};

struct StageCost {
    double flops, mem, time;
    bool compute_bound;
};

// Per-stage costs of Table "cost_model" for scheme s on (M,N,K);
// ceil quotients for non-divisible shapes.  fused: Combine H fused into the
// GEMM.  b_static: Combine B done offline -> zero cost.
void stage_costs(const Scheme& s, double M, double N, double K, const Profile& hw, bool fused,
                 bool b_static, StageCost out[4]);
double gemm_intensity(double M, double N, double K);          // Eq. stdgemm LHS
double estimate_time_std(double M, double N, double K, const Profile& hw);
double estimate_time(const Scheme& s, double M, double N, double K, const Profile& hw, bool fused,
                     bool b_static);
double condition_lhs(const Scheme& s, double M, double N, double K, bool fused);  // P:250 / P:260

struct DecisionResult {
    int scheme_id;          // SCHEME_CLASSICAL if the standard GEMM wins
    bool memory_bound;      // Eq. stdgemm held -> early return
    double t_std, t_choice;
    std::vector<std::pair<int, double>> candidates;   // (scheme id, predicted time)
};

// select: Eq. stdgemm early exit, else argmin of estimate_time over
// {classical} U candidates; ties -> classical, then lower id.
DecisionResult decide(const std::vector<int>& candidate_ids, double M, double N, double K,
                      const Profile& hw, bool fused, bool b_static);

// The same selection with this build's calibrated B200 cost model (see
// decision.cpp); elem_bytes = storage bytes of the dtype.
double estimate_time_b200(const Scheme& s, double M, double N, double K, const Profile& hw, bool fused,
                          bool b_static, double elem_bytes);
DecisionResult decide_b200(const std::vector<int>& candidate_ids, double M, double N, double K,
                           const Profile& hw, bool fused, bool b_static, double elem_bytes);

// Built-in B200 profile per dtype (0 bf16, 1 fp16, 2 tf32, 3 fp32), overridable
// through the environment variable LCMA_PROFILE="flops_mul=..,flops_add=..,beta_elems=..".
Profile default_profile(int dtype);

}  // namespace lcma
