#pragma once

#include <vector>

#include "ctx.cuh"
#include "gemm_tf32x3.cuh"

namespace spngd {

struct FactorPlan {
  std::vector<GemmProblem> probs;
  std::vector<GemmWorkItem> items;
  std::vector<SyrkReduceTask> reduce;
  int n_slots = 0;
  int kchunk = 0;
};

int plan_factors(const spngd_factor_req* reqs, int n, FactorPlan& plan);
int run_factors(spngd_ctx* ctx, const GemmProblem* d_probs, const GemmWorkItem* d_items, int n_items,
                float* d_partials, const SyrkReduceTask* d_reduce, int n_reduce);
int launch_bn_moments(spngd_ctx* ctx, const spngd_bn_moments_req* d_reqs, int n, int64_t max_c);

}  // namespace spngd
