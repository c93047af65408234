#pragma once

#include <vector>

#include "ctx.cuh"
#include "gemm_tf32x3.cuh"

namespace spngd {

struct RepackTask {  // conv/FC capture -> K-contiguous dim x (n*hw) matrix
  const float* src;
  float* dst;
  int64_t n, dim, hw;
};

struct FactorPlan {
  std::vector<RepackTask> repacks;
  size_t repack_floats = 0;
  int64_t repack_max = 0;  // largest element count of one repack
  std::vector<GemmProblem> probs;
  std::vector<GemmWorkItem> items;
  std::vector<SyrkReduceTask> reduce;
  int n_slots = 0;
  int kchunk = 0;
  // 2-CTA SYRK: items of pair-eligible problems come first (n_pair of them,
  // in cluster pairs); every filtered item list keeps that order.
  std::vector<char> pair_prob;
  int n_pair = 0;
};

// `ws` receives the repacked captures (sizing pass when null: only
// repack_floats is meaningful).
int plan_factors(const spngd_factor_req* reqs, int n, FactorPlan& plan, float* ws = nullptr);
int launch_repack(spngd_ctx* ctx, const RepackTask* d_tasks, int n, int64_t max_elems);
// Leading items of `items` that belong to the 2-CTA kernel.
int count_pair_items(const FactorPlan& plan, const std::vector<GemmWorkItem>& items);
int run_factors(spngd_ctx* ctx, const FactorPlan& plan, const GemmProblem* d_probs, int n_pair,
                const GemmWorkItem* d_items, int n_items, float* d_partials, const SyrkReduceTask* d_reduce,
                int n_reduce);
// The factor SYRK launch alone.
// Items [0, n_pair) run on the 2-CTA kernel, the rest on the single-CTA engine.
int launch_factor_gemm(spngd_ctx* ctx, const FactorPlan& plan, const GemmProblem* d_probs, int n_pair,
                       const GemmWorkItem* d_items, int n_items, float* d_partials, cudaStream_t stream);
int launch_bn_moments(spngd_ctx* ctx, const spngd_bn_moments_req* d_reqs, int n, int64_t max_c);

struct BnGradPayloadTask {  // grad_payload's BN branch (dist.cpp:364-371)
  const float* gg;
  const float* gb;
  int64_t m, c;
  float* out;  // 2c: gamma then beta
};
int launch_bn_grad_payload(spngd_ctx* ctx, const BnGradPayloadTask* d_tasks, int n, int64_t max_c);
int launch_im2col(spngd_ctx* ctx, const spngd_im2col_req* d_reqs, int n);
// SHAPE_MISMATCH unless positive and (a, hw >= 0) c_in k^2 == a, h_out w_out == hw.
int check_conv_geom(const spngd_conv_geom& g, int64_t a, int64_t hw);

}  // namespace spngd
