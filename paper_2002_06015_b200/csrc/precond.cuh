#pragma once

#include <vector>

#include "ctx.cuh"
#include "gemm_tf32x3.cuh"

namespace spngd {

struct RescaleTask {  // rescale_weights + velocity fix, one FC/Conv layer
  float* W;
  float* V;
  int64_t n;
  const double* norm2;
  double target;  // sqrt(2 * d_out)
};

struct PrecondPlan {
  std::vector<GemmProblem> probs1, probs2;
  std::vector<GemmWorkItem> items1, items2;
  std::vector<RescaleTask> rescale;
  size_t tmp_floats = 0;    // P1^T scratch
  int n_norms = 0;
};

// Builds the two grouped GEMM launches P1^T = A^-1 dW^T and
// P^T = P1^T G^-1 (EPI_UPDATE).  `tmp` holds the P1^T buffers (sizing pass when
// null) and `norms` one double per request.
int plan_precondition(const spngd_precond_req* reqs, int n, double eta, double momentum, float* tmp,
                      double* norms, PrecondPlan& plan, const float* scal = nullptr);
int run_precondition(spngd_ctx* ctx, const PrecondPlan& plan, const GemmProblem* d_p1, const GemmWorkItem* d_i1,
                     const GemmProblem* d_p2, const GemmWorkItem* d_i2, const RescaleTask* d_rescale,
                     double* d_norms);

struct BnUpdateTask {
  spngd_bn_update_req r;
};
int launch_bn_update(spngd_ctx* ctx, const spngd_bn_update_req* d_reqs, int n, int64_t max_c, double lambda,
                     double eta, double momentum, const float* scal = nullptr);
int launch_stat_distance(spngd_ctx* ctx, const spngd_stat_req* d_reqs, int n, int64_t max_rows);

}  // namespace spngd
