#pragma once

#include <vector>

#include "ctx.cuh"
#include "gemm_tf32x3.cuh"

namespace spngd {

struct BaseTask {   // n <= 128 diagonal block: L = chol(M), T = L^-1 -> Tlow, T^T -> Tup
  const float* m;
  float* tlow;
  float* tup;
  int64_t ld;
  int32_t n;
  int32_t pad_;
};

struct UnpackTask {  // dense = unpack(packed) + damp * I
  const float* packed;
  int64_t n;
  const float* damp_dev;  // overrides damp when non-null
  float damp;
  int32_t pad_;
  float* dense;
  int64_t ld;
};

struct PackTask {
  const float* dense;
  int64_t ld;
  int64_t n;
  float* packed;
};

struct PiTask {  // damp_and_invert's pi and the two dampings (fisher.cpp:221-226)
  const float* A;
  const float* G;
  int64_t a, g;
  double sqrt_lambda;
  float* dampA;
  float* dampG;
  float* pi_out;
};

struct InverseRound {
  int item_off, item_cnt;
  int base_off, base_cnt;
};

// Schedule of the Schur-complement recursion for a batch of dense matrices.
struct InversePlan {
  std::vector<GemmProblem> probs;
  std::vector<GemmWorkItem> items;
  std::vector<BaseTask> bases;
  std::vector<InverseRound> rounds;
  size_t workspace_floats = 0;
};

struct DenseMatrix {
  float* ptr;     // in: M + dI (dense symmetric); out: (M + dI)^-1
  float* tlow;    // workspace n x ld, zero above the diagonal: L^-1
  float* tup;     // workspace n x ld, zero below the diagonal: L^-T
  int64_t ld;
  int64_t n;
};

// Builds the plan; temporaries are carved from `workspace` (may be null for a
// sizing pass, in which case only workspace_floats is meaningful).
// form_inverse = false stops after the factors: tlow = L^-1 and tup = L^-T
// (the optimizer preconditions with them directly); ptr is scratch then.
void plan_inverse(const std::vector<DenseMatrix>& mats, float* workspace, InversePlan& plan, bool form_inverse = true);
// X = Tup Tup^T -> m.ptr (the lauum step alone), synchronous.
int materialize_inverse(spngd_ctx* ctx, const DenseMatrix& m);

int launch_pi(spngd_ctx* ctx, const PiTask* d_tasks, int n);
int launch_unpack(spngd_ctx* ctx, const UnpackTask* d_tasks, int n, int64_t max_n);
int launch_pack(spngd_ctx* ctx, const PackTask* d_tasks, int n, int64_t max_n);
int launch_base(spngd_ctx* ctx, const BaseTask* d_tasks, int n);
// Runs all rounds; d_probs/d_items/d_bases are the device copies of the plan.
int run_inverse(spngd_ctx* ctx, const InversePlan& plan, const GemmProblem* d_probs, const GemmWorkItem* d_items,
                const BaseTask* d_bases);

}  // namespace spngd
