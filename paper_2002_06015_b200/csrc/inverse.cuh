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
  int32_t inject;   // test hook (SPNGD_TEST_FAIL_N): report a non-positive pivot
  int* info;        // per-matrix status word (NotPositiveDefinite), may be null
};

struct UnpackTask {  // dense = unpack(packed) + damp * I
  const float* packed;
  int64_t n;
  const float* damp_dev;  // overrides damp when non-null
  float damp;
  int32_t pad_;
  float* dense;
  int64_t ld;
  int* info;        // per-matrix status word (non-finite input), may be null
};

struct PackTask {    // finite check of the dense result (+ pack when `packed`)
  const float* dense;
  int64_t ld;
  int64_t n;
  float* packed;     // may be null: check only
  int* info;
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
  int item_off, item_cnt;  // items [item_off, item_off + pair_cnt) run on the 2-CTA kernel
  int base_off, base_cnt;
  int pair_cnt;
};

// Schedule of the Schur-complement recursion for a batch of dense matrices.
struct InversePlan {
  std::vector<GemmProblem> probs;
  std::vector<GemmWorkItem> items;
  std::vector<BaseTask> bases;
  std::vector<InverseRound> rounds;
  size_t workspace_floats = 0;
  // Upper bound of items.size() for any subset of the matrices (each round's
  // 2-CTA / single-CTA choice can differ for a subset): sizes re-plan buffers.
  size_t item_bound = 0;
};

struct DenseMatrix {
  float* ptr;     // in: M + dI (dense symmetric); out: (M + dI)^-1
  float* tlow;    // workspace n x ld, zero above the diagonal: L^-1
  float* tup;     // workspace n x ld, zero below the diagonal: L^-T
  int64_t ld;
  int64_t n;
  int* info = nullptr;  // per-matrix status word for the leaves
};

// Builds the plan; temporaries are carved from `workspace` (may be null for a
// sizing pass, in which case only workspace_floats is meaningful).
// form_inverse = false stops after the factors: tlow = L^-1 and tup = L^-T
// (the optimizer preconditions with them directly); ptr is scratch then.
void plan_inverse(const std::vector<DenseMatrix>& mats, float* workspace, InversePlan& plan, bool form_inverse = true);
// X = Tup Tup^T -> m.ptr (the lauum step alone), synchronous.
int materialize_inverse(spngd_ctx* ctx, const DenseMatrix& m);

// ---- accuracy refinement of explicit inverses (refine.cu) ------------------
// The fp32 Cholesky inverse has forward error ~3e-9 * cond(M + dI) (measured,
// DESIGN.md §4).  ||M + dI||_F / d bounds cond from above (lambda_min >= d for
// PSD M); above kRefineCond one refinement step X1 = X0 + X0 (I - M X0) with
// the residual formed from exact tf32 splits (M = Mh + Mr, K-concatenated,
// error ~2^-33 per product) brings the error to ~1e-5.
struct FroTask {
  const float* packed;
  int64_t n;
  const float* damp_dev;  // overrides damp when non-null
  float damp;
  int32_t pad_;
  double* sumsq;          // out: ||M + dI||_F^2 (accumulated)
};
struct RefineJob {
  const float* packed;    // M (packed), the same input the inverse read
  int64_t n;
  float damp;             // the fp32 damping the inverse used
  float* X;               // dense (n x ld) inverse X0 in, refined symmetric X1 out
  int64_t ld;
};
double refine_threshold();  // kRefineCond or SPNGD_REFINE_COND (<0: never, 0: always)
int launch_fro(spngd_ctx* ctx, const FroTask* d_tasks, int n, int64_t max_n);
// Refines every job in place (grouped launches); scratch comes from `scratch`.
int refine_inverses(spngd_ctx* ctx, DeviceScratch& scratch, const std::vector<RefineJob>& jobs);

int launch_pi(spngd_ctx* ctx, const PiTask* d_tasks, int n);
int launch_unpack(spngd_ctx* ctx, const UnpackTask* d_tasks, int n, int64_t max_n);
int launch_pack(spngd_ctx* ctx, const PackTask* d_tasks, int n, int64_t max_n);
int launch_base(spngd_ctx* ctx, const BaseTask* d_tasks, int n);
// Runs all rounds; d_probs/d_items/d_bases are the device copies of the plan.
int run_inverse(spngd_ctx* ctx, const InversePlan& plan, const GemmProblem* d_probs, const GemmWorkItem* d_items,
                const BaseTask* d_bases);

}  // namespace spngd
