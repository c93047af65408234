#pragma once

#include <vector>

#include "ctx.cuh"
#include "gemm_tf32x3.cuh"

namespace spngd {

constexpr int kMaxPeers = 7;  // one process per GPU, <= 8 GPUs per box

struct RescaleTask {  // rescale_weights + velocity fix, one FC/Conv layer
  float* W;
  float* V;
  int64_t n;
  const double* norm2;
  double target;  // sqrt(2 * d_out)
  // P2P all-gather (spngd_opt_attach_peers): W'' is also stored to the same
  // offset of every peer's replica buffer over NVLink (Stage 5 fused in)
  float* peers[kMaxPeers];
  int32_t n_peers;
  int32_t pad_;
};

// Owned replica range -> every peer's replica buffer (NVLink stores), for the
// layers whose final weights are not produced by the rescale pass.
struct PeerCopyTask {
  const float* src;
  float* dst[kMaxPeers];
  int32_t n_peers;
  int32_t pad_;
  int64_t n;
};
int launch_peer_copy(spngd_ctx* ctx, const PeerCopyTask* d_tasks, int n, int64_t max_n);

// Parameters the wave schedule updates before every inverse is known good
// (early precondition parts): saved at step start, restored in phase 4 when
// the step failed, so a failed step changes no parameter (dist.cpp:597-601).
struct SnapTask {
  float* live;
  float* save;
  int64_t n;
};
// restore = false: save <- live; restore = true: live <- save iff *d_status.
int launch_snapshot(spngd_ctx* ctx, const SnapTask* d_tasks, int n, int64_t max_n, bool restore);

// Owner side of the fused reduce-scatter: out = mean over the `world` source
// slots (slot q at in + q * slot_stride), summed in ascending rank order
// like reduce_scatter_v (dist.cpp:204-213).
struct SlotMeanTask {
  const float* in;
  float* out;
  int64_t slot_stride;
  int64_t n;
  int32_t world;
  int32_t pad_;
};
int launch_slot_mean(spngd_ctx* ctx, const SlotMeanTask* d_tasks, int n, int64_t max_n);

struct PrecondPlan {
  // Grouped GEMM launches in order: dense inverses -> 2 (P1^T = A^-1 dW^T,
  // P^T = P1^T G^-1 with EPI_UPDATE); triangular factors -> 4 (see
  // plan_precondition).
  int stages = 2;
  std::vector<GemmProblem> probs[4];
  std::vector<GemmWorkItem> items[4];   // per stage: the 2-CTA pair items first (n_pair)
  int n_pair[4] = {0, 0, 0, 0};
  std::vector<RescaleTask> rescale;
  size_t tmp_floats = 0;    // intermediate products
  int n_norms = 0;
};

// Triangular factors of the damped inverses (A + dI)^-1 = T_A^T T_A: lower
// T = L^-1 and upper T^T, same leading dimension as the request's lda / ldg.
struct PrecondTri {
  const float* tlA;
  const float* tuA;
  const float* tlG;
  const float* tuG;
};

// Builds the grouped GEMM launches of P = G^-1 dW A^-1 fused with the
// update.  `tmp` holds the intermediates (sizing pass when null), `norms` one
// double per request.  With `tri` (one entry per request) the inverses are
// never formed: P^T = T_A^T T_A dW^T T_G^T T_G as four half-flop triangular
// GEMMs, reqs[i].Ainv / Ginv unused.
int plan_precondition(const spngd_precond_req* reqs, int n, double eta, double momentum, float* tmp,
                      double* norms, PrecondPlan& plan, const float* scal = nullptr,
                      const PrecondTri* tri = nullptr);
int run_precondition(spngd_ctx* ctx, const PrecondPlan& plan, GemmProblem* const* d_probs,
                     GemmWorkItem* const* d_items, const RescaleTask* d_rescale, double* d_norms);
// Stages [q0, q1) only; `finish` also zeroes the norms first and runs the
// rescale pass after (the stages before the last write only temporaries).
int run_precondition_stages(spngd_ctx* ctx, const PrecondPlan& plan, GemmProblem* const* d_probs,
                            GemmWorkItem* const* d_items, const RescaleTask* d_rescale, double* d_norms, int q0, int q1,
                            bool finish);

struct BnUpdateTask {
  spngd_bn_update_req r;
};
int launch_bn_update(spngd_ctx* ctx, const spngd_bn_update_req* d_reqs, int n, int64_t max_c, double lambda,
                     double eta, double momentum, const float* scal = nullptr);
// Plain-gradient update of one layer (ngd_step with blocks == nullptr,
// fisher.cpp:320-333, 348-356): W' = W - eta g + m V, V' = W' - W.
struct SgdTask {
  float* W;
  float* V;
  const float* g;
  int64_t n;
};
int launch_sgd_update(spngd_ctx* ctx, const SgdTask* d_tasks, int n, const float* scal);
// SingularBlock check of every BN channel before any parameter is written.
int launch_bn_det_check(spngd_ctx* ctx, const spngd_bn_update_req* d_reqs, int n, int64_t max_c, double lambda);
// world > 1: all ranks adopt the largest status word (d_flag: one device double).
int agree_status(spngd_ctx* ctx, double* d_flag);
// One similarity job: the public request plus, on the optimizer path, the
// snapshot slot the statistic rotates into (x2 <- x1 <- x).  The kernel writes
// rot[q] = x[q] right after reading x2[q] (rot is x2's slot when it exists), so
// the rotation costs no separate copy pass.
struct StatJob {
  spngd_stat_req r;
  float* rot;  // NULL: no rotation (public entry point)
};
int launch_stat_distance(spngd_ctx* ctx, const StatJob* d_jobs, int n, int64_t max_rows);

}  // namespace spngd
