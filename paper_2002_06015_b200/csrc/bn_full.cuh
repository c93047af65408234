#pragma once
// Full 2c x 2c BatchNorm block (BnMode::Full), shared by the one-shot entry
// points (bn_full.cu) and the whole step (opt.cu).
#include "ctx.cuh"

namespace spngd {

// build_bn_full's per-sample vector u = (g_gamma0, g_beta0, g_gamma1, ...)
// (fisher.cpp:204-208), one row of 2c per sample.
struct InterleaveTask {
  const float* gg;
  const float* gb;
  float* u;  // (hi - lo) x 2c
  int64_t c, lo, hi;
};
int launch_bn_interleave(spngd_ctx* ctx, const InterleaveTask* d_tasks, int n, int64_t max_total);
// v = F_inv u (dense finv, ld), then the BN momentum update (or pg/pb out
// only when gamma == NULL); `scal` = device {eta, momentum} overrides.
int launch_bn_full_update(spngd_ctx* ctx, const spngd_bn_full_update_req* d_reqs, int n, int64_t max_dim, double eta,
                          double momentum, const float* scal);

}  // namespace spngd
