// the full 2c x 2c BatchNorm Fisher block (BnMode::Full).
//   build_bn_full        (fisher.cpp:187-216): interleave (gg, gb) -> u (M x 2c),
//                        then the 3xTF32 SYRK engine builds F = mean u u^T (packed).
//   damp_bn_full         (fisher.cpp:248-253): spngd_spd_inverse_batched(F, lambda).
//   precondition_bn_full (fisher.cpp:278-296) + ngd_step's BN branch
//                        (fisher.cpp:346-359): one warp per output row of
//                        F_inv * u_grad, then the momentum update of gamma/beta.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "bn_full.cuh"
#include "ctx.cuh"
#include "factor.cuh"

namespace spngd {
namespace {

__global__ void bn_interleave_kernel(const InterleaveTask* __restrict__ tasks) {
  const InterleaveTask t = tasks[blockIdx.y];
  const int64_t total = (t.hi - t.lo) * t.c;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t s = q / t.c, ch = q - s * t.c;
    const int64_t src = (t.lo + s) * t.c + ch;
    t.u[s * 2 * t.c + 2 * ch] = t.gg[src];
    t.u[s * 2 * t.c + 2 * ch + 1] = t.gb[src];
  }
}

__global__ void bn_full_update_kernel(const spngd_bn_full_update_req* __restrict__ reqs, double eta, double momentum,
                                      const float* __restrict__ scal, const int* __restrict__ status) {
  if (*status) return;  // see rescale_kernel (precond.cu)
  if (scal) {
    eta = scal[0];
    momentum = scal[1];
  }
  const spngd_bn_full_update_req r = reqs[blockIdx.y];
  const int lane = threadIdx.x & 31;
  const int64_t dim = 2 * r.c;
  const int64_t warp = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t nw = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t i = warp; i < dim; i += nw) {
    // v_i = sum_j F_inv[i][j] u_j with u interleaved (gamma_0, beta_0, gamma_1, ...)
    double acc = 0.0;
    const float* row = r.finv + i * r.ld;
    for (int64_t j = lane; j < dim; j += 32) {
      const float u = (j & 1) ? r.grad[r.c + (j >> 1)] : r.grad[j >> 1];
      acc += double(row[j]) * double(u);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const int64_t ch = i >> 1;
      const bool is_beta = i & 1;
      float* w = is_beta ? r.beta + ch : r.gamma + ch;
      float* v = is_beta ? r.vbeta + ch : r.vgamma + ch;
      const float p = float(acc);
      if (is_beta ? r.pb_out != nullptr : r.pg_out != nullptr) (is_beta ? r.pb_out : r.pg_out)[ch] = p;
      if (!r.gamma) continue;  // precondition_bn_full only
      const float w0 = *w;
      const float nw = float(double(w0) - eta * double(p) + momentum * double(*v));  // fisher.cpp:356-357
      *w = nw;
      *v = nw - w0;                                                                    // fisher.cpp:358-359
    }
  }
}

}  // namespace

int launch_bn_interleave(spngd_ctx* ctx, const InterleaveTask* d_tasks, int n, int64_t max_total) {
  if (n <= 0) return SPNGD_OK;
  dim3 grid(unsigned(std::min<int64_t>(std::max<int64_t>((max_total + 255) / 256, 1), 1024)), unsigned(n));
  bn_interleave_kernel<<<grid, 256, 0, ctx->stream>>>(d_tasks);
  SPNGD_CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return SPNGD_OK;
}

int launch_bn_full_update(spngd_ctx* ctx, const spngd_bn_full_update_req* d_reqs, int n, int64_t max_dim, double eta,
                          double momentum, const float* scal) {
  if (n <= 0) return SPNGD_OK;
  dim3 grid(unsigned(std::min<int64_t>((max_dim + 7) / 8, 1024)), unsigned(n));
  bn_full_update_kernel<<<grid, 256, 0, ctx->stream>>>(d_reqs, eta, momentum, scal, ctx->d_status);
  SPNGD_CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return SPNGD_OK;
}

}  // namespace spngd

using namespace spngd;

extern "C" int spngd_bn_full_moments_batched(spngd_ctx* ctx, int n, const spngd_bn_full_req* reqs) {
  SPNGD_CTX_SCOPE(ctx);
  if (!ctx || (n > 0 && !reqs)) return fail(SPNGD_ERR_INVALID, "spngd_bn_full_moments_batched: null argument");
  if (n == 0) return SPNGD_OK;
  DeviceScratch scratch(ctx);
  std::vector<InterleaveTask> il;
  std::vector<spngd_factor_req> fr;
  int64_t max_total = 0;
  for (int i = 0; i < n; ++i) {
    const spngd_bn_full_req& r = reqs[i];
    if (r.lo < 0 || r.hi <= r.lo) return fail(SPNGD_ERR_EMPTY_BATCH, "build_bn_full: empty sample range");
    if (r.c <= 0) return fail(SPNGD_ERR_SHAPE_MISMATCH, "build_bn_full: c must be > 0");
    if (!r.gg || !r.gb || !r.packed_out) return fail(SPNGD_ERR_EMPTY_BATCH, "build_bn_full: no captured gradients");
    const int64_t m = r.hi - r.lo;
    float* u = scratch.alloc<float>(size_t(m * 2 * r.c));
    if (!u) return fail(SPNGD_ERR_CUDA, "build_bn_full: scratch allocation failed");
    il.push_back({r.gg, r.gb, u, r.c, r.lo, r.hi});
    // FC layout (element (row i, sample s) = u[s * dim + i]), scale 1/m.
    fr.push_back({u, 2 * r.c, 1, 0, 0, m, 1.0 / double(m), r.packed_out});
    max_total = std::max(max_total, m * r.c);
  }
  auto* d_il = scratch.upload(il);
  int rc = launch_bn_interleave(ctx, d_il, n, max_total);
  if (rc) return rc;
  return spngd_factor_sym_batched(ctx, n, fr.data());  // the SYRK engine, then sync
}

extern "C" int spngd_bn_full_solve_update_batched(spngd_ctx* ctx, int n, const spngd_bn_full_update_req* reqs,
                                                  double eta, double momentum) {
  SPNGD_CTX_SCOPE(ctx);
  if (!ctx || (n > 0 && !reqs)) return fail(SPNGD_ERR_INVALID, "spngd_bn_full_solve_update_batched: null argument");
  if (n == 0) return SPNGD_OK;
  int64_t max_dim = 0;
  for (int i = 0; i < n; ++i) {
    const auto& r = reqs[i];
    if (r.c <= 0 || r.ld < 2 * r.c) return fail(SPNGD_ERR_SHAPE_MISMATCH, "precondition_bn_full: gradient length mismatch");
    if (!r.finv) return fail(SPNGD_ERR_STALE_BEYOND_LIMIT, "precondition_bn_full: block never inverted");
    const bool upd = r.gamma || r.beta || r.vgamma || r.vbeta;
    if (!r.grad || (upd && !(r.gamma && r.beta && r.vgamma && r.vbeta)) || (!upd && !(r.pg_out && r.pb_out)))
      return fail(SPNGD_ERR_INVALID, "bn_full_update: null pointer");
    max_dim = std::max(max_dim, 2 * r.c);
  }
  DeviceScratch scratch(ctx);
  std::vector<spngd_bn_full_update_req> v(reqs, reqs + n);
  auto* d = scratch.upload(v);
  int rc = launch_bn_full_update(ctx, d, n, max_dim, eta, momentum, nullptr);
  if (rc) return rc;
  return spngd_ctx_sync(ctx);
}
