// fused BN per-sample reduction.  The reference captures the
// per-sample BN parameter gradients in the backward (src/net.cpp:467-475):
//   gg[s][ch] = sum_p dY[s][ch*S+p] * xhat[s][ch*S+p],  gb[s][ch] = sum_p dY[s][ch*S+p]
// This kernel reads dY and xhat once (the only large traffic: 2 * M*c*S*4 B)
// and writes the M x c captures the step consumes.  One warp per (sample,
// channel) segment; float4 loads when S % 4 == 0 (segments then start 16-byte
// aligned), 4 independent loads in flight per lane, fp32 lane partials
// reduced pairwise by shuffles.  Layers are batched in one launch through a
// prefix table of segment counts.  HBM-bound: the roofline is bytes read / HBM
// bandwidth.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "bn_reduce.cuh"
#include "ctx.cuh"

namespace spngd {
namespace {

struct BnGradTask {
  spngd_bn_grad_req r;
  int64_t seg0;  // first global segment of this task
};

constexpr int kWarpsPerBlock = 8;

__device__ __forceinline__ void warp_sum2(float& a, float& b) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32) bn_grad_reduce_kernel(const BnGradTask* __restrict__ tasks,
                                                                            int n_tasks, int64_t n_segs) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = int64_t(blockIdx.x) * kWarpsPerBlock + (threadIdx.x >> 5);
  const int64_t nwarps = int64_t(gridDim.x) * kWarpsPerBlock;
  int t = 0;
  for (int64_t g = warp0; g < n_segs; g += nwarps) {
    while (t + 1 < n_tasks && g >= tasks[t + 1].seg0) ++t;  // segments ascend per warp
    const spngd_bn_grad_req r = tasks[t].r;
    const int64_t q = g - tasks[t].seg0;  // = s * c + ch
    const int64_t S = r.S;
    const float* dy = r.dy + q * S;
    const float* xh = r.xhat + q * S;
    float dot = 0.f, sum = 0.f;
    if ((S & 3) == 0) {
      const float4* d4 = reinterpret_cast<const float4*>(dy);
      const float4* x4 = reinterpret_cast<const float4*>(xh);
      const int64_t n4 = S >> 2;
      int64_t i = lane;
      for (; i + 96 < n4; i += 128) {  // 4 float4 of each array in flight per lane
        float4 a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a[u] = __ldcs(d4 + i + 32 * u);
          b[u] = __ldcs(x4 + i + 32 * u);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          dot = fmaf(a[u].x, b[u].x, fmaf(a[u].y, b[u].y, fmaf(a[u].z, b[u].z, fmaf(a[u].w, b[u].w, dot))));
          sum += (a[u].x + a[u].y) + (a[u].z + a[u].w);
        }
      }
      for (; i < n4; i += 32) {
        const float4 a = __ldcs(d4 + i), b = __ldcs(x4 + i);
        dot = fmaf(a.x, b.x, fmaf(a.y, b.y, fmaf(a.z, b.z, fmaf(a.w, b.w, dot))));
        sum += (a.x + a.y) + (a.z + a.w);
      }
    } else {
      for (int64_t i = lane; i < S; i += 32) {
        const float a = __ldcs(dy + i), b = __ldcs(xh + i);
        dot = fmaf(a, b, dot);
        sum += a;
      }
    }
    warp_sum2(dot, sum);
    if (lane == 0) {
      r.gg[q] = dot;
      r.gb[q] = sum;
    }
  }
}

// ---- fused: dY, x_hat -> per-sample (g_gamma, g_beta), 3c moments, payload --
// One launch per step for every BN layer: the per-sample
// reduction above (net.cpp:467-475), build_bn_block's moments
// (fisher.cpp:147-185, interleaved 3c payload dist.cpp:283-292) and
// grad_payload's BN branch [sum_s g_gamma / m | sum_s g_beta / m]
// (dist.cpp:364-371).  Work items are (layer, channel, sample chunk) sized to
// ~64 KB of dY + x_hat each, one warp per item; the chunk partials (fp64) go to
// slots and the last chunk of a channel to finish (an atomic counter, reset for
// the next launch) sums them in chunk order -- deterministic, no fp atomics.
__device__ __forceinline__ void segment_reduce(const float* dy, const float* xh, int64_t S, int lane, float& dot,
                                               float& sum) {
  dot = 0.f;
  sum = 0.f;
  if ((S & 3) == 0 && ((reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(xh)) & 15) == 0) {
    const float4* d4 = reinterpret_cast<const float4*>(dy);
    const float4* x4 = reinterpret_cast<const float4*>(xh);
    const int64_t n4 = S >> 2;
    int64_t i = lane;
    for (; i + 96 < n4; i += 128) {
      float4 a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = __ldcs(d4 + i + 32 * u);
        b[u] = __ldcs(x4 + i + 32 * u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        dot = fmaf(a[u].x, b[u].x, fmaf(a[u].y, b[u].y, fmaf(a[u].z, b[u].z, fmaf(a[u].w, b[u].w, dot))));
        sum += (a[u].x + a[u].y) + (a[u].z + a[u].w);
      }
    }
    for (; i < n4; i += 32) {
      const float4 a = __ldcs(d4 + i), b = __ldcs(x4 + i);
      dot = fmaf(a.x, b.x, fmaf(a.y, b.y, fmaf(a.z, b.z, fmaf(a.w, b.w, dot))));
      sum += (a.x + a.y) + (a.z + a.w);
    }
  } else {
    for (int64_t i = lane; i < S; i += 32) {
      const float a = __ldcs(dy + i), b = __ldcs(xh + i);
      dot = fmaf(a, b, dot);
      sum += a;
    }
  }
  warp_sum2(dot, sum);
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32) bn_backward_stats_kernel(const BnxTask* __restrict__ tasks,
                                                                               const BnxItem* __restrict__ items,
                                                                               int64_t n_items, double* slots,
                                                                               int* counters) {
  const int lane = threadIdx.x & 31;
  const int64_t w = int64_t(blockIdx.x) * kWarpsPerBlock + (threadIdx.x >> 5);
  if (w >= n_items) return;
  const BnxItem it = items[w];
  const BnxTask t = tasks[it.task];
  const int64_t S = t.S, c = t.c;
  double p[5] = {0, 0, 0, 0, 0};  // sum gg^2, gg gb, gb^2, gg, gb
  for (int32_t s = it.s0; s < it.s1; ++s) {
    const int64_t q = int64_t(s) * c + it.ch;
    float dot, sum;
    segment_reduce(t.dy + q * S, t.xh + q * S, S, lane, dot, sum);
    if (lane == 0) {
      if (t.gg) t.gg[q] = dot;
      if (t.gb) t.gb[q] = sum;
    }
    const double g = dot, b = sum;  // the fp32 capture values, as build_bn_block reads them
    p[0] += g * g;
    p[1] += g * b;
    p[2] += b * b;
    p[3] += g;
    p[4] += b;
  }
  if (lane != 0) return;
  const int64_t nch = t.nchunks;
  double* slot = slots + 5 * (t.slot0 + int64_t(it.ch) * nch + it.chunk);
#pragma unroll
  for (int k = 0; k < 5; ++k) slot[k] = p[k];
  if (nch == 1) {
    // single chunk: finish directly
  } else {
    __threadfence();
    const int done = atomicAdd(counters + t.chan0 + it.ch, 1);
    if (done != nch - 1) return;
    __threadfence();
    const double* base = slots + 5 * (t.slot0 + int64_t(it.ch) * nch);
#pragma unroll
    for (int k = 0; k < 5; ++k) p[k] = 0.0;
    for (int64_t j = 0; j < nch; ++j)
#pragma unroll
      for (int k = 0; k < 5; ++k) p[k] += __ldcg(base + 5 * j + k);
    counters[t.chan0 + it.ch] = 0;  // ready for the next launch (graph replay)
  }
  const double inv = 1.0 / double(t.M);
  if (t.out3c) {
    t.out3c[3 * it.ch + 0] = float(p[0] * inv);
    t.out3c[3 * it.ch + 1] = float(p[1] * inv);
    t.out3c[3 * it.ch + 2] = float(p[2] * inv);
  }
  if (t.payload) {
    t.payload[it.ch] = float(p[3] * inv);
    t.payload[c + it.ch] = float(p[4] * inv);
  }
}

}  // namespace

int plan_bn_backward(const std::vector<spngd_bn_backward_req>& reqs, BnxPlan& plan) {
  plan = BnxPlan();
  constexpr int64_t kItemBytes = 64 << 10;
  for (size_t i = 0; i < reqs.size(); ++i) {
    const spngd_bn_backward_req& r = reqs[i];
    if (r.M <= 0) return fail(SPNGD_ERR_EMPTY_BATCH, "bn backward statistics: request %zu: empty batch", i);
    if (r.c <= 0 || r.S <= 0) return fail(SPNGD_ERR_SHAPE_MISMATCH, "bn backward statistics: request %zu: bad shape", i);
    if (!r.dy || !r.xhat) return fail(SPNGD_ERR_INVALID, "bn backward statistics: request %zu: null input", i);
    const int64_t per = std::max<int64_t>(1, kItemBytes / (8 * r.S));  // samples per chunk
    const int64_t nch = (r.M + per - 1) / per;
    BnxTask t{r.dy, r.xhat, r.M, r.c, r.S, r.gg, r.gb, r.out3c, r.payload, int32_t(nch), 0, plan.slots, plan.channels};
    plan.tasks.push_back(t);
    for (int64_t ch = 0; ch < r.c; ++ch)
      for (int64_t k = 0; k < nch; ++k)
        plan.items.push_back({int32_t(i), int32_t(ch), int32_t(k * per), int32_t(std::min(r.M, (k + 1) * per)),
                              int32_t(k), 0});
    plan.slots += r.c * nch;
    plan.channels += r.c;
    plan.bytes += 2 * r.M * r.c * r.S * int64_t(sizeof(float));
  }
  return SPNGD_OK;
}

int launch_bn_backward(spngd_ctx* ctx, const BnxTask* d_tasks, const BnxItem* d_items, int64_t n_items, double* d_slots,
                       int* d_counters) {
  if (n_items <= 0) return SPNGD_OK;
  const int64_t blocks = (n_items + kWarpsPerBlock - 1) / kWarpsPerBlock;
  bn_backward_stats_kernel<<<unsigned(blocks), kWarpsPerBlock * 32, 0, ctx->stream>>>(d_tasks, d_items, n_items,
                                                                                      d_slots, d_counters);
  SPNGD_CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return SPNGD_OK;
}

}  // namespace spngd

using namespace spngd;

extern "C" int spngd_bn_backward_stats_batched(spngd_ctx* ctx, int n, const spngd_bn_backward_req* reqs) {
  SPNGD_CTX_SCOPE(ctx);
  if (!ctx || (n > 0 && !reqs)) return fail(SPNGD_ERR_INVALID, "spngd_bn_backward_stats_batched: null argument");
  if (n == 0) return SPNGD_OK;
  BnxPlan plan;
  int rc = plan_bn_backward(std::vector<spngd_bn_backward_req>(reqs, reqs + n), plan);
  if (rc) return rc;
  DeviceScratch scratch(ctx);
  auto* d_tasks = scratch.upload(plan.tasks);
  auto* d_items = scratch.upload(plan.items);
  double* d_slots = scratch.alloc<double>(size_t(5 * plan.slots));
  int* d_cnt = scratch.alloc<int>(size_t(plan.channels));
  if (!d_tasks || !d_items || !d_slots || !d_cnt) return fail(SPNGD_ERR_CUDA, "bn backward statistics: allocation failed");
  SPNGD_CUDA_TRY(cudaMemsetAsync(d_cnt, 0, sizeof(int) * plan.channels, ctx->stream));
  rc = launch_bn_backward(ctx, d_tasks, d_items, int64_t(plan.items.size()), d_slots, d_cnt);
  if (rc) return rc;
  return spngd_ctx_sync(ctx);
}

extern "C" int spngd_bn_grad_reduce_batched(spngd_ctx* ctx, int n, const spngd_bn_grad_req* reqs) {
  SPNGD_CTX_SCOPE(ctx);
  if (!ctx || (n > 0 && !reqs)) return fail(SPNGD_ERR_INVALID, "spngd_bn_grad_reduce_batched: null argument");
  std::vector<BnGradTask> tasks;
  int64_t segs = 0;
  for (int i = 0; i < n; ++i) {
    const spngd_bn_grad_req& r = reqs[i];
    if (r.M <= 0) return fail(SPNGD_ERR_EMPTY_BATCH, "bn_grad_reduce: empty batch");
    if (r.c <= 0 || r.S <= 0) return fail(SPNGD_ERR_SHAPE_MISMATCH, "bn_grad_reduce: bad shape");
    if (!r.dy || !r.xhat || !r.gg || !r.gb) return fail(SPNGD_ERR_INVALID, "bn_grad_reduce: null pointer");
    tasks.push_back({r, segs});
    segs += r.M * r.c;
  }
  if (segs == 0) return SPNGD_OK;
  DeviceScratch scratch(ctx);
  auto* d = scratch.upload(tasks);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  const int64_t blocks = std::min<int64_t>((segs + kWarpsPerBlock - 1) / kWarpsPerBlock, int64_t(sms) * 8);
  bn_grad_reduce_kernel<<<unsigned(blocks), kWarpsPerBlock * 32, 0, ctx->stream>>>(d, int(tasks.size()), segs);
  SPNGD_CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return spngd_ctx_sync(ctx);
}
