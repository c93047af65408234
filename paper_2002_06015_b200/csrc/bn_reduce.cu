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

}  // namespace
}  // namespace spngd

using namespace spngd;

extern "C" int spngd_bn_grad_reduce_batched(spngd_ctx* ctx, int n, const spngd_bn_grad_req* reqs) {
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
