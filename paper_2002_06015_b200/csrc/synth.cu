// Synthetic-input generator for tests and the benchmark harness (not part of
// the optimizer step).  Counter-based: element i of stream `key` is a
// Box-Muller normal from two splitmix64 draws (src/rng.cpp:9-14, :36-45), the
// same formula as oracle/spngd_oracle.cpp:or_synth_normal, so every GPU
// generates its shard in place and captures never cross PCIe.
// Conv captures are materialised in the reference's stacked im2col layout
// (src/net.cpp:199-219, row = ch*k*k + ky*k + kx, zero padding).
#include <cuda_runtime.h>

#include "ctx.cuh"

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__device__ __forceinline__ float synth_normal(uint64_t key, uint64_t c) {
  const uint64_t b1 = mix64(key ^ (2 * c)), b2 = mix64(key ^ (2 * c + 1));
  const double u1 = (double(b1 >> 11) + 1.0) * 0x1.0p-53;
  const double u2 = double(b2 >> 11) * 0x1.0p-53;
  return float(sqrt(-2.0 * log(u1)) * cospi(2.0 * u2));
}

__global__ void normal_kernel(float* out, int64_t n, uint64_t key, float scale, float shift, int relu) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    float v = synth_normal(key, uint64_t(i)) * scale + shift;
    if (relu) v = fmaxf(v, 0.f);
    out[i] = v;
  }
}

// out[(s*c*k*k + row)*ho*wo + col] = relu?(x[s, ch, iy, ix]) with x ~ N(0,1)
// drawn at counter s*c*h*w + (ch*h + iy)*w + ix; 0 in the padding.
__global__ void conv_capture_kernel(float* out, int64_t batch, int64_t c, int64_t h, int64_t w, int64_t k,
                                    int64_t stride, int64_t pad, uint64_t key, int relu, float scale, float shift) {
  const int64_t ho = (h + 2 * pad - k) / stride + 1, wo = (w + 2 * pad - k) / stride + 1;
  const int64_t rows = c * k * k, hw = ho * wo;
  const int64_t total = batch * rows * hw;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t col = e % hw;
    const int64_t rs = e / hw;
    const int64_t row = rs % rows, s = rs / rows;
    const int64_t ch = row / (k * k), kyx = row % (k * k), ky = kyx / k, kx = kyx % k;
    const int64_t oy = col / wo, ox = col % wo;
    const int64_t iy = oy * stride + ky - pad, ix = ox * stride + kx - pad;
    float v = 0.f;
    if (iy >= 0 && iy < h && ix >= 0 && ix < w) {
      v = synth_normal(key, uint64_t(((s * c + ch) * h + iy) * w + ix)) * scale + shift;
      if (relu) v = fmaxf(v, 0.f);
    }
    out[e] = v;
  }
}

// BN per-sample gradient pairs: g ~ N(0,1), b = 0.6 g + 0.8 N(0,1)
// (tests/acceptance.cpp:192-204).
__global__ void bn_pairs_kernel(float* gg, float* gb, int64_t n, uint64_t key) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const float g = synth_normal(key, uint64_t(2 * i));
    const float z = synth_normal(key, uint64_t(2 * i + 1));
    gg[i] = g;
    gb[i] = 0.6f * g + 0.8f * z;
  }
}

unsigned grid_for(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return unsigned(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

}  // namespace

extern "C" {

int spngd_synth_normal(spngd_ctx* ctx, float* out, int64_t n, uint64_t key, float scale, float shift, int relu) {
  SPNGD_CTX_SCOPE(ctx);
  if (!ctx || !out) return spngd::fail(SPNGD_ERR_INVALID, "synth: null");
  normal_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(out, n, key, scale, shift, relu);
  SPNGD_CUDA_TRY(cudaGetLastError());
  return SPNGD_OK;
}

int spngd_synth_conv_capture(spngd_ctx* ctx, float* out, int64_t batch, int64_t c, int64_t h, int64_t w, int64_t k,
                             int64_t stride, int64_t pad, uint64_t key, int relu, float scale, float shift) {
  SPNGD_CTX_SCOPE(ctx);
  if (!ctx || !out) return spngd::fail(SPNGD_ERR_INVALID, "synth: null");
  const int64_t ho = (h + 2 * pad - k) / stride + 1, wo = (w + 2 * pad - k) / stride + 1;
  const int64_t total = batch * c * k * k * ho * wo;
  conv_capture_kernel<<<grid_for(total), 256, 0, ctx->stream>>>(out, batch, c, h, w, k, stride, pad, key, relu, scale,
                                                              shift);
  SPNGD_CUDA_TRY(cudaGetLastError());
  return SPNGD_OK;
}

int spngd_synth_bn_pairs(spngd_ctx* ctx, float* gg, float* gb, int64_t n, uint64_t key) {
  SPNGD_CTX_SCOPE(ctx);
  if (!ctx || !gg || !gb) return spngd::fail(SPNGD_ERR_INVALID, "synth: null");
  bn_pairs_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(gg, gb, n, key);
  SPNGD_CUDA_TRY(cudaGetLastError());
  return SPNGD_OK;
}

}  // extern "C"
