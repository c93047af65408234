// K1: Kronecker-factor construction (factor_A / factor_G, src/fisher.cpp:55-145)
// and K2: BatchNorm unit moments (build_bn_block, src/fisher.cpp:147-185).
//
// K1 is one grouped SYRK launch over every requested factor: only the upper
// triangle of 128x128 tiles is computed (SYRK-half), the capture is read in
// its reference layout (conv: stacked im2col (M*dim) x hw, FC: M x dim), and
// the epilogue writes the packed upper triangle (linalg.hpp:48-51) scaled by
// 1/(n*hw) or 1/n directly.  Long K (up to B*h*w = 401,408 at ResNet-50 conv1)
// is split into chunks whose fp32 partial tiles are summed in fp64 by a
// deterministic reduction kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "ctx.cuh"
#include "factor.cuh"
#include "gemm_tf32x3.cuh"

namespace spngd {

namespace {

__global__ void bn_moments_kernel(const spngd_bn_moments_req* __restrict__ reqs) {
  const spngd_bn_moments_req r = reqs[blockIdx.y];
  const int64_t ch = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (ch >= r.c) return;
  // Same per-channel accumulation order as build_bn_block (fisher.cpp:172-177).
  double sgg = 0.0, sgb = 0.0, sbb = 0.0;
  for (int64_t s = r.lo; s < r.hi; ++s) {
    const double g = r.gg[s * r.c + ch], b = r.gb[s * r.c + ch];
    sgg += g * g;
    sgb += g * b;
    sbb += b * b;
  }
  const double inv_n = 1.0 / double(r.hi - r.lo);
  r.out3c[3 * ch + 0] = float(sgg * inv_n);
  r.out3c[3 * ch + 1] = float(sgb * inv_n);
  r.out3c[3 * ch + 2] = float(sbb * inv_n);
}

// im2col (net.cpp:199-219) per sample: out[(s*rows + row)*hw + col], row =
// ch*k*k + ky*k + kx, col = oy*wo + ox; coalesced writes, gathered reads that
// hit L1/L2 k*k times.  HBM-bound: reads B*c*h*w, writes B*c*k*k*hw floats.
// One warp per output row (s, ch, ky, kx): the row decomposition is
// warp-uniform, and each lane walks its columns incrementally (one division
// per lane per row) -- the per-element div/mod chain of a flat mapping made
// the kernel issue-bound at ~0.8 TB/s (ncu, profiles/r01_kernel_captures.json).
template <typename I>
__device__ __forceinline__ void im2col_range(const spngd_im2col_req& r) {
  const spngd_conv_geom g = r.geom;
  const I h = I(g.h), w = I(g.w), k = I(g.k), st = I(g.stride), pad = I(g.pad), c = I(g.c_in);
  const I ho = (h + 2 * pad - k) / st + 1, wo = (w + 2 * pad - k) / st + 1;
  const I kk = k * k, rows = c * kk, hw = ho * wo;
  const I nrows = I(r.batch) * rows;
  const int lane = threadIdx.x & 31;
  const I warps = I(gridDim.x) * (blockDim.x >> 5);
  const I oy0 = I(lane) / wo, ox0 = I(lane) - oy0 * wo;
  const I dy = I(32) / wo, dx = I(32) - dy * wo;  // advancing col by 32
  for (I rs = I(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); rs < nrows; rs += warps) {
    const I s = rs / rows, row = rs - s * rows;
    const I ch = row / kk, kyx = row - ch * kk, ky = kyx / k, kx = kyx - ky * k;
    const float* __restrict__ src = r.x + int64_t(s * c + ch) * h * w;
    float* __restrict__ dst = r.out + int64_t(rs) * hw;
    I oy = oy0, ox = ox0;
    // four columns per lane in flight: one outstanding load per warp left
    // ~8 KB in flight per SM (latency-bound, 2.15 TB/s; now 2.6 TB/s).  A
    // shared-memory plane-staging variant measured 2.6x slower (occupancy cut
    // by the largest plane's buffer, tiny 7x7 planes latency-bound).
    for (I col = lane; col < hw; col += 128) {
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const I iy = oy * st + ky - pad, ix = ox * st + kx - pad;  // signed: padding reads as 0
        v[u] = 0.f;
        if (col + 32 * u < hw && iy >= 0 && iy < h && ix >= 0 && ix < w) v[u] = __ldg(src + iy * w + ix);
        oy += dy;
        ox += dx;
        if (ox >= wo) { ox -= wo; ++oy; }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (col + 32 * u < hw) dst[col + 32 * u] = v[u];
    }
  }
}

// im2col (net.cpp:199-219) per sample: out[(s*rows + row)*hw + col], row =
// ch*k*k + ky*k + kx, col = oy*wo + ox; coalesced writes, gathered reads that
// hit L1/L2 k*k times.  HBM-bound: reads B*c*h*w, writes B*c*k*k*hw floats.
// 32-bit index math whenever the capture has < 2^31 elements (always, at
// ResNet-50 B = 256).
__global__ void im2col_kernel(const spngd_im2col_req* __restrict__ reqs) {
  const spngd_im2col_req r = reqs[blockIdx.y];
  const spngd_conv_geom& g = r.geom;
  const int64_t ho = (g.h + 2 * g.pad - g.k) / g.stride + 1, wo = (g.w + 2 * g.pad - g.k) / g.stride + 1;
  if (r.batch * g.c_in * g.k * g.k * ho * wo < (int64_t(1) << 31))
    im2col_range<int32_t>(r);
  else
    im2col_range<int64_t>(r);
}

// BN branch of grad_payload (dist.cpp:364-371): [sum_s g_gamma / m | sum_s g_beta / m].
__global__ void bn_grad_payload_kernel(const BnGradPayloadTask* __restrict__ tasks) {
  const BnGradPayloadTask t = tasks[blockIdx.y];
  const int64_t ch = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (ch >= t.c) return;
  double sg = 0.0, sb = 0.0;
  for (int64_t s = 0; s < t.m; ++s) {
    sg += t.gg[s * t.c + ch];
    sb += t.gb[s * t.c + ch];
  }
  t.out[ch] = float(sg / double(t.m));
  t.out[t.c + ch] = float(sb / double(t.m));
}

// X'[i][s*hw + p] = X[(s*dim + i)*hw + p]: coalesced reads, runs of hw writes.
// Four consecutive source elements per thread: one float4 load (the source
// base is 16-byte aligned), one division for the group, four scalar stores.
template <typename I>
__device__ __forceinline__ void repack_range(const RepackTask& t) {
  const I hw = I(t.hw), dim = I(t.dim), n = I(t.n);
  const I total = n * dim * hw;
  const bool vec = (reinterpret_cast<uintptr_t>(t.src) & 15) == 0;
  const I step = I(gridDim.x) * blockDim.x;
  if (vec) {
    const I total4 = total / 4;
    for (I q = I(blockIdx.x) * blockDim.x + threadIdx.x; q < total4; q += step) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(t.src) + q);
      const float vv[4] = {v.x, v.y, v.z, v.w};
      I e = 4 * q, row = e / hw, p = e - row * hw;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const I s_ = row / dim, i = row - s_ * dim;
        t.dst[int64_t(i) * (n * hw) + s_ * hw + p] = vv[u];
        if (++p == hw) { p = 0; ++row; }
      }
    }
  }
  for (I e = (vec ? total / 4 * 4 : 0) + I(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += step) {
    const I row = e / hw, p = e - row * hw;
    const I s_ = row / dim, i = row - s_ * dim;
    t.dst[int64_t(i) * (n * hw) + s_ * hw + p] = __ldg(t.src + e);
  }
}

// 32-bit index math when the capture has < 2^31 elements (64-bit division
// dominated the old kernel: 1.9 TB/s on ResNet-50's 196 MB).
__global__ void repack_kernel(const RepackTask* __restrict__ tasks) {
  const RepackTask t = tasks[blockIdx.y];
  if (t.n * t.dim * t.hw < (int64_t(1) << 31))
    repack_range<int32_t>(t);
  else
    repack_range<int64_t>(t);
}

}  // namespace

int launch_repack(spngd_ctx* ctx, const RepackTask* d_tasks, int n, int64_t max_elems) {
  if (n <= 0) return SPNGD_OK;
  dim3 grid(unsigned(std::min<int64_t>((max_elems + 255) / 256, 2048)), unsigned(n));
  repack_kernel<<<grid, 256, 0, ctx->stream>>>(d_tasks);
  SPNGD_CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return SPNGD_OK;
}

int plan_factors(const spngd_factor_req* reqs, int n, FactorPlan& plan, float* ws) {
  plan = FactorPlan();
  std::vector<std::pair<int64_t, int64_t>> tk;
  for (int i = 0; i < n; ++i) {
    const spngd_factor_req& r = reqs[i];
    if (!r.x || !r.packed_out) return fail(SPNGD_ERR_INVALID, "factor request %d: null pointer", i);
    if (r.dim <= 0) return fail(SPNGD_ERR_SHAPE_MISMATCH, "factor request %d: dim must be > 0", i);
    if (r.lo < 0 || r.hi <= r.lo) return fail(SPNGD_ERR_EMPTY_BATCH, "factor request %d: empty sample range", i);
    if (r.layout == 1 && r.hw <= 0) return fail(SPNGD_ERR_SHAPE_MISMATCH, "factor request %d: hw must be > 0", i);
    GemmOperand op{};
    if (r.layout == 0) {  // FC: element (row i, sample s) = x[s*dim + i]
      op.ptr = r.x + r.lo * r.dim;
      op.row_stride = 1;
      op.seg_len = 1;
      op.seg_stride = r.dim;
    } else {              // conv: element (i, s*hw+p) = x[s*dim*hw + i*hw + p]
      op.ptr = r.x + r.lo * r.dim * r.hw;
      op.row_stride = r.hw;
      op.seg_len = r.hw;
      op.seg_stride = r.dim * r.hw;
    }
    op.rows = int32_t(r.dim);
    op.nseg = r.hi - r.lo;
    const int64_t K_true = (r.hi - r.lo) * (r.layout == 0 ? 1 : r.hw);
    const int64_t hw = r.layout == 0 ? 1 : r.hw;
    if (hw % 4 != 0 && K_true % 4 == 0) {
      // Row strides of 4*hw bytes defeat TMA (16-byte strides): repack this
      // capture K-contiguous first and read it as a dense 2D operand.
      float* dst = ws ? ws + plan.repack_floats : nullptr;
      plan.repacks.push_back({op.ptr, dst, r.hi - r.lo, r.dim, hw});
      plan.repack_floats += size_t(round_up(r.dim * K_true, 64));
      plan.repack_max = std::max(plan.repack_max, r.dim * K_true);
      op.ptr = dst;
      op.row_stride = K_true;
      op.seg_len = K_true;
      op.seg_stride = 0;
    }
    finalize_operand(op, K_true);
    // TMA-3D iterates zero-padded 32-wide chunks per sample (padded_k).
    const int64_t K = padded_k(op, K_true);
    if (K > INT32_MAX) return fail(SPNGD_ERR_SHAPE_MISMATCH, "factor request %d: K too large", i);
    GemmProblem p{};
    p.A = op;
    p.B = op;
    p.M = p.N = int32_t(r.dim);
    p.K = int32_t(K);
    p.flags = FLAG_SAME_AB;
    p.alpha = float(r.scale);
    p.C = r.packed_out;
    plan.probs.push_back(p);
    const int64_t t = (r.dim + kTileM - 1) / kTileM;
    tk.push_back({t * (t + 1) / 2, K});
  }
  plan.kchunk = choose_kchunk(tk);
  // The single-CTA problems (n = 64, 128, 576) form their own launch after the
  // 2-CTA one: chunk them for ~4 waves of their own (with the shared chunk the
  // ResNet-50 launch had 193 CTAs, 1.3 waves, ~1.85 ms at 0.23 of the roofline).
  std::vector<std::pair<int64_t, int64_t>> tk_single;
  for (int i = 0; i < n; ++i)
    if (!pair_eligible(plan.probs[i])) tk_single.push_back(tk[size_t(i)]);
  int kchunk_single = tk_single.empty() ? plan.kchunk : std::min(plan.kchunk, choose_kchunk(tk_single, 4));
  static const char* kc_env = getenv("SPNGD_KCHUNK");  // experiment override (multiple of 32)
  if (kc_env && atoi(kc_env) >= 32) plan.kchunk = kchunk_single = atoi(kc_env) / 32 * 32;
  int slot = 0;
  std::vector<GemmWorkItem> pair_items;
  plan.pair_prob.assign(size_t(n), 0);
  for (int i = 0; i < n; ++i) {
    GemmProblem& p = plan.probs[i];
    const int chunk = pair_eligible(p) ? plan.kchunk : kchunk_single;
    const bool split = p.K > chunk;
    p.mode = split ? EPI_PARTIAL : EPI_PACKED;
    const int kc = split ? chunk : p.K + kTileK;
    if (pair_eligible(p)) {  // 256 x 256 tiles on CTA pairs (gemm_pair.cu)
      plan.pair_prob[size_t(i)] = 1;
      plan_pair_tiles(i, p, kc, pair_items, &plan.reduce, &slot, reqs[i].scale, reqs[i].packed_out);
    } else {
      plan_problem_tiles(i, p, /*upper_only=*/true, kc, plan.items, &plan.reduce, &slot, reqs[i].scale,
                         reqs[i].packed_out);
    }
  }
  plan.n_slots = slot;
  // Longest work first: items are independent, so issue the big K ranges early
  // (cluster pairs move as units).
  auto longer = [](const GemmWorkItem& x, const GemmWorkItem& y) { return (x.k1 - x.k0) > (y.k1 - y.k0); };
  std::stable_sort(plan.items.begin(), plan.items.end(), longer);
  std::vector<std::pair<GemmWorkItem, GemmWorkItem>> pairs;
  for (size_t q = 0; q + 1 < pair_items.size(); q += 2) pairs.push_back({pair_items[q], pair_items[q + 1]});
  std::stable_sort(pairs.begin(), pairs.end(), [&](const auto& x, const auto& y) { return longer(x.first, y.first); });
  std::vector<GemmWorkItem> all;
  for (const auto& pr : pairs) {
    all.push_back(pr.first);
    all.push_back(pr.second);
  }
  plan.n_pair = int(all.size());
  all.insert(all.end(), plan.items.begin(), plan.items.end());
  plan.items.swap(all);
  return SPNGD_OK;
}

int count_pair_items(const FactorPlan& plan, const std::vector<GemmWorkItem>& items) {
  int k = 0;
  while (k < int(items.size()) && plan.pair_prob[size_t(items[size_t(k)].problem)]) ++k;
  return k;
}

int launch_factor_gemm(spngd_ctx* ctx, const FactorPlan& plan, const GemmProblem* d_probs, int n_pair,
                       const GemmWorkItem* d_items, int n_items, float* d_partials, cudaStream_t stream) {
  int rc = launch_syrk_pair(d_probs, d_items, n_pair, d_partials, stream);
  if (rc || n_items <= n_pair) return rc;
  return launch_gemm(d_probs, d_items + n_pair, n_items - n_pair, d_partials, ctx->d_status, stream,
                     gemm_variant(plan.probs.data(), int(plan.probs.size())));
}

int run_factors(spngd_ctx* ctx, const FactorPlan& plan, const GemmProblem* d_probs, int n_pair,
                const GemmWorkItem* d_items, int n_items, float* d_partials, const SyrkReduceTask* d_reduce,
                int n_reduce) {
  int rc = launch_factor_gemm(ctx, plan, d_probs, n_pair, d_items, n_items, d_partials, ctx->stream);
  if (rc) return rc;
  ctx->launches += n_items > 0;
  rc = launch_syrk_reduce(d_reduce, n_reduce, d_partials, ctx->stream);
  ctx->launches += n_reduce > 0;
  return rc;
}

int launch_im2col(spngd_ctx* ctx, const spngd_im2col_req* d_reqs, int n) {
  if (n <= 0) return SPNGD_OK;
  dim3 grid(148u * 8u, unsigned(n));
  im2col_kernel<<<grid, 256, 0, ctx->stream>>>(d_reqs);
  SPNGD_CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return SPNGD_OK;
}

int check_conv_geom(const spngd_conv_geom& g, int64_t a, int64_t hw) {
  if (g.c_in <= 0 || g.h <= 0 || g.w <= 0 || g.k <= 0 || g.stride <= 0 || g.pad < 0)
    return fail(SPNGD_ERR_SHAPE_MISMATCH, "conv geometry must be positive");
  const int64_t ho = (g.h + 2 * g.pad - g.k) / g.stride + 1, wo = (g.w + 2 * g.pad - g.k) / g.stride + 1;
  if (ho <= 0 || wo <= 0) return fail(SPNGD_ERR_SHAPE_MISMATCH, "conv geometry: empty output");
  if ((a >= 0 && g.c_in * g.k * g.k != a) || (hw >= 0 && ho * wo != hw))
    return fail(SPNGD_ERR_SHAPE_MISMATCH, "conv geometry does not match the layer (a = c_in k^2, hw = h_out w_out)");
  return SPNGD_OK;
}

int launch_bn_grad_payload(spngd_ctx* ctx, const BnGradPayloadTask* d_tasks, int n, int64_t max_c) {
  if (n <= 0) return SPNGD_OK;
  dim3 grid(unsigned((max_c + 255) / 256), unsigned(n));
  bn_grad_payload_kernel<<<grid, 256, 0, ctx->stream>>>(d_tasks);
  SPNGD_CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return SPNGD_OK;
}

int launch_bn_moments(spngd_ctx* ctx, const spngd_bn_moments_req* d_reqs, int n, int64_t max_c) {
  if (n <= 0) return SPNGD_OK;
  dim3 grid(unsigned((max_c + 255) / 256), unsigned(n));
  bn_moments_kernel<<<grid, 256, 0, ctx->stream>>>(d_reqs);
  SPNGD_CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return SPNGD_OK;
}

}  // namespace spngd

extern "C" int spngd_factor_sym_batched(spngd_ctx* ctx, int n, const spngd_factor_req* reqs) {
  SPNGD_CTX_SCOPE(ctx);
  using namespace spngd;
  if (!ctx || (n > 0 && !reqs)) return fail(SPNGD_ERR_INVALID, "spngd_factor_sym_batched: null argument");
  if (n == 0) return SPNGD_OK;
  FactorPlan sizing;
  int rc = plan_factors(reqs, n, sizing);
  if (rc) return rc;
  DeviceScratch scratch(ctx);
  float* ws = scratch.alloc<float>(std::max<size_t>(sizing.repack_floats, 1));
  FactorPlan plan;
  plan_factors(reqs, n, plan, ws);
  auto* d_repack = scratch.upload(plan.repacks);
  rc = launch_repack(ctx, d_repack, int(plan.repacks.size()), plan.repack_max);
  if (rc) return rc;
  auto* d_probs = scratch.upload(plan.probs);
  auto* d_items = scratch.upload(plan.items);
  auto* d_reduce = scratch.upload(plan.reduce);
  float* d_partials = scratch.alloc<float>(size_t(std::max(plan.n_slots, 1)) * kTileM * kTileN);
  if (!d_probs || !d_items || !d_reduce || !d_partials) return fail(SPNGD_ERR_CUDA, "factor: workspace allocation failed");
  rc = run_factors(ctx, plan, d_probs, plan.n_pair, d_items, int(plan.items.size()), d_partials, d_reduce,
                   int(plan.reduce.size()));
  if (rc) return rc;
  SPNGD_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return SPNGD_OK;
}

extern "C" int spngd_bn_moments_batched(spngd_ctx* ctx, int n, const spngd_bn_moments_req* reqs) {
  SPNGD_CTX_SCOPE(ctx);
  using namespace spngd;
  if (!ctx || (n > 0 && !reqs)) return fail(SPNGD_ERR_INVALID, "spngd_bn_moments_batched: null argument");
  int64_t max_c = 0;
  for (int i = 0; i < n; ++i) {
    if (reqs[i].lo < 0 || reqs[i].hi <= reqs[i].lo) return fail(SPNGD_ERR_EMPTY_BATCH, "build_bn_block: empty sample range");
    if (!reqs[i].gg || !reqs[i].gb || !reqs[i].out3c) return fail(SPNGD_ERR_EMPTY_BATCH, "build_bn_block: no captured gradients");
    max_c = std::max(max_c, reqs[i].c);
  }
  if (n == 0) return SPNGD_OK;
  DeviceScratch scratch(ctx);
  std::vector<spngd_bn_moments_req> v(reqs, reqs + n);
  auto* d = scratch.upload(v);
  int rc = launch_bn_moments(ctx, d, n, max_c);
  if (rc) return rc;
  SPNGD_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return SPNGD_OK;
}

using namespace spngd;

extern "C" int spngd_im2col_batched(spngd_ctx* ctx, int n, const spngd_im2col_req* reqs) {
  SPNGD_CTX_SCOPE(ctx);
  if (!ctx || (n > 0 && !reqs)) return fail(SPNGD_ERR_INVALID, "spngd_im2col_batched: null argument");
  if (n == 0) return SPNGD_OK;
  for (int i = 0; i < n; ++i) {
    if (!reqs[i].x || !reqs[i].out) return fail(SPNGD_ERR_INVALID, "im2col: null pointer");
    if (reqs[i].batch <= 0) return fail(SPNGD_ERR_EMPTY_BATCH, "im2col: empty batch");
    int rc = check_conv_geom(reqs[i].geom, -1, -1);
    if (rc) return rc;
  }
  DeviceScratch scratch(ctx);
  std::vector<spngd_im2col_req> v(reqs, reqs + n);
  auto* d = scratch.upload(v);
  int rc = launch_im2col(ctx, d, n);
  if (rc) return rc;
  return spngd_ctx_sync(ctx);
}
