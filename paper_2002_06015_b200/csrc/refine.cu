// Accuracy refinement of the explicit damped inverse (spd_inverse,
// src/linalg.cpp:29-48, where Eigen's LLT + solve(I) runs in fp64).
//
// The fp32 recursive Cholesky inverse (inverse.cu) has a forward error of
// about 3e-9 * cond(M + dI) (measured on post-ReLU factors):
// it passes the 1e-4 gate up to cond ~3e4, but the rank-deficient K < n
// factors of the config-5 sweep reach cond 4.7e4 at n = 4608.  For those one
// step of iterative refinement is applied:
//
//   R'^T = X0' M - I            (residual, formed exactly enough)
//   X1   = X0 - X0 R'           (correction; R' is small, so 3xTF32 is ample)
//   X    = (X1 + X1^T) / 2      (the reference's symmetrization)
//
// The residual must be formed in better than fp32 (an fp32 residual gains
// only ~2x).  With M = Mh + Mr (Mh = tf32 truncation of M, Mr = M - Mh exact
// in fp32) the 3xTF32 engine's products over the K-concatenation
//   [X0 | X0] . [Mh | Mr]^T
// are  Xl Mh + Xh Mh  (Mh has no lo part)  +  Xl Mm + Xh Ml + Xh Mm  (Mr = Mm
// + Ml exactly), i.e. X0' M up to the Xl Ml term (2^-33 relative), where X0'
// = Xh + Xl is the 22-bit split of X0 the engine uses anyway.  Accumulation
// is the engine's per-stage round-to-nearest drain.  Measured (numpy
// emulation, n = 2048 / 4608 post-ReLU K = n/2): 1.6e-4 / 2.6e-4 (LAPACK
// fp32) -> ~2e-5 / ~3e-5 after the step.
//
// Whether to refine is decided per matrix from ||M + dI||_F / d, an upper
// bound of cond(M + dI) (lambda_min >= d for PSD M, ||.||_2 <= ||.||_F).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>

#include "ctx.cuh"
#include "inverse.cuh"

namespace spngd {

namespace {

constexpr double kRefineCond = 1.5e4;  // predicted error 3e-9 * cond = 4.5e-5 at the threshold

__global__ void fro_kernel(const FroTask* __restrict__ tasks) {
  const FroTask t = tasks[blockIdx.y];
  const float d = t.damp_dev ? t.damp_dev[0] : t.damp;
  double s = 0.0;
  for (int64_t i = blockIdx.x; i < t.n; i += gridDim.x) {
    const float* row = t.packed + packed_offset(t.n, i, i);  // (i, i .. n-1)
    const int64_t len = t.n - i;
    for (int64_t j = threadIdx.x; j < len; j += blockDim.x) {
      const double v = j == 0 ? double(row[0] + d) : double(row[j]);
      s += (j == 0 ? 1.0 : 2.0) * v * v;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) tot += red[w];
    atomicAdd(t.sumsq, tot);
  }
}

struct SplitTask {
  const float* Md;   // dense M + dI (n x ld)
  const float* X0;   // dense inverse (n x ld)
  float* Mcat;       // n x 2ld: [Mh | Mr]
  float* Xcat;       // n x 2ld: [X0 | X0]
  float* Iden;       // n x ld identity
  int64_t n, ld;
};

// Elementwise, float4 over the ld-wide rows (ld % 32 == 0); columns >= n are
// zero in every output so the padded K range contributes nothing.
__global__ void refine_split_kernel(const SplitTask* __restrict__ tasks) {
  const SplitTask t = tasks[blockIdx.y];
  const int64_t q4 = t.ld / 4, total = t.n * q4;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / q4, j0 = (e - i * q4) * 4;
    float m[4], x[4], h[4], r[4], id[4];
    const float4 mv = *reinterpret_cast<const float4*>(t.Md + i * t.ld + j0);
    const float4 xv = *reinterpret_cast<const float4*>(t.X0 + i * t.ld + j0);
    m[0] = mv.x; m[1] = mv.y; m[2] = mv.z; m[3] = mv.w;
    x[0] = xv.x; x[1] = xv.y; x[2] = xv.z; x[3] = xv.w;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const bool in = j0 + c < t.n;
      if (!in) m[c] = x[c] = 0.f;
      h[c] = __uint_as_float(__float_as_uint(m[c]) & 0xffffe000u);
      r[c] = m[c] - h[c];  // exact
      id[c] = (j0 + c == i) ? 1.f : 0.f;
    }
    float* mc = t.Mcat + i * 2 * t.ld + j0;
    float* xc = t.Xcat + i * 2 * t.ld + j0;
    *reinterpret_cast<float4*>(mc) = make_float4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<float4*>(mc + t.ld) = make_float4(r[0], r[1], r[2], r[3]);
    *reinterpret_cast<float4*>(xc) = make_float4(x[0], x[1], x[2], x[3]);
    *reinterpret_cast<float4*>(xc + t.ld) = make_float4(x[0], x[1], x[2], x[3]);
    *reinterpret_cast<float4*>(t.Iden + i * t.ld + j0) = make_float4(id[0], id[1], id[2], id[3]);
  }
}

struct SymTask {
  const float* X1;   // n x ld
  float* X;          // n x ld: (X1 + X1^T) / 2
  int64_t n, ld;
};

// 32 x 32 tiles of the upper triangle: tile (ti, tj) and its mirror are both
// staged so every global access is a row access.
__global__ void symmetrize_kernel(const SymTask* __restrict__ tasks) {
  const SymTask t = tasks[blockIdx.y];
  __shared__ float a[32][33], b[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int64_t tn = (t.n + 31) / 32;
  for (int64_t tt = blockIdx.x; tt < tn * tn; tt += gridDim.x) {
    const int64_t ti = tt / tn, tj = tt - ti * tn;
    if (ti > tj) continue;
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int li = ty + 8 * q;
      const int64_t i = ti * 32 + li, j = tj * 32 + tx;  // tile (ti, tj)
      a[li][tx] = (i < t.n && j < t.n) ? t.X1[i * t.ld + j] : 0.f;
      const int64_t i2 = tj * 32 + li, j2 = ti * 32 + tx;  // tile (tj, ti)
      b[li][tx] = (i2 < t.n && j2 < t.n) ? t.X1[i2 * t.ld + j2] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int li = ty + 8 * q;
      const int64_t i = ti * 32 + li, j = tj * 32 + tx;
      const float v = 0.5f * (a[li][tx] + b[tx][li]);
      if (i < t.n && j < t.n) t.X[i * t.ld + j] = v;
      const int64_t i2 = tj * 32 + li, j2 = ti * 32 + tx;
      if (ti != tj && i2 < t.n && j2 < t.n) t.X[i2 * t.ld + j2] = 0.5f * (b[li][tx] + a[tx][li]);
    }
  }
}

GemmOperand dense_operand(const float* ptr, int64_t ld, int64_t rows, int64_t K) {
  GemmOperand o{};
  o.ptr = ptr;
  o.row_stride = ld;
  o.seg_len = K;
  o.seg_stride = 0;
  o.rows = int32_t(rows);
  finalize_operand(o, K);
  return o;
}

GemmProblem dense_problem(const GemmOperand& a, const GemmOperand& b, int64_t M, int64_t N, int64_t K, float alpha,
                          float beta, const float* Cin, float* C, int64_t ldc) {
  GemmProblem p{};
  p.A = a;
  p.B = b;
  p.M = int32_t(M); p.N = int32_t(N); p.K = int32_t(K);
  p.mode = EPI_DENSE;
  p.alpha = alpha; p.beta = beta;
  p.C = C; p.Cin = Cin; p.ldc = ldc;
  return p;
}

}  // namespace

double refine_threshold() {
  static const double t = [] {
    const char* e = getenv("SPNGD_REFINE_COND");
    if (!e) return kRefineCond;
    const double v = atof(e);
    return v < 0 ? INFINITY : v;
  }();
  return t;
}

int launch_fro(spngd_ctx* ctx, const FroTask* d_tasks, int n, int64_t max_n) {
  if (n <= 0) return SPNGD_OK;
  dim3 grid(unsigned(std::min<int64_t>(std::max<int64_t>(max_n, 1), 256)), unsigned(n));
  fro_kernel<<<grid, 256, 0, ctx->stream>>>(d_tasks);
  SPNGD_CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return SPNGD_OK;
}

namespace {

// One grouped GEMM over `probs`: the 2-CTA 256 x 256 kernel for the problems it
// covers without waste, the 128 x 256 kernel for the rest.
int launch_dense_group(spngd_ctx* ctx, DeviceScratch& scratch, const std::vector<GemmProblem>& probs) {
  std::vector<GemmWorkItem> pair, single_elig, single;
  for (size_t q = 0; q < probs.size(); ++q) {
    int slot = 0;
    if (!no_pair_inv() && pair_eligible_dense(probs[q])) {
      plan_pair_dense(int(q), probs[q], pair);
      plan_problem_tiles(int(q), probs[q], false, probs[q].K + kTileK, single_elig, nullptr, &slot, 1.0, nullptr);
    } else {
      plan_problem_tiles(int(q), probs[q], false, probs[q].K + kTileK, single, nullptr, &slot, 1.0, nullptr);
    }
  }
  if (!pair_group_wins(int64_t(pair.size()), int64_t(single_elig.size()), int64_t(single.size()))) {
    pair.clear();
    single.insert(single.begin(), single_elig.begin(), single_elig.end());
  }
  auto* d_probs = scratch.upload(probs);
  auto* d_pair = pair.empty() ? nullptr : scratch.upload(pair);
  auto* d_single = single.empty() ? nullptr : scratch.upload(single);
  if (!d_probs || (!pair.empty() && !d_pair) || (!single.empty() && !d_single))
    return fail(SPNGD_ERR_CUDA, "refine: descriptor upload failed");
  int rc = SPNGD_OK;
  if (!pair.empty()) {
    if ((rc = launch_syrk_pair(d_probs, d_pair, int(pair.size()), nullptr, ctx->stream, ctx->d_status))) return rc;
    ctx->launches++;
  }
  if (!single.empty()) {
    rc = launch_gemm(d_probs, d_single, int(single.size()), nullptr, ctx->d_status, ctx->stream,
                     gemm_variant(probs.data(), int(probs.size())));
    if (rc) return rc;
    ctx->launches++;
  }
  return SPNGD_OK;
}

}  // namespace

int refine_inverses(spngd_ctx* ctx, DeviceScratch& scratch, const std::vector<RefineJob>& jobs) {
  if (jobs.empty()) return SPNGD_OK;
  std::vector<UnpackTask> unpack;
  std::vector<SplitTask> split;
  std::vector<SymTask> sym;
  std::vector<GemmProblem> p1, p2;
  int64_t max_n = 0, max_elems = 0;
  for (const RefineJob& j : jobs) {
    const int64_t n = j.n, ld = j.ld;
    float* Md = scratch.alloc<float>(size_t(n) * ld);
    float* Mcat = scratch.alloc<float>(size_t(n) * 2 * ld);
    float* Xcat = scratch.alloc<float>(size_t(n) * 2 * ld);
    float* Iden = scratch.alloc<float>(size_t(n) * ld);
    float* X1 = scratch.alloc<float>(size_t(n) * ld);
    if (!Md || !Mcat || !Xcat || !Iden || !X1) return fail(SPNGD_ERR_CUDA, "refine: scratch allocation failed");
    float* RT = Md;  // M + dI is dead once split
    unpack.push_back({j.packed, n, nullptr, j.damp, 0, Md, ld, nullptr});
    split.push_back({Md, j.X, Mcat, Xcat, Iden, n, ld});
    // R'^T = X0' M - I  (rows of Xcat x rows of Mcat, K = 2 ld)
    p1.push_back(dense_problem(dense_operand(Xcat, 2 * ld, n, 2 * ld), dense_operand(Mcat, 2 * ld, n, 2 * ld), n, n,
                               2 * ld, 1.f, -1.f, Iden, RT, ld));
    // X1 = X0 - X0 R'   (B rows = rows of R'^T)
    p2.push_back(dense_problem(dense_operand(j.X, ld, n, n), dense_operand(RT, ld, n, n), n, n, n, -1.f, 1.f, j.X,
                               X1, ld));
    sym.push_back({X1, j.X, n, ld});
    max_n = std::max(max_n, n);
    max_elems = std::max(max_elems, n * ld);
  }
  auto* d_unpack = scratch.upload(unpack);
  auto* d_split = scratch.upload(split);
  auto* d_sym = scratch.upload(sym);
  if (!d_unpack || !d_split || !d_sym) return fail(SPNGD_ERR_CUDA, "refine: descriptor upload failed");
  int rc = launch_unpack(ctx, d_unpack, int(unpack.size()), max_n);
  if (rc) return rc;
  {
    const int64_t q4 = max_elems / 4;
    dim3 grid(unsigned(std::min<int64_t>((q4 + 255) / 256, 4 * kNumSMs)), unsigned(split.size()));
    refine_split_kernel<<<grid, 256, 0, ctx->stream>>>(d_split);
    SPNGD_CUDA_TRY(cudaGetLastError());
    ctx->launches++;
  }
  if ((rc = launch_dense_group(ctx, scratch, p1))) return rc;
  if ((rc = launch_dense_group(ctx, scratch, p2))) return rc;
  {
    const int64_t tn = (max_n + 31) / 32;
    dim3 grid(unsigned(std::min<int64_t>(tn * tn, 1024)), unsigned(sym.size()));
    symmetrize_kernel<<<grid, 256, 0, ctx->stream>>>(d_sym);
    SPNGD_CUDA_TRY(cudaGetLastError());
    ctx->launches++;
  }
  return SPNGD_OK;
}

}  // namespace spngd
