// K3/K4: damped SPD inverse (spd_inverse, src/linalg.cpp:29-48;
// damp_and_invert, src/fisher.cpp:218-228).
//
// (M + dI)^-1 = L^-T L^-1 with L = chol(M + dI), like the reference's
// Eigen::LLT + solve(I), computed by a recursive blocked Cholesky that carries
// T = L^-1 along (n^3 flops: potrf n^3/3 + trtri n^3/3 + lauum n^3/3):
//     M = [A B^T-block ; B C]:  chol(A) -> T11 (recurse),
//     L21 = B T11^T,  S = C - L21 L21^T,  U^T = T11^T L21^T,
//     chol(S) -> T22 (recurse),  T21 = -T22 U,      finally X = T^T T.
// Every update is a K-major GEMM on the 3xTF32 tcgen05 engine; triangular
// operands trim the K range per tile.  Leaves (n <= 128) run one CTA that
// factors in fp32 registers and forms T by forward elimination.  Explicit
// inverses of ill-conditioned matrices get one refinement step (refine.cu).  A
// non-positive or non-finite pivot raises NotPositiveDefinite (the LLT
// failure of linalg.cpp:37-40).  X is written upper-tile + mirrored, so the
// result is exactly symmetric as the reference's 0.5 (X + X^T) makes it.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "ctx.cuh"
#include "inverse.cuh"

namespace spngd {

namespace {

constexpr int kBaseMax = 128;
constexpr int kLeafWarps = 8;           // warp w owns rows 4 w + t + 32 g (t, g = 0..3)
constexpr int kBaseThreads = 32 * kLeafWarps;
constexpr int kLd = kBaseMax + 1;       // padded smem row (floats)
// staging [128][129] | published rows R [3][4][64] float2 | -L columns [3][128] float4
constexpr size_t kBaseSmem = size_t(kBaseMax) * kLd * sizeof(float) + 3 * 4 * 64 * sizeof(float2) +
                             3 * kBaseMax * sizeof(float4);

__device__ __forceinline__ float pivot_rsqrt(float p, bool& bad) {
  if (!(p > 0.f) || !isfinite(p)) {
    bad = true;
    p = 1.f;
  }
  const float inv = rsqrtf(p);
  return inv * fmaf(-0.5f * p, inv * inv, 1.5f);  // MUFU rsqrt + one Newton step
}

// One CTA per leaf (n <= 128): Cholesky by blocked column elimination with
// T = L^-1 formed in the same pass; the whole 128x128 working matrix X sits in
// registers (thread (w, l) holds rows 4w + t + 32g, columns 2l + 64p + {0,1}).
//
// Block b (rows/columns K = 4b..4b+3, one barrier): the warp owning rows K
// takes the 4x4 Schur block D = X_KK (already updated by blocks < b), forms
// L_d = chol(D) and T_d = L_d^-1 redundantly in every lane, and publishes
//     R = T_d * X~_K.     (X~_K = rows K with the K columns replaced by I)
// R holds T_Kj for j < 4b+4 (T_d itself in the K columns) and L_jK for j beyond
// (the trailing part of X is kept symmetric, so row K = column K there).  Every
// later row i then applies  X_i. -= L_iK R  with its K entries zeroed first:
// the Schur update for trailing columns, and for columns already eliminated
// the forward elimination T_ij = -(1/L_ii) sum_{k=j}^{i-1} L_ik T_kj carried
// column-block-wise (the 1/L_ii arrives when row i's block publishes).  After
// the last block the lower triangle of X is T.  Updates are packed fp32x2
// FMAs; fp32 storage and arithmetic (LAPACK spotrf/strtri class).
#ifdef SPNGD_GEMM_TRACE_BUILD
__device__ long long g_leaf_trace[8];
#define LEAF_STAMP(i) \
  do {                \
    if (blockIdx.x == 0 && threadIdx.x == 0) g_leaf_trace[i] = clock64(); \
  } while (0)
#else
#define LEAF_STAMP(i) \
  do {                \
  } while (0)
#endif

struct LeafBufs {
  float2* R;   // [3][4][64]: published rows by column pair
  float4* L;   // [3][128]:  (-L_i,4b .. -L_i,4b+3) by row i
};

// Apply block b (column pair group P = b >> 4, pairs 2b, 2b+1 in lanes lk0,
// lk0+1) to rows (G, t = 0..3) of this thread.
template <int G, int P>
__device__ __forceinline__ void leaf_apply(float2 (&x)[4][4][2], const float2 (&r)[4][2], const float4* lcol,
                                           int row0, float m) {
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const float4 nl = lcol[row0 + t];
    x[G][t][P] = __fmul2_rn(x[G][t][P], make_float2(m, m));
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      float2 v = x[G][t][p];
      v = __ffma2_rn(make_float2(nl.x, nl.x), r[0][p], v);
      v = __ffma2_rn(make_float2(nl.y, nl.y), r[1][p], v);
      v = __ffma2_rn(make_float2(nl.z, nl.z), r[2][p], v);
      v = __ffma2_rn(make_float2(nl.w, nl.w), r[3][p], v);
      x[G][t][p] = v;
    }
  }
}

// Row slots Gs..3 (slot Gs skipped when !first: already applied by the publisher).
template <int Gs, int P>
__device__ __forceinline__ void leaf_apply_rest(float2 (&x)[4][4][2], const float2 (&r)[4][2], const float4* lcol,
                                                int row0, float m, bool first) {
  if (first) leaf_apply<Gs, P>(x, r, lcol, row0 + 32 * Gs, m);
  if constexpr (Gs < 3) leaf_apply_rest<Gs + 1, P>(x, r, lcol, row0, m, true);
}

// Factor and publish block b = 8 G + warp (rows slot G of this warp).
template <int G>
__device__ __forceinline__ void leaf_publish(float2 (&x)[4][4][2], int b, int lane, float2* R, float4* L, bool& bad) {
  constexpr int P = G >> 1;
  const int lk0 = (2 * b) & 31;
  // D = X_KK gathered into every lane: lane lk0 holds columns (4b, 4b+1), lane
  // lk0 + 1 columns (4b+2, 4b+3).
  float d[4][4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    d[t][0] = __shfl_sync(0xffffffffu, x[G][t][P].x, lk0);
    d[t][1] = __shfl_sync(0xffffffffu, x[G][t][P].y, lk0);
    d[t][2] = __shfl_sync(0xffffffffu, x[G][t][P].x, lk0 + 1);
    d[t][3] = __shfl_sync(0xffffffffu, x[G][t][P].y, lk0 + 1);
  }
  // L_d = chol(D), T_d = L_d^-1 (lower; r_t = 1 / L_tt).
  const float r0 = pivot_rsqrt(d[0][0], bad);
  const float l10 = d[1][0] * r0, l20 = d[2][0] * r0, l30 = d[3][0] * r0;
  const float r1 = pivot_rsqrt(fmaf(-l10, l10, d[1][1]), bad);
  const float l21 = fmaf(-l20, l10, d[2][1]) * r1, l31 = fmaf(-l30, l10, d[3][1]) * r1;
  const float r2 = pivot_rsqrt(fmaf(-l21, l21, fmaf(-l20, l20, d[2][2])), bad);
  const float l32 = fmaf(-l31, l21, fmaf(-l30, l20, d[3][2])) * r2;
  const float r3 = pivot_rsqrt(fmaf(-l32, l32, fmaf(-l31, l31, fmaf(-l30, l30, d[3][3]))), bad);
  const float t10 = -r1 * l10 * r0;
  const float t21 = -r2 * l21 * r1;
  const float t20 = -r2 * fmaf(l21, t10, l20 * r0);
  const float t32 = -r3 * l32 * r2;
  const float t31 = -r3 * fmaf(l32, t21, l31 * r1);
  const float t30 = -r3 * fmaf(l32, t20, fmaf(l31, t10, l30 * r0));
  // X~: the block's own columns become the identity.
  if (lane == lk0) {
    x[G][0][P] = make_float2(1.f, 0.f);
    x[G][1][P] = make_float2(0.f, 1.f);
    x[G][2][P] = make_float2(0.f, 0.f);
    x[G][3][P] = make_float2(0.f, 0.f);
  } else if (lane == lk0 + 1) {
    x[G][0][P] = make_float2(0.f, 0.f);
    x[G][1][P] = make_float2(0.f, 0.f);
    x[G][2][P] = make_float2(1.f, 0.f);
    x[G][3][P] = make_float2(0.f, 1.f);
  }
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const float2 x0 = x[G][0][p], x1 = x[G][1][p], x2 = x[G][2][p], x3 = x[G][3][p];
    const float2 y0 = __fmul2_rn(make_float2(r0, r0), x0);
    const float2 y1 = __ffma2_rn(make_float2(r1, r1), x1, __fmul2_rn(make_float2(t10, t10), x0));
    const float2 y2 = __ffma2_rn(make_float2(r2, r2), x2,
                                 __ffma2_rn(make_float2(t21, t21), x1, __fmul2_rn(make_float2(t20, t20), x0)));
    const float2 y3 = __ffma2_rn(
        make_float2(r3, r3), x3,
        __ffma2_rn(make_float2(t32, t32), x2,
                   __ffma2_rn(make_float2(t31, t31), x1, __fmul2_rn(make_float2(t30, t30), x0))));
    x[G][0][p] = y0;
    x[G][1][p] = y1;
    x[G][2][p] = y2;
    x[G][3][p] = y3;
#pragma unroll
    for (int t = 0; t < 4; ++t) R[t * 64 + 32 * p + lane] = x[G][t][p];
    L[2 * lane + 64 * p] = make_float4(-y0.x, -y1.x, -y2.x, -y3.x);
    L[2 * lane + 64 * p + 1] = make_float4(-y0.y, -y1.y, -y2.y, -y3.y);
  }
  __syncwarp();  // the publishing warp reads its own rows next without waiting at the barrier
}

// Blocks b = 8 G + wp, wp = 0..7 (G static: which register rows can still be
// active and which column pair group holds the block are compile-time).  The
// warp owning block b + 1 applies block b to those rows first and publishes,
// then finishes its other rows while the CTA is still consuming block b; it
// only arrives at the barrier (it needs nothing newer than its own rows).
// Barrier ids alternate by parity so an arrive-only warp is never counted
// twice in one barrier instance.
template <int G>
__device__ __forceinline__ void leaf_blocks(float2 (&x)[4][4][2], int nb, int warp, int lane, LeafBufs buf,
                                            bool& bad) {
  constexpr int P = G >> 1;
  for (int wp = 0; wp < kLeafWarps; ++wp) {
    const int b = kLeafWarps * G + wp;
    if (b >= nb) return;
    // published rows rotate over three buffers: the producer of block b + 1
    // arrives as soon as it has published and may still be applying block b
    // while the producer of b + 2 writes the next buffer
    const float2* Rb = buf.R + (b % 3) * 256;
    const float4* Lb = buf.L + (b % 3) * kBaseMax;
    float2 r[4][2];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int p = 0; p < 2; ++p) r[t][p] = Rb[t * 64 + 32 * p + lane];
    const float m = ((lane >> 1) == (b & 15)) ? 0.f : 1.f;  // zero the block's own columns first
    const int b1 = b + 1;
    const bool producer = b1 < nb && warp == (b1 & (kLeafWarps - 1));
    float2* Rn = buf.R + (b1 % 3) * 256;
    float4* Ln = buf.L + (b1 % 3) * kBaseMax;
    if (producer) {
      if (wp < kLeafWarps - 1) {
        leaf_apply<G, P>(x, r, Lb, 4 * warp + 32 * G, m);
        leaf_publish<G>(x, b1, lane, Rn, Ln, bad);
      } else if constexpr (G < 3) {
        leaf_apply<G + 1, P>(x, r, Lb, 4 * warp + 32 * (G + 1), m);
        leaf_publish<G + 1>(x, b1, lane, Rn, Ln, bad);
      }
      // block b1 is published: release the other warps before finishing this
      // warp's remaining rows (the critical path is publish -> barrier -> publish)
      asm volatile("bar.arrive %0, %1;" ::"r"(1 + (b1 & 1)), "r"(kBaseThreads) : "memory");
    }
    if ((warp > wp) && !(producer && wp < kLeafWarps - 1)) leaf_apply<G, P>(x, r, Lb, 4 * warp + 32 * G, m);
    if constexpr (G < 3) leaf_apply_rest<G + 1, P>(x, r, Lb, 4 * warp, m, !(producer && wp == kLeafWarps - 1));
    if (!producer) asm volatile("bar.sync %0, %1;" ::"r"(1 + (b1 & 1)), "r"(kBaseThreads) : "memory");
  }
  if constexpr (G < 3) leaf_blocks<G + 1>(x, nb, warp, lane, buf, bad);
}

__global__ void __launch_bounds__(kBaseThreads, 1) base_chol_inv_kernel(const BaseTask* __restrict__ tasks, int* status) {
  LEAF_STAMP(0);
  extern __shared__ __align__(16) uint8_t base_smem[];
  float* S = reinterpret_cast<float*>(base_smem);  // [128][129] staging (M in, T out)
  LeafBufs buf;
  buf.R = reinterpret_cast<float2*>(S + kBaseMax * kLd);
  buf.L = reinterpret_cast<float4*>(buf.R + 3 * 4 * 64);
  const BaseTask t = tasks[blockIdx.x];
  const int n = t.n;
  // PDL: the task table is static; the matrix comes from the previous kernel.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // Stage M's lower triangle (identity beyond n): warp w rows w + 8 q, lane
  // columns 32 c + l; all loads of a thread in flight before any store.
  {
    constexpr int kRows = kBaseMax / kLeafWarps;
    float v[4][kRows];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int q = 0; q < kRows; ++q) {
        const int i = warp + kLeafWarps * q, j = 32 * c + lane;
        v[c][q] = (i == j) ? 1.f : 0.f;
        if (i < n && j < n && j <= i) v[c][q] = __ldg(t.m + int64_t(i) * t.ld + j);
      }
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int q = 0; q < kRows; ++q) {
        const int i = warp + kLeafWarps * q, j = 32 * c + lane;
        if (j <= i) S[i * kLd + j] = v[c][q];
      }
  }
  __syncthreads();
  // Registers: the full symmetric matrix (upper read mirrored).
  float2 x[4][4][2];
#pragma unroll
  for (int g = 0; g < 4; ++g)
#pragma unroll
    for (int tt = 0; tt < 4; ++tt)
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int i = 4 * warp + tt + 32 * g, j = 2 * lane + 64 * p;
        x[g][tt][p].x = j <= i ? S[i * kLd + j] : S[j * kLd + i];
        x[g][tt][p].y = j + 1 <= i ? S[i * kLd + j + 1] : S[(j + 1) * kLd + i];
      }
  LEAF_STAMP(1);
  bool bad = false;
  const int nb = (n + 3) / 4;  // padded rows/columns are identity: inert
  if (warp == 0) leaf_publish<0>(x, 0, lane, buf.R, buf.L, bad);
  __syncthreads();
  leaf_blocks<0>(x, nb, warp, lane, buf, bad);
  LEAF_STAMP(2);
  if (bad || t.inject) {
    set_status(status, SPNGD_ERR_NOT_POSITIVE_DEFINITE);
    if (t.info && threadIdx.x % 32 == 0) *t.info = SPNGD_ERR_NOT_POSITIVE_DEFINITE;
  }
  // T = lower triangle of X -> staging (zeros above the diagonal).
#pragma unroll
  for (int g = 0; g < 4; ++g)
#pragma unroll
    for (int tt = 0; tt < 4; ++tt)
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int i = 4 * warp + tt + 32 * g, j = 2 * lane + 64 * p;
        S[i * kLd + j] = j <= i ? x[g][tt][p].x : 0.f;
        S[i * kLd + j + 1] = j + 1 <= i ? x[g][tt][p].y : 0.f;
      }
  __syncthreads();
  float* T = S;
  // Stores: tlow row i = T row i (zeros above the diagonal are T's own), tup
  // row i = T column i (read transposed from smem); float4 per lane where the
  // chunk lies inside the block.
  {
    const int j0 = 4 * lane;
    const bool vst = (t.ld & 3) == 0 && (reinterpret_cast<uintptr_t>(t.tlow) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(t.tup) & 15) == 0;
    for (int i = warp; i < n; i += kBaseThreads / 32) {
      if (j0 >= n) continue;
      float lo[4], up[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int j = j0 + c;
        lo[c] = (j <= i && j < n) ? T[i * kLd + j] : 0.f;
        up[c] = (j >= i && j < n) ? T[j * kLd + i] : 0.f;
      }
      float* dl = t.tlow + int64_t(i) * t.ld + j0;
      float* du = t.tup + int64_t(i) * t.ld + j0;
      if (vst && j0 + 3 < n) {
        *reinterpret_cast<float4*>(dl) = make_float4(lo[0], lo[1], lo[2], lo[3]);
        *reinterpret_cast<float4*>(du) = make_float4(up[0], up[1], up[2], up[3]);
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int j = j0 + c;
          if (j < n && j <= i) dl[c] = lo[c];
          if (j < n && j >= i) du[c] = up[c];
        }
      }
    }
  }
  LEAF_STAMP(3);
}

__global__ void pi_kernel(const PiTask* __restrict__ tasks) {
  const PiTask t = tasks[blockIdx.x];
  double sa = 0.0, sg = 0.0;
  for (int64_t i = threadIdx.x; i < t.a; i += blockDim.x) sa += double(t.A[packed_offset(t.a, i, i)]);
  for (int64_t i = threadIdx.x; i < t.g; i += blockDim.x) sg += double(t.G[packed_offset(t.g, i, i)]);
  __shared__ double ra[32], rg[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    sg += __shfl_xor_sync(0xffffffffu, sg, o);
  }
  if ((threadIdx.x & 31) == 0) { ra[threadIdx.x >> 5] = sa; rg[threadIdx.x >> 5] = sg; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ta = 0, tg = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) { ta += ra[w]; tg += rg[w]; }
    const double ea = ta / double(t.a), eg = tg / double(t.g);      // avg_eigenvalue, linalg.cpp:64-69
    const double pi = (ea < 1e-12 || eg < 1e-12) ? 1.0 : sqrt(ea / eg);  // fisher.cpp:223
    t.dampA[0] = float(pi * t.sqrt_lambda);
    t.dampG[0] = float(t.sqrt_lambda / pi);
    if (t.pi_out) t.pi_out[0] = float(pi);
  }
}

// dense = unpack(packed) + d I, by 32x32 tiles of the upper triangle so both
// the packed reads and the mirrored (transposed) dense writes are coalesced.
// Blocks walk the upper tiles only (triangular index), two tiles per pass so
// eight loads per thread are in flight (one tile per pass over all tn^2
// tiles, half of them skipped, was latency-bound at 2.4 TB/s).  32-bit index
// math whenever the dense square fits (every ResNet-50 factor).
template <typename I>
__device__ __forceinline__ void upper_tile(I u, I tn, I& ti, I& tj) {
  // row-major over the upper triangle: row r starts at r*tn - r(r-1)/2
  const double b = 2.0 * double(tn) + 1.0;
  I r = I((b - sqrt(b * b - 8.0 * double(u))) * 0.5);
  if (r < 0) r = 0;
  while (r > 0 && r * tn - r * (r - 1) / 2 > u) --r;
  while ((r + 1) * tn - (r + 1) * r / 2 <= u) ++r;
  ti = r;
  tj = r + (u - (r * tn - r * (r - 1) / 2));
}

template <typename I>
__device__ __forceinline__ bool unpack_damp_tiles(const UnpackTask& t, float (*s)[32][33]) {
  const float d = t.damp_dev ? t.damp_dev[0] : t.damp;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const I n = I(t.n), ld = I(t.ld);
  const I tn = (n + 31) / 32, nt = tn * (tn + 1) / 2;
  bool bad = false;
  for (I u0 = I(blockIdx.x) * 2; u0 < nt; u0 += I(gridDim.x) * 2) {
    I ti[2], tj[2];
    float v[2][4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const I u = u0 + h < nt ? u0 + h : u0;
      upper_tile<I>(u, tn, ti[h], tj[h]);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const I i = ti[h] * 32 + ty + 8 * q, j = tj[h] * 32 + tx;
        float x = 0.f;
        if (i < n && j < n && j >= i) {
          x = t.packed[i * n - i * (i - 1) / 2 + (j - i)];
          bad |= !isfinite(x);
          if (i == j) x += d;
        }
        v[h][q] = x;
      }
    }
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int q = 0; q < 4; ++q) s[h][ty + 8 * q][tx] = v[h][q];
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (u0 + h >= nt) break;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int li = ty + 8 * q;
        const I i = ti[h] * 32 + li, j = tj[h] * 32 + tx;
        if (i < n && j < n) t.dense[i * ld + j] = (j >= i) ? s[h][li][tx] : s[h][tx][li];
        if (ti[h] != tj[h]) {
          const I r = tj[h] * 32 + li, c = ti[h] * 32 + tx;  // transposed tile
          if (r < n && c < n) t.dense[r * ld + c] = s[h][tx][li];
        }
      }
    }
  }
  return bad;
}

__global__ void unpack_damp_kernel(const UnpackTask* __restrict__ tasks, int* status) {
  const UnpackTask t = tasks[blockIdx.y];
  __shared__ float s[2][32][33];
  const int64_t span = (t.ld > t.n ? t.ld : t.n) * (t.n + 32);
  const bool bad = span < (int64_t(1) << 31) ? unpack_damp_tiles<int32_t>(t, s) : unpack_damp_tiles<int64_t>(t, s);
  if (bad) {
    set_status(status, SPNGD_ERR_NOT_POSITIVE_DEFINITE);
    if (t.info) *t.info = SPNGD_ERR_NOT_POSITIVE_DEFINITE;
  }
}

__global__ void pack_kernel(const PackTask* __restrict__ tasks, int* status) {
  const PackTask t = tasks[blockIdx.y];
  bool bad = false;
  for (int64_t i = blockIdx.x; i < t.n; i += gridDim.x) {
    const int64_t base = i * t.n - i * (i - 1) / 2;
    for (int64_t j = i + threadIdx.x; j < t.n; j += blockDim.x) {
      const float v = t.dense[i * t.ld + j];
      bad |= !isfinite(v);
      if (t.packed) t.packed[base + (j - i)] = v;
    }
  }
  if (bad) {  // spd_inverse's "inverse has non-finite entries" (linalg.cpp:41-43)
    set_status(status, SPNGD_ERR_NOT_POSITIVE_DEFINITE);
    if (t.info) *t.info = SPNGD_ERR_NOT_POSITIVE_DEFINITE;
  }
}

// ---------------------------------------------------------------- planning
struct Op {
  int kind;  // 0 base, 1 gemm
  BaseTask base;
  GemmProblem prob;
  bool upper;
  GemmProblem prob2;  // optional independent GEMM in the same round
  bool upper2;
  bool has2;
};

int64_t split_point(int64_t n) {
  // Keep the leading block a multiple of the 128-row MMA tile when possible.
  int64_t n1 = round_up((n + 1) / 2, n > 2 * kBaseMax ? 128 : 32);
  if (n1 >= n) n1 = n - 1;
  return n1;
}

GemmOperand dense_op(const float* ptr, int64_t ld, int64_t rows, int64_t K) {
  GemmOperand o{};
  o.ptr = ptr;
  o.row_stride = ld;
  o.seg_len = std::max<int64_t>(K, 1);
  o.seg_stride = 0;
  o.rows = int32_t(rows);
  finalize_operand(o, K);
  return o;
}

struct Gen {
  float* ws;
  size_t used = 0;
  float* take(size_t n) {
    float* p = ws ? ws + used : nullptr;
    used += round_up(int64_t(n), 64);
    return p;
  }
};

template <typename T>
T* at(T* base, int64_t ld, int64_t r, int64_t c) {
  return base ? base + r * ld + c : nullptr;
}

Op gemm_op(const GemmOperand& a, const GemmOperand& b, int64_t M, int64_t N, int64_t K, int32_t flags, int32_t ktri,
           float alpha, float beta, float* C, int64_t ldc, float* CT = nullptr, int64_t ldct = 0, bool upper = false) {
  Op o{};
  o.kind = 1;
  o.upper = upper;
  GemmProblem& p = o.prob;
  p.A = a;
  p.B = b;
  p.M = int32_t(M); p.N = int32_t(N); p.K = int32_t(K);
  p.mode = EPI_DENSE; p.flags = flags; p.ktri = ktri;
  p.alpha = alpha; p.beta = beta;
  p.C = C; p.Cin = C; p.ldc = ldc; p.CT = CT; p.ldct = ldct;
  return o;
}

// Cholesky + running inverse of the diagonal block at `off` of size n.
void gen_chol(const DenseMatrix& m, int64_t off, int64_t n, Gen& g, std::vector<Op>& ops) {
  const int64_t ld = m.ld;
  if (n <= kBaseMax) {
    Op o{};
    o.kind = 0;
    o.base = BaseTask{at(m.ptr, ld, off, off), at(m.tlow, ld, off, off), at(m.tup, ld, off, off), ld, int32_t(n), 0,
                      m.info};
    ops.push_back(o);
    return;
  }
  const int64_t n1 = split_point(n), n2 = n - n1, o2 = off + n1;
  gen_chol(m, off, n1, g, ops);
  const int64_t ldl = round_up(n1, 32), ldu = round_up(n2, 32);
  float* L21 = g.take(size_t(n2) * ldl);
  float* Ut = g.take(size_t(n1) * ldu);
  // L21 = B T11^T  (B = M[o2.., off..]); T11 lower -> K band k <= j
  ops.push_back(gemm_op(dense_op(at(m.ptr, ld, o2, off), ld, n2, n1), dense_op(at(m.tlow, ld, off, off), ld, n1, n1),
                        n2, n1, n1, 0, KTRI_B_LOWER, 1.f, 0.f, L21, ldl));
  // S = C - L21 L21^T (symmetric, in place) and, independent of it in the
  // same round, U^T = T11^T L21^T (T11^T upper -> K band k >= j).
  Op s = gemm_op(dense_op(L21, ldl, n2, n1), dense_op(L21, ldl, n2, n1), n2, n2, n1, FLAG_SAME_AB | FLAG_SYM_MIRROR, 0,
                 -1.f, 1.f, at(m.ptr, ld, o2, o2), ld, nullptr, 0, true);
  const Op u = gemm_op(dense_op(at(m.tup, ld, off, off), ld, n1, n1), dense_op(L21, ldl, n2, n1), n1, n2, n1, 0,
                       KTRI_A_UPPER, 1.f, 0.f, Ut, ldu);
  s.prob2 = u.prob;
  s.upper2 = false;
  s.has2 = true;
  ops.push_back(s);
  gen_chol(m, o2, n2, g, ops);
  // T21 = -T22 U (+ T21^T into the upper factor); T22 lower -> K band k <= i
  ops.push_back(gemm_op(dense_op(at(m.tlow, ld, o2, o2), ld, n2, n2), dense_op(Ut, ldu, n1, n2), n2, n1, n2,
                        FLAG_TRANS, KTRI_A_LOWER, -1.f, 0.f, at(m.tlow, ld, o2, off), ld, at(m.tup, ld, off, o2), ld));
}

Op lauum_op(const DenseMatrix& m) {
  // X = T^T T = Tup Tup^T; row i of Tup is zero for k < i.
  return gemm_op(dense_op(m.tup, m.ld, m.n, m.n), dense_op(m.tup, m.ld, m.n, m.n), m.n, m.n, m.n,
                 FLAG_SAME_AB | FLAG_SYM_MIRROR, KTRI_A_UPPER | KTRI_B_UPPER, 1.f, 0.f, m.ptr, m.ld, nullptr, 0, true);
}

void gen_ops(const DenseMatrix& m, Gen& g, std::vector<Op>& ops, bool form_inverse) {
  gen_chol(m, 0, m.n, g, ops);
  if (form_inverse) ops.push_back(lauum_op(m));
}

}  // namespace

void plan_inverse(const std::vector<DenseMatrix>& mats, float* workspace, InversePlan& plan, bool form_inverse) {
  plan = InversePlan();
  Gen g{workspace};
  std::vector<std::vector<Op>> per(mats.size());
  size_t max_ops = 0;
  for (size_t m = 0; m < mats.size(); ++m) {
    gen_ops(mats[m], g, per[m], form_inverse);
    max_ops = std::max(max_ops, per[m].size());
  }
  // Failure-path test hook: the last leaf of every n == SPNGD_TEST_FAIL_N
  // matrix reports a non-positive pivot (the failure found at the very end of
  // its recursion, after earlier classes' parameters could have been written).
  const long long fail_n = getenv("SPNGD_TEST_FAIL_N") ? atoll(getenv("SPNGD_TEST_FAIL_N")) : -1;
  for (size_t m = 0; m < mats.size(); ++m)
    if (mats[m].n == fail_n)
      for (size_t r = per[m].size(); r-- > 0;)
        if (per[m][r].kind == 0) {
          per[m][r].base.inject = 1;
          break;
        }
  plan.workspace_floats = g.used;
  // Round r runs op r of every matrix: one base launch + the grouped GEMMs,
  // the 2-CTA 256 x 256 kernel's items first (pair_cnt), then the 128 x 256 ones.
  for (size_t r = 0; r < max_ops; ++r) {
    InverseRound rd{int(plan.items.size()), 0, int(plan.bases.size()), 0, 0};
    // eligible problems planned both ways, the rest single; the round goes to
    // the pair kernel only when that is faster at wave granularity
    std::vector<GemmWorkItem> pair, single_elig, single;
    for (size_t m = 0; m < mats.size(); ++m) {
      if (r >= per[m].size()) continue;
      const Op& o = per[m][r];
      if (o.kind == 0) {
        plan.bases.push_back(o.base);
        continue;
      }
      for (int h = 0; h < (o.has2 ? 2 : 1); ++h) {
        const GemmProblem& p = h ? o.prob2 : o.prob;
        const bool upper = h ? o.upper2 : o.upper;
        const int pi = int(plan.probs.size());
        plan.probs.push_back(p);
        int slot = 0;
        if (!no_pair_inv() && pair_eligible_dense(p, upper)) {
          plan_pair_dense(pi, p, pair, upper);
          plan_problem_tiles(pi, p, upper, p.K + kTileK, single_elig, nullptr, &slot, 1.0, nullptr);
        } else {
          plan_problem_tiles(pi, p, upper, p.K + kTileK, single, nullptr, &slot, 1.0, nullptr);
        }
      }
    }
    plan.item_bound += std::max(pair.size(), single_elig.size()) + single.size();
    if (pair_group_wins(int64_t(pair.size()), int64_t(single_elig.size()), int64_t(single.size())))
      plan.items.insert(plan.items.end(), pair.begin(), pair.end());
    else
      single.insert(single.begin(), single_elig.begin(), single_elig.end());
    rd.pair_cnt = int(plan.items.size()) - rd.item_off;
    plan.items.insert(plan.items.end(), single.begin(), single.end());
    rd.item_cnt = int(plan.items.size()) - rd.item_off;
    rd.base_cnt = int(plan.bases.size()) - rd.base_off;
    plan.rounds.push_back(rd);
  }
}

int launch_pi(spngd_ctx* ctx, const PiTask* d_tasks, int n) {
  if (n <= 0) return SPNGD_OK;
  pi_kernel<<<n, 256, 0, ctx->stream>>>(d_tasks);
  SPNGD_CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return SPNGD_OK;
}

int launch_unpack(spngd_ctx* ctx, const UnpackTask* d_tasks, int n, int64_t max_n) {
  if (n <= 0) return SPNGD_OK;
  const int64_t tn = (max_n + 31) / 32;
  dim3 grid(unsigned(std::min<int64_t>((tn * (tn + 1) / 2 + 1) / 2, 1024)), unsigned(n));
  unpack_damp_kernel<<<grid, 256, 0, ctx->stream>>>(d_tasks, ctx->d_status);
  SPNGD_CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return SPNGD_OK;
}

int launch_pack(spngd_ctx* ctx, const PackTask* d_tasks, int n, int64_t max_n) {
  if (n <= 0) return SPNGD_OK;
  dim3 grid(unsigned(std::min<int64_t>(max_n, 512)), unsigned(n));
  pack_kernel<<<grid, 256, 0, ctx->stream>>>(d_tasks, ctx->d_status);
  SPNGD_CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return SPNGD_OK;
}

int launch_base(spngd_ctx* ctx, const BaseTask* d_tasks, int n) {
  if (n <= 0) return SPNGD_OK;
  static bool attr = false;
  if (!attr) {
    SPNGD_CUDA_TRY(cudaFuncSetAttribute(base_chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(kBaseSmem)));
    attr = true;
  }
  {
    static const bool pdl = getenv("SPNGD_NO_PDL") == nullptr;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(n));
    cfg.blockDim = dim3(kBaseThreads);
    cfg.dynamicSmemBytes = kBaseSmem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    attr[1].id = cudaLaunchAttributePriority;
    attr[1].val.priority = ctx->launch_prio;
    cfg.attrs = attr;
    cfg.numAttrs = ctx->launch_prio ? 2 : 1;
    SPNGD_CUDA_TRY(cudaLaunchKernelEx(&cfg, base_chol_inv_kernel, d_tasks, ctx->d_status));
  }
  SPNGD_CUDA_TRY(cudaGetLastError());
#ifdef SPNGD_GEMM_TRACE_BUILD
  static int printed = 0;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(ctx->stream, &cap);
  if (getenv("SPNGD_GEMM_TRACE") && cap == cudaStreamCaptureStatusNone && printed++ < 6) {
    long long h[8];
    cudaStreamSynchronize(ctx->stream);
    cudaMemcpyFromSymbol(h, g_leaf_trace, sizeof(h));
    printf("leaf launch (%d leaves): load %lld eliminate %lld store %lld cycles\n", n, h[1] - h[0], h[2] - h[1],
           h[3] - h[2]);
  }
#endif
  ctx->launches++;
  return SPNGD_OK;
}

int materialize_inverse(spngd_ctx* ctx, const DenseMatrix& m) {
  const Op op = lauum_op(m);
  std::vector<GemmWorkItem> items;
  int slot = 0;
  plan_problem_tiles(0, op.prob, op.upper, op.prob.K + kTileK, items, nullptr, &slot, 1.0, nullptr);
  DeviceScratch scratch(ctx);
  std::vector<GemmProblem> probs{op.prob};
  auto* d_probs = scratch.upload(probs);
  auto* d_items = scratch.upload(items);
  if (!d_probs || !d_items) return fail(SPNGD_ERR_CUDA, "materialize_inverse: scratch upload failed");
  int rc = launch_gemm(d_probs, d_items, int(items.size()), nullptr, ctx->d_status, ctx->stream,
                       gemm_variant(probs.data(), 1));
  if (rc) return rc;
  ctx->launches++;
  return spngd_ctx_sync(ctx);
}

int run_inverse(spngd_ctx* ctx, const InversePlan& plan, const GemmProblem* d_probs, const GemmWorkItem* d_items,
                const BaseTask* d_bases) {
  const uint32_t variant = gemm_variant(plan.probs.data(), int(plan.probs.size()));
  g_gemm_launch_prio = ctx->launch_prio;
  int rc = SPNGD_OK;
  for (const InverseRound& r : plan.rounds) {
    rc = launch_base(ctx, d_bases + r.base_off, r.base_cnt);
    if (rc) break;
    if (r.pair_cnt > 0) {
      rc = launch_syrk_pair(d_probs, d_items + r.item_off, r.pair_cnt, nullptr, ctx->stream, ctx->d_status);
      if (rc) break;
      ctx->launches++;
    }
    if (r.item_cnt > r.pair_cnt) {
      rc = launch_gemm(d_probs, d_items + r.item_off + r.pair_cnt, r.item_cnt - r.pair_cnt, nullptr, ctx->d_status,
                       ctx->stream, variant);
      if (rc) break;
      ctx->launches++;
    }
  }
  g_gemm_launch_prio = 0;
  return rc;
}

}  // namespace spngd

using namespace spngd;

namespace {

// One matrix of a batched explicit-inverse call.
struct InvItem {
  const float* packed;
  int64_t n;
  float damp;             // host damping (unused when damp_dev)
  const float* damp_dev;  // device damping (damp_and_invert's pi-scaled values)
  float* dense;           // n x ld output (or scratch)
  int64_t ld;
  float* packed_out;      // may be null
  int req;                // request index (info[] slot)
  int side;               // 0: spd_inverse / A factor, 1: G factor
};

// unpack + damping, recursive Cholesky inverse, refinement of the
// ill-conditioned ones, finite check + pack; per-matrix status in info[req]
// (host array of n_req, may be null).  Synchronous.
int batched_inverse(spngd_ctx* ctx, DeviceScratch& scratch, std::vector<InvItem>& items, const PiTask* d_pis,
                    int n_pis, int n_req, int* info, const char* who) {
  const int nm = int(items.size());
  int* d_info = scratch.alloc<int>(nm);
  double* d_fro = scratch.alloc<double>(nm);
  float* d_damp = scratch.alloc<float>(nm);
  if (!d_info || !d_fro || !d_damp) return fail(SPNGD_ERR_CUDA, "%s: allocation failed", who);
  SPNGD_CUDA_TRY(cudaMemsetAsync(d_info, 0, sizeof(int) * nm, ctx->stream));
  SPNGD_CUDA_TRY(cudaMemsetAsync(d_fro, 0, sizeof(double) * nm, ctx->stream));
  std::vector<DenseMatrix> mats;
  std::vector<UnpackTask> unpack;
  std::vector<FroTask> fro;
  std::vector<PackTask> pack;
  int64_t max_n = 0;
  for (int q = 0; q < nm; ++q) {
    InvItem& it = items[q];
    float* tl = scratch.alloc<float>(size_t(it.n) * it.ld);
    float* tu = scratch.alloc<float>(size_t(it.n) * it.ld);
    if (!tl || !tu) return fail(SPNGD_ERR_CUDA, "%s: allocation failed", who);
    SPNGD_CUDA_TRY(cudaMemsetAsync(tl, 0, sizeof(float) * it.n * it.ld, ctx->stream));
    SPNGD_CUDA_TRY(cudaMemsetAsync(tu, 0, sizeof(float) * it.n * it.ld, ctx->stream));
    mats.push_back({it.dense, tl, tu, it.ld, it.n, d_info + q});
    unpack.push_back({it.packed, it.n, it.damp_dev, it.damp, 0, it.dense, it.ld, d_info + q});
    fro.push_back({it.packed, it.n, it.damp_dev, it.damp, 0, d_fro + q});
    pack.push_back({it.dense, it.ld, it.n, it.packed_out, d_info + q});
    max_n = std::max(max_n, it.n);
  }
  InversePlan sizing;
  plan_inverse(mats, nullptr, sizing);
  float* ws = scratch.alloc<float>(std::max<size_t>(sizing.workspace_floats, 1));
  InversePlan plan;
  plan_inverse(mats, ws, plan);
  auto* d_unpack = scratch.upload(unpack);
  auto* d_fro_t = scratch.upload(fro);
  auto* d_probs = scratch.upload(plan.probs);
  auto* d_items = scratch.upload(plan.items);
  auto* d_bases = scratch.upload(plan.bases);
  int rc = launch_pi(ctx, d_pis, n_pis);
  if (!rc) rc = launch_unpack(ctx, d_unpack, nm, max_n);
  if (!rc) rc = launch_fro(ctx, d_fro_t, nm, max_n);
  if (!rc) rc = run_inverse(ctx, plan, d_probs, d_items, d_bases);
  if (rc) return rc;
  // refine the matrices whose cond bound ||M + dI||_F / d passes the threshold
  const double thr = refine_threshold();
  if (std::isfinite(thr)) {
    std::vector<double> h_fro(nm);
    std::vector<int> h_info(nm);
    std::vector<float> h_damp(nm);
    for (int q = 0; q < nm; ++q)
      if (items[q].damp_dev)
        SPNGD_CUDA_TRY(cudaMemcpyAsync(d_damp + q, items[q].damp_dev, sizeof(float), cudaMemcpyDeviceToDevice,
                                       ctx->stream));
    SPNGD_CUDA_TRY(cudaMemcpyAsync(h_fro.data(), d_fro, sizeof(double) * nm, cudaMemcpyDeviceToHost, ctx->stream));
    SPNGD_CUDA_TRY(cudaMemcpyAsync(h_info.data(), d_info, sizeof(int) * nm, cudaMemcpyDeviceToHost, ctx->stream));
    SPNGD_CUDA_TRY(cudaMemcpyAsync(h_damp.data(), d_damp, sizeof(float) * nm, cudaMemcpyDeviceToHost, ctx->stream));
    SPNGD_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    std::vector<RefineJob> jobs;
    for (int q = 0; q < nm; ++q) {
      const float d = items[q].damp_dev ? h_damp[q] : items[q].damp;
      if (h_info[q] || !(d > 0.f)) continue;
      if (std::sqrt(h_fro[q]) / double(d) > thr) jobs.push_back({items[q].packed, items[q].n, d, items[q].dense, items[q].ld});
    }
    rc = refine_inverses(ctx, scratch, jobs);
    if (rc) return rc;
  }
  auto* d_pack = scratch.upload(pack);
  rc = launch_pack(ctx, d_pack, nm, max_n);
  if (rc) return rc;
  std::vector<int> h_info(nm);
  SPNGD_CUDA_TRY(cudaMemcpyAsync(h_info.data(), d_info, sizeof(int) * nm, cudaMemcpyDeviceToHost, ctx->stream));
  rc = spngd_ctx_sync(ctx);
  if (info)
    for (int r = 0; r < n_req; ++r) info[r] = 0;
  int first = -1;
  for (int q = 0; q < nm; ++q) {
    if (!h_info[q]) continue;
    if (info && !info[items[q].req]) info[items[q].req] = h_info[q];
    if (first < 0) first = q;
  }
  if (first >= 0) {  // name the failing factor the way layer_tag does (fisher.cpp:48-51)
    const InvItem& f = items[first];
    const char* side = f.side ? "G factor" : (std::strcmp(who, "damp_and_invert") == 0 ? "A factor" : "matrix");
    return fail(h_info[first], "%s: request %d (%s, n=%lld): Cholesky factorization failed -- non-positive pivot or "
                "non-finite entries", who, f.req, side, (long long)f.n);
  }
  return rc;
}

}  // namespace

extern "C" int spngd_spd_inverse_batched(spngd_ctx* ctx, int n, const spngd_spd_req* reqs, int* info) {
  SPNGD_CTX_SCOPE(ctx);
  if (!ctx || (n > 0 && !reqs)) return fail(SPNGD_ERR_INVALID, "spngd_spd_inverse_batched: null argument");
  if (n == 0) return SPNGD_OK;
  DeviceScratch scratch(ctx);
  std::vector<InvItem> items;
  for (int i = 0; i < n; ++i) {
    const spngd_spd_req& r = reqs[i];
    if (r.n <= 0) return fail(SPNGD_ERR_SHAPE_MISMATCH, "spd_inverse: request %d: empty matrix", i);
    if (!r.packed || (!r.dense_out && !r.packed_out)) return fail(SPNGD_ERR_INVALID, "spd_inverse: request %d: null pointer", i);
    if (r.dense_out && r.ld < r.n) return fail(SPNGD_ERR_SHAPE_MISMATCH, "spd_inverse: request %d: ld < n", i);
    float* dense = r.dense_out;
    int64_t ld = r.ld;
    if (!dense) {
      ld = round_up(r.n, 32);
      dense = scratch.alloc<float>(size_t(r.n) * ld);
      if (!dense) return fail(SPNGD_ERR_CUDA, "spd_inverse: allocation failed");
    }
    items.push_back({r.packed, r.n, r.damping, r.damping_dev, dense, ld, r.packed_out, i, 0});
  }
  return batched_inverse(ctx, scratch, items, nullptr, 0, n, info, "spd_inverse");
}

extern "C" int spngd_damp_and_invert_batched(spngd_ctx* ctx, int n, const spngd_kron_req* reqs, double lambda,
                                             int* info) {
  SPNGD_CTX_SCOPE(ctx);
  if (!ctx || (n > 0 && !reqs)) return fail(SPNGD_ERR_INVALID, "spngd_damp_and_invert_batched: null argument");
  if (!(lambda > 0.0)) return fail(SPNGD_ERR_NOT_POSITIVE_DEFINITE, "damp_and_invert: lambda must be > 0");
  if (n == 0) return SPNGD_OK;
  DeviceScratch scratch(ctx);
  float* damps = scratch.alloc<float>(2 * n);
  if (!damps) return fail(SPNGD_ERR_CUDA, "damp_and_invert: allocation failed");
  std::vector<PiTask> pis;
  std::vector<InvItem> items;
  for (int i = 0; i < n; ++i) {
    const spngd_kron_req& r = reqs[i];
    if (r.a <= 0 || r.g <= 0) return fail(SPNGD_ERR_SHAPE_MISMATCH, "avg_eigenvalue: request %d: empty matrix", i);
    if (!r.A_packed || !r.G_packed) return fail(SPNGD_ERR_INVALID, "damp_and_invert: request %d: null factor", i);
    pis.push_back({r.A_packed, r.G_packed, r.a, r.g, std::sqrt(lambda), damps + 2 * i, damps + 2 * i + 1, r.pi_out});
    const float* in[2] = {r.A_packed, r.G_packed};
    float* dn[2] = {r.Ainv_dense, r.Ginv_dense};
    int64_t lds[2] = {r.lda, r.ldg};
    float* pk[2] = {r.Ainv_packed, r.Ginv_packed};
    int64_t dims[2] = {r.a, r.g};
    for (int s = 0; s < 2; ++s) {
      float* dense = dn[s];
      int64_t ld = lds[s];
      if (dense && ld < dims[s]) return fail(SPNGD_ERR_SHAPE_MISMATCH, "damp_and_invert: request %d: ld < n", i);
      if (!dense) {
        ld = round_up(dims[s], 32);
        dense = scratch.alloc<float>(size_t(dims[s]) * ld);
        if (!dense) return fail(SPNGD_ERR_CUDA, "damp_and_invert: allocation failed");
      }
      items.push_back({in[s], dims[s], 0.f, damps + 2 * i + s, dense, ld, pk[s], i, s});
    }
  }
  auto* d_pis = scratch.upload(pis);
  if (!d_pis) return fail(SPNGD_ERR_CUDA, "damp_and_invert: upload failed");
  return batched_inverse(ctx, scratch, items, d_pis, int(pis.size()), n, info, "damp_and_invert");
}
