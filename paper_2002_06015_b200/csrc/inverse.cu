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
// factors in fp64 registers and forms T by forward elimination.  A
// non-positive or non-finite pivot raises NotPositiveDefinite (the LLT
// failure of linalg.cpp:37-40).  X is written upper-tile + mirrored, so the
// result is exactly symmetric as the reference's 0.5 (X + X^T) makes it.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "ctx.cuh"
#include "inverse.cuh"

namespace spngd {

namespace {

constexpr int kBaseMax = 128;
constexpr int kPB = 32;                 // panel width = one warp of rows
constexpr int kBaseThreads = 256;
constexpr int kLd = kBaseMax + 1;       // padded smem row (floats)
constexpr int kNb = kBaseMax / kPB;
constexpr size_t kBaseSmem = (2 * size_t(kBaseMax) * kLd + size_t(kNb) * kPB * kPB + kBaseMax) * sizeof(float);

// Compile-time-unrolled steps of the 32x32 diagonal factorization (rows in
// lanes) and of the column substitution, so `row`/`col` stay in registers.
// Step K with its pivot p = A_KK (already broadcast) and inv = 1/sqrt(p).
// The next pivot depends only on column K+1, so it is updated and the next
// broadcast + rsqrt issued before the remaining rank-1 columns of this step:
// the serial pivot chain overlaps the bulk of the shuffles.
__device__ __forceinline__ float pivot_rsqrt(float p, bool& bad) {
  if (!(p > 0.f) || !isfinite(p)) {
    bad = true;
    p = 1.f;
  }
  const float inv = rsqrtf(p);
  return inv * fmaf(-0.5f * p, inv * inv, 1.5f);  // MUFU rsqrt + one Newton step
}

template <int K>
__device__ __forceinline__ void diag_chol_step(float (&row)[32], int lane, float* rdiag, bool& bad, float p,
                                               float inv) {
  if (lane == K) rdiag[K] = inv;
  row[K] = (lane == K) ? p * inv : (lane > K ? row[K] * inv : row[K]);
  if constexpr (K + 1 < 32) {
    const float l1 = __shfl_sync(0xffffffffu, row[K], K + 1);
    row[K + 1] = (lane >= K + 1) ? fmaf(-row[K], l1, row[K + 1]) : row[K + 1];
    const float pn = __shfl_sync(0xffffffffu, row[K + 1], K + 1);  // next pivot
    const float invn = pivot_rsqrt(pn, bad);
#pragma unroll
    for (int j = K + 2; j < 32; ++j) {
      const float ljk = __shfl_sync(0xffffffffu, row[K], j);
      row[j] = (lane >= j) ? fmaf(-row[K], ljk, row[j]) : row[j];
    }
    diag_chol_step<K + 1>(row, lane, rdiag, bad, pn, invn);
  }
}

template <int I>
__device__ __forceinline__ void diag_subst_step(float (&col)[32], const float* Ld, int ld, const float* rdiag,
                                                int lane) {
  float a0 = (I == lane) ? 1.f : 0.f, a1 = 0.f;
#pragma unroll
  for (int p = 0; p < I; ++p) {
    if (p & 1) a1 = fmaf(-Ld[I * ld + p], col[p], a1);
    else a0 = fmaf(-Ld[I * ld + p], col[p], a0);
  }
  col[I] = (I < lane) ? 0.f : (a0 + a1) * rdiag[I];
  if constexpr (I + 1 < 32) diag_subst_step<I + 1>(col, Ld, ld, rdiag, lane);
}

// One CTA per leaf (n <= 128): blocked right-looking Cholesky with 32-column
// panels.  Warp 0 factors each 32x32 diagonal block with rows in lanes and
// columns broadcast by shuffle, then inverts it by forward substitution; all
// warps solve the panel and apply the SYRK trailing update on 4x4 register
// tiles; finally T = L^-1 by blocked forward substitution.  fp32 storage and
// FMA (LAPACK spotrf class).
#ifdef SPNGD_GEMM_TRACE_BUILD
__device__ long long g_leaf_trace[32];
#define LEAF_STAMP(i) \
  do {                \
    if (blockIdx.x == 0 && threadIdx.x == 0) g_leaf_trace[i] = clock64(); \
  } while (0)
#else
#define LEAF_STAMP(i) \
  do {                \
  } while (0)
#endif

__global__ void __launch_bounds__(kBaseThreads, 1) base_chol_inv_kernel(const BaseTask* __restrict__ tasks, int* status) {
  LEAF_STAMP(0);
  extern __shared__ __align__(16) uint8_t base_smem[];
  float* A = reinterpret_cast<float*>(base_smem);   // [128][129], lower = M -> L
  float* T = A + kBaseMax * kLd;                    // [128][129], T = L^-1
  float* R = T + kBaseMax * kLd;                    // [4][32][32] scratch
  float* rdiag = R + kNb * kPB * kPB;               // [128] 1 / L_ii
  const BaseTask t = tasks[blockIdx.x];
  const int n = t.n;
  // PDL: the task table is static; the matrix comes from the previous kernel.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int np = (n + kPB - 1) / kPB * kPB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // Load M's lower triangle: warp w owns rows w + 8 q, lane l columns
  // 32 cc + l (coalesced 128-byte rows, conflict-free smem stores); all 64
  // loads of a warp are in flight before any store.  Identity padding beyond
  // n is inert.
  {
    float v[kNb][kBaseMax / 8];
#pragma unroll
    for (int cc = 0; cc < kNb; ++cc)
#pragma unroll
      for (int q = 0; q < kBaseMax / 8; ++q) {
        const int i = warp + 8 * q, j = 32 * cc + lane;
        v[cc][q] = (i == j) ? 1.f : 0.f;
        if (i < n && j < n && j <= i) v[cc][q] = __ldg(t.m + int64_t(i) * t.ld + j);
      }
#pragma unroll
    for (int cc = 0; cc < kNb; ++cc)
#pragma unroll
      for (int q = 0; q < kBaseMax / 8; ++q) {
        const int i = warp + 8 * q, j = 32 * cc + lane;
        if (i < np && j < np) {
          A[i * kLd + j] = v[cc][q];
          T[i * kLd + j] = 0.f;
        }
      }
  }
  __syncthreads();
  LEAF_STAMP(1);
  bool bad = false;
  const int nblk = np / kPB;
  for (int kb = 0; kb < nblk; ++kb) {
    const int k0 = kb * kPB;
    if (warp == 0) {
      // (1) 32x32 diagonal block: lane i owns row i in registers; column k is
      //     broadcast by shuffle.
      float row[kPB];
#pragma unroll
      for (int j = 0; j < kPB; ++j) row[j] = (j <= lane) ? A[(k0 + lane) * kLd + k0 + j] : 0.f;
      if (kb == 0) LEAF_STAMP(20);
      {
        const float p0 = __shfl_sync(0xffffffffu, row[0], 0);
        diag_chol_step<0>(row, lane, rdiag + k0, bad, p0, pivot_rsqrt(p0, bad));
      }
      if (kb == 0) LEAF_STAMP(21);
#pragma unroll
      for (int j = 0; j < kPB; ++j)
        if (j <= lane) A[(k0 + lane) * kLd + k0 + j] = row[j];
      __syncwarp();
      if (kb == 0) LEAF_STAMP(22);
      // Column `lane` of L_dd^-1 (forward substitution), into T's diagonal block.
      float col[kPB];
      diag_subst_step<0>(col, A + k0 * kLd + k0, kLd, rdiag + k0, lane);
      if (kb == 0) LEAF_STAMP(23);
#pragma unroll
      for (int i = 0; i < kPB; ++i) T[(k0 + i) * kLd + k0 + lane] = col[i];
      if (kb == 0) LEAF_STAMP(24);
    }
    __syncthreads();
    LEAF_STAMP(2 + 3 * kb);
    const int m = np - k0 - kPB;  // trailing size
    if (m > 0) {
      // (2) panel: L[i][k0+j] = sum_{p<=j} A[i][k0+p] Dinv[j][p] (Dinv = T's
      //     diagonal block, lower) on 4x4 register tiles: thread (rg, cg) owns
      //     rows k0+32+4rg.. and columns 4cg..; 8 shared loads per 16 FMA.
      {
        const int ntiles = (m / 4) * 8;
        float acc[4][4] = {};
        const int rg = tid >> 3, cg = tid & 7;
        const int i0 = k0 + kPB + 4 * rg, j0 = 4 * cg;
        if (tid < ntiles) {
#pragma unroll 4
          for (int p = 0; p < kPB; ++p) {
            float a[4], d[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              a[q] = A[(i0 + q) * kLd + k0 + p];
              d[q] = (p <= j0 + q) ? T[(k0 + j0 + q) * kLd + k0 + p] : 0.f;
            }
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
              for (int y = 0; y < 4; ++y) acc[x][y] = fmaf(a[x], d[y], acc[x][y]);
          }
        }
        __syncthreads();  // every read of the panel precedes its in-place overwrite
        if (tid < ntiles)
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) A[(i0 + x) * kLd + k0 + j0 + y] = acc[x][y];
      }
      __syncthreads();
      LEAF_STAMP(3 + 3 * kb);
      // (3) trailing SYRK on 4x4 register tiles of the lower triangle.
      const int mt = m / 4;
      const int ntiles = mt * (mt + 1) / 2;
      for (int tt = tid; tt < ntiles; tt += kBaseThreads) {
        int ti = int((sqrtf(8.f * tt + 1.f) - 1.f) * 0.5f);
        while ((ti + 1) * (ti + 2) / 2 <= tt) ++ti;
        while (ti * (ti + 1) / 2 > tt) --ti;
        const int tj = tt - ti * (ti + 1) / 2;
        const int i0 = k0 + kPB + 4 * ti, j0 = k0 + kPB + 4 * tj;
        float acc[4][4] = {};
#pragma unroll 8
        for (int p = 0; p < kPB; ++p) {
          float a[4], b[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            a[q] = A[(i0 + q) * kLd + k0 + p];
            b[q] = A[(j0 + q) * kLd + k0 + p];
          }
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) acc[x][y] = fmaf(a[x], b[y], acc[x][y]);
        }
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y)
            if (j0 + y <= i0 + x) A[(i0 + x) * kLd + j0 + y] -= acc[x][y];
      }
      __syncthreads();
      LEAF_STAMP(4 + 3 * kb);
    }
  }
  // (4) T = L^-1 off-diagonal 32x32 blocks, block row by block row, on 4x4
  //     register tiles (thread = (jb, tr, tc), 64 tiles per block):
  //     R[jb] = sum_{p in [32 jb, 32 ib)} L[ib][p] T[p][jb],  T[ib][jb] = -T[ib][ib] R[jb].
  for (int ib = 1; ib < nblk; ++ib) {
    const int jb = tid >> 6, tr = (tid >> 3) & 7, tc = tid & 7;
    const bool act = jb < ib;
    const int r0 = ib * kPB + 4 * tr, c0 = jb * kPB + 4 * tc;
    float acc[4][4] = {};
    if (act) {
      for (int p = jb * kPB; p < ib * kPB; ++p) {
        float l[4], tv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          l[q] = A[(r0 + q) * kLd + p];
          tv[q] = T[p * kLd + c0 + q];
        }
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) acc[x][y] = fmaf(l[x], tv[y], acc[x][y]);
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) R[(jb * kPB + 4 * tr + x) * kPB + 4 * tc + y] = acc[x][y];
    }
    __syncthreads();
    if (act) {
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = 0.f;
      const int qmax = 4 * tr + 4;  // T[ib][ib] is lower: row 4tr+x uses q <= 4tr+x
      for (int q = 0; q < qmax; ++q) {
        float d[4], rv[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) d[x] = (q <= 4 * tr + x) ? T[(r0 + x) * kLd + ib * kPB + q] : 0.f;
#pragma unroll
        for (int y = 0; y < 4; ++y) rv[y] = R[(jb * kPB + q) * kPB + 4 * tc + y];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) acc[x][y] = fmaf(d[x], rv[y], acc[x][y]);
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) T[(r0 + x) * kLd + c0 + y] = -acc[x][y];
    }
    __syncthreads();
    LEAF_STAMP(14 + ib);
  }
  if (bad) set_status(status, SPNGD_ERR_NOT_POSITIVE_DEFINITE);
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
  __syncthreads();
  LEAF_STAMP(18);
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
__global__ void unpack_damp_kernel(const UnpackTask* __restrict__ tasks, int* status) {
  const UnpackTask t = tasks[blockIdx.y];
  const float d = t.damp_dev ? t.damp_dev[0] : t.damp;
  __shared__ float s[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int64_t tn = (t.n + 31) / 32;
  bool bad = false;
  for (int64_t tt = blockIdx.x; tt < tn * tn; tt += gridDim.x) {
    const int64_t ti = tt / tn, tj = tt % tn;
    if (ti > tj) continue;
    __syncthreads();
    for (int q = 0; q < 4; ++q) {
      const int64_t i = ti * 32 + ty + 8 * q, j = tj * 32 + tx;
      float v = 0.f;
      if (i < t.n && j < t.n && j >= i) {
        v = t.packed[i * t.n - i * (i - 1) / 2 + (j - i)];
        bad |= !isfinite(v);
        if (i == j) v += d;
      }
      s[ty + 8 * q][tx] = v;
    }
    __syncthreads();
    for (int q = 0; q < 4; ++q) {
      const int li = ty + 8 * q;
      const int64_t i = ti * 32 + li, j = tj * 32 + tx;
      if (i < t.n && j < t.n) t.dense[i * t.ld + j] = (j >= i) ? s[li][tx] : s[tx][li];
      if (ti != tj) {
        const int64_t r = tj * 32 + li, c = ti * 32 + tx;  // transposed tile
        if (r < t.n && c < t.n) t.dense[r * t.ld + c] = s[tx][li];
      }
    }
  }
  if (bad) set_status(status, SPNGD_ERR_NOT_POSITIVE_DEFINITE);
}

__global__ void pack_kernel(const PackTask* __restrict__ tasks, int* status) {
  const PackTask t = tasks[blockIdx.y];
  bool bad = false;
  for (int64_t i = blockIdx.x; i < t.n; i += gridDim.x) {
    const int64_t base = i * t.n - i * (i - 1) / 2;
    for (int64_t j = i + threadIdx.x; j < t.n; j += blockDim.x) {
      const float v = t.dense[i * t.ld + j];
      bad |= !isfinite(v);
      t.packed[base + (j - i)] = v;
    }
  }
  if (bad) set_status(status, SPNGD_ERR_NOT_POSITIVE_DEFINITE);
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
    o.base = BaseTask{at(m.ptr, ld, off, off), at(m.tlow, ld, off, off), at(m.tup, ld, off, off), ld, int32_t(n), 0};
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

void gen_ops(const DenseMatrix& m, Gen& g, std::vector<Op>& ops) {
  gen_chol(m, 0, m.n, g, ops);
  // X = T^T T = Tup Tup^T; row i of Tup is zero for k < i.
  ops.push_back(gemm_op(dense_op(m.tup, m.ld, m.n, m.n), dense_op(m.tup, m.ld, m.n, m.n), m.n, m.n, m.n,
                        FLAG_SAME_AB | FLAG_SYM_MIRROR, KTRI_A_UPPER | KTRI_B_UPPER, 1.f, 0.f, m.ptr, m.ld, nullptr, 0,
                        true));
}

}  // namespace

void plan_inverse(const std::vector<DenseMatrix>& mats, float* workspace, InversePlan& plan) {
  plan = InversePlan();
  Gen g{workspace};
  std::vector<std::vector<Op>> per(mats.size());
  size_t max_ops = 0;
  for (size_t m = 0; m < mats.size(); ++m) {
    gen_ops(mats[m], g, per[m]);
    max_ops = std::max(max_ops, per[m].size());
  }
  plan.workspace_floats = g.used;
  // Round r runs op r of every matrix: one base launch + one grouped GEMM.
  for (size_t r = 0; r < max_ops; ++r) {
    InverseRound rd{int(plan.items.size()), 0, int(plan.bases.size()), 0};
    for (size_t m = 0; m < mats.size(); ++m) {
      if (r >= per[m].size()) continue;
      const Op& o = per[m][r];
      if (o.kind == 0) {
        plan.bases.push_back(o.base);
      } else {
        const int pi = int(plan.probs.size());
        plan.probs.push_back(o.prob);
        int slot = 0;
        plan_problem_tiles(pi, o.prob, o.upper, o.prob.K + kTileK, plan.items, nullptr, &slot, 1.0, nullptr);
        if (o.has2) {
          const int pj = int(plan.probs.size());
          plan.probs.push_back(o.prob2);
          plan_problem_tiles(pj, o.prob2, o.upper2, o.prob2.K + kTileK, plan.items, nullptr, &slot, 1.0, nullptr);
        }
      }
    }
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
  dim3 grid(unsigned(std::min<int64_t>(tn * tn, 1024)), unsigned(n));
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
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SPNGD_CUDA_TRY(cudaLaunchKernelEx(&cfg, base_chol_inv_kernel, d_tasks, ctx->d_status));
  }
  SPNGD_CUDA_TRY(cudaGetLastError());
#ifdef SPNGD_GEMM_TRACE_BUILD
  static int printed = 0;
  if (getenv("SPNGD_GEMM_TRACE") && printed++ < 6) {
    long long h[32];
    cudaStreamSynchronize(ctx->stream);
    cudaMemcpyFromSymbol(h, g_leaf_trace, sizeof(h));
    printf("leaf launch (%d leaves): load %lld", n, h[1] - h[0]);
    for (int kb = 0; kb < 4; ++kb) printf(" | kb%d diag %lld panel %lld syrk %lld", kb, h[2 + 3 * kb] - h[0], h[3 + 3 * kb] - h[0], h[4 + 3 * kb] - h[0]);
    printf(" | T rows %lld %lld %lld | store %lld\n", h[15] - h[0], h[16] - h[0], h[17] - h[0], h[18] - h[0]);
    printf("   kb0 diag: rows-in %lld chol %lld store %lld subst %lld T-store %lld\n", h[20] - h[1], h[21] - h[20],
           h[22] - h[21], h[23] - h[22], h[24] - h[23]);
  }
#endif
  ctx->launches++;
  return SPNGD_OK;
}

int run_inverse(spngd_ctx* ctx, const InversePlan& plan, const GemmProblem* d_probs, const GemmWorkItem* d_items,
                const BaseTask* d_bases) {
  const uint32_t variant = gemm_variant(plan.probs.data(), int(plan.probs.size()));
  for (const InverseRound& r : plan.rounds) {
    int rc = launch_base(ctx, d_bases + r.base_off, r.base_cnt);
    if (rc) return rc;
    if (r.item_cnt > 0) {
      rc = launch_gemm(d_probs, d_items + r.item_off, r.item_cnt, nullptr, ctx->d_status, ctx->stream, variant);
      if (rc) return rc;
      ctx->launches++;
    }
  }
  return SPNGD_OK;
}

}  // namespace spngd

using namespace spngd;

extern "C" int spngd_spd_inverse_batched(spngd_ctx* ctx, int n, const spngd_spd_req* reqs) {
  if (!ctx || (n > 0 && !reqs)) return fail(SPNGD_ERR_INVALID, "spngd_spd_inverse_batched: null argument");
  if (n == 0) return SPNGD_OK;
  DeviceScratch scratch(ctx);
  std::vector<DenseMatrix> mats;
  std::vector<UnpackTask> unpack;
  std::vector<PackTask> pack;
  int64_t max_n = 0;
  for (int i = 0; i < n; ++i) {
    const spngd_spd_req& r = reqs[i];
    if (r.n <= 0) return fail(SPNGD_ERR_SHAPE_MISMATCH, "spd_inverse: empty matrix");
    if (!r.packed || (!r.dense_out && !r.packed_out)) return fail(SPNGD_ERR_INVALID, "spd_inverse: null pointer");
    if (r.dense_out && r.ld < r.n) return fail(SPNGD_ERR_SHAPE_MISMATCH, "spd_inverse: ld < n");
    float* dense = r.dense_out;
    int64_t ld = r.ld;
    if (!dense) {
      ld = round_up(r.n, 32);
      dense = scratch.alloc<float>(size_t(r.n) * ld);
      if (!dense) return fail(SPNGD_ERR_CUDA, "spd_inverse: allocation failed");
    }
    float* tl = scratch.alloc<float>(size_t(r.n) * ld);
    float* tu = scratch.alloc<float>(size_t(r.n) * ld);
    if (!tl || !tu) return fail(SPNGD_ERR_CUDA, "spd_inverse: allocation failed");
    cudaMemsetAsync(tl, 0, sizeof(float) * r.n * ld, ctx->stream);
    cudaMemsetAsync(tu, 0, sizeof(float) * r.n * ld, ctx->stream);
    mats.push_back({dense, tl, tu, ld, r.n});
    unpack.push_back({r.packed, r.n, r.damping_dev, r.damping, 0, dense, ld});
    if (r.packed_out) pack.push_back({dense, ld, r.n, r.packed_out});
    max_n = std::max(max_n, r.n);
  }
  InversePlan sizing;
  plan_inverse(mats, nullptr, sizing);
  float* ws = scratch.alloc<float>(std::max<size_t>(sizing.workspace_floats, 1));
  InversePlan plan;
  plan_inverse(mats, ws, plan);
  auto* d_unpack = scratch.upload(unpack);
  auto* d_pack = scratch.upload(pack);
  auto* d_probs = scratch.upload(plan.probs);
  auto* d_items = scratch.upload(plan.items);
  auto* d_bases = scratch.upload(plan.bases);
  int rc = launch_unpack(ctx, d_unpack, int(unpack.size()), max_n);
  if (!rc) rc = run_inverse(ctx, plan, d_probs, d_items, d_bases);
  if (!rc) rc = launch_pack(ctx, d_pack, int(pack.size()), max_n);
  if (rc) return rc;
  return spngd_ctx_sync(ctx);
}

extern "C" int spngd_damp_and_invert_batched(spngd_ctx* ctx, int n, const spngd_kron_req* reqs, double lambda) {
  if (!ctx || (n > 0 && !reqs)) return fail(SPNGD_ERR_INVALID, "spngd_damp_and_invert_batched: null argument");
  if (!(lambda > 0.0)) return fail(SPNGD_ERR_NOT_POSITIVE_DEFINITE, "damp_and_invert: lambda must be > 0");
  if (n == 0) return SPNGD_OK;
  DeviceScratch scratch(ctx);
  float* damps = scratch.alloc<float>(2 * n);
  std::vector<PiTask> pis;
  std::vector<DenseMatrix> mats;
  std::vector<UnpackTask> unpack;
  std::vector<PackTask> pack;
  int64_t max_n = 0;
  for (int i = 0; i < n; ++i) {
    const spngd_kron_req& r = reqs[i];
    if (r.a <= 0 || r.g <= 0) return fail(SPNGD_ERR_SHAPE_MISMATCH, "avg_eigenvalue: empty matrix");
    if (!r.A_packed || !r.G_packed) return fail(SPNGD_ERR_INVALID, "damp_and_invert: null factor");
    pis.push_back({r.A_packed, r.G_packed, r.a, r.g, std::sqrt(lambda), damps + 2 * i, damps + 2 * i + 1, r.pi_out});
    const float* in[2] = {r.A_packed, r.G_packed};
    float* dn[2] = {r.Ainv_dense, r.Ginv_dense};
    int64_t lds[2] = {r.lda, r.ldg};
    float* pk[2] = {r.Ainv_packed, r.Ginv_packed};
    int64_t dims[2] = {r.a, r.g};
    for (int s = 0; s < 2; ++s) {
      float* dense = dn[s];
      int64_t ld = lds[s];
      if (dense && ld < dims[s]) return fail(SPNGD_ERR_SHAPE_MISMATCH, "damp_and_invert: ld < n");
      if (!dense) {
        ld = round_up(dims[s], 32);
        dense = scratch.alloc<float>(size_t(dims[s]) * ld);
      }
      float* tl = scratch.alloc<float>(size_t(dims[s]) * ld);
      float* tu = scratch.alloc<float>(size_t(dims[s]) * ld);
      if (!dense || !tl || !tu) return fail(SPNGD_ERR_CUDA, "damp_and_invert: allocation failed");
      cudaMemsetAsync(tl, 0, sizeof(float) * dims[s] * ld, ctx->stream);
      cudaMemsetAsync(tu, 0, sizeof(float) * dims[s] * ld, ctx->stream);
      mats.push_back({dense, tl, tu, ld, dims[s]});
      unpack.push_back({in[s], dims[s], damps + 2 * i + s, 0.f, 0, dense, ld});
      if (pk[s]) pack.push_back({dense, ld, dims[s], pk[s]});
      max_n = std::max(max_n, dims[s]);
    }
  }
  InversePlan sizing;
  plan_inverse(mats, nullptr, sizing);
  float* ws = scratch.alloc<float>(std::max<size_t>(sizing.workspace_floats, 1));
  InversePlan plan;
  plan_inverse(mats, ws, plan);
  auto* d_pis = scratch.upload(pis);
  auto* d_unpack = scratch.upload(unpack);
  auto* d_pack = scratch.upload(pack);
  auto* d_probs = scratch.upload(plan.probs);
  auto* d_items = scratch.upload(plan.items);
  auto* d_bases = scratch.upload(plan.bases);
  int rc = launch_pi(ctx, d_pis, int(pis.size()));
  if (!rc) rc = launch_unpack(ctx, d_unpack, int(unpack.size()), max_n);
  if (!rc) rc = run_inverse(ctx, plan, d_probs, d_items, d_bases);
  if (!rc) rc = launch_pack(ctx, d_pack, int(pack.size()), max_n);
  if (rc) return rc;
  return spngd_ctx_sync(ctx);
}
