// K5/K6: precondition (src/fisher.cpp:255-257 -> kron_matvec, src/linalg.cpp:58-62)
// fused with ngd_step's FC/Conv update (src/fisher.cpp:332-333) and the
// rescale + velocity fix (src/schemes.cpp:116-119, src/dist.cpp:621-632).
// K7: unit-wise BatchNorm 2x2 solve + update (src/fisher.cpp:259-276, 336-357).
// K8: stale-statistics similarity norms (include/spngd/stale.hpp:23-64).
//
// P = G^-1 dW A^-1 runs as back-to-back grouped 3xTF32 GEMMs over all
// layers, with K-major operands thanks to the symmetry of the inverses:
//   GEMM1  P1^T[j,i] = sum_k A^-1[j,k] dW[i,k]      (M=a, N=g, K=a)
//   GEMM2  P^T [j,i] = sum_k P1^T[j,k] G^-1[i,k]    (M=a, N=g, K=g)
// or, inside the optimizer, from the triangular factors T = L^-1 without
// ever forming the inverses (four half-flop GEMMs, plan_precondition).
// The last GEMM's epilogue walks the P^T tile column-wise, i.e. along rows of the
// g x a weight, so W' = W - eta P + m V and V' = W' - W are coalesced and
// ||W'||_F^2 is reduced on the fly for the rescale pass.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "ctx.cuh"
#include "precond.cuh"

namespace spngd {

namespace {

// Every parameter-mutating kernel of Stage 4/5 returns without writing when the
// context status word is set (an inverse, unpack or BN determinant failed
// earlier in the step): the reference throws in damp_and_invert /
// precondition_bn before ngd_step, so its parameters stay unchanged
// (dist.cpp:597-601).  The status stays set until spngd_ctx_sync reports it.
__global__ void rescale_kernel(const RescaleTask* __restrict__ tasks, const int* __restrict__ status) {
  if (*status) return;
  const RescaleTask t = tasks[blockIdx.y];
  const double nrm = sqrt(t.norm2[0]);
  const float s = float(t.target / (nrm + 1e-9));  // schemes.cpp:117-118
  const int64_t n4 = (t.n % 4 == 0 && (reinterpret_cast<uintptr_t>(t.W) % 16 == 0) &&
                      (reinterpret_cast<uintptr_t>(t.V) % 16 == 0))
                         ? t.n / 4
                         : 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n4; q += stride) {
    float4 w = reinterpret_cast<float4*>(t.W)[q];
    float4 v = reinterpret_cast<float4*>(t.V)[q];
    // V'' = W'' - W_old = W'' - (W' - V')   (dist.cpp:626-630)
    float4 nw = make_float4(s * w.x, s * w.y, s * w.z, s * w.w);
    v = make_float4(nw.x - w.x + v.x, nw.y - w.y + v.y, nw.z - w.z + v.z, nw.w - w.w + v.w);
    reinterpret_cast<float4*>(t.W)[q] = nw;
    reinterpret_cast<float4*>(t.V)[q] = v;
    for (int p = 0; p < t.n_peers; ++p) reinterpret_cast<float4*>(t.peers[p])[q] = nw;  // Stage 5 over NVLink
  }
  for (int64_t i = 4 * n4 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < t.n; i += stride) {
    const float w = t.W[i], nw = s * w;
    t.V[i] = nw - w + t.V[i];
    t.W[i] = nw;
    for (int p = 0; p < t.n_peers; ++p) t.peers[p][i] = nw;
  }
  if (t.n_peers) __threadfence_system();
}

__global__ void peer_copy_kernel(const PeerCopyTask* __restrict__ tasks, const int* __restrict__ status) {
  if (*status) return;
  const PeerCopyTask t = tasks[blockIdx.y];
  const bool vec = t.n % 4 == 0 && (reinterpret_cast<uintptr_t>(t.src) & 15) == 0;
  const int64_t n4 = vec ? t.n / 4 : 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n4; q += stride) {
    const float4 v = reinterpret_cast<const float4*>(t.src)[q];
    for (int p = 0; p < t.n_peers; ++p) reinterpret_cast<float4*>(t.dst[p])[q] = v;
  }
  for (int64_t i = 4 * n4 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < t.n; i += stride)
    for (int p = 0; p < t.n_peers; ++p) t.dst[p][i] = t.src[i];
  __threadfence_system();
}

__global__ void snapshot_kernel(const SnapTask* __restrict__ tasks, bool restore, const int* __restrict__ status) {
  if (restore && *status == 0) return;
  const SnapTask t = tasks[blockIdx.y];
  const float* src = restore ? t.save : t.live;
  float* dst = restore ? t.live : t.save;
  const bool vec = t.n % 4 == 0 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  const int64_t n4 = vec ? t.n / 4 : 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n4; q += stride)
    reinterpret_cast<float4*>(dst)[q] = reinterpret_cast<const float4*>(src)[q];
  for (int64_t i = 4 * n4 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < t.n; i += stride) dst[i] = src[i];
}

__global__ void bn_update_kernel(const spngd_bn_update_req* __restrict__ reqs, double lambda, double eta,
                                 double momentum, const float* scal, int* status) {
  if (*status) return;  // includes a singular block found by bn_det_check_kernel
  if (scal) {
    eta = scal[0];
    momentum = scal[1];
  }
  const spngd_bn_update_req r = reqs[blockIdx.y];
  const int64_t ch = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (ch >= r.c) return;
  // inv2x2(fgg + lambda, fgb, fgb, fbb + lambda)  (linalg.cpp:50-56, fisher.cpp:268-270)
  const double a = double(r.m3c[3 * ch]) + lambda, b = double(r.m3c[3 * ch + 1]);
  const double d = double(r.m3c[3 * ch + 2]) + lambda;
  const double det = a * d - b * b;
  if (fabs(det) < 1e-30) {
    set_status(status, SPNGD_ERR_SINGULAR_BLOCK);
    return;
  }
  const double ia = d / det, ib = -b / det, id = a / det;
  const double gg = r.grad[ch], gb = r.grad[r.c + ch];
  const double pg = ia * gg + ib * gb, pb = ib * gg + id * gb;
  if (r.pg_out) r.pg_out[ch] = float(pg);
  if (r.pb_out) r.pb_out[ch] = float(pb);
  if (r.gamma) {
    // np = p - eta * delta + momentum * v ; nv = np - p   (fisher.cpp:353-356)
    const float g0 = r.gamma[ch], b0 = r.beta[ch];
    const float ng = float(double(g0) - eta * pg + momentum * double(r.vgamma[ch]));
    const float nb = float(double(b0) - eta * pb + momentum * double(r.vbeta[ch]));
    r.gamma[ch] = ng;
    r.beta[ch] = nb;
    r.vgamma[ch] = ng - g0;
    r.vbeta[ch] = nb - b0;
  }
}

// damp_bn's SingularBlock (fisher.cpp:230-246, linalg.cpp:50-56) for every
// channel before any parameter is touched, so a singular channel aborts the
// whole update like the reference's throw.
__global__ void bn_det_check_kernel(const spngd_bn_update_req* __restrict__ reqs, double lambda, int* status) {
  const spngd_bn_update_req r = reqs[blockIdx.y];
  for (int64_t ch = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; ch < r.c; ch += int64_t(gridDim.x) * blockDim.x) {
    const double a = double(r.m3c[3 * ch]) + lambda, b = double(r.m3c[3 * ch + 1]);
    const double d = double(r.m3c[3 * ch + 2]) + lambda;
    if (fabs(a * d - b * b) < 1e-30) set_status(status, SPNGD_ERR_SINGULAR_BLOCK);
  }
}

// world > 1: every rank adopts the largest status of any rank before Stage 4
// mutates parameters (16^code summed over <= 8 ranks decodes exactly).
__global__ void status_encode_kernel(const int* status, double* flag) {
  flag[0] = *status ? pow(16.0, double(*status)) : 0.0;
}
__global__ void status_decode_kernel(int* status, const double* flag) {
  if (flag[0] > 0.0 && *status == 0) *status = int(floor(log(flag[0]) / log(16.0) + 1e-9));
}

// HBM-bound: 16 bytes in / 8 out per element; float4 when every pointer is
// 16-byte aligned and n % 4 == 0 (true for the owner-major 64-float entries).
__global__ void sgd_update_kernel(const SgdTask* __restrict__ tasks, const float* __restrict__ scal,
                                  const int* __restrict__ status) {
  if (*status) return;
  const SgdTask t = tasks[blockIdx.y];
  const double eta = scal[0], mom = scal[1];
  const bool vec = t.n % 4 == 0 && ((reinterpret_cast<uintptr_t>(t.W) | reinterpret_cast<uintptr_t>(t.V) |
                                     reinterpret_cast<uintptr_t>(t.g)) & 15) == 0;
  const int64_t n4 = vec ? t.n / 4 : 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  auto upd = [&](float w, float v, float g, float& nw, float& nv) {
    nw = float(double(w) - eta * double(g) + mom * double(v));  // fisher.cpp:332
    nv = nw - w;                                                 // fisher.cpp:333
  };
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n4; q += stride) {
    const float4 w = reinterpret_cast<const float4*>(t.W)[q];
    const float4 v = reinterpret_cast<const float4*>(t.V)[q];
    const float4 g = __ldg(reinterpret_cast<const float4*>(t.g) + q);
    float4 nw, nv;
    upd(w.x, v.x, g.x, nw.x, nv.x);
    upd(w.y, v.y, g.y, nw.y, nv.y);
    upd(w.z, v.z, g.z, nw.z, nv.z);
    upd(w.w, v.w, g.w, nw.w, nv.w);
    reinterpret_cast<float4*>(t.W)[q] = nw;
    reinterpret_cast<float4*>(t.V)[q] = nv;
  }
  for (int64_t i = 4 * n4 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < t.n; i += stride) {
    float nw, nv;
    upd(t.W[i], t.V[i], t.g[i], nw, nv);
    t.W[i] = nw;
    t.V[i] = nv;
  }
}

// Weighted norms of x - x1, x1, x - x2, x2 (weights 1 on the diagonal, 2 off it
// for packed statistics; 1,2,1 for BN 3c payloads), stale.hpp:23-64.
__global__ void stat_distance_kernel(const StatJob* __restrict__ jobs) {
  const spngd_stat_req r = jobs[blockIdx.y].r;
  // rot may alias r.x2 (the fused snapshot rotation writes x into x2's slot):
  // no __restrict__; every element is read by the same thread before that
  // thread overwrites it, so the rotation is race-free.
  float* rot = jobs[blockIdx.y].rot;
  double acc[4] = {0, 0, 0, 0};
  if (r.kind == 0) {
    for (int64_t i = blockIdx.x; i < r.n; i += gridDim.x) {
      const int64_t base = i * r.n - i * (i - 1) / 2;
      for (int64_t j = i + threadIdx.x; j < r.n; j += blockDim.x) {
        const double w = (i == j) ? 1.0 : 2.0;
        const double x = r.x[base + j - i];
        if (r.x1) {
          const double y = r.x1[base + j - i];
          acc[0] += w * (x - y) * (x - y);
          acc[1] += w * y * y;
        }
        if (r.x2) {
          const double y = r.x2[base + j - i];
          acc[2] += w * (x - y) * (x - y);
          acc[3] += w * y * y;
        }
        if (rot) rot[base + j - i] = float(x);
      }
    }
  } else {
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < 3 * r.n; q += int64_t(gridDim.x) * blockDim.x) {
      const double w = (q % 3 == 1) ? 2.0 : 1.0;
      const double x = r.x[q];
      if (r.x1) { const double y = r.x1[q]; acc[0] += w * (x - y) * (x - y); acc[1] += w * y * y; }
      if (r.x2) { const double y = r.x2[q]; acc[2] += w * (x - y) * (x - y); acc[3] += w * y * y; }
      if (rot) rot[q] = float(x);
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
  // Warps that saw no entries skip their atomics: most of the grid's blocks
  // (small statistics, short tails) had nothing to add and stalled at exit
  // draining four atomics each (ncu: drain was the top stall reason).
  if ((threadIdx.x & 31) == 0 && (acc[0] != 0.0 || acc[1] != 0.0 || acc[2] != 0.0 || acc[3] != 0.0))
    for (int k = 0; k < 4; ++k) atomicAdd(r.out4 + k, acc[k]);
}

// The distance kernel accumulates weighted squares; the public entry point
// returns the norms themselves (weighted_norm, stale.hpp:49-51).
__global__ void stat_sqrt_kernel(const StatJob* __restrict__ jobs, int n) {
  for (int i = threadIdx.x; i < 4 * n; i += blockDim.x) {
    double* o = jobs[i >> 2].r.out4 + (i & 3);
    *o = sqrt(fmax(*o, 0.0));
  }
}

GemmOperand dense_operand(const float* ptr, int64_t ld, int64_t rows, int64_t K) {
  GemmOperand o{};
  o.ptr = ptr;
  o.row_stride = ld;
  o.seg_len = std::max<int64_t>(K, 1);
  o.rows = int32_t(rows);
  finalize_operand(o, K);
  return o;
}

}  // namespace

int plan_precondition(const spngd_precond_req* reqs, int n, double eta, double momentum, float* tmp,
                      double* norms, PrecondPlan& plan, const float* scal, const PrecondTri* tri) {
  plan = PrecondPlan();
  plan.stages = tri ? 4 : 2;
  std::vector<std::vector<GemmWorkItem>> pair_items[4];  // per stage, per problem: cluster-pair items
  std::vector<GemmWorkItem> elig_single[4];  // the same problems as 128 x 128 tiles
  size_t off = 0;
  auto take = [&](int64_t floats) {
    float* p = tmp ? tmp + off : nullptr;
    off += size_t(round_up(floats, 64));
    return p;
  };
  for (int i = 0; i < n; ++i) {
    const spngd_precond_req& r = reqs[i];
    if (r.g <= 0 || r.a <= 0) return fail(SPNGD_ERR_SHAPE_MISMATCH, "kron_matvec: empty operand");
    if (!r.dW || (!tri && (!r.Ginv || !r.Ainv))) return fail(SPNGD_ERR_INVALID, "precondition: null pointer");
    if (tri && (!tri[i].tlA || !tri[i].tuA || !tri[i].tlG || !tri[i].tuG))
      return fail(SPNGD_ERR_INVALID, "precondition: null triangular factor");
    if (r.ldg < r.g || r.lda < r.a) return fail(SPNGD_ERR_SHAPE_MISMATCH, "kron_matvec: X must be dim(G) x dim(A)");
    if (r.W && !r.V) return fail(SPNGD_ERR_INVALID, "ngd_step: velocity missing");
    const int64_t ldp = round_up(r.g, 4);
    GemmProblem st[4]{};
    auto dense = [](GemmProblem& p, int64_t M, int64_t N, int64_t K, int32_t ktri, float* C, int64_t ldc) {
      p.M = int32_t(M); p.N = int32_t(N); p.K = int32_t(K);
      p.mode = EPI_DENSE; p.alpha = 1.f; p.beta = 0.f; p.ktri = ktri;
      p.C = C; p.ldc = ldc;
    };
    GemmProblem* last = nullptr;
    if (!tri) {
      //   P1^T[j,i] = sum_k A^-1[j,k] dW[i,k]      (M=a, N=g, K=a)
      //   P^T [j,i] = sum_k P1^T[j,k] G^-1[i,k]    (M=a, N=g, K=g)
      float* p1t = take(r.a * ldp);
      st[0].A = dense_operand(r.Ainv, r.lda, r.a, r.a);
      st[0].B = dense_operand(r.dW, r.a, r.g, r.a);
      dense(st[0], r.a, r.g, r.a, 0, p1t, ldp);
      st[1].A = dense_operand(p1t, ldp, r.a, r.g);
      st[1].B = dense_operand(r.Ginv, r.ldg, r.g, r.g);
      last = &st[1];
    } else {
      // (A + dI)^-1 = T_A^T T_A, (G + dI)^-1 = T_G^T T_G, T lower (tl), T^T upper (tu):
      //   Q^T [i,m] = sum_k dW[i,k]   T_A[m,k]     (M=g, N=a, K=a; B lower)
      //   P1^T[j,i] = sum_m T_A^T[j,m] Q^T[i,m]     (M=a, N=g, K=a; A upper)
      //   R   [j,l] = sum_k P1^T[j,k] T_G[l,k]     (M=a, N=g, K=g; B lower)
      //   P^T [j,i] = sum_l R[j,l]   T_G^T[i,l]    (M=a, N=g, K=g; B upper)
      const int64_t ldq = round_up(r.a, 4);
      float* qt = take(r.g * ldq);
      float* p1t = take(r.a * ldp);
      float* rr = take(r.a * ldp);
      st[0].A = dense_operand(r.dW, r.a, r.g, r.a);
      st[0].B = dense_operand(tri[i].tlA, r.lda, r.a, r.a);
      dense(st[0], r.g, r.a, r.a, KTRI_B_LOWER, qt, ldq);
      st[1].A = dense_operand(tri[i].tuA, r.lda, r.a, r.a);
      st[1].B = dense_operand(qt, ldq, r.g, r.a);
      dense(st[1], r.a, r.g, r.a, KTRI_A_UPPER, p1t, ldp);
      st[2].A = dense_operand(p1t, ldp, r.a, r.g);
      st[2].B = dense_operand(tri[i].tlG, r.ldg, r.g, r.g);
      dense(st[2], r.a, r.g, r.g, KTRI_B_LOWER, rr, ldp);
      st[3].A = dense_operand(rr, ldp, r.a, r.g);
      st[3].B = dense_operand(tri[i].tuG, r.ldg, r.g, r.g);
      st[3].ktri = KTRI_B_UPPER;
      last = &st[3];
    }
    GemmProblem& pu = *last;
    pu.M = int32_t(r.a); pu.N = int32_t(r.g); pu.K = int32_t(r.g);
    pu.mode = EPI_UPDATE; pu.alpha = 1.f;
    pu.W = r.W; pu.V = r.V; pu.P_out = r.P_out;
    pu.eta = float(eta); pu.momentum = float(momentum);
    pu.scal = scal;
    pu.norm2 = (r.W && r.rescale && norms) ? norms + i : nullptr;
    const int idx = int(plan.probs[0].size());
    for (int q = 0; q < plan.stages; ++q) {
      plan.probs[q].push_back(st[q]);
      int slot = 0;
      if (pair_eligible_dense(st[q])) {  // 256 x 256 tiles on CTA pairs (gemm_pair.cu), or not (below)
        pair_items[q].push_back({});
        plan_pair_dense(idx, st[q], pair_items[q].back());
        plan_problem_tiles(idx, st[q], false, st[q].K + kTileK, elig_single[q], nullptr, &slot, 1.0, nullptr);
      } else {
        plan_problem_tiles(idx, st[q], false, st[q].K + kTileK, plan.items[q], nullptr, &slot, 1.0, nullptr);
      }
    }
    if (r.W && r.rescale)
      plan.rescale.push_back({r.W, r.V, r.g * r.a, norms ? norms + i : nullptr, std::sqrt(2.0 * double(r.g))});
  }
  plan.tmp_floats = off;
  plan.n_norms = n;
  auto longest = [](const GemmWorkItem& x, const GemmWorkItem& y) { return (x.k1 - x.k0) > (y.k1 - y.k0); };
  for (int q = 0; q < plan.stages; ++q) {
    // the stage takes the 2-CTA kernel only when that is faster at wave
    // granularity (a stage with ~one wave of 128 x 128 tiles finishes sooner
    // on it: the 4608-wide layers' stages were 1.4x longer on pairs)
    size_t npair = 0;
    for (const auto& v : pair_items[q]) npair += v.size();
    static const bool always = getenv("SPNGD_PRE_PAIR_ALWAYS") != nullptr;  // A/B experiments
    if (!always && !pair_group_wins(int64_t(npair), int64_t(elig_single[q].size()), int64_t(plan.items[q].size()))) {
      pair_items[q].clear();
      plan.items[q].insert(plan.items[q].end(), elig_single[q].begin(), elig_single[q].end());
    }
    std::stable_sort(plan.items[q].begin(), plan.items[q].end(), longest);
    std::vector<std::pair<GemmWorkItem, GemmWorkItem>> pairs;  // longest first, pairs as units
    for (const auto& v : pair_items[q])
      for (size_t k = 0; k + 1 < v.size(); k += 2) pairs.push_back({v[k], v[k + 1]});
    std::stable_sort(pairs.begin(), pairs.end(), [&](const auto& x, const auto& y) { return longest(x.first, y.first); });
    std::vector<GemmWorkItem> all;
    for (const auto& pr : pairs) {
      all.push_back(pr.first);
      all.push_back(pr.second);
    }
    plan.n_pair[q] = int(all.size());
    all.insert(all.end(), plan.items[q].begin(), plan.items[q].end());
    plan.items[q].swap(all);
  }
  return SPNGD_OK;
}

int run_precondition(spngd_ctx* ctx, const PrecondPlan& plan, GemmProblem* const* d_probs,
                     GemmWorkItem* const* d_items, const RescaleTask* d_rescale, double* d_norms) {
  return run_precondition_stages(ctx, plan, d_probs, d_items, d_rescale, d_norms, 0, plan.stages, true);
}

int run_precondition_stages(spngd_ctx* ctx, const PrecondPlan& plan, GemmProblem* const* d_probs,
                            GemmWorkItem* const* d_items, const RescaleTask* d_rescale, double* d_norms, int q0, int q1,
                            bool finish) {
  if (finish && d_norms && plan.n_norms > 0)
    SPNGD_CUDA_TRY(cudaMemsetAsync(d_norms, 0, sizeof(double) * plan.n_norms, ctx->stream));
  for (int q = q0; q < q1; ++q) {
    const int np = plan.n_pair[q], n = int(plan.items[q].size());
    int rc = launch_syrk_pair(d_probs[q], d_items[q], np, nullptr, ctx->stream, ctx->d_status);
    ctx->launches += np > 0;
    if (!rc && n > np)
      rc = launch_gemm(d_probs[q], d_items[q] + np, n - np, nullptr, ctx->d_status, ctx->stream,
                       gemm_variant(plan.probs[q].data(), int(plan.probs[q].size())));
    if (rc) return rc;
    ctx->launches += n > np;
  }
  if (finish && !plan.rescale.empty()) {
    dim3 grid(296, unsigned(plan.rescale.size()));
    rescale_kernel<<<grid, 256, 0, ctx->stream>>>(d_rescale, ctx->d_status);
    SPNGD_CUDA_TRY(cudaGetLastError());
    ctx->launches++;
  }
  return SPNGD_OK;
}

namespace {
__global__ void slot_mean_kernel(const SlotMeanTask* __restrict__ tasks) {
  const SlotMeanTask t = tasks[blockIdx.y];
  const float inv = 1.f / float(t.world);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < t.n; i += stride) {
    float acc = t.in[i];
    for (int q = 1; q < t.world; ++q) acc += t.in[q * t.slot_stride + i];
    t.out[i] = acc * inv;
  }
}
}  // namespace

int launch_slot_mean(spngd_ctx* ctx, const SlotMeanTask* d_tasks, int n, int64_t max_n) {
  if (n <= 0) return SPNGD_OK;
  dim3 grid(unsigned(std::min<int64_t>(std::max<int64_t>((max_n + 255) / 256, 1), 296)), unsigned(n));
  slot_mean_kernel<<<grid, 256, 0, ctx->stream>>>(d_tasks);
  SPNGD_CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return SPNGD_OK;
}

int launch_peer_copy(spngd_ctx* ctx, const PeerCopyTask* d_tasks, int n, int64_t max_n) {
  if (n <= 0) return SPNGD_OK;
  dim3 grid(unsigned(std::min<int64_t>(std::max<int64_t>((max_n / 4 + 255) / 256, 1), 296)), unsigned(n));
  peer_copy_kernel<<<grid, 256, 0, ctx->stream>>>(d_tasks, ctx->d_status);
  SPNGD_CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return SPNGD_OK;
}

int launch_snapshot(spngd_ctx* ctx, const SnapTask* d_tasks, int n, int64_t max_n, bool restore) {
  if (n <= 0) return SPNGD_OK;
  dim3 grid(unsigned(std::min<int64_t>(std::max<int64_t>((max_n / 4 + 255) / 256, 1), 2 * kNumSMs)), unsigned(n));
  snapshot_kernel<<<grid, 256, 0, ctx->stream>>>(d_tasks, restore, ctx->d_status);
  SPNGD_CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return SPNGD_OK;
}

int launch_bn_update(spngd_ctx* ctx, const spngd_bn_update_req* d_reqs, int n, int64_t max_c, double lambda,
                     double eta, double momentum, const float* scal) {
  if (n <= 0) return SPNGD_OK;
  dim3 grid(unsigned((max_c + 255) / 256), unsigned(n));
  bn_update_kernel<<<grid, 256, 0, ctx->stream>>>(d_reqs, lambda, eta, momentum, scal, ctx->d_status);
  SPNGD_CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return SPNGD_OK;
}

int launch_bn_det_check(spngd_ctx* ctx, const spngd_bn_update_req* d_reqs, int n, int64_t max_c, double lambda) {
  if (n <= 0) return SPNGD_OK;
  dim3 grid(unsigned(std::min<int64_t>((max_c + 255) / 256, 64)), unsigned(n));
  bn_det_check_kernel<<<grid, 256, 0, ctx->stream>>>(d_reqs, lambda, ctx->d_status);
  SPNGD_CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return SPNGD_OK;
}

int agree_status(spngd_ctx* ctx, double* d_flag) {
  if (ctx->world <= 1) return SPNGD_OK;
  status_encode_kernel<<<1, 1, 0, ctx->stream>>>(ctx->d_status, d_flag);
  SPNGD_CUDA_TRY(cudaGetLastError());
  int rc = comm_allreduce_sum_f64(ctx, d_flag, 1);
  if (rc) return rc;
  status_decode_kernel<<<1, 1, 0, ctx->stream>>>(ctx->d_status, d_flag);
  SPNGD_CUDA_TRY(cudaGetLastError());
  ctx->launches += 2;
  return SPNGD_OK;
}

int launch_sgd_update(spngd_ctx* ctx, const SgdTask* d_tasks, int n, const float* scal) {
  if (n <= 0) return SPNGD_OK;
  dim3 grid(296u, unsigned(n));  // 2 x 148 SMs
  sgd_update_kernel<<<grid, 256, 0, ctx->stream>>>(d_tasks, scal, ctx->d_status);
  SPNGD_CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return SPNGD_OK;
}

int launch_stat_distance(spngd_ctx* ctx, const StatJob* d_jobs, int n, int64_t max_rows) {
  if (n <= 0) return SPNGD_OK;
  dim3 grid(unsigned(std::min<int64_t>(std::max<int64_t>(max_rows, 1), 256)), unsigned(n));
  stat_distance_kernel<<<grid, 256, 0, ctx->stream>>>(d_jobs);
  SPNGD_CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return SPNGD_OK;
}

}  // namespace spngd

using namespace spngd;

extern "C" int spngd_precondition_update_batched(spngd_ctx* ctx, int n, const spngd_precond_req* reqs, double eta,
                                                 double momentum) {
  SPNGD_CTX_SCOPE(ctx);
  if (!ctx || (n > 0 && !reqs)) return fail(SPNGD_ERR_INVALID, "spngd_precondition_update_batched: null argument");
  if (n == 0) return SPNGD_OK;
  PrecondPlan sizing;
  int rc = plan_precondition(reqs, n, eta, momentum, nullptr, nullptr, sizing);
  if (rc) return rc;
  DeviceScratch scratch(ctx);
  float* tmp = scratch.alloc<float>(sizing.tmp_floats);
  double* norms = scratch.alloc<double>(n);
  PrecondPlan plan;
  plan_precondition(reqs, n, eta, momentum, tmp, norms, plan);
  GemmProblem* d_p[4] = {};
  GemmWorkItem* d_i[4] = {};
  for (int q = 0; q < plan.stages; ++q) {
    d_p[q] = scratch.upload(plan.probs[q]);
    d_i[q] = scratch.upload(plan.items[q]);
  }
  auto* d_rs = scratch.upload(plan.rescale);
  rc = run_precondition(ctx, plan, d_p, d_i, d_rs, norms);
  if (rc) return rc;
  return spngd_ctx_sync(ctx);
}

extern "C" int spngd_bn_solve_update_batched(spngd_ctx* ctx, int n, const spngd_bn_update_req* reqs, double lambda,
                                             double eta, double momentum) {
  SPNGD_CTX_SCOPE(ctx);
  if (!ctx || (n > 0 && !reqs)) return fail(SPNGD_ERR_INVALID, "spngd_bn_solve_update_batched: null argument");
  int64_t max_c = 0;
  for (int i = 0; i < n; ++i) {
    if (!reqs[i].m3c || !reqs[i].grad) return fail(SPNGD_ERR_INVALID, "precondition_bn: null pointer");
    if (reqs[i].gamma && (!reqs[i].beta || !reqs[i].vgamma || !reqs[i].vbeta))
      return fail(SPNGD_ERR_INVALID, "ngd_step: BN state incomplete");
    max_c = std::max(max_c, reqs[i].c);
  }
  if (n == 0) return SPNGD_OK;
  DeviceScratch scratch(ctx);
  std::vector<spngd_bn_update_req> v(reqs, reqs + n);
  auto* d = scratch.upload(v);
  int rc = launch_bn_det_check(ctx, d, n, max_c, lambda);
  if (!rc) rc = launch_bn_update(ctx, d, n, max_c, lambda, eta, momentum);
  if (rc) return rc;
  return spngd_ctx_sync(ctx);
}

extern "C" int spngd_stat_distance_batched(spngd_ctx* ctx, int n, const spngd_stat_req* reqs) {
  SPNGD_CTX_SCOPE(ctx);
  if (!ctx || (n > 0 && !reqs)) return fail(SPNGD_ERR_INVALID, "spngd_stat_distance_batched: null argument");
  int64_t max_rows = 0;
  for (int i = 0; i < n; ++i) {
    if (!reqs[i].x || !reqs[i].out4) return fail(SPNGD_ERR_INVALID, "similar: null pointer");
    max_rows = std::max(max_rows, reqs[i].kind == 0 ? reqs[i].n : (3 * reqs[i].n + 255) / 256);
    SPNGD_CUDA_TRY(cudaMemsetAsync(reqs[i].out4, 0, 4 * sizeof(double), ctx->stream));
  }
  if (n == 0) return SPNGD_OK;
  DeviceScratch scratch(ctx);
  std::vector<StatJob> v(n);
  for (int i = 0; i < n; ++i) v[i] = StatJob{reqs[i], nullptr};
  auto* d = scratch.upload(v);
  int rc = launch_stat_distance(ctx, d, n, max_rows);
  if (rc) return rc;
  stat_sqrt_kernel<<<1, 128, 0, ctx->stream>>>(d, n);
  SPNGD_CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return spngd_ctx_sync(ctx);
}
