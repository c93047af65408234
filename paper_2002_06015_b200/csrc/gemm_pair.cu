// sm_100a 2-CTA (cta_group::2) 3xTF32 SYRK: 256 x 256 output tiles for the
// large Kronecker factors (K1, mean_outer, fisher.cpp:55-75).
//
// Why: the single-CTA engine (gemm_tf32x3.cu) moves 32 KB of operands per
// 128x128x32 stage and is bound by operand delivery per SM (~14-15 B/cycle of
// the 42 B/cycle it would need at full MMA rate; neither a deeper ring nor
// larger TMA boxes helped, profiles/r02_ring).  A CTA pair on one TPC computes
// a 256x256 tile with one M=256, N=256 tcgen05.mma per product: each CTA loads
// its 128 A rows and HALF of the B tile (128 rows), the same 32 KB per stage,
// for twice the MMA work -- half the operand bytes per flop.
//
// Layout per CTA and 32-k stage (3 stages, 64 KB each):
//   A raw (= A hi) | A lo | B raw (= B hi) | B lo        (SS-form MMAs)
// TMEM: two 256-column fp32 accumulators (each CTA holds its 128 rows x 256),
// drained into round-to-nearest registers after every stage exactly as in the
// single-CTA engine, so the RZ accumulation bias stays bounded by one stage.
// Diagonal super-tiles (A rows == B rows in each CTA) load one tile per stage.
//
// Roles (512 threads per CTA, registers rebalanced with setmaxnreg): warps
// 0-3 producers (TMA of the A tile and the B half, both lo planes), warp 4 of
// the leader (cluster rank 0) issues the MMAs and does nothing else (a warp
// that also drains blocks on the tensor core's issue queue and delays the
// drains the next MMAs wait for), warps 8-15 drain (184 registers: 128 fp32
// accumulators per thread, lane quarter warp % 4, column half (warp - 8) / 4).
// Pair synchronisation: the producers of both CTAs arrive on the leader's
// `full` barrier (remote mbarrier arrive); the leader's commits are multicast
// to both CTAs' `empty` and `tmem_full`; drain warps of both CTAs arrive on
// the leader's `tmem_empty`.  Epilogues (packed triangle / split-K partials)
// per CTA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "gemm_tf32x3.cuh"

namespace spngd {

namespace {

constexpr int kPS = 3;                          // stages
constexpr int kPOp = kTileM * kTileK * 4;       // 16 KB: one 128 x 32 fp32 plane
constexpr int kPStage = 4 * kPOp;               // A raw | A lo | B raw | B lo
constexpr int kPEpi = 2 * kTileN + 4;           // epilogue tile row stride (floats)
constexpr int kPThreads = 512;

struct __align__(64) PairCtl {
  uint64_t raw[kPS];         // TMA arrival of this CTA's A tile (+ B half)
  uint64_t full[kPS];        // leader: 2 arrivals (the producer group of each CTA)
  uint64_t empty[kPS];       // multicast commit: stage free
  uint64_t tmem_full[2];     // multicast commit
  uint64_t tmem_empty[2];    // leader: 16 drain-warp arrivals (8 per CTA)
  uint32_t tmem_base;
  int32_t pad;
  GemmProblem prob;
  GemmWorkItem item;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAITC_%=: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Arrive on the leader's copy of `bar` (local when this CTA is the leader).
__device__ __forceinline__ void arrive_leader(uint64_t* bar, bool leader) {
  if (leader) {
    mbar_arrive(bar);
  } else {
    const uint32_t remote = map_to_rank(smem_u32(bar), 0);
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
  }
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "n"(512)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(512) : "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T across the pair (M = 256: 128 rows per CTA).
__device__ __forceinline__ void umma_pair_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void load_tile(const GemmOperand& op, const CUtensorMap* map, uint32_t dst, int32_t tq,
                                          int32_t row0, uint64_t* bar) {
  if (op.mode == OP_TMA2D) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(tq * kTileK), "r"(row0), "r"(smem_u32(bar))
        : "memory");
  } else {
    const int32_t seg = tq / op.cps, ch = tq - seg * op.cps;
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(ch * kTileK), "r"(row0), "r"(seg), "r"(smem_u32(bar))
        : "memory");
  }
}
__device__ __forceinline__ void tmem_ld_x32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

#ifdef SPNGD_GEMM_TRACE_BUILD
// make TRACE=1 + SPNGD_GEMM_TRACE=1: clock64 stamps of the first pair's stages
// {TMA issued, landed, full arrived (producers), MMA issued (leader), drained}
__device__ long long g_pair_trace[2][64][5];
#define PAIR_STAMP(cond, cta, it, k) \
  do {                               \
    if ((cond) && blockIdx.x < 2 && (it) < 64) g_pair_trace[cta][it][k] = clock64(); \
  } while (0)
#else
#define PAIR_STAMP(cond, cta, it, k) \
  do {                               \
  } while (0)
#endif

// Lo plane of a 128 x 32 swizzled fp32 tile: rows rbase + 16 j, 16-byte chunk c.
__device__ __forceinline__ void lo_plane(const uint8_t* src, uint8_t* dst, int rbase, int c) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int r = rbase + 16 * j;
    const uint32_t off = r * 128 + ((c ^ (r & 7)) << 4);
    const float4 x = *reinterpret_cast<const float4*>(src + off);
    float4 l;
    l.x = tf32_lo(x.x);
    l.y = tf32_lo(x.y);
    l.z = tf32_lo(x.z);
    l.w = tf32_lo(x.w);
    *reinterpret_cast<float4*>(dst + off) = l;
  }
}

// Work item of CTA r of a pair: tm = 2 I + r (its 128-row tile), tn = 2 J (the
// first of its two 128-column tiles), slot = first of 2 partial slots (split-K).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPThreads, 1)
    syrk_pair_kernel(const GemmProblem* __restrict__ probs, const GemmWorkItem* __restrict__ items,
                     float* __restrict__ partials, int* status) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  PairCtl* ctl = reinterpret_cast<PairCtl*>(smem + kPS * kPStage);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;

  if (threadIdx.x == 0) ctl->item = items[blockIdx.x];
  __syncthreads();
  {
    const int32_t* src = reinterpret_cast<const int32_t*>(probs + ctl->item.problem);
    int32_t* dst = reinterpret_cast<int32_t*>(&ctl->prob);
    for (int i = threadIdx.x; i < int(sizeof(GemmProblem) / 4); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();  // the cooperative descriptor copy is complete before anyone reads it
  const GemmWorkItem item0 = ctl->item;
  // SYRK super-diagonal tile: A rows == B rows in both CTAs, one load per stage
  const bool diag = (ctl->prob.flags & FLAG_SAME_AB) && (item0.tm >> 1) == (item0.tn >> 1);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPS; ++s) {
      mbar_init(&ctl->raw[s], 1);
      mbar_init(&ctl->full[s], 2);
      mbar_init(&ctl->empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ctl->tmem_full[b], 1);
      mbar_init(&ctl->tmem_empty[b], 16);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == 4) tmem_alloc_pair(&ctl->tmem_base);
  tc_fence_before();
  cluster_sync_all();  // both CTAs' barriers and the pair's TMEM exist before any remote use
  tc_fence_after();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t tmem = ctl->tmem_base;
  const GemmWorkItem item = ctl->item;
  const GemmProblem& prob = ctl->prob;
  const int n_iters = (item.k1 - item.k0 + kTileK - 1) / kTileK;
  float* T = reinterpret_cast<float*>(smem);

  if (warp >= 8) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 184;" ::: "memory");
    // ---------------------------------------- drain (warps 8-15)
    const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
    const uint32_t col_base = ((warp - 8) >> 2) * 128;
    float acc[128];
#pragma unroll
    for (int j = 0; j < 128; ++j) acc[j] = 0.f;
    for (int j = 0; j < n_iters; ++j) {
      const int b = j & 1;
      mbar_wait(&ctl->tmem_full[b], (j >> 1) & 1);
      tc_fence_after();
      PAIR_STAMP(warp == 8 && lane == 0, rank, j, 4);
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        uint32_t v[32];
        tmem_ld_x32_nowait(tmem + lane_base + b * 256 + col_base + 32 * h, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int q = 0; q < 32; ++q) acc[32 * h + q] += __uint_as_float(v[q]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_leader(&ctl->tmem_empty[b], leader);
    }
    // every MMA of this CTA's accumulator has completed: the stage ring is free
    asm volatile("bar.sync 1, 256;" ::: "memory");
    const int r = (warp & 3) * 32 + lane;
    float4* trow = reinterpret_cast<float4*>(T + r * kPEpi + col_base);
#pragma unroll
    for (int j = 0; j < 32; ++j) trow[j] = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
    asm volatile("setmaxnreg.dec.sync.aligned.u32 128;" ::: "memory");  // uniform again for the epilogue
  } else if (warp >= 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;" ::: "memory");
    // ---------------------------------------- MMA issue (leader warp 4 only)
    if (warp == 4 && leader) {
      constexpr uint32_t idesc = umma_idesc_tf32(2 * kTileM, 2 * kTileN);  // M = 256 across the pair, N = 256
      for (int it = 0; it < n_iters; ++it) {
        const int s = it % kPS, b = it & 1;
        mbar_wait_cluster(&ctl->full[s], (it / kPS) & 1);
        if (it >= 2) mbar_wait_cluster(&ctl->tmem_empty[b], ((it >> 1) + 1) & 1);
        tc_fence_after();
        PAIR_STAMP(lane == 0, 0, it, 3);
        if (lane == 0) {
          const uint32_t base = smem_u32(smem + s * kPStage);
          const uint32_t a_hi = base, a_lo = base + kPOp;
          const uint32_t b_hi = diag ? a_hi : base + 2 * kPOp, b_lo = diag ? a_lo : base + 3 * kPOp;
          const uint32_t dt = tmem + b * 256;
#pragma unroll
          for (int kk = 0; kk < kTileK / 8; ++kk) {
            const uint32_t koff = kk * 32;  // 8 tf32 = 32 bytes along the swizzled row
            const uint64_t dah = umma_desc_k_sw128(a_hi + koff), dal = umma_desc_k_sw128(a_lo + koff);
            const uint64_t dbh = umma_desc_k_sw128(b_hi + koff), dbl = umma_desc_k_sw128(b_lo + koff);
            umma_pair_ss(dt, dal, dbh, idesc, kk > 0 ? 1u : 0u);
            umma_pair_ss(dt, dah, dbl, idesc, 1u);
            umma_pair_ss(dt, dah, dbh, idesc, 1u);
          }
          commit_pair(&ctl->empty[s]);
          commit_pair(&ctl->tmem_full[b]);
        }
        __syncwarp();
      }
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 128;" ::: "memory");
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 80;" ::: "memory");
    // ------------------------------------------------------------ producers (warps 0-3)
    const int t = threadIdx.x;
    const int c = t & 7, rbase = t >> 3;
    const CUtensorMap* amap = &probs[item.problem].A.tmap;
    const CUtensorMap* bmap = &probs[item.problem].B.tmap;
    // A: this CTA's 128 rows; B: this CTA's half (128 rows) of the 256-row B tile
    const int32_t arow = item.tm * kTileM, brow = (item.tn + int32_t(rank)) * kTileN;
    const int32_t tq0 = item.k0 / kTileK;
    const uint32_t bytes = diag ? kPOp : 2 * kPOp;
    // implicit im2col operands (raw conv inputs) are gathered by all 128
    // producer threads with cp.async (one commit group per stage)
    const bool gather = prob.A.mode == OP_IM2COL;
    auto load = [&](int q) {
      const int ps = q % kPS;
      PAIR_STAMP(t == 0, rank, q, 0);
      const uint32_t st = smem_u32(smem + ps * kPStage);
      if (gather) {
        const int32_t kb = item.k0 + q * kTileK;
        im2col_stage(prob.A.ptr, prob.A.geo, prob.A.rows, arow, kb, item.k1, st, warp, lane);
        if (!diag) im2col_stage(prob.B.ptr, prob.B.geo, prob.B.rows, brow, kb, item.k1, st + 2 * kPOp, warp, lane);
        return;
      }
      expect_tx(&ctl->raw[ps], bytes);
      load_tile(prob.A, amap, st, tq0 + q, arow, &ctl->raw[ps]);
      if (!diag) load_tile(prob.B, bmap, st + 2 * kPOp, tq0 + q, brow, &ctl->raw[ps]);
    };
    if (gather) {
      for (int q = 0; q < kPS - 1; ++q) {
        if (q < n_iters) load(q);
        asm volatile("cp.async.commit_group;" ::: "memory");
      }
    } else if (t == 0) {
      asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(reinterpret_cast<uint64_t>(amap))
                   : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(amap)) : "memory");
      if (!diag) {
        asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(reinterpret_cast<uint64_t>(bmap))
                     : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(bmap)) : "memory");
      }
      for (int q = 0; q < kPS - 1 && q < n_iters; ++q) load(q);
    }
    for (int it = 0; it < n_iters; ++it) {
      const int s = it % kPS;
      uint8_t* stage = smem + s * kPStage;
      if (gather) {
        asm volatile("cp.async.wait_group %0;" ::"n"(kPS - 2) : "memory");
        asm volatile("bar.sync 2, 128;" ::: "memory");  // rows span other threads' copies
      } else {
        mbar_wait(&ctl->raw[s], (it / kPS) & 1);
      }
      PAIR_STAMP(t == 0, rank, it, 1);
      lo_plane(stage, stage + kPOp, rbase, c);
      if (!diag) lo_plane(stage + 2 * kPOp, stage + 3 * kPOp, rbase, c);
      fence_proxy_async_smem();
      asm volatile("bar.sync 2, 128;" ::: "memory");
      if (t == 0) {
        PAIR_STAMP(true, rank, it, 2);
        arrive_leader(&ctl->full[s], leader);
      }
      const int nx = it + kPS - 1;  // refill the slot the MMAs of stage it-1 released
      if (gather) {
        if (nx < n_iters) {
          mbar_wait(&ctl->empty[nx % kPS], ((nx / kPS) & 1) ^ 1);
          load(nx);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      } else if (t == 0 && nx < n_iters) {
        mbar_wait(&ctl->empty[nx % kPS], ((nx / kPS) & 1) ^ 1);
        load(nx);
      }
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 128;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the pair's MMAs, commits and remote arrivals are all done
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc_pair(tmem);
  }

  // ------------------------------------------------------------ epilogue (this CTA's 128 x 256)
  const int tid = threadIdx.x;
  const int64_t n = prob.M;
  const int64_t m0 = int64_t(item.tm) * kTileM, n0 = int64_t(item.tn) * kTileN;
  if (prob.mode == EPI_PARTIAL) {
    if (item.slot < 0) return;
    // sub-tile q (columns 128 q..) -> slot + q; rows/columns outside the
    // triangle are written too (the reduction only reads kept tiles)
    for (int p = tid; p < 8192; p += kPThreads) {  // 8192 float4 chunks
      const int r = p >> 6, cc = (p & 63) * 4;
      const int q = cc >> 7;
      float4* dst = reinterpret_cast<float4*>(partials + (int64_t(item.slot) + q) * kTileM * kTileN);
      dst[r * 32 + ((cc & 127) >> 2)] = *reinterpret_cast<const float4*>(T + r * kPEpi + cc);
    }
  } else if (prob.mode == EPI_PACKED) {  // alpha * acc -> packed upper triangle
    float* C = prob.C;
    const float alpha = prob.alpha;
    for (int p = tid; p < 8192; p += kPThreads) {
      const int r = p >> 6, cc = (p & 63) * 4;
      const int64_t i = m0 + r;
      if (i >= n) continue;
      const int64_t rb = packed_offset(n, i, i) - i;
      const float4 v = *reinterpret_cast<const float4*>(T + r * kPEpi + cc);
      const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t jj = n0 + cc + q;
        if (jj < n && i <= jj) C[rb + jj] = alpha * vv[q];
      }
    }
  } else if (prob.mode == EPI_DENSE) {
    // C = alpha acc + beta Cin row-major; FLAG_SYM_MIRROR writes i <= j and
    // mirrors to (j, i); FLAG_TRANS also writes CT[j][i] (the inverse recursion)
    float* C = prob.C;
    const float* Cin = prob.Cin;
    const float alpha = prob.alpha, beta = prob.beta;
    const int64_t M = prob.M, N = prob.N, ldc = prob.ldc;
    const bool mirror = (prob.flags & FLAG_SYM_MIRROR) != 0, trans = (prob.flags & FLAG_TRANS) != 0;
    const bool has_cin = beta != 0.f;
    const bool vec = ((reinterpret_cast<uintptr_t>(C) | (has_cin ? reinterpret_cast<uintptr_t>(Cin) : 0)) & 15) == 0 &&
                     (ldc & 3) == 0;
    for (int p = tid; p < 8192; p += kPThreads) {
      const int r = p >> 6, cc = (p & 63) * 4;
      const int64_t i = m0 + r, j = n0 + cc;
      if (i >= M || j >= N) continue;
      float4* tp = reinterpret_cast<float4*>(T + r * kPEpi + cc);
      float4 v = *tp;
      float4 ci = make_float4(0.f, 0.f, 0.f, 0.f);  // Cin first: C and Cin may alias
      if (has_cin) {
        if (vec && j + 3 < N) {
          ci = *reinterpret_cast<const float4*>(Cin + i * ldc + j);
        } else {
          const float* src = Cin + i * ldc + j;
          ci.x = src[0];
          if (j + 1 < N) ci.y = src[1];
          if (j + 2 < N) ci.z = src[2];
          if (j + 3 < N) ci.w = src[3];
        }
      }
      v = make_float4(alpha * v.x + beta * ci.x, alpha * v.y + beta * ci.y, alpha * v.z + beta * ci.z,
                      alpha * v.w + beta * ci.w);
      *tp = v;
      float* dst = C + i * ldc + j;
      if (vec && j + 3 < N && (!mirror || i <= j)) {
        *reinterpret_cast<float4*>(dst) = v;
      } else {
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (j + q < N && (!mirror || i <= j + q)) dst[q] = vv[q];
      }
    }
    if (mirror || trans) {
      __syncthreads();
      float* dstT = mirror ? C : prob.CT;
      const int64_t ldt = mirror ? ldc : prob.ldct;
      const bool vt = (reinterpret_cast<uintptr_t>(dstT) & 15) == 0 && (ldt & 3) == 0;
      for (int p = tid; p < 8192; p += kPThreads) {
        // 16 columns x 2 row quads per warp: conflict-free column reads of T
        const int wk = p >> 5, ln = p & 31;
        const int c = (wk & 15) * 16 + (ln & 15);
        const int r = ((wk >> 4) * 2 + (ln >> 4)) * 4;
        const int64_t i = m0 + r, j = n0 + c;  // writes dstT[j][i .. i+3]
        if (j >= N || i >= M) continue;
        const float4 v = make_float4(T[r * kPEpi + c], T[(r + 1) * kPEpi + c], T[(r + 2) * kPEpi + c],
                                     T[(r + 3) * kPEpi + c]);
        float* dst = dstT + j * ldt + i;
        if (vt && i + 3 < M && (!mirror || i + 3 < j)) {
          *reinterpret_cast<float4*>(dst) = v;
        } else {
          const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (i + q < M && (!mirror || i + q < j)) dst[q] = vv[q];
        }
      }
    }
  } else if (prob.mode == EPI_UPDATE) {
    // P^T tile (rows: a-index j = m0 + r, columns: g-index i = n0 + c) ->
    // W' = W - eta P + m V, V' = W' - W (fisher.cpp:332-333) along weight rows
    // W[i * a + j], plus the ||W'||^2 partials of the rescale.  Nothing is
    // written after a failed inverse / BN check (status word, precond.cu).
    if (prob.W && status && *reinterpret_cast<volatile int*>(status)) return;
    const int64_t a = prob.M, N = prob.N;
    const float alpha = prob.alpha;
    const float eta = prob.scal ? prob.scal[0] : prob.eta;
    const float mom = prob.scal ? prob.scal[1] : prob.momentum;
    float* W = prob.W;
    float* V = prob.V;
    float* Pout = prob.P_out;
    const bool vec = (a & 3) == 0 && (!W || ((reinterpret_cast<uintptr_t>(W) | reinterpret_cast<uintptr_t>(V)) & 15) == 0) &&
                     (!Pout || (reinterpret_cast<uintptr_t>(Pout) & 15) == 0);
    double ss = 0.0;
    for (int p = tid; p < 8192; p += kPThreads) {
      // 16 columns x 2 row quads per warp: conflict-free column reads of T
      const int wk = p >> 5, ln = p & 31;
      const int c = (wk & 15) * 16 + (ln & 15);
      const int r = ((wk >> 4) * 2 + (ln >> 4)) * 4;
      const int64_t j = m0 + r, i = n0 + c;
      if (i >= N || j >= a) continue;
      const float t0 = T[r * kPEpi + c], t1 = T[(r + 1) * kPEpi + c], t2 = T[(r + 2) * kPEpi + c],
                  t3 = T[(r + 3) * kPEpi + c];
      const float pp[4] = {alpha * t0, alpha * t1, alpha * t2, alpha * t3};
      const int64_t o = i * a + j;
      const int nq = (a - j) >= 4 ? 4 : int(a - j);
      if (vec && nq == 4) {
        if (Pout) *reinterpret_cast<float4*>(Pout + o) = make_float4(pp[0], pp[1], pp[2], pp[3]);
        if (W) {
          const float4 w = *reinterpret_cast<const float4*>(W + o), vl = *reinterpret_cast<const float4*>(V + o);
          const float4 nw = make_float4(w.x - eta * pp[0] + mom * vl.x, w.y - eta * pp[1] + mom * vl.y,
                                        w.z - eta * pp[2] + mom * vl.z, w.w - eta * pp[3] + mom * vl.w);
          *reinterpret_cast<float4*>(W + o) = nw;
          *reinterpret_cast<float4*>(V + o) = make_float4(nw.x - w.x, nw.y - w.y, nw.z - w.z, nw.w - w.w);
          ss += double(nw.x) * nw.x + double(nw.y) * nw.y + double(nw.z) * nw.z + double(nw.w) * nw.w;
        }
      } else {
        for (int q = 0; q < nq; ++q) {
          if (Pout) Pout[o + q] = pp[q];
          if (W) {
            const float w = W[o + q];
            const float nw = w - eta * pp[q] + mom * V[o + q];
            W[o + q] = nw;
            V[o + q] = nw - w;
            ss += double(nw) * nw;
          }
        }
      }
    }
    if (prob.norm2) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0 && ss != 0.0) atomicAdd(prob.norm2, ss);
    }
  }
}

}  // namespace

bool pair_eligible(const GemmProblem& p) {
  static const bool off = getenv("SPNGD_NO_PAIR") != nullptr;
  if (off || !(p.flags & FLAG_SAME_AB)) return false;
  if (p.A.mode != OP_TMA2D && p.A.mode != OP_TMA3D) return false;
  // 256-row super-tiles cover the triangle with more (partly empty) MMA work
  // than 128-row tiles; the pair runs ~1.45x the single-CTA rate on the same
  // work (ncu: tensor pipe 45.6% vs 38.6%, ResNet-50 B=32), so it wins while
  // its sub-tile count stays within 1.35x (n = 147, 256, 512, >= 1024; not 64,
  // 128, 576)
  const int64_t t = (p.M + kTileM - 1) / kTileM, ts = (p.M + 2 * kTileM - 1) / (2 * kTileM);
  return double(2 * ts * (ts + 1)) <= 1.35 * double(t * (t + 1) / 2);
}

int plan_pair_tiles(int problem_index, const GemmProblem& p, int kchunk, std::vector<GemmWorkItem>& items,
                    std::vector<SyrkReduceTask>* reduce, int* next_slot, double reduce_scale, float* packed_out) {
  const int t128 = (p.M + kTileM - 1) / kTileM;
  const int ts = (p.M + 2 * kTileM - 1) / (2 * kTileM);
  const bool whole = kchunk >= p.K;
  kchunk = std::max(kTileK, (kchunk / kTileK) * kTileK);
  const int nchunks = whole ? 1 : std::max(1, (p.K + kchunk - 1) / kchunk);
  struct Pair {
    int I, J, s0, s1;
  };
  std::vector<Pair> pairs;
  int used = 0;
  for (int J = 0; J < ts; ++J)
    for (int I = 0; I <= J; ++I) {
      Pair pr{I, J, -1, -1};
      if (nchunks > 1) {
        for (int r = 0; r < 2; ++r) {
          const int s0 = *next_slot;
          *next_slot += 2 * nchunks;
          used += 2 * nchunks;
          (r ? pr.s1 : pr.s0) = s0;
          const int tm = 2 * I + r;
          for (int q = 0; q < 2; ++q) {
            const int tn = 2 * J + q;
            if (tm < t128 && tn < t128 && tm <= tn && reduce)
              reduce->push_back({tm, tn, s0 + q, nchunks, p.M, 2, reduce_scale, packed_out});
          }
        }
      }
      pairs.push_back(pr);
    }
  // chunk-major so the pairs running together share panels in L2
  for (int q = 0; q < nchunks; ++q) {
    const int k0 = q * kchunk, k1 = nchunks == 1 ? p.K : std::min(p.K, k0 + kchunk);
    for (const Pair& pr : pairs)
      for (int r = 0; r < 2; ++r)
        items.push_back({problem_index, 2 * pr.I + r, 2 * pr.J, k0, k1,
                         nchunks == 1 ? -1 : (r ? pr.s1 : pr.s0) + 2 * q});
  }
  return used;
}

bool pair_eligible_dense(const GemmProblem& p, bool upper_only) {
  static const bool off = getenv("SPNGD_NO_PAIR") != nullptr;
  if (off || (p.mode != EPI_DENSE && p.mode != EPI_UPDATE)) return false;
  if ((p.A.mode != OP_TMA2D && p.A.mode != OP_TMA3D) || (p.B.mode != OP_TMA2D && p.B.mode != OP_TMA3D)) return false;
  if (p.M < 256 || p.N < 256) return false;
  const int64_t tm = (p.M + kTileM - 1) / kTileM, tn = (p.N + kTileN - 1) / kTileN;
  const int64_t sm = (p.M + 2 * kTileM - 1) / (2 * kTileM), sn = (p.N + 2 * kTileN - 1) / (2 * kTileN);
  if (upper_only)  // square, upper super-tiles (symmetric results)
    return double(2 * sm * (sm + 1)) <= 1.35 * double(tm * (tm + 1) / 2);
  return double(4 * sm * sn) <= 1.25 * double(tm * tn);
}

int plan_pair_dense(int problem_index, const GemmProblem& p, std::vector<GemmWorkItem>& items, bool upper_only) {
  const int sm = (p.M + 2 * kTileM - 1) / (2 * kTileM), sn = (p.N + 2 * kTileN - 1) / (2 * kTileN);
  for (int I = 0; I < sm; ++I)
    for (int J = upper_only ? I : 0; J < sn; ++J) {
      int k0 = 0, k1 = p.K;  // triangular operands: the band of the whole 256 x 256 tile
      if (p.ktri & KTRI_A_LOWER) k1 = std::min(k1, (2 * I + 2) * kTileM);
      if (p.ktri & KTRI_A_UPPER) k0 = std::max(k0, 2 * I * kTileM);
      if (p.ktri & KTRI_B_LOWER) k1 = std::min(k1, (2 * J + 2) * kTileN);
      if (p.ktri & KTRI_B_UPPER) k0 = std::max(k0, 2 * J * kTileN);
      if (k1 < k0) k1 = k0;
      for (int r = 0; r < 2; ++r) items.push_back({problem_index, 2 * I + r, 2 * J, k0, k1, -1});
    }
  return 0;
}

bool pair_group_wins(int64_t pair_ctas, int64_t single_ctas, int64_t rest_ctas) {
  if (pair_ctas <= 0) return false;
  auto waves = [](int64_t c) { return double((c + kNumSMs - 1) / kNumSMs); };
  return 1.45 * waves(pair_ctas) + waves(rest_ctas) < waves(single_ctas + rest_ctas);
}

size_t gemm_pair_smem_bytes() { return size_t(kPS) * kPStage + sizeof(PairCtl) + 1024; }

int launch_syrk_pair(const GemmProblem* d_probs, const GemmWorkItem* d_items, int n_items, float* d_partials,
                     cudaStream_t stream, int* d_status) {
  if (n_items <= 0) return SPNGD_OK;
  static bool attr_set = false;
  const size_t smem = gemm_pair_smem_bytes();
  if (!attr_set) {
    SPNGD_CUDA_TRY(cudaFuncSetAttribute(syrk_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr_set = true;
  }
  static const bool pdl = getenv("SPNGD_NO_PDL") == nullptr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(n_items));
  cfg.blockDim = dim3(kPThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, syrk_pair_kernel, d_probs, d_items, d_partials, d_status);
  if (e != cudaSuccess) return fail(SPNGD_ERR_CUDA, "syrk_pair launch failed: %s", cudaGetErrorString(e));
#ifdef SPNGD_GEMM_TRACE_BUILD
  static int printed = 0;
  if (getenv("SPNGD_GEMM_TRACE") && printed++ < 3) {
    long long h[2][64][5];
    cudaStreamSynchronize(stream);
    cudaMemcpyFromSymbol(h, g_pair_trace, sizeof(h));
    printf("pair launch %d (%d CTAs): CTA r: stage issue landed full | mma_issue drained (cycles rel. to CTA 0's first issue)\n",
           printed - 1, n_items);
    const long long t0 = h[0][0][0];
    for (int q = 0; q < 24; ++q)
      printf("  %2d  r0 %7lld %7lld %7lld | r1 %7lld %7lld %7lld | mma %7lld  drained r0 %7lld r1 %7lld\n", q,
             h[0][q][0] - t0, h[0][q][1] - t0, h[0][q][2] - t0, h[1][q][0] - t0, h[1][q][1] - t0, h[1][q][2] - t0,
             h[0][q][3] - t0, h[0][q][4] - t0, h[1][q][4] - t0);
  }
#endif
  return SPNGD_OK;
}

}  // namespace spngd
