// sm_100a grouped 3xTF32 GEMM on tcgen05 tensor cores with TMEM accumulators.
//
// CTA layout (512 threads, one CTA per SM):
//   warps 0-3   producers of the A tile (128 rows x 32 k per stage)
//   warps 4-7   producers of the B tile (idle on SYRK diagonal tiles)
//   warps 8-15  accumulator drain (TMEM -> round-to-nearest fp32 registers);
//               warp 8 also allocates TMEM and issues tcgen05.mma (one lane)
// Producers read fp32 from HBM/L2 (coalesced float4 when the layout allows),
// derive the tf32 lo plane (the raw fp32 tile doubles as the hi operand since
// the tensor core truncates to tf32) into 128B-swizzled K-major smem tiles;
// the MMA thread issues
// hi*hi + hi*lo + lo*hi per 8-wide k step (3xTF32 = fp32-accurate products,
// SURVEY.md §7.3).  mbarrier full/empty rings pipeline kStages smem stages;
// tcgen05.commit releases smem slots.
// The tensor core's fp32 accumulator rounds toward zero on every MMA, which
// biases long sums (measured ~1e-8 * K relative).  Each 32-deep stage
// therefore accumulates into one of two TMEM buffers that the producer warps
// drain right after (tcgen05.ld 32x32b) into round-to-nearest fp32 registers,
// so the truncation bias is bounded by one stage (~4e-7) at any K.
// Epilogue: registers -> padded smem tile -> coalesced global writes in the
// order each epilogue mode needs.
#include <cuda_runtime.h>

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "gemm_tf32x3.cuh"

namespace spngd {

namespace {

constexpr int kOperandBytes = kTileM * kTileK * 4;     // 16 KB (128 rows x 128 B)
constexpr int kStageBytes = 3 * kOperandBytes;         // A raw, B raw (= B hi), B lo
// Epilogue tile row stride: 132 floats keeps rows 16-byte aligned (float4
// row access is conflict-free) and makes the (16 columns x 2 row-quads) column
// access of the transposed/update stores conflict-free too (528 = 16 mod 32).
constexpr int kEpiStride = kTileN + 4;
constexpr int kTmemCols = 512;  // 2 x 128 accumulator columns + kStages x (A hi | A lo) x 32
constexpr uint32_t kTmemA = 256;                       // first A-operand column

struct __align__(64) SmemCtl {
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t tmem_full[2];
  uint64_t tmem_empty[2];
  uint64_t raw[2][kStages];  // TMA raw-tile arrival per operand (A, B)
  uint32_t tmem_base;
  int32_t pad;
  GemmProblem prob;
  GemmWorkItem item;
};

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// Per-thread cursor over the segmented K axis: k = s * seg_len + p.  Advanced
// incrementally (no 64-bit division in the main loop).
struct KCursor {
  int64_t s;
  int32_t p;
  int32_t k;  // absolute k of the chunk start
};

__device__ __forceinline__ KCursor cursor_at(const GemmOperand& op, int32_t k) {
  KCursor c;
  c.k = k;
  if (op.seg_len == 1) {
    c.s = k;
    c.p = 0;
  } else {
    c.s = k / op.seg_len;
    c.p = int32_t(k - c.s * op.seg_len);
  }
  return c;
}

__device__ __forceinline__ void cursor_advance(const GemmOperand& op, KCursor& c, int32_t dk) {
  c.k += dk;
  if (op.seg_len == 1) {
    c.s += dk;
    return;
  }
  c.p += dk;
  while (c.p >= op.seg_len) {
    c.p -= int32_t(op.seg_len);
    ++c.s;
  }
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1, int32_t c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// Issues the async copies of k .. k+3 for the 8 rows (r0 + 16 j) this thread
// feeds into the swizzled fp32 plane at `plane` (zero-filled outside).
__device__ __forceinline__ void issue_stage(const GemmOperand& op, int32_t r0, int rbase, int c, const KCursor& cur,
                                           int32_t kend, uint32_t plane) {
  if (op.vec && cur.k + 3 < kend) {
    const float* base = op.ptr + cur.s * op.seg_stride + cur.p;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int32_t r = r0 + 16 * j;
      const int rl = rbase + 16 * j;
      const uint32_t dst = plane + rl * 128 + ((c ^ (rl & 7)) << 4);
      const bool ok = r < op.rows;
      cp_async16(dst, ok ? base + int64_t(r) * op.row_stride : op.ptr, ok ? 16u : 0u);
    }
    return;
  }
  int64_t off[4];
  bool ok[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    ok[e] = cur.k + e < kend;
    if (op.seg_len == 1) {
      off[e] = (cur.s + e) * op.seg_stride;
    } else {
      int64_t ss = cur.s;
      int32_t pp = cur.p + e;
      if (pp >= op.seg_len) { pp -= int32_t(op.seg_len); ++ss; }
      off[e] = ss * op.seg_stride + pp;
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int32_t r = r0 + 16 * j;
    const int rl = rbase + 16 * j;
    const uint32_t dst = plane + rl * 128 + ((c ^ (rl & 7)) << 4);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const bool v = r < op.rows && ok[e];
      cp_async4(dst + 4 * e, v ? op.ptr + off[e] + int64_t(r) * op.row_stride : op.ptr, v ? 4u : 0u);
    }
  }
}

// kModes: bit set of the GemmEpi modes compiled in; kAsync: the cp.async
// (OP_ASYNC) operand path is compiled in.  Each launch gets the smallest
// variant its problems need: the inverse recursion issues ~100 short launches
// per matrix that each start with a cold instruction cache, so code size is
// latency.
template <uint32_t kModes, bool kAsync>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tf32x3_kernel(const GemmProblem* __restrict__ probs, const GemmWorkItem* __restrict__ items,
                       float* __restrict__ partials, int* status, long long* trace) {
  // trace (debug): for CTAs < 4, stages < 64: [cta][stage][4] clock64 stamps
  // {A TMA issued, A raw landed, MMA saw full, drain saw MMA done}.
#ifdef SPNGD_GEMM_TRACE_BUILD
  long long* tr = (trace && blockIdx.x < 4) ? trace + blockIdx.x * 264 : nullptr;
  long long* meta = tr ? tr + 256 : nullptr;  // entry, setup, tmem, mma-end, prod-end, epi-start, epi-end, epi-mid
#define TRACE_STAMP(cond, slot) \
  do {                          \
    if (cond) slot = clock64(); \
  } while (0)
#else
#define TRACE_STAMP(cond, slot) \
  do {                          \
  } while (0)
#endif
  TRACE_STAMP(meta && threadIdx.x == 0, meta[0]);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the SWIZZLE_128B atoms.
  // Offset from the __shared__ array itself (not via uintptr_t) so every
  // derived pointer keeps the shared address space: LDS/STS, not generic
  // LD/ST (which cost ~10k cycles per epilogue tile and slowed `prob` reads).
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  SmemCtl* ctl = reinterpret_cast<SmemCtl*>(smem + kStages * kStageBytes);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    ctl->item = items[blockIdx.x];
  }
  __syncthreads();
  {
    // Cooperative copy of the problem descriptor.
    const int32_t* src = reinterpret_cast<const int32_t*>(probs + ctl->item.problem);
    int32_t* dst = reinterpret_cast<int32_t*>(&ctl->prob);
    for (int i = threadIdx.x; i < int(sizeof(GemmProblem) / 4); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();

  const GemmWorkItem item = ctl->item;
  const GemmProblem& prob = ctl->prob;
  const bool same_ab = (prob.flags & FLAG_SAME_AB) != 0;
  const bool diag_shared = same_ab && item.tm == item.tn;
  const int n_iters = (item.k1 - item.k0 + kTileK - 1) / kTileK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&ctl->full[s], diag_shared ? 128 : 256);
      mbar_init(&ctl->empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ctl->tmem_full[b], 1);
      mbar_init(&ctl->tmem_empty[b], 256);
      for (int q = 0; q < kStages; ++q) mbar_init(&ctl->raw[b][q], 1);
    }
    mbar_fence_init();
  }
  TRACE_STAMP(meta && threadIdx.x == 0, meta[1]);
  if (warp == 8) tmem_alloc<kTmemCols>(&ctl->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ctl->tmem_base;
  TRACE_STAMP(meta && threadIdx.x == 0, meta[2]);
  // Programmatic dependent launch: everything above reads only the static
  // plan, so it overlaps the tail of the previous kernel; operand data is read
  // only after the prerequisite grid completed.  Let the next kernel start its
  // own prologue now.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  float* T = reinterpret_cast<float*>(smem);  // 128 x 129 fp32 epilogue tile, reuses the stage ring
  if (warp >= 8) {
    // ---------------------------------------- MMA issue (warp 8) + drain (8-15)
    // Drain warp w reads TMEM lanes 32*(w%4).. (the tcgen05 lane-access rule),
    // columns 64*((w-8)/4)..+63 of each stage's accumulator buffer into
    // round-to-nearest fp32 registers.
    const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
    const uint32_t col_base = ((warp - 8) >> 2) * 64;
    float acc[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) acc[j] = 0.f;
    auto drain = [&](int j) {
      const int b = j & 1;
      mbar_wait(&ctl->tmem_full[b], (j >> 1) & 1);
      tc_fence_after();
      TRACE_STAMP(warp == 8 && lane == 0 && tr && j < 64, tr[j * 4 + 3]);
      {
        float v[32];
        tmem_ld_32x32b_x32(tmem + lane_base + b * 128 + col_base, v);
#pragma unroll
        for (int q = 0; q < 32; ++q) acc[q] += v[q];
        tmem_ld_32x32b_x32(tmem + lane_base + b * 128 + col_base + 32, v);
#pragma unroll
        for (int q = 0; q < 32; ++q) acc[32 + q] += v[q];
      }
      tc_fence_before();
      mbar_arrive(&ctl->tmem_empty[b]);
    };
    constexpr uint32_t idesc = umma_idesc_tf32(kTileM, kTileN);
    auto issue_mma = [&](int it) {
      const int slot = it % kStages;
      const uint32_t round = it / kStages;
      const int b = it & 1;
      mbar_wait(&ctl->full[slot], round & 1);
      if (it >= 2) mbar_wait(&ctl->tmem_empty[b], ((it >> 1) + 1) & 1);
      tc_fence_after();
      TRACE_STAMP(lane == 0 && tr && it < 64, tr[it * 4 + 2]);
      if (lane == 0) {
        const uint32_t base = smem_u32(smem + slot * kStageBytes);
        const uint32_t b_hi = diag_shared ? base : base + kOperandBytes;
        const uint32_t b_lo = base + 2 * kOperandBytes;
        const uint32_t a_hi = tmem + kTmemA + slot * 64, a_lo = a_hi + 32;
        const uint32_t dt = tmem + b * 128;
#pragma unroll
        for (int kk = 0; kk < kTileK / 8; ++kk) {
          const uint32_t koff = kk * 32;  // 8 tf32 = 32 bytes along the swizzled row
          const uint64_t dbh = umma_desc_k_sw128(b_hi + koff), dbl = umma_desc_k_sw128(b_lo + koff);
          umma_tf32_ts(dt, a_lo + kk * 8, dbh, idesc, kk > 0 ? 1u : 0u);
          umma_tf32_ts(dt, a_hi + kk * 8, dbl, idesc, 1u);
          umma_tf32_ts(dt, a_hi + kk * 8, dbh, idesc, 1u);
        }
        umma_commit(&ctl->empty[slot]);
        umma_commit(&ctl->tmem_full[b]);
      }
      __syncwarp();
    };
    if (warp == 8) {
      for (int it = 0; it < n_iters; ++it) {
        issue_mma(it);
        if (it >= 1) drain(it - 1);
      }
      if (n_iters >= 1) drain(n_iters - 1);
      TRACE_STAMP(meta && lane == 0, meta[3]);
    } else {
      for (int j = 0; j < n_iters; ++j) drain(j);
    }
    // All MMAs have completed (last tmem_full), so the stage ring is free.
    asm volatile("bar.sync 1, 256;" ::: "memory");
    const int r = (warp & 3) * 32 + lane;
    float4* trow = reinterpret_cast<float4*>(T + r * kEpiStride + col_base);
#pragma unroll
    for (int j = 0; j < 16; ++j) trow[j] = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
  } else if (warp < 8) {
    // --------------------------------------------------------------- producers
    const bool is_b = warp >= 4;
    const bool produce = !(is_b && diag_shared);
    const GemmOperand& op = is_b ? prob.B : prob.A;
    const int t = threadIdx.x & 127;
    const int c = t & 7;           // cp.async: 16-byte chunk within the 128-byte row
    const int rbase = t >> 3;      // cp.async: 0..15
    const int32_t row0 = (is_b ? item.tn : item.tm) * kTileM;
    const uint32_t raw_off = is_b ? kOperandBytes : 0;
    const uint32_t blo_off = 2 * kOperandBytes;
    // Raw fp32 tiles land three stages ahead -- by TMA (one elected thread,
    // mbarrier complete_tx) when the layout allows, else by per-thread
    // cp.async.  A: each thread takes one row, writes tf32 hi/lo into TMEM
    // (lane = row) for the TS-form MMA.  B: the raw tile is the hi operand (the
    // tensor core truncates fp32 to tf32), each thread derives the lo plane
    // for its 8 16-byte chunks.
    const int32_t r0 = row0 + rbase;
    const bool tma = !kAsync || (op.mode == OP_TMA2D || op.mode == OP_TMA3D);
    const bool im2col = kAsync && op.mode == OP_IM2COL;
    const CUtensorMap* tmap = is_b ? &probs[item.problem].B.tmap : &probs[item.problem].A.tmap;
    uint64_t* raw = ctl->raw[is_b ? 1 : 0];
    KCursor cur{};
    int32_t tq = 0;  // TMA: 32-wide chunk index of the next stage
    auto issue = [&](int it) {
      const int slot = it % kStages;
      const uint32_t plane = smem_u32(smem + slot * kStageBytes + raw_off);
      if (tma) {
        if (t == 0) {
          TRACE_STAMP(tr && !is_b && it < 64, tr[it * 4 + 0]);
          mbar_expect_tx(&raw[slot], kOperandBytes);
          if (op.mode == OP_TMA2D) {
            tma_load_2d(plane, tmap, tq * kTileK, row0, &raw[slot]);
          } else {
            const int32_t seg = tq / op.cps, ch = tq - seg * op.cps;
            tma_load_3d(plane, tmap, ch * kTileK, row0, seg, &raw[slot]);
          }
        }
        ++tq;
      } else if constexpr (kAsync) {
        if (im2col) im2col_stage(op.ptr, op.geo, op.rows, row0, cur.k - 4 * c, item.k1, plane, warp & 3, lane);
        else issue_stage(op, r0, rbase, c, cur, item.k1, plane);
        cursor_advance(op, cur, kTileK);
      }
    };
    auto convert_a = [&](int it) {
      const int slot = it % kStages;
      uint8_t* stage = smem + slot * kStageBytes;
      const int r = t;  // row of the tile == TMEM lane
      float x[32], h[32];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 v = *reinterpret_cast<const float4*>(stage + raw_off + r * 128 + ((q ^ (r & 7)) << 4));
        x[4 * q] = v.x; x[4 * q + 1] = v.y; x[4 * q + 2] = v.z; x[4 * q + 3] = v.w;
      }
#pragma unroll
      for (int q = 0; q < 32; ++q) h[q] = __uint_as_float(__float_as_uint(x[q]) & 0xffffe000u);
      const uint32_t ta = tmem + (uint32_t(warp * 32) << 16) + kTmemA + slot * 64;
      tmem_st_32x32b_x32(ta, h);
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        uint32_t l;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(x[q] - h[q]));
        x[q] = __uint_as_float(l);
      }
      tmem_st_32x32b_x32(ta + 32, x);
      if (diag_shared) {  // the same rows are the B operand: lo plane in smem too
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(stage + blo_off + r * 128 + ((q ^ (r & 7)) << 4)) =
              make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
        fence_proxy_async_smem();
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&ctl->full[slot]);
    };
    auto convert_b = [&](int it) {
      const int slot = it % kStages;
      uint8_t* stage = smem + slot * kStageBytes;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int r = rbase + 16 * j;
        const uint32_t off = r * 128 + ((c ^ (r & 7)) << 4);
        const float4 x = *reinterpret_cast<const float4*>(stage + raw_off + off);
        float4 l;
        l.x = tf32_lo(x.x);
        l.y = tf32_lo(x.y);
        l.z = tf32_lo(x.z);
        l.w = tf32_lo(x.w);
        *reinterpret_cast<float4*>(stage + blo_off + off) = l;
      }
      fence_proxy_async_smem();
      mbar_arrive(&ctl->full[slot]);
    };
    if (produce) {
      if (tma) {
        tq = item.k0 / kTileK;
        if (t == 0) {
          // Descriptors live in global memory written by host copies; one-shot
          // entry points reuse pooled addresses for new descriptors, so the
          // tensormap proxy must re-acquire them (stale descriptor cache).
          asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(reinterpret_cast<uint64_t>(tmap))
                       : "memory");
          asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
        }
      } else if constexpr (kAsync) {
        cur = cursor_at(op, item.k0 + 4 * c);
      }
#pragma unroll
      for (int q = 0; q < kStages - 1; ++q) {
        if (q < n_iters) issue(q);
        if constexpr (kAsync) cp_async_commit();
      }
    }
    for (int it = 0; it < n_iters; ++it) {
      if (produce) {
        if (tma) {
          mbar_wait(&raw[it % kStages], (it / kStages) & 1);
          TRACE_STAMP(tr && !is_b && t == 0 && it < 64, tr[it * 4 + 1]);
        } else if constexpr (kAsync) {
          cp_async_wait<kStages - 2>();
          // rows span other threads' copies (A always, B when gathered by rows)
          if (!is_b) asm volatile("bar.sync 2, 128;" ::: "memory");
          else if (im2col) asm volatile("bar.sync 3, 128;" ::: "memory");
        }
        if (is_b) convert_b(it);
        else convert_a(it);
        const int nx = it + kStages - 1;
        if (nx < n_iters) {
          if (!tma || t == 0) mbar_wait(&ctl->empty[nx % kStages], ((nx / kStages) & 1) ^ 1);
          issue(nx);
        }
        if constexpr (kAsync) cp_async_commit();
      }
    }
    TRACE_STAMP(meta && threadIdx.x == 0, meta[4]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
  TRACE_STAMP(meta && threadIdx.x == 0, meta[5]);

  const int tid = threadIdx.x;
  const int nthr = blockDim.x;
  const int32_t m0 = item.tm * kTileM, n0 = item.tn * kTileN;
  // Epilogue arguments live in registers: `prob` sits in shared memory and
  // every generic global store could alias it, which made the compiler reload
  // prob fields after each store (measured 10-16k cycles per tile).
  struct {
    int32_t mode, flags, M, N;
    float alpha, beta, eta, momentum;
    float* C;
    const float* Cin;
    int64_t ldc;
    float* CT;
    int64_t ldct;
    float* W;
    float* V;
    float* P_out;
    double* norm2;
    const float* scal;
  } e{prob.mode, prob.flags, prob.M, prob.N, prob.alpha, prob.beta, prob.eta, prob.momentum, prob.C, prob.Cin,
      prob.ldc, prob.CT, prob.ldct, prob.W, prob.V, prob.P_out, prob.norm2, prob.scal};
  // Work is split in float4 chunks, 8 per thread (4096 per tile).  Row chunks
  // (r, c4) read T rows; column chunks (c, r4) read 4 rows of one column in
  // the (16 columns x 2 row-quads) lane layout.  In-bounds, aligned chunks use
  // 16-byte global accesses; ragged or masked chunks fall back to scalars.
  auto row_chunk = [&](int k, int& r, int& c) {
    const int p = tid + k * kGemmThreads;
    r = p >> 5;
    c = (p & 31) * 4;
  };
  auto col_chunk = [&](int k, int& c, int& r) {
    const int p = tid + k * kGemmThreads;
    const int wk = p >> 5, ln = p & 31;
    c = (wk & 7) * 16 + (ln & 15);
    r = ((wk >> 3) * 2 + (ln >> 4)) * 4;
  };
  auto t_col4 = [&](int r, int c) {
    return make_float4(T[r * kEpiStride + c], T[(r + 1) * kEpiStride + c], T[(r + 2) * kEpiStride + c],
                       T[(r + 3) * kEpiStride + c]);
  };
  auto aligned16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  switch (e.mode) {
    case EPI_PARTIAL: if constexpr ((kModes >> EPI_PARTIAL) & 1) {
      float4* dst = reinterpret_cast<float4*>(partials + int64_t(item.slot) * kTileM * kTileN);
#pragma unroll 4
      for (int k = 0; k < 8; ++k) {
        int r, c;
        row_chunk(k, r, c);
        dst[r * 32 + (c >> 2)] = *reinterpret_cast<const float4*>(T + r * kEpiStride + c);
      }
      break;
    }
    case EPI_PACKED: if constexpr ((kModes >> EPI_PACKED) & 1) {
      const int64_t n = e.M;
#pragma unroll 2
      for (int k = 0; k < 8; ++k) {
        int r, c;
        row_chunk(k, r, c);
        const int64_t i = m0 + r;
        if (i >= e.M) continue;
        const int64_t rb = packed_offset(n, i, i) - i;  // offset of (i, j) = rb + j
        const float4 v = *reinterpret_cast<const float4*>(T + r * kEpiStride + c);
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t jj = n0 + c + q;
          if (jj < e.N && i <= jj) e.C[rb + jj] = e.alpha * vv[q];
        }
      }
      break;
    }
    case EPI_DENSE: if constexpr ((kModes >> EPI_DENSE) & 1) {
      const bool mirror = (e.flags & FLAG_SYM_MIRROR) != 0;
      const bool has_cin = e.beta != 0.f;
      const bool vec = aligned16(e.C) && (!has_cin || aligned16(e.Cin)) && (e.ldc & 3) == 0;
#pragma unroll 1
      for (int k0 = 0; k0 < 8; k0 += 4) {
        float4 cin[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {  // Cin loads first: C and Cin may alias
          int r, c;
          row_chunk(k0 + u, r, c);
          const int64_t i = m0 + r, j = n0 + c;
          cin[u] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (!has_cin || i >= e.M) continue;
          const float* src = e.Cin + i * e.ldc + j;
          if (vec && j + 3 < e.N) {
            cin[u] = __ldg(reinterpret_cast<const float4*>(src));
          } else {
            if (j < e.N) cin[u].x = src[0];
            if (j + 1 < e.N) cin[u].y = src[1];
            if (j + 2 < e.N) cin[u].z = src[2];
            if (j + 3 < e.N) cin[u].w = src[3];
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          int r, c;
          row_chunk(k0 + u, r, c);
          const int64_t i = m0 + r, j = n0 + c;
          if (i >= e.M) continue;
          float4* tp = reinterpret_cast<float4*>(T + r * kEpiStride + c);
          float4 v = *tp;
          v.x = e.alpha * v.x + e.beta * cin[u].x;
          v.y = e.alpha * v.y + e.beta * cin[u].y;
          v.z = e.alpha * v.z + e.beta * cin[u].z;
          v.w = e.alpha * v.w + e.beta * cin[u].w;
          *tp = v;
          float* dst = e.C + i * e.ldc + j;
          if (vec && j + 3 < e.N && (!mirror || i <= j)) {
            *reinterpret_cast<float4*>(dst) = v;
          } else {
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (j + q < e.N && (!mirror || i <= j + q)) dst[q] = vv[q];
          }
        }
      }
      TRACE_STAMP(meta && tid == 0, meta[7]);
      if (mirror || (e.flags & FLAG_TRANS)) {
        __syncthreads();
        float* dstT = mirror ? e.C : e.CT;
        const int64_t ldt = mirror ? e.ldc : e.ldct;
        const bool vt = aligned16(dstT) && (ldt & 3) == 0;
#pragma unroll 2
        for (int k = 0; k < 8; ++k) {
          int c, r;
          col_chunk(k, c, r);
          const int64_t i = m0 + r, j = n0 + c;  // writes dstT[j][i .. i+3]
          if (j >= e.N) continue;
          const float4 v = t_col4(r, c);
          float* dst = dstT + j * ldt + i;
          if (vt && i + 3 < e.M && (!mirror || i + 3 < j)) {
            *reinterpret_cast<float4*>(dst) = v;
          } else {
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (i + q < e.M && (!mirror || i + q < j)) dst[q] = vv[q];
          }
        }
      }
      break;
    }
    case EPI_UPDATE: if constexpr ((kModes >> EPI_UPDATE) & 1) {
      // No parameter writes after a failed inverse / BN check (precond.cu).
      if (e.W && status && *reinterpret_cast<volatile int*>(status)) break;
      // Tile of P^T: rows = a-index (M = a), cols = g-index.  W is g x a
      // row-major, so element (i = n0+c, j = m0+r) lives at W[i*a + j]:
      // column chunks of T are contiguous in W.
      const int64_t a = e.M;
      const float eta = e.scal ? e.scal[0] : e.eta;
      const float mom = e.scal ? e.scal[1] : e.momentum;
      const bool vec = (a & 3) == 0 && (!e.W || (aligned16(e.W) && aligned16(e.V))) && (!e.P_out || aligned16(e.P_out));
      double ss = 0.0;
#pragma unroll 1
      for (int k0 = 0; k0 < 8; k0 += 4) {
        float4 w[4], vel[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {  // all loads first (W/V are also stored)
          int c, r;
          col_chunk(k0 + u, c, r);
          const int64_t j = m0 + r, i = n0 + c;
          w[u] = vel[u] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (!e.W || i >= e.N || j >= a) continue;
          const int64_t o = i * a + j;
          if (vec && j + 3 < a) {
            w[u] = __ldg(reinterpret_cast<const float4*>(e.W + o));
            vel[u] = __ldg(reinterpret_cast<const float4*>(e.V + o));
          } else {
            float* wp = &w[u].x;
            float* vp = &vel[u].x;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (j + q < a) {
                wp[q] = e.W[o + q];
                vp[q] = e.V[o + q];
              }
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          int c, r;
          col_chunk(k0 + u, c, r);
          const int64_t j = m0 + r, i = n0 + c;
          if (i >= e.N || j >= a) continue;
          const float4 t = t_col4(r, c);
          const float4 p = make_float4(e.alpha * t.x, e.alpha * t.y, e.alpha * t.z, e.alpha * t.w);
          float4 nw, nv;
          nw.x = w[u].x - eta * p.x + mom * vel[u].x;  // fisher.cpp:332
          nw.y = w[u].y - eta * p.y + mom * vel[u].y;
          nw.z = w[u].z - eta * p.z + mom * vel[u].z;
          nw.w = w[u].w - eta * p.w + mom * vel[u].w;
          nv = make_float4(nw.x - w[u].x, nw.y - w[u].y, nw.z - w[u].z, nw.w - w[u].w);  // fisher.cpp:333
          const int64_t o = i * a + j;
          const int nq = (a - j) >= 4 ? 4 : int(a - j);
          if (vec && nq == 4) {
            if (e.P_out) *reinterpret_cast<float4*>(e.P_out + o) = p;
            if (e.W) {
              *reinterpret_cast<float4*>(e.W + o) = nw;
              *reinterpret_cast<float4*>(e.V + o) = nv;
            }
          } else {
            const float pp[4] = {p.x, p.y, p.z, p.w}, ww[4] = {nw.x, nw.y, nw.z, nw.w}, vv[4] = {nv.x, nv.y, nv.z, nv.w};
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (q < nq) {
                if (e.P_out) e.P_out[o + q] = pp[q];
                if (e.W) {
                  e.W[o + q] = ww[q];
                  e.V[o + q] = vv[q];
                }
              }
          }
          if (e.W) {
            const float ww[4] = {nw.x, nw.y, nw.z, nw.w};
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (q < nq) ss += double(ww[q]) * double(ww[q]);
          }
        }
      }
      if (e.norm2) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        if (lane == 0) atomicAdd(e.norm2, ss);
      }
      break;
    }
    default:
      if (tid == 0) set_status(status, SPNGD_ERR_INVALID);
  }
#ifdef SPNGD_GEMM_TRACE_BUILD
  if (meta) {
    __syncthreads();
    if (tid == 0) meta[6] = clock64();
  }
#endif
}

// Split-K reduction: block (task, y) sums rows 16y .. 16y+15 of one tile's
// partial slots in fp64, float4 loads with four slots in flight per thread
// (the one-block-per-tile loop over slots was latency-bound: ~1 ms for the
// last wave's factors inside the step).
constexpr int kReduceRows = 16;
__global__ void __launch_bounds__(256) syrk_reduce_kernel(const SyrkReduceTask* __restrict__ tasks,
                                                          const float* __restrict__ partials) {
  const SyrkReduceTask t = tasks[blockIdx.x];
  const int64_t n = t.n;
  const int r0 = blockIdx.y * kReduceRows;
  const int64_t i_first = int64_t(t.tm) * kTileM + r0, j_last = int64_t(t.tn) * kTileN + kTileN - 1;
  if (i_first >= n || i_first > j_last) return;
  const int64_t step4 = int64_t(t.stride > 1 ? t.stride : 1) * (kTileM * kTileN / 4);
  for (int v = threadIdx.x; v < kReduceRows * (kTileN / 4); v += blockDim.x) {
    const int r = r0 + (v >> 5), c = (v & 31) * 4;
    const int64_t i = int64_t(t.tm) * kTileM + r, j = int64_t(t.tn) * kTileN + c;
    if (i >= n || j >= n || j + 3 < i) continue;
    const float4* p = reinterpret_cast<const float4*>(partials + int64_t(t.slot0) * kTileM * kTileN + r * kTileN + c);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int q = 0;
    for (; q + 4 <= t.nslots; q += 4) {
      float4 x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = __ldcs(p + (q + u) * step4);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        s0 += double(x[u].x); s1 += double(x[u].y); s2 += double(x[u].z); s3 += double(x[u].w);
      }
    }
    for (; q < t.nslots; ++q) {
      const float4 x = __ldcs(p + q * step4);
      s0 += double(x.x); s1 += double(x.y); s2 += double(x.z); s3 += double(x.w);
    }
    const double sv[4] = {s0, s1, s2, s3};
    float* out = t.packed_out + packed_offset(n, i, j);  // row i is contiguous from (i, i)
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (j + e < n && j + e >= i) out[e] = float(sv[e] * t.scale);
  }
}

}  // namespace

namespace {
PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}
}  // namespace

void make_im2col_operand(GemmOperand& op, const float* x, int c, int h, int w, int k, int stride, int pad) {
  Im2colGeo g{};
  g.c = c; g.h = h; g.w = w; g.k = k; g.stride = stride; g.pad = pad;
  g.wo = (w + 2 * pad - k) / stride + 1;
  const int ho = (h + 2 * pad - k) / stride + 1;
  g.hw = ho * g.wo;
  g.seg_pad = op.mode == OP_TMA3D ? op.cps * 32 : g.hw;  // the k order the operand had
  op.geo = g;
  op.ptr = x;
  op.mode = OP_IM2COL;
  op.vec = 0;
}

void finalize_operand(GemmOperand& op, int64_t K, bool allow_tma) {
  const uintptr_t addr = reinterpret_cast<uintptr_t>(op.ptr);
  op.vec = (addr % 16 == 0) && (op.seg_len % 4 == 0) && (op.row_stride % 4 == 0) && (op.seg_stride % 4 == 0);
  op.mode = OP_ASYNC;
  op.cps = 0;
  static const bool no_tma = getenv("SPNGD_NO_TMA") != nullptr;
  if (no_tma || !allow_tma || !op.ptr || addr % 16 != 0 || op.rows <= 0) return;
  auto encode = tma_encode_fn();
  if (!encode) return;
  const bool dense = (K < 0) || (op.seg_len >= K && op.seg_stride == 0);
  cuuint32_t box[3] = {32, 128, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r;
  if (dense) {
    if (op.row_stride % 4 != 0 || K <= 0) return;
    cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(op.rows)};
    cuuint64_t strides[1] = {cuuint64_t(op.row_stride) * 4};
    r = encode(&op.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(op.ptr), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS) op.mode = OP_TMA2D;
  } else {
    if (op.seg_len % 4 != 0 || op.row_stride % 4 != 0 || op.seg_stride % 4 != 0 || op.nseg <= 0) return;
    cuuint64_t dims[3] = {cuuint64_t(op.seg_len), cuuint64_t(op.rows), cuuint64_t(op.nseg)};
    cuuint64_t strides[2] = {cuuint64_t(op.row_stride) * 4, cuuint64_t(op.seg_stride) * 4};
    r = encode(&op.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(op.ptr), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS) {
      op.mode = OP_TMA3D;
      op.cps = int32_t((op.seg_len + 31) / 32);
    }
  }
}

size_t gemm_smem_bytes() { return size_t(kStages) * kStageBytes + sizeof(SmemCtl) + 1024; }

thread_local int g_gemm_launch_prio = 0;

uint32_t gemm_variant(const GemmProblem* probs, int n) {
  uint32_t v = 0;
  for (int i = 0; i < n; ++i) {
    v |= 1u << probs[i].mode;
    if (probs[i].A.mode == OP_ASYNC || probs[i].B.mode == OP_ASYNC || probs[i].A.mode == OP_IM2COL ||
        probs[i].B.mode == OP_IM2COL)
      v |= kVariantAsync;
  }
  return v;
}

namespace {
using GemmKernelFn = void (*)(const GemmProblem*, const GemmWorkItem*, float*, int*, long long*);

template <uint32_t kModes, bool kAsync>
GemmKernelFn gemm_instance(size_t smem, int* err) {
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(gemm_tf32x3_kernel<kModes, kAsync>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(smem)) != cudaSuccess) {
      *err = 1;
      return nullptr;
    }
    attr_set = true;
  }
  return gemm_tf32x3_kernel<kModes, kAsync>;
}

// The variants the planners produce (factor: PARTIAL|PACKED; inverse rounds
// and precondition GEMM1: DENSE; precondition GEMM2: UPDATE), each with and
// without the cp.async operand path; anything else runs the full kernel.
GemmKernelFn select_gemm(uint32_t variant, size_t smem, int* err) {
  constexpr uint32_t kPart = 1u << EPI_PARTIAL, kPack = 1u << EPI_PACKED, kDense = 1u << EPI_DENSE,
                     kUpd = 1u << EPI_UPDATE;
  const bool async = variant & kVariantAsync;
  const uint32_t modes = variant & 0xFu;
  if ((modes & ~(kPart | kPack)) == 0)
    return async ? gemm_instance<kPart | kPack, true>(smem, err) : gemm_instance<kPart | kPack, false>(smem, err);
  if (modes == kDense)
    return async ? gemm_instance<kDense, true>(smem, err) : gemm_instance<kDense, false>(smem, err);
  if (modes == kUpd) return async ? gemm_instance<kUpd, true>(smem, err) : gemm_instance<kUpd, false>(smem, err);
  return gemm_instance<0xFu, true>(smem, err);
}
}  // namespace

int launch_gemm(const GemmProblem* d_probs, const GemmWorkItem* d_items, int n_items, float* d_partials,
                int* d_status, cudaStream_t stream, uint32_t variant) {
  if (n_items <= 0) return SPNGD_OK;
  const size_t smem = gemm_smem_bytes();
  int aerr = 0;
  GemmKernelFn kern = select_gemm(variant, smem, &aerr);
  if (aerr) return fail(SPNGD_ERR_CUDA, "gemm smem attribute failed");
  static long long* trace = nullptr;
#ifdef SPNGD_GEMM_TRACE_BUILD
  static const bool want_trace = getenv("SPNGD_GEMM_TRACE") != nullptr;
#else
  constexpr bool want_trace = false;
#endif
  if (want_trace && !trace) {
    cudaMalloc(&trace, 4 * 264 * sizeof(long long));
    cudaMemset(trace, 0, 4 * 264 * sizeof(long long));
  }
  {
    // Launched with programmatic stream serialization (PDL): the kernel waits
    // on griddepcontrol.wait before touching data of earlier kernels.
    static const bool pdl = getenv("SPNGD_NO_PDL") == nullptr;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(n_items));
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    attr[1].id = cudaLaunchAttributePriority;
    attr[1].val.priority = g_gemm_launch_prio;
    cfg.attrs = attr;
    cfg.numAttrs = g_gemm_launch_prio ? 2 : 1;
    cudaError_t le = cudaLaunchKernelEx(&cfg, kern, d_probs, d_items, d_partials, d_status, trace);
    if (le != cudaSuccess) return fail(SPNGD_ERR_CUDA, "gemm launch failed: %s", cudaGetErrorString(le));
  }
  if (want_trace) {
    static int printed = 0;
    if (printed++ < 12) {
      long long h[4 * 264];
      cudaStreamSynchronize(stream);
      cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost);
      const long long* m = h + 256;

      printf("gemm launch %d items %d: setup %lld tmem %lld mainloop(mma) %lld prod %lld epi-start %lld epi-mid %lld epi-end %lld cycles\n",
             printed - 1, n_items, m[1] - m[0], m[2] - m[0], m[3] - m[0], m[4] - m[0], m[5] - m[0], m[7] ? m[7] - m[0] : -1, m[6] - m[0]);
      for (int b = 0; b < (n_items >= 4 && printed <= 2 ? 2 : 1); ++b) {
        const long long t0 = h[b * 264];
        printf("trace cta %d (cycles rel. to first TMA issue; first issue at +%lld from entry): stage issue raw full mma_done\n", b,
               h[b * 264] - h[b * 264 + 256]);
        for (int q = 0; q < 24; ++q) {
          const long long* e = h + b * 264 + q * 4;
          if (!e[0] && !e[2]) break;
          printf("  %2d %8lld %8lld %8lld %8lld\n", q, e[0] ? e[0] - t0 : -1, e[1] ? e[1] - t0 : -1,
                 e[2] ? e[2] - t0 : -1, e[3] ? e[3] - t0 : -1);
        }
      }
      cudaMemset(trace, 0, 4 * 264 * sizeof(long long));
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(kern));
    return fail(SPNGD_ERR_CUDA, "gemm launch failed: %s (regs %d, maxThreads %d, static smem %zu, dyn smem %zu)",
                cudaGetErrorString(e), fa.numRegs, fa.maxThreadsPerBlock, fa.sharedSizeBytes, smem);
  }
  return SPNGD_OK;
}

int launch_syrk_reduce(const SyrkReduceTask* d_tasks, int n_tasks, const float* d_partials, cudaStream_t stream) {
  if (n_tasks <= 0) return SPNGD_OK;
  syrk_reduce_kernel<<<dim3(unsigned(n_tasks), kTileM / kReduceRows), 256, 0, stream>>>(d_tasks, d_partials);
  SPNGD_CUDA_TRY(cudaGetLastError());
  return SPNGD_OK;
}

int plan_problem_tiles(int problem_index, const GemmProblem& p, bool upper_only, int kchunk,
                       std::vector<GemmWorkItem>& items, std::vector<SyrkReduceTask>* reduce, int* next_slot,
                       double reduce_scale, float* packed_out) {
  const int tiles_m = (p.M + kTileM - 1) / kTileM;
  const int tiles_n = (p.N + kTileN - 1) / kTileN;
  const bool whole = kchunk >= p.K;  // no split-K (callers pass K + kTileK)
  kchunk = std::max(kTileK, (kchunk / kTileK) * kTileK);
  const int nchunks = whole ? 1 : std::max(1, (p.K + kchunk - 1) / kchunk);
  int used = 0;
  struct SplitTile {
    int tm, tn, slot0;
  };
  std::vector<SplitTile> split_tiles;
  for (int tm = 0; tm < tiles_m; ++tm)
    for (int tn = upper_only ? tm : 0; tn < tiles_n; ++tn) {
      if (p.ktri) {  // triangular operands: one item over the nonzero K band
        int k0 = 0, k1 = p.K;
        if (p.ktri & KTRI_A_LOWER) k1 = std::min(k1, (tm + 1) * kTileM);
        if (p.ktri & KTRI_A_UPPER) k0 = std::max(k0, tm * kTileM);
        if (p.ktri & KTRI_B_LOWER) k1 = std::min(k1, (tn + 1) * kTileN);
        if (p.ktri & KTRI_B_UPPER) k0 = std::max(k0, tn * kTileN);
        if (k1 < k0) k1 = k0;
        items.push_back({problem_index, tm, tn, k0, k1, -1});
        continue;
      }
      if (nchunks == 1) {
        items.push_back({problem_index, tm, tn, 0, p.K, -1});
        continue;
      }
      // split-K: reserve this tile's slots now; the items are emitted below
      // chunk-major so CTAs running together share A/B panels in L2.
      const int slot0 = *next_slot;
      *next_slot += nchunks;
      used += nchunks;
      if (reduce) reduce->push_back({tm, tn, slot0, nchunks, p.M, 0, reduce_scale, packed_out});
      split_tiles.push_back({tm, tn, slot0});
    }
  for (int q = 0; q < nchunks && !split_tiles.empty(); ++q) {
    const int k0 = q * kchunk, k1 = std::min(p.K, k0 + kchunk);
    for (const auto& st : split_tiles) items.push_back({problem_index, st.tm, st.tn, k0, k1, st.slot0 + q});
  }
  return used;
}

}  // namespace spngd
