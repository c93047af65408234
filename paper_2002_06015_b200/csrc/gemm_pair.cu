// sm_100a 2-CTA (cta_group::2) 3xTF32 SYRK for the factor construction.
//
// A CTA pair (cluster of 2 on one TPC) computes two vertically adjacent
// 128x128 output tiles (rows tm, tm+1) of the same column tile tn with one
// M=256 tcgen05.mma per product: each CTA keeps its own 128 A rows (tf32
// hi/lo in its TMEM, TS form) and loads only HALF of the shared B tile (64
// rows) into its smem; the pair's tensor cores read both halves.  Per CTA and
// 32-deep stage the loads drop from 32 KB (A 16 + B 16) to 24 KB (A 16 + B 8)
// for the same MMA work, and the smem ring deepens from 4 to 6 stages -- the
// single-CTA kernel is bound by operand delivery per SM.
//
// Status: correct (tests/test_gpu_kernels.py factor cases pass with it) but
// measured SLOWER than the single-CTA kernel on ResNet-50 (10.0 vs 7.7 ms;
// 3 accumulator buffers / 2 A slots: 10.8 ms) -- every stage waits on the
// slower CTA of the pair plus remote-arrive latency, and sub-diagonal pair
// partners add ~15% tiles.  Opt-in with SPNGD_PAIR=1 until that is fixed.
//
// Roles per CTA (512 threads): warps 0-3 A (TMA + split into TMEM), warps
// 4-6 B half (TMA + lo plane), warp 7 MMA issue (leader), warps 8-15 drain (per-stage double-buffered
// TMEM accumulators into round-to-nearest fp32 registers, as in the single-CTA
// kernel, so the RZ accumulation bias stays bounded by one stage).  Synchronisation across the pair: each
// group of the peer signals the leader's `full` barrier with one remote
// mbarrier arrive; the leader's commits are multicast to both CTAs' `empty`,
// TMEM-slot and `tmem_full` barriers; drain warps of both CTAs arrive on the
// leader's `tmem_empty`.  Epilogues (packed / split-K partial) are per CTA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "gemm_tf32x3.cuh"

namespace spngd {

namespace {

constexpr int kPS = 6;                          // smem ring stages
constexpr int kPASlots = 4;                     // TMEM A hi|lo slots (64 columns each)
constexpr int kPAcc = 2;                        // TMEM accumulator buffers (128 columns each)
constexpr int kPABytes = kTileM * kTileK * 4;   // 16 KB: 128 A rows x 32 k
constexpr int kPBBytes = 64 * kTileK * 4;       // 8 KB: 64 B rows x 32 k (this CTA's half)
constexpr int kPStage = kPABytes + 2 * kPBBytes;  // A raw | B raw (hi) | B lo
constexpr int kPEpi = kTileN + 4;               // epilogue tile row stride (floats)
constexpr uint32_t kPTmemA = kPAcc * 128;
constexpr int kPEpiThreads = 512;               // all 16 warps share the epilogue

struct __align__(64) PairCtl {
  uint64_t raw_a[kPS];
  uint64_t raw_b[kPS];
  uint64_t full[kPS];        // leader: 4 arrivals (A, B groups of both CTAs)
  uint64_t empty[kPS];       // multicast commit: B raw/lo slot free
  uint64_t ta_empty[kPASlots];
  uint64_t tmem_full[kPAcc];
  uint64_t tmem_empty[kPAcc];  // leader: 16 drain-warp arrivals (8 per CTA)
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
      "{\n.reg .pred p;\nWAITC: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Arrive on the leader's barrier (local when this CTA is the leader).
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
__device__ __forceinline__ void umma_pair_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
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
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma3d(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1, int32_t c2,
                                      uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void load_tile(const GemmOperand& op, const CUtensorMap* map, uint32_t dst, int32_t tq,
                                          int32_t row0, uint64_t* bar, uint32_t bytes) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  expect_tx(bar, bytes);
  if (op.mode == OP_TMA2D) {
    tma2d(dst, map, tq * kTileK, row0, bar);
  } else {
    const int32_t seg = tq / op.cps, ch = tq - seg * op.cps;
    tma3d(dst, map, ch * kTileK, row0, seg, bar);
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    gemm_pair_kernel(const GemmProblem* __restrict__ probs, const CUtensorMap* __restrict__ halfmaps,
                     const GemmWorkItem* __restrict__ items, float* __restrict__ partials) {
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
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPS; ++s) {
      mbar_init(&ctl->raw_a[s], 1);
      mbar_init(&ctl->raw_b[s], 1);
      mbar_init(&ctl->full[s], 4);
      mbar_init(&ctl->empty[s], 1);
    }
    for (int s = 0; s < kPASlots; ++s) mbar_init(&ctl->ta_empty[s], 1);
    for (int b = 0; b < kPAcc; ++b) {
      mbar_init(&ctl->tmem_full[b], 1);
      mbar_init(&ctl->tmem_empty[b], 16);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == 8) tmem_alloc_pair(&ctl->tmem_base);
  tc_fence_before();
  cluster_sync_all();  // both CTAs' barriers and the pair's TMEM exist before any remote use
  tc_fence_after();
  const uint32_t tmem = ctl->tmem_base;
  const GemmWorkItem item = ctl->item;
  const GemmProblem& prob = ctl->prob;
  const int n_iters = (item.k1 - item.k0 + kTileK - 1) / kTileK;
  float* T = reinterpret_cast<float*>(smem);

  if (warp == 7) {
    // ------------------------------------------------ MMA issue (leader CTA, one lane)
    if (leader) {
    constexpr uint32_t idesc = umma_idesc_tf32(2 * kTileM, kTileN);  // M = 256 across the pair
      auto issue_mma = [&](int it) {
        const int s = it % kPS, sa = it % kPASlots, b = it % kPAcc;
        mbar_wait_cluster(&ctl->full[s], (it / kPS) & 1);
        if (it >= kPAcc) mbar_wait_cluster(&ctl->tmem_empty[b], ((it / kPAcc) + 1) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t base = smem_u32(smem + s * kPStage);
          const uint32_t b_hi = base + kPABytes, b_lo = b_hi + kPBBytes;
          const uint32_t a_hi = tmem + kPTmemA + sa * 64, a_lo = a_hi + 32;
          const uint32_t dt = tmem + b * 128;
#pragma unroll
          for (int kk = 0; kk < kTileK / 8; ++kk) {
            const uint32_t koff = kk * 32;
            const uint64_t dbh = umma_desc_k_sw128(b_hi + koff), dbl = umma_desc_k_sw128(b_lo + koff);
            umma_pair_ts(dt, a_lo + kk * 8, dbh, idesc, kk > 0 ? 1u : 0u);
            umma_pair_ts(dt, a_hi + kk * 8, dbl, idesc, 1u);
            umma_pair_ts(dt, a_hi + kk * 8, dbh, idesc, 1u);
          }
          commit_pair(&ctl->empty[s]);
          commit_pair(&ctl->ta_empty[sa]);
          commit_pair(&ctl->tmem_full[b]);
        }
        __syncwarp();
      };
      for (int it = 0; it < n_iters; ++it) issue_mma(it);
    }
  } else if (warp >= 8) {
    // ------------------------------------------------ drain (8-15)
    const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
    const uint32_t col_base = ((warp - 8) >> 2) * 64;
    float acc[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) acc[j] = 0.f;
    auto drain = [&](int j) {
      const int b = j % kPAcc;
      mbar_wait(&ctl->tmem_full[b], (j / kPAcc) & 1);
      tc_fence_after();
#pragma unroll
      for (int h = 0; h < 4; ++h) {  // 16 columns at a time keeps the drain inside 128 registers
        float v[16];
        tmem_ld_32x32b_x16(tmem + lane_base + b * 128 + col_base + 16 * h, v);
#pragma unroll
        for (int q = 0; q < 16; ++q) acc[16 * h + q] += v[q];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_leader(&ctl->tmem_empty[b], leader);
    };
    for (int j = 0; j < n_iters; ++j) drain(j);
    asm volatile("bar.sync 1, 256;" ::: "memory");
    const int r = (warp & 3) * 32 + lane;
    float4* trow = reinterpret_cast<float4*>(T + r * kPEpi + col_base);
#pragma unroll
    for (int j = 0; j < 16; ++j) trow[j] = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
  } else {
    // ------------------------------------------------------------ producers
    const bool is_b = warp >= 4;  // B half: warps 4-6 (96 threads); warp 7 issues MMAs
    const int t = is_b ? threadIdx.x - 128 : threadIdx.x;
    const GemmOperand& op = is_b ? prob.B : prob.A;
    const CUtensorMap* map = is_b ? halfmaps + item.problem : &probs[item.problem].A.tmap;
    const int32_t row0 = is_b ? item.tn * kTileN + int32_t(rank) * 64 : item.tm * kTileM;
    const uint32_t off = is_b ? kPABytes : 0;
    const uint32_t bytes = is_b ? kPBBytes : kPABytes;
    uint64_t* raw = is_b ? ctl->raw_b : ctl->raw_a;
    const int32_t tq0 = item.k0 / kTileK;
    if (t == 0) {
      asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(reinterpret_cast<uint64_t>(map))
                   : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
      // A slots free up after conversion, B slots after the MMA: prefill the whole ring
      // with A, all but one stage with B (its refill trails the MMA by one stage).
      const int pre = is_b ? kPS - 1 : kPS;
      for (int q = 0; q < pre && q < n_iters; ++q)
        load_tile(op, map, smem_u32(smem + q * kPStage + off), tq0 + q, row0, &raw[q], bytes);
    }
    for (int it = 0; it < n_iters; ++it) {
      const int s = it % kPS;
      uint8_t* stage = smem + s * kPStage;
      mbar_wait(&raw[s], (it / kPS) & 1);
      if (!is_b) {
        const int sa = it % kPASlots;
        if (it >= kPASlots) mbar_wait(&ctl->ta_empty[sa], ((it / kPASlots) & 1) ^ 1);
        tc_fence_after();
        const int rr = t;
        float x[32], h[32];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 v = *reinterpret_cast<const float4*>(stage + rr * 128 + ((q ^ (rr & 7)) << 4));
          x[4 * q] = v.x; x[4 * q + 1] = v.y; x[4 * q + 2] = v.z; x[4 * q + 3] = v.w;
        }
#pragma unroll
        for (int q = 0; q < 32; ++q) h[q] = __uint_as_float(__float_as_uint(x[q]) & 0xffffe000u);
        const uint32_t ta = tmem + (uint32_t(warp * 32) << 16) + kPTmemA + sa * 64;
        tmem_st_32x32b_x32(ta, h);
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          uint32_t l;
          asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(x[q] - h[q]));
          x[q] = __uint_as_float(l);
        }
        tmem_st_32x32b_x32(ta + 32, x);
        tmem_wait_st();
        tc_fence_before();
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (t == 0) {
          arrive_leader(&ctl->full[s], leader);
          if (it + kPS < n_iters)  // the raw A slot is consumed: refill kPS stages ahead
            load_tile(op, map, smem_u32(stage + off), tq0 + it + kPS, row0, &raw[s], bytes);
        }
      } else {
        // lo plane of this CTA's 64 B rows: 512 16-byte chunks over 96 threads
        for (int idx = t; idx < 512; idx += 96) {
          const int r = idx >> 3, c = idx & 7;
          const uint32_t o = r * 128 + ((c ^ (r & 7)) << 4);
          const float4 xv = *reinterpret_cast<const float4*>(stage + kPABytes + o);
          float4 l;
          l.x = tf32_lo(xv.x);
          l.y = tf32_lo(xv.y);
          l.z = tf32_lo(xv.z);
          l.w = tf32_lo(xv.w);
          *reinterpret_cast<float4*>(stage + kPABytes + kPBBytes + o) = l;
        }
        fence_proxy_async_smem();
        asm volatile("bar.sync 3, 96;" ::: "memory");
        if (t == 0) {
          arrive_leader(&ctl->full[s], leader);
          const int nx = it + kPS - 1;  // refill the slot the MMA of stage it-1 released (fresh at it = 0)
          if (nx < n_iters) {
            const int ps = nx % kPS;
            mbar_wait(&ctl->empty[ps], ((nx / kPS) & 1) ^ 1);
            load_tile(op, map, smem_u32(smem + ps * kPStage + off), tq0 + nx, row0, &raw[ps], bytes);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the pair's MMAs, commits and remote arrivals are all done
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc_pair(tmem);
  }

  // ------------------------------------------------------------ epilogue (per CTA tile)
  const int tid = threadIdx.x;
  const int32_t m0 = item.tm * kTileM, n0 = item.tn * kTileN;
  if (prob.mode == EPI_PARTIAL) {
    if (item.slot < 0) return;  // pair partner below the diagonal: nothing to keep
    float4* dst = reinterpret_cast<float4*>(partials + int64_t(item.slot) * kTileM * kTileN);
#pragma unroll 4
    for (int k = 0; k < 8; ++k) {
      const int p = tid + k * kPEpiThreads;
      const int r = p >> 5, c = (p & 31) * 4;
      dst[r * 32 + (c >> 2)] = *reinterpret_cast<const float4*>(T + r * kPEpi + c);
    }
  } else {  // EPI_PACKED
    float* C = prob.C;
    const int64_t n = prob.M;
    const float alpha = prob.alpha;
    for (int k = 0; k < 8; ++k) {
      const int p = tid + k * kPEpiThreads;
      const int r = p >> 5, c = (p & 31) * 4;
      const int64_t i = m0 + r;
      if (i >= n) continue;
      const int64_t rb = packed_offset(n, i, i) - i;
      const float4 v = *reinterpret_cast<const float4*>(T + r * kPEpi + c);
      const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t jj = n0 + c + q;
        if (jj < n && i <= jj) C[rb + jj] = alpha * vv[q];
      }
    }
  }
}

}  // namespace

size_t gemm_pair_smem_bytes() { return size_t(kPS) * kPStage + sizeof(PairCtl) + 1024; }

int encode_half_map(const GemmOperand& op, int64_t K, CUtensorMap* out);  // gemm_tf32x3.cu

int launch_gemm_pair(const GemmProblem* d_probs, const CUtensorMap* d_halfmaps, const GemmWorkItem* d_items,
                     int n_items, float* d_partials, cudaStream_t stream) {
  if (n_items <= 0) return SPNGD_OK;
  static bool attr_set = false;
  const size_t smem = gemm_pair_smem_bytes();
  if (!attr_set) {
    SPNGD_CUDA_TRY(cudaFuncSetAttribute(gemm_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr_set = true;
  }
  gemm_pair_kernel<<<n_items, kGemmThreads, smem, stream>>>(d_probs, d_halfmaps, d_items, d_partials);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SPNGD_ERR_CUDA, "gemm_pair launch failed: %s", cudaGetErrorString(e));
  return SPNGD_OK;
}

}  // namespace spngd
