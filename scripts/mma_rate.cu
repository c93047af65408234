// tcgen05.mma issue-rate microbenchmark (not part of the product).
// One CTA per SM; lane 0 of warp 0 issues N back-to-back MMAs on resident
// smem/TMEM operands and waits for completion.  Reports cycles per MMA for
// kind::tf32 (SS and TS forms) and kind::f16 (SS), M=128, N in {64,128,256}.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2002_06015_b200/csrc -I include \
//        -o scripts/mma_rate.bin scripts/mma_rate.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#include "common.cuh"

using namespace spngd;

__device__ __forceinline__ void umma_f16_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__host__ __device__ constexpr uint32_t idesc_f16(uint32_t M, uint32_t N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);  // f32 D, bf16 A/B
}

// GEMM-like stage: 4 k-steps x 3 TS MMAs (lo*hi, hi*lo, hi*hi) + 3 commits,
// alternating two accumulators and 4 B slots like the factor kernel.
__device__ volatile int g_stop;
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}
__global__ void __launch_bounds__(512, 1) stage_kernel(int stages, int commits, unsigned long long* out, int bg, const float* gsrc, size_t gfloats) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar[4];
  __shared__ uint64_t tbar[4];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) {
    uint32_t h = uint32_t(i) * 2654435761u + blockIdx.x;
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    reinterpret_cast<float*>(smem)[i] = (bg & 8) ? float(h) * 2.3283064e-10f - 0.5f : 0.f;
  }
  if (threadIdx.x == 0) {
    for (int q = 0; q < 4; ++q) { mbar_init(&bar[q], 1); mbar_init(&tbar[q], 1); }
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc<512>(&tbase);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (bg & 8) {  // random A operand columns in TMEM (all 4 warps cover the 128 lanes)
    float v[32];
    for (int q = 0; q < 32; ++q) v[q] = float((threadIdx.x * 37 + q * 11) % 97) * 0.01f - 0.48f;
    const uint32_t lb = uint32_t(warp * 32) << 16;
    for (int c = 256; c < 512; c += 32) tmem_st_32x32b_x32(tmem + lb + c, v);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0 && lane == 0) {
    constexpr uint32_t idesc = umma_idesc_tf32(128, 128);
    long long t0 = clock64();
    for (int it = 0; it < stages; ++it) {
      const uint32_t bslot = smem_u32(smem + (it % 4) * 32768);
      const uint32_t b_hi = bslot, b_lo = bslot + 16384;
      const uint32_t a_hi = tmem + 256 + (it % 4) * 64, a_lo = a_hi + 32;
      const uint32_t dt = tmem + (it & 1) * 128;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t dbh = umma_desc_k_sw128(b_hi + kk * 32), dbl = umma_desc_k_sw128(b_lo + kk * 32);
        umma_tf32_ts(dt, a_lo + kk * 8, dbh, idesc, kk > 0 ? 1u : 0u);
        umma_tf32_ts(dt, a_hi + kk * 8, dbl, idesc, 1u);
        umma_tf32_ts(dt, a_hi + kk * 8, dbh, idesc, 1u);
      }
      if (commits > 0) umma_commit(&bar[0]);
      if (commits > 1) umma_commit(&bar[1]);
      if (commits > 2) umma_commit(&bar[2]);
    }
    long long t1 = clock64();
    umma_commit(&bar[3]);
    mbar_wait(&bar[3], 0);
    long long t2 = clock64();
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = t2 - t0;
  }
  if (warp >= 1 && warp <= 2 && (bg & 16)) {  // heavy TMA: 2 issuers, 16 KB copies, 4-deep each, L2-resident source
    if (lane == 0) {
      long long tend = clock64() + (long long)stages * 800;
      size_t off = size_t(blockIdx.x * 2 + warp) * 4096 * 37;
      unsigned long long bytes = 0;
      uint64_t* tb = &tbar[(warp - 1) * 2];
      for (int i = 0; clock64() < tend; ++i) {
        const int s = i & 1;
        if (i >= 2) mbar_wait(&tb[s], ((i >> 1) - 1) & 1);
        mbar_expect_tx(&tb[s], 16384);
        bulk_g2s(smem_u32(smem + 131072 + ((warp - 1) * 2 + s) * 16384 - (bg & 128 ? 0 : 65536)), gsrc + (off % (gfloats - 4096)), 16384, &tb[s]);
        off += 4096 * 149;
        bytes += 16384;
      }
      out[2 * 4096 + blockIdx.x * 2 + (warp - 1)] = bytes;
    }
  } else if (warp >= 4 && (warp & 3) == 0 && (bg & 32)) {  // ALU-busy warps on the MMA warp's SMSP
    long long tend = clock64() + (long long)stages * 800;
    float a0 = threadIdx.x, a1 = 1.f, a2 = 2.f, a3 = 3.f;
    while (clock64() < tend) {
#pragma unroll 16
      for (int q = 0; q < 64; ++q) { a0 = fmaf(a0, 1.0001f, a1); a1 = fmaf(a1, 0.9999f, a2); a2 = fmaf(a2, 1.0001f, a3); a3 = fmaf(a3, 0.9999f, a0); }
    }
    if (a0 + a1 + a2 + a3 == 1.2345f) out[0] = 0;
  } else if (warp >= 4 && (warp & 3) == 0 && (bg & 64)) {  // spinning mbarrier waiters on the MMA warp's SMSP
    long long tend = clock64() + (long long)stages * 800;
    while (clock64() < tend) { mbar_wait(&bar[2], 1); }
  } else if (warp > 0 && warp < 4 && (bg & 7)) {
    // background load for ~ the MMA duration: bg bit 1 STTM, 2 LDTM, 4 LDS/STS
    float v[32];
    for (int q = 0; q < 32; ++q) v[q] = float(q);
    const uint32_t lb = uint32_t(warp * 32) << 16;
    long long tend = clock64() + (long long)stages * 800;
    float sink = 0.f;
    float* sm = reinterpret_cast<float*>(smem) + 40960 / 4 * 0;
    while (clock64() < tend) {
      if (bg & 1) { tmem_st_32x32b_x32(tmem + lb + 384, v); tmem_wait_st(); }
      if (bg & 2) { float w[32]; tmem_ld_32x32b_x32(tmem + lb + 128, w); for (int q = 0; q < 32; ++q) sink += w[q]; }
      if (bg & 4) {
        for (int q = 0; q < 8; ++q) {
          float4 x = reinterpret_cast<float4*>(sm)[(threadIdx.x + q * 128) & 4095];
          reinterpret_cast<float4*>(sm)[((threadIdx.x + q * 128) & 4095) + 4096] = x;
          sink += x.x;
        }
      }
    }
    if (sink == 12345.f) out[0] = 0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int KIND, int N>  // KIND 0 tf32 SS, 1 tf32 TS, 2 bf16 SS
__global__ void __launch_bounds__(128, 1) rate_kernel(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc<512>(&tbase);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp == 0 && lane == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const uint64_t da = umma_desc_k_sw128(a), db = umma_desc_k_sw128(b);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (KIND == 0) umma_tf32(tmem, da, db, umma_idesc_tf32(128, N), i > 0);
      if (KIND == 1) umma_tf32_ts(tmem, tmem + 256, db, umma_idesc_tf32(128, N), i > 0);
      if (KIND == 2) umma_f16_ss(tmem, da, db, idesc_f16(128, N), i > 0);
    }
    long long t1 = clock64();
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = t2 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int KIND, int N>
void run(const char* name, int nsm) {
  unsigned long long* d;
  cudaMalloc(&d, nsm * 16);
  auto k = rate_kernel<KIND, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  const int iters = 4096;
  for (int rep = 0; rep < 2; ++rep) k<<<nsm, 128, 66 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(e));
    return;
  }
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double kdim = KIND == 2 ? 16 : 8;
  const double flops = 2.0 * 128 * N * kdim;
  printf("%-10s N=%3d: issue %.1f cyc/MMA, complete %.1f cyc/MMA -> %.0f flop/cyc/SM (%d SMs)\n", name, N,
         double(h[0]) / iters, double(h[1]) / iters, flops * iters / double(h[1]), nsm);
  cudaFree(d);
}

void run_stage(int commits, int nsm, int bg = 0) {
  unsigned long long* d;
  static float* g = nullptr;
  const size_t gf = size_t(1) << 22;
  if (!g) { cudaMalloc(&g, gf * 4); cudaMemset(g, 0, gf * 4); }
  cudaMalloc(&d, nsm * 16);
  cudaFuncSetAttribute(stage_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 161 * 1024);
  const int stages = 20000;
  for (int rep = 0; rep < 2; ++rep) stage_kernel<<<nsm, 512, 161 * 1024>>>(stages, commits, d, bg, g, gf);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("stage: %s\n", cudaGetErrorString(e)); return; }
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  unsigned long long tb[2];
  cudaMemcpy(tb, d + 2 * 4096, 16, cudaMemcpyDeviceToHost);
  printf("gemm-like stage (12 TS MMAs, %d commits, bg %d): issue %.0f cyc/stage, complete %.0f cyc/stage (%d SMs); TMA %.1f B/cyc\n", commits, bg,
         double(h[0]) / stages, double(h[1]) / stages, nsm, double(tb[0] + tb[1]) / double(h[1]));
  cudaMemset(d, 0, 4096 * 16 * 4);
  cudaFree(d);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int bg : {0, 16, 16 | 128, 16 | 8}) run_stage(3, nsm, bg);
  return 0;
  for (int g : {1, 0}) {
    const int n = g ? 1 : nsm;
    printf("--- grid %d\n", n);
    run<0, 64>("tf32 SS", n);
    run<0, 128>("tf32 SS", n);
    run<0, 256>("tf32 SS", n);
    run<1, 64>("tf32 TS", n);
    run<1, 128>("tf32 TS", n);
    run<1, 256>("tf32 TS", n);
    run<2, 128>("bf16 SS", n);
    run<2, 256>("bf16 SS", n);
  }
  return 0;
}
