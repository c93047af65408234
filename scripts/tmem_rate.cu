// TMEM load throughput microbenchmark (not part of the product): how fast can
// W warps drain tcgen05 accumulators (tcgen05.ld 32x32b.x32) per SM?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2002_06015_b200/csrc -I include \
//        -o scripts/tmem_rate.bin scripts/tmem_rate.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#include "common.cuh"

using namespace spngd;

__device__ __forceinline__ void ld_x32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
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

// mode 0: x32 + wait per load (the factor kernel's drain); mode 1: 2 x x32 then one wait
__global__ void __launch_bounds__(512, 1) tmem_kernel(int warps, int iters, int mode, unsigned long long* out,
                                                      float* sink) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  float acc = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  if (warp < warps) {
    const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
    const uint32_t col0 = ((warp >> 2) * 64) & 511;
    for (int i = 0; i < iters; ++i) {
      const uint32_t col = (col0 + (i & 3) * 128) & 511;
      uint32_t a[32], b[32];
      if (mode == 0) {
        ld_x32_nowait(tmem + lane_base + col, a);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        ld_x32_nowait(tmem + lane_base + col + 32, b);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      } else {
        ld_x32_nowait(tmem + lane_base + col, a);
        ld_x32_nowait(tmem + lane_base + col + 32, b);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      }
#pragma unroll
      for (int q = 0; q < 32; ++q) acc += __uint_as_float(a[q]) + __uint_as_float(b[q]);
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  if (acc == 1.2345f) sink[threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, nsm * sizeof(unsigned long long));
  cudaMalloc(&sink, 512 * sizeof(float));
  const int iters = 4096;
  for (int mode = 0; mode < 2; ++mode)
    for (int w : {1, 2, 4, 8, 12, 16}) {
      for (int rep = 0; rep < 2; ++rep) tmem_kernel<<<nsm, 512>>>(w, iters, mode, d, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      unsigned long long h[256];
      cudaMemcpy(h, d, nsm * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
      const double bytes = double(w) * 32 * 64 * 4 * iters;
      printf("mode %d (%s) warps %2d: %.1f B/cycle/SM  (%llu cycles; one 128x128 fp32 drain = %.0f cycles)\n", mode,
             mode ? "2 loads, 1 wait" : "wait per load", w, bytes / double(mx), mx, 65536.0 / (bytes / double(mx)));
    }
  return 0;
}
