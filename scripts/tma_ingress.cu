// Per-SM TMA ingress microbenchmark (not part of the product).
// One CTA per SM streams boxes from a global fp32 matrix into a smem ring and
// reports bytes/cycle/SM for several box shapes and in-flight depths.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_ingress scripts/tma_ingress.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)),
               "r"(bytes));
}
__device__ int g_waitkind;
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  if (g_waitkind == 1) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(ok) : "r"((uint32_t)__cvta_generic_to_shared(b)), "r"(ph) : "memory");
    return;
  }
  if (g_waitkind == 2) {
    asm volatile(
        "{\n.reg .pred p;\nW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n@!p bra W2;\n}\n" ::"r"(
            (uint32_t)__cvta_generic_to_shared(b)),
        "r"(ph), "r"(20));
    return;
  }
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
          (uint32_t)__cvta_generic_to_shared(b)),
      "r"(ph));
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"((uint32_t)__cvta_generic_to_shared(b))
      : "memory");
}
__device__ __forceinline__ void bulk1d(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(b))
               : "memory");
}

// mode 0: 2D tensor box {bw, br}; mode 1: 1D bulk copy of box bytes.
__global__ void __launch_bounds__(128) stream_kernel(const __grid_constant__ CUtensorMap m, const float* src,
                                                    int rows, int cols, int bw, int br, int depth, int iters,
                                                    int mode, int per, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[16];
  const uint32_t box = uint32_t(bw) * br * 4;
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) mbar_init(&bar[i], mode == 2 ? 128 : 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (mode == 2) {  // LDGSTS: 128 threads, 16 B each per op, arrive via cp.async.mbarrier.arrive
    const size_t total = size_t(rows) * cols * 4;
    long long t0 = clock64();
    for (int it = 0; it < iters + depth; ++it) {
      if (it < iters) {
        const int s = it % depth;
        if (it >= depth) mbar_wait(&bar[s], ((it - depth) / depth) & 1);
        const size_t base = (size_t(blockIdx.x) * 7919 + size_t(it) * 131) * box % total;
        const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem + size_t(s) * box);
        for (uint32_t o = threadIdx.x * 16; o < box; o += 128 * 16)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + o),
                       "l"(reinterpret_cast<const uint8_t*>(src) + (base + o) % total));
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&bar[s])));
      }
    }
    for (int it = iters - depth; it < iters; ++it) mbar_wait(&bar[it % depth], (it / depth) & 1);
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    return;
  }
  if (threadIdx.x != 0) return;
  const int tiles_c = cols / bw, tiles_r = rows / br;
  const int ntile = tiles_c * tiles_r;
  auto issue = [&](int it) {
    const int s = it % depth;
    const int t = (blockIdx.x * 7919 + it * 131) % ntile;
    const int tr = t / tiles_c, tc = t % tiles_c;
    mbar_expect(&bar[s], box);
    if (mode == 0 && per > 1) {
      for (int p = 0; p < per; ++p)
        tma2d(smem + size_t(s) * box + size_t(p) * (box / per), &m, tc * bw, tr * br + p * (br / per), &bar[s]);
    } else if (mode == 0)
      tma2d(smem + size_t(s) * box, &m, tc * bw, tr * br, &bar[s]);
    else
      bulk1d(smem + size_t(s) * box, reinterpret_cast<const uint8_t*>(src) + (size_t(t) * box) % (size_t(rows) * cols * 4),
             box, &bar[s]);
  };
  for (int i = 0; i < depth && i < iters; ++i) issue(i);
  long long t0 = clock64();
  unsigned long long bad = 0;
  for (int it = 0; it < iters; ++it) {
    mbar_wait(&bar[it % depth], (it / depth) & 1);
    if (mode == 1) {  // first word of the box must equal src at the box origin
      const int t = (blockIdx.x * 7919 + it * 131) % ntile;
      const size_t off = (size_t(t) * box) % (size_t(rows) * cols * 4);
      const float want = *reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(src) + off);
      const float got = *reinterpret_cast<const float*>(smem + size_t(it % depth) * box);
      bad += (want != got);
    }
    if (it + depth < iters) issue(it + depth);
  }
  long long t1 = clock64();
  cyc[blockIdx.x] = (t1 - t0) | (bad << 48);
}

__global__ void fill(float* p, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    uint32_t h = uint32_t(i) * 2654435761u ^ uint32_t(i >> 32) * 40503u;
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    p[i] = float(h) * 2.3283064e-10f - 0.5f;
  }
}

int main() {
  typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  Enc enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* cyc;
  cudaMalloc(&cyc, nsm * 8);
  struct Cfg { int rows, cols, bw, br, depth, mode, sw; const char* what; int per; };
  std::vector<Cfg> cfgs;
  for (int big = 0; big < 2; ++big) {
    int rows = big ? 32768 : 4096, cols = big ? 8192 : 1024;
    for (int depth : {2, 4, 6}) {
      cfgs.push_back({rows, cols, 32, 64, depth, 0, 3, "2d 32x64 (8KB)", 1});
      cfgs.push_back({rows, cols, 32, 128, depth, 0, 3, "2d 32x128 (16KB)", 1});
      cfgs.push_back({rows, cols, 32, 256, depth, 0, 3, "2d 32x256 (32KB)", 1});
      cfgs.push_back({rows, cols, 32, 256, depth, 0, 3, "2x 2d 32x128 /bar", 2});
      cfgs.push_back({rows, cols, 32, 256, depth, 0, 3, "4x 2d 32x64 /bar", 4});
      cfgs.push_back({rows, cols, 128, 128, depth, 1, 0, "bulk1d 64KB", 1});
      // wide-row boxes (no swizzle): does the per-row request rate bound ingress?
      cfgs.push_back({rows, cols, 64, 128, depth, 0, 0, "2d 64x128 noswz (32KB)", 1});
      cfgs.push_back({rows, cols, 128, 64, depth, 0, 0, "2d 128x64 noswz (32KB)", 1});
      cfgs.push_back({rows, cols, 256, 32, depth, 0, 0, "2d 256x32 noswz (32KB)", 1});
      cfgs.push_back({rows, cols, 32, 256, depth, 0, 0, "2d 32x256 noswz (32KB)", 1});
      cfgs.push_back({rows, cols, 128, 32, depth, 1, 0, "bulk1d 16KB", 1});
      cfgs.push_back({rows, cols, 32, 128, depth, 2, 0, "ldgsts 16KB", 1});
      cfgs.push_back({rows, cols, 32, 256, depth, 2, 0, "ldgsts 32KB", 1});
    }
  }
  float* src;
  cudaMalloc(&src, size_t(32768) * 8192 * 4);
  fill<<<1184, 256>>>(src, size_t(32768) * 8192);
  for (int wk = 0; wk < 3; ++wk) {
  cudaMemcpyToSymbol(g_waitkind, &wk, 4);
  printf("=== wait kind %d (0 try_wait, 1 test_wait spin, 2 try_wait hint 20ns)\n", wk);
  for (auto& c : cfgs) {
    if (c.depth == 6) continue;
    CUtensorMap m;
    cuuint64_t dims[2] = {cuuint64_t(c.cols), cuuint64_t(c.rows)};
    cuuint64_t strides[1] = {cuuint64_t(c.cols) * 4};
    cuuint32_t box[2] = {cuuint32_t(c.bw), cuuint32_t(c.br / c.per)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     c.sw == 3 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS && c.mode == 0) { printf("%s encode failed %d\n", c.what, r); continue; }
    size_t smem = size_t(c.bw) * c.br * 4 * c.depth;
    if (smem > 200 * 1024) continue;
    if (cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess) { printf("attr failed\n"); return 1; }
    const int iters = 400;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      if (rep == 1) cudaEventRecord(e0);
      stream_kernel<<<nsm, 128, smem>>>(m, src, c.rows, c.cols, c.bw, c.br, c.depth, iters, c.mode, c.per, cyc);
    }
    cudaEventRecord(e1);
    if (cudaGetLastError() != cudaSuccess) { printf("%s: launch failed\n", c.what); return 1; }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", c.what, cudaGetErrorString(e)); return 1; }
    std::vector<unsigned long long> h(nsm);
    cudaMemcpy(h.data(), cyc, nsm * 8, cudaMemcpyDeviceToHost);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    double mean = 0, mx = 0;
    unsigned long long nbad = 0;
    for (auto& v : h) { nbad += v >> 48; v &= (1ull << 48) - 1; }
    for (auto v : h) { mean += double(v) / nsm; mx = v > mx ? v : mx; }
    double bytes = double(c.bw) * c.br * 4 * iters;
    printf("%-5s %-20s depth %d inflight %3zu KB: %6.1f B/cyc/SM (mean)  %6.1f (slowest)  lat~%6.0f cyc/box*depth\n", c.rows > 4096 ? "DRAM" : "L2", c.what,
           c.depth, smem / 1024, bytes / mean, bytes / mx, mean / iters * c.depth);
    printf("      event %.3f ms -> %.1f GB/s chip, %.0f MHz implied, bad %llu\n", ms, bytes * nsm / ms / 1e6, mx / ms / 1e3, nbad);
  }
  }
  return 0;
}
