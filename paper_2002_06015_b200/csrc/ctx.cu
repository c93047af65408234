// Context lifecycle, error reporting and small shared host utilities.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "ctx.cuh"

namespace {
thread_local char g_last_error[1024] = "";
}

namespace spngd {

thread_local spngd_ctx* g_cur_ctx = nullptr;

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
  if (g_cur_ctx) snprintf(g_cur_ctx->last_error, sizeof(g_cur_ctx->last_error), "%s", g_last_error);
  return code;
}

int fail_cuda(cudaError_t e, const char* what) {
  return fail(SPNGD_ERR_CUDA, "CUDA error %s (%s) in %s", cudaGetErrorName(e), cudaGetErrorString(e), what);
}

int choose_kchunk(const std::vector<std::pair<int64_t, int64_t>>& tiles_and_k, int waves) {
  double work = 0;
  for (auto& tk : tiles_and_k) work += double(tk.first) * double(tk.second);
  const double target_items = double(kNumSMs) * waves;
  int64_t chunk = int64_t(work / target_items);
  chunk = std::max<int64_t>(chunk, 1024);
  chunk = (chunk + 31) / 32 * 32;
  return int(std::min<int64_t>(chunk, 1 << 30));
}

}  // namespace spngd

extern "C" {

const char* spngd_last_error(void) { return g_last_error; }
const char* spngd_ctx_last_error(const spngd_ctx* ctx) { return ctx ? ctx->last_error : ""; }
const char* spngd_version(void) { return "spngd_b200 0.1 (sm_100a, tcgen05 3xTF32)"; }

int spngd_ctx_create(int device, void* stream, spngd_ctx** out) {
  if (!out) return spngd::fail(SPNGD_ERR_INVALID, "spngd_ctx_create: out is NULL");
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return spngd::fail(SPNGD_ERR_CUDA, "spngd_ctx_create: no CUDA device (%s); there is no CPU fallback",
                       cudaGetErrorString(e));
  SPNGD_CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  SPNGD_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return spngd::fail(SPNGD_ERR_CUDA, "spngd_ctx_create: device %d is sm_%d%d, need sm_100 (B200)", device,
                       prop.major, prop.minor);
  auto* c = new spngd_ctx();
  c->device = device;
  // A private stream-ordered pool for DeviceScratch, kept cached across calls
  // (release threshold = max) without touching the device's default pool,
  // which other cudaMallocAsync users (e.g. PyTorch's async allocator) share.
  {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaError_t pe = cudaMemPoolCreate(&c->pool, &props);
    if (pe != cudaSuccess) {
      delete c;
      return spngd::fail_cuda(pe, "cudaMemPoolCreate");
    }
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  if (stream) {
    c->stream = static_cast<cudaStream_t>(stream);
  } else {
    SPNGD_CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  SPNGD_CUDA_TRY(cudaMalloc(&c->d_status, sizeof(int)));
  SPNGD_CUDA_TRY(cudaMemset(c->d_status, 0, sizeof(int)));
  SPNGD_CUDA_TRY(cudaMallocHost(&c->h_status, sizeof(int)));
  *out = c;
  return SPNGD_OK;
}

void spngd_ctx_destroy(spngd_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->d_status) cudaFree(ctx->d_status);
  if (ctx->h_status) cudaFreeHost(ctx->h_status);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  spngd::comm_destroy(ctx);
  if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
  delete ctx;
}

int spngd_copy(spngd_ctx* ctx, void* dst, const void* src, size_t bytes) {
  SPNGD_CTX_SCOPE(ctx);
  if (!ctx) return spngd::fail(SPNGD_ERR_INVALID, "spngd_copy: ctx is NULL");
  SPNGD_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream));
  return SPNGD_OK;
}

int spngd_host_alloc(void** out, size_t bytes) {
  SPNGD_CUDA_TRY(cudaMallocHost(out, bytes));
  return SPNGD_OK;
}

void spngd_host_free(void* p) { cudaFreeHost(p); }

int spngd_event_time(spngd_ctx* ctx, void** ev_pair, int record_second, float* ms) {
  SPNGD_CTX_SCOPE(ctx);
  // Harness helper: ev_pair[0] created+recorded on first call, ev_pair[1] on second.
  if (!ctx || !ev_pair) return spngd::fail(SPNGD_ERR_INVALID, "spngd_event_time: bad argument");
  cudaEvent_t* e = reinterpret_cast<cudaEvent_t*>(ev_pair);
  if (!e[0]) SPNGD_CUDA_TRY(cudaEventCreate(&e[0]));
  if (!e[1]) SPNGD_CUDA_TRY(cudaEventCreate(&e[1]));
  if (!record_second) {
    SPNGD_CUDA_TRY(cudaEventRecord(e[0], ctx->stream));
    return SPNGD_OK;
  }
  SPNGD_CUDA_TRY(cudaEventRecord(e[1], ctx->stream));
  SPNGD_CUDA_TRY(cudaEventSynchronize(e[1]));
  SPNGD_CUDA_TRY(cudaEventElapsedTime(ms, e[0], e[1]));
  return SPNGD_OK;
}

void* spngd_ctx_stream(spngd_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int spngd_ctx_sync(spngd_ctx* ctx) {
  SPNGD_CTX_SCOPE(ctx);
  if (!ctx) return spngd::fail(SPNGD_ERR_INVALID, "spngd_ctx_sync: ctx is NULL");
  SPNGD_CUDA_TRY(cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  SPNGD_CUDA_TRY(cudaMemsetAsync(ctx->d_status, 0, sizeof(int), ctx->stream));
  SPNGD_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  const int s = *ctx->h_status;
  switch (s) {
    case SPNGD_OK:
      return SPNGD_OK;
    case SPNGD_ERR_NOT_POSITIVE_DEFINITE:
      return spngd::fail(s, "spd_inverse: Cholesky/Schur pivot not positive or non-finite entries");
    case SPNGD_ERR_SINGULAR_BLOCK:
      return spngd::fail(s, "inv2x2: determinant below 1e-30");
    default:
      return spngd::fail(s, "device-side error %d", s);
  }
}

}  // extern "C"
