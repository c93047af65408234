// Context, device workspace and descriptor upload helpers.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <string>
#include <vector>

#include "common.cuh"
#include "spngd_b200.h"

struct ncclComm;

struct spngd_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int* d_status = nullptr;      // device-side error word
  int* h_status = nullptr;      // pinned mirror
  ncclComm* comm = nullptr;
  int world = 1, rank = 0;
  int64_t launches = 0;         // kernels launched through this context
  int launch_prio = 0;          // != 0: cudaLaunchAttributePriority of the recursion kernels
  cudaMemPool_t pool = nullptr; // private stream-ordered pool of DeviceScratch (kept cached)
  char last_error[1024] = "";   // spngd_ctx_last_error: the last failure of a call on this context
};

namespace spngd {

// The context of the ABI call running on this thread: fail() also records the
// message there (spngd_ctx_last_error).
extern thread_local spngd_ctx* g_cur_ctx;
struct CtxScope {
  spngd_ctx* prev;
  explicit CtxScope(spngd_ctx* c) : prev(g_cur_ctx) { g_cur_ctx = c ? c : prev; }
  ~CtxScope() { g_cur_ctx = prev; }
};
#define SPNGD_CTX_SCOPE(c) ::spngd::CtxScope spngd_ctx_scope_(c)

// Stream-ordered scratch buffer from the context's private pool, released at scope exit.
class DeviceScratch {
 public:
  DeviceScratch(spngd_ctx* ctx) : ctx_(ctx) {}
  ~DeviceScratch() {
    for (void* p : ptrs_) cudaFreeAsync(p, ctx_->stream);
  }
  template <typename T>
  T* alloc(size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    if (cudaMallocFromPoolAsync(&p, count * sizeof(T), ctx_->pool, ctx_->stream) != cudaSuccess) return nullptr;
    static const bool poison = getenv("SPNGD_POISON_SCRATCH") != nullptr;  // debug: NaN-fill fresh scratch
    if (poison) cudaMemsetAsync(p, 0xff, count * sizeof(T), ctx_->stream);
    ptrs_.push_back(p);
    return static_cast<T*>(p);
  }
  template <typename T>
  T* upload(const std::vector<T>& v) {
    T* d = alloc<T>(v.size());
    if (d && !v.empty()) cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, ctx_->stream);
    return d;
  }

 private:
  spngd_ctx* ctx_;
  std::vector<void*> ptrs_;
};

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// Chooses the split-K chunk so a grouped launch has ~`waves` work items per SM.
void comm_destroy(spngd_ctx* ctx);  // comm.cu
struct OwnerReduce {
  const float* send;
  float* recv;
  int64_t count;
  int root;
};
int comm_reduce_to_owners(spngd_ctx* ctx, const std::vector<OwnerReduce>& ops);  // comm.cu
int comm_allreduce_sum_f64(spngd_ctx* ctx, double* buf, int64_t count);        // comm.cu

int choose_kchunk(const std::vector<std::pair<int64_t, int64_t>>& tiles_and_k, int waves = 6);

}  // namespace spngd
