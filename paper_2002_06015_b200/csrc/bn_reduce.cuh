// Fused BN backward statistics: plan + launch shared by the
// public entry point and the optimizer step (bn_reduce.cu).
#pragma once

#include <vector>

#include "ctx.cuh"

namespace spngd {

struct BnxTask {
  const float* dy;
  const float* xh;
  int64_t M, c, S;
  float* gg;        // per-sample captures (may be null)
  float* gb;
  float* out3c;     // build_bn_block moments, interleaved 3c (may be null)
  float* payload;   // grad_payload BN branch [c gamma | c beta] (may be null)
  int32_t nchunks;  // sample chunks per channel
  int32_t pad_;
  int64_t slot0;    // first chunk slot of this task
  int64_t chan0;    // first channel counter of this task
};

struct BnxItem {
  int32_t task, ch, s0, s1, chunk, pad_;
};

struct BnxPlan {
  std::vector<BnxTask> tasks;
  std::vector<BnxItem> items;
  int64_t slots = 0, channels = 0, bytes = 0;
};

int plan_bn_backward(const std::vector<spngd_bn_backward_req>& reqs, BnxPlan& plan);
// d_counters: plan.channels ints, zero before the first launch (the kernel
// resets them); d_slots: 5 * plan.slots doubles.
int launch_bn_backward(spngd_ctx* ctx, const BnxTask* d_tasks, const BnxItem* d_items, int64_t n_items, double* d_slots,
                       int* d_counters);

}  // namespace spngd
