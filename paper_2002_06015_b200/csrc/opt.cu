// The whole SP-NGD optimizer step on one rank: Stages 2-5 of
// accumulate_microsteps (src/dist.cpp:406-675) with n = 1 micro-step.
//
//   factors + BN moments (local shard)  -> RS send buffer, owner-major
//   ncclReduceScatter(avg)               -> owner receives the shard means
//   pi, damping, Cholesky inverse        (owned Kronecker layers)
//   precondition + momentum + rescale    (owned FC/Conv layers, in place in
//   BN 2x2 solve + update                 the all-gather buffer)
//   ncclAllGather (in place)             -> every rank's weight replicas
//
// Ownership is LPT-balanced on a^3 + g^3 + 2g^2 a + 2 g a^2 instead of the
// reference's round-robin li % K (dist.cpp:147-153); ownership never changes
// numerics.  All plans (GEMM problems, tiles, tasks) are built once at creation
// and stay device-resident; a step is a fixed sequence of launches on the
// context stream, bracketed by CUDA events per phase.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "ctx.cuh"
#include "factor.cuh"
#include "inverse.cuh"
#include "precond.cuh"

using namespace spngd;

namespace {

template <typename T>
T* dev_upload(const std::vector<T>& v, std::vector<void*>& owned) {
  if (v.empty()) return nullptr;
  T* d = nullptr;
  if (cudaMalloc(&d, v.size() * sizeof(T)) != cudaSuccess) return nullptr;
  cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  owned.push_back(d);
  return d;
}

struct LayerState {
  spngd_layer_desc d;
  int owner = 0;
  // captures (inputs)
  float* act = nullptr;
  float* grad = nullptr;
  float* gg = nullptr;
  float* gb = nullptr;
  // RS send offsets (floats within this owner's segment)
  int64_t off_A = -1, off_G = -1, off_M = -1, off_dW = -1;
  // AG offsets (within the owner segment)
  int64_t off_W = -1;
  // owner-local
  float* V = nullptr;
  float* Ainv = nullptr; int64_t lda = 0;
  float* Ginv = nullptr; int64_t ldg = 0;
};

}  // namespace

struct spngd_opt {
  spngd_ctx* ctx = nullptr;
  spngd_opt_config cfg{};
  std::vector<LayerState> layers;
  int world = 1, rank = 0;
  int64_t seg_rs = 0, seg_ag = 0;  // per-owner padded segment sizes (floats)
  float* rs_send = nullptr;        // world * seg_rs
  float* rs_recv = nullptr;        // seg_rs (== rs_send when world == 1)
  float* ag = nullptr;             // world * seg_ag
  std::vector<void*> owned;        // every device allocation
  // plans
  FactorPlan fplan;
  GemmProblem* d_fprobs = nullptr; GemmWorkItem* d_fitems = nullptr; SyrkReduceTask* d_freduce = nullptr;
  RepackTask* d_repack = nullptr;
  float* d_partials = nullptr;
  std::vector<spngd_bn_moments_req> bnm;
  spngd_bn_moments_req* d_bnm = nullptr; int64_t bnm_maxc = 0;
  std::vector<PiTask> pis; PiTask* d_pis = nullptr;
  std::vector<UnpackTask> unpacks; UnpackTask* d_unpacks = nullptr; int64_t max_n = 0;
  struct InvClass {  // one recursion schedule per matrix size class, on its own stream
    InversePlan plan;
    GemmProblem* d_probs = nullptr;
    GemmWorkItem* d_items = nullptr;
    BaseTask* d_bases = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;
  };
  std::vector<InvClass> inv;
  cudaEvent_t inv_fork = nullptr;
  float* d_scal = nullptr;         // {eta, momentum} read by the update kernels
  cudaGraph_t graphs[6] = {};
  cudaGraphExec_t graph_exec[6] = {};
  bool use_graph = true;
  bool graphs_ready = false;
  PrecondPlan pplan;
  GemmProblem *d_p1 = nullptr, *d_p2 = nullptr; GemmWorkItem *d_i1 = nullptr, *d_i2 = nullptr;
  RescaleTask* d_rescale = nullptr; double* d_norms = nullptr;
  std::vector<spngd_bn_update_req> bnu; spngd_bn_update_req* d_bnu = nullptr; int64_t bnu_maxc = 0;
  float* d_damps = nullptr;
  cudaEvent_t ev[7] = {};
  int64_t launches = 0;
  bool timed = false;

  float* alloc(size_t floats, bool zero = false) {
    void* p = nullptr;
    if (floats == 0) floats = 1;
    if (cudaMalloc(&p, floats * sizeof(float)) != cudaSuccess) return nullptr;
    if (zero) cudaMemset(p, 0, floats * sizeof(float));
    owned.push_back(p);
    return static_cast<float*>(p);
  }
  ~spngd_opt() {
    for (int i = 0; i < 6; ++i) {
      if (graph_exec[i]) cudaGraphExecDestroy(graph_exec[i]);
      if (graphs[i]) cudaGraphDestroy(graphs[i]);
    }
    for (auto& c : inv) {
      if (c.done) cudaEventDestroy(c.done);
      if (c.stream) cudaStreamDestroy(c.stream);
    }
    if (inv_fork) cudaEventDestroy(inv_fork);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (void* p : owned) cudaFree(p);
  }
};

namespace {

double layer_cost(const spngd_layer_desc& d) {
  if (d.kind == SPNGD_BN) return double(d.g);
  const double a = double(d.a), g = double(d.g);
  return a * a * a + g * g * g + 2 * g * g * a + 2 * g * a * a;
}

int build(spngd_opt* o, const spngd_layer_desc* descs, int n) {
  const int W = o->world;
  std::vector<spngd_layout_entry> lay(n);
  int rc0 = spngd_plan_layout(descs, n, W, lay.data(), &o->seg_rs, &o->seg_ag);
  if (rc0) return rc0;
  o->layers.resize(n);
  for (int li = 0; li < n; ++li) {
    LayerState& L = o->layers[li];
    L.d = descs[li];
    L.owner = lay[li].owner;
    L.off_A = lay[li].off_A;
    L.off_G = lay[li].off_G;
    L.off_M = lay[li].off_M;
    L.off_dW = lay[li].off_dW;
    L.off_W = lay[li].off_W;
  }
  o->rs_send = o->alloc(size_t(W) * o->seg_rs, true);
  o->rs_recv = (W == 1) ? o->rs_send : o->alloc(o->seg_rs, true);
  o->ag = o->alloc(size_t(W) * o->seg_ag, true);
  if (!o->rs_send || !o->rs_recv || !o->ag) return fail(SPNGD_ERR_CUDA, "opt: buffer allocation failed");

  const int64_t B = o->cfg.batch;
  std::vector<spngd_factor_req> freqs;
  std::vector<DenseMatrix> mats;
  std::vector<spngd_precond_req> preqs;
  int n_owned_kron = 0;
  for (int li = 0; li < n; ++li) {
    LayerState& L = o->layers[li];
    float* seg = o->rs_send + int64_t(L.owner) * o->seg_rs;
    if (L.d.kind == SPNGD_BN) {
      const int64_t c = L.d.g;
      L.gg = o->alloc(size_t(B * c));
      L.gb = o->alloc(size_t(B * c));
      o->bnm.push_back({L.gg, L.gb, c, 0, B, seg + L.off_M});
      o->bnm_maxc = std::max(o->bnm_maxc, c);
    } else {
      const bool conv = L.d.kind == SPNGD_CONV;
      const int64_t hw = conv ? L.d.hw : 1;
      L.act = o->alloc(size_t(B * L.d.a * hw));
      L.grad = o->alloc(size_t(B * L.d.g * hw));
      if (!L.act || !L.grad) return fail(SPNGD_ERR_CUDA, "opt: capture allocation failed");
      const double nb = double(B);
      freqs.push_back({L.act, L.d.a, hw, conv ? 1 : 0, 0, B, conv ? 1.0 / (nb * double(hw)) : 1.0 / nb, seg + L.off_A});
      freqs.push_back({L.grad, L.d.g, hw, conv ? 1 : 0, 0, B, 1.0 / nb, seg + L.off_G});
    }
  }
  // ---- owner-local state and plans
  o->d_damps = o->alloc(2 * size_t(n));
  o->d_norms = reinterpret_cast<double*>(o->alloc(2 * size_t(n)));
  for (int li = 0; li < n; ++li) {
    LayerState& L = o->layers[li];
    if (L.owner != o->rank) continue;
    float* wseg = o->ag + int64_t(o->rank) * o->seg_ag;
    if (L.d.kind == SPNGD_BN) {
      const int64_t c = L.d.g;
      L.V = o->alloc(size_t(2 * c), true);
      spngd_bn_update_req r{};
      r.m3c = o->rs_recv + L.off_M;
      r.grad = o->rs_recv + L.off_dW;
      r.c = c;
      r.gamma = wseg + L.off_W;
      r.beta = wseg + L.off_W + c;
      r.vgamma = L.V;
      r.vbeta = L.V + c;
      o->bnu.push_back(r);
      o->bnu_maxc = std::max(o->bnu_maxc, c);
      continue;
    }
    const int64_t a = L.d.a, g = L.d.g;
    L.lda = round_up(a, 32);
    L.ldg = round_up(g, 32);
    L.Ainv = o->alloc(size_t(a * L.lda));
    L.Ginv = o->alloc(size_t(g * L.ldg));
    float* tla = o->alloc(size_t(a * L.lda), true);
    float* tua = o->alloc(size_t(a * L.lda), true);
    float* tlg = o->alloc(size_t(g * L.ldg), true);
    float* tug = o->alloc(size_t(g * L.ldg), true);
    L.V = o->alloc(size_t(g * a), true);
    if (!L.Ainv || !L.Ginv || !tla || !tua || !tlg || !tug || !L.V)
      return fail(SPNGD_ERR_CUDA, "opt: owner state allocation failed");
    float* dA = o->d_damps + 2 * li;
    float* dG = dA + 1;
    o->pis.push_back({o->rs_recv + L.off_A, o->rs_recv + L.off_G, a, g, std::sqrt(o->cfg.lambda), dA, dG, nullptr});
    o->unpacks.push_back({o->rs_recv + L.off_A, a, dA, 0.f, 0, L.Ainv, L.lda});
    o->unpacks.push_back({o->rs_recv + L.off_G, g, dG, 0.f, 0, L.Ginv, L.ldg});
    o->max_n = std::max({o->max_n, a, g});
    mats.push_back({L.Ainv, tla, tua, L.lda, a});
    mats.push_back({L.Ginv, tlg, tug, L.ldg, g});
    spngd_precond_req pr{};
    pr.Ginv = L.Ginv; pr.ldg = L.ldg;
    pr.Ainv = L.Ainv; pr.lda = L.lda;
    pr.dW = o->rs_recv + L.off_dW;
    pr.g = g; pr.a = a;
    pr.W = wseg + L.off_W;
    pr.V = L.V;
    pr.rescale = o->cfg.rescale;
    preqs.push_back(pr);
    ++n_owned_kron;
  }
  std::vector<void*>& own = o->owned;
  // factor plan (all layers, local shard)
  FactorPlan fsz;
  int rc = plan_factors(freqs.data(), int(freqs.size()), fsz);
  if (rc) return rc;
  float* fws = o->alloc(fsz.repack_floats);
  rc = plan_factors(freqs.data(), int(freqs.size()), o->fplan, fws);
  if (rc) return rc;
  o->d_repack = dev_upload(o->fplan.repacks, own);
  o->d_fprobs = dev_upload(o->fplan.probs, own);
  o->d_fitems = dev_upload(o->fplan.items, own);
  o->d_freduce = dev_upload(o->fplan.reduce, own);
  o->d_partials = o->alloc(size_t(std::max(o->fplan.n_slots, 1)) * kTileM * kTileN);
  o->d_bnm = dev_upload(o->bnm, own);
  o->d_pis = dev_upload(o->pis, own);
  o->d_unpacks = dev_upload(o->unpacks, own);
  // inverse plans: one per matrix size class (owned matrices of equal n share
  // identical recursion schedules and batch into the same launches); classes
  // run concurrently on their own streams.
  {
    std::vector<int64_t> sizes;
    for (const auto& m : mats) sizes.push_back(m.n);
    std::sort(sizes.begin(), sizes.end());
    sizes.erase(std::unique(sizes.begin(), sizes.end()), sizes.end());
    std::reverse(sizes.begin(), sizes.end());  // largest (critical path) first
    for (int64_t n : sizes) {
      std::vector<DenseMatrix> cls;
      for (const auto& m : mats)
        if (m.n == n) cls.push_back(m);
      o->inv.emplace_back();
      spngd_opt::InvClass& c = o->inv.back();
      InversePlan sizing;
      plan_inverse(cls, nullptr, sizing);
      float* ws = o->alloc(sizing.workspace_floats);
      plan_inverse(cls, ws, c.plan);
      c.d_probs = dev_upload(c.plan.probs, own);
      c.d_items = dev_upload(c.plan.items, own);
      c.d_bases = dev_upload(c.plan.bases, own);
      SPNGD_CUDA_TRY(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
      SPNGD_CUDA_TRY(cudaEventCreateWithFlags(&c.done, cudaEventDisableTiming));
    }
    SPNGD_CUDA_TRY(cudaEventCreateWithFlags(&o->inv_fork, cudaEventDisableTiming));
  }
  o->d_scal = o->alloc(2);
  o->use_graph = getenv("SPNGD_NO_GRAPH") == nullptr;
  // precondition plan
  PrecondPlan psz;
  rc = plan_precondition(preqs.data(), int(preqs.size()), 0.0, 0.0, nullptr, nullptr, psz);
  if (rc) return rc;
  float* ptmp = o->alloc(psz.tmp_floats);
  rc = plan_precondition(preqs.data(), int(preqs.size()), 0.0, 0.0, ptmp, o->d_norms, o->pplan, o->d_scal);
  if (rc) return rc;
  o->d_p1 = dev_upload(o->pplan.probs1, own);
  o->d_i1 = dev_upload(o->pplan.items1, own);
  o->d_p2 = dev_upload(o->pplan.probs2, own);
  o->d_i2 = dev_upload(o->pplan.items2, own);
  o->d_rescale = dev_upload(o->pplan.rescale, own);
  o->d_bnu = dev_upload(o->bnu, own);
  for (auto& e : o->ev) SPNGD_CUDA_TRY(cudaEventCreate(&e));
  SPNGD_CUDA_TRY(cudaDeviceSynchronize());
  return SPNGD_OK;
}

}  // namespace

extern "C" {

int spngd_plan_layout(const spngd_layer_desc* descs, int n, int W, spngd_layout_entry* out, int64_t* seg_rs,
                      int64_t* seg_ag) {
  if (!descs || !out || n <= 0 || W < 1) return fail(SPNGD_ERR_INVALID, "spngd_plan_layout: bad argument");
  // ownership: LPT on inverse + precondition cost, deterministic tie-break
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int x, int y) { return layer_cost(descs[x]) > layer_cost(descs[y]); });
  std::vector<double> load(W, 0.0);
  for (int li : order) {
    const int r = int(std::min_element(load.begin(), load.end()) - load.begin());
    out[li].owner = r;
    load[r] += layer_cost(descs[li]);
  }
  // owner-major segment layout, 64-float aligned entries, in layer order
  std::vector<int64_t> rs_fill(W, 0), ag_fill(W, 0);
  auto place = [](int64_t& fill, int64_t cnt) {
    const int64_t off = fill;
    fill += round_up(cnt, 64);
    return off;
  };
  for (int li = 0; li < n; ++li) {
    spngd_layout_entry& e = out[li];
    const spngd_layer_desc& d = descs[li];
    const int r = e.owner;
    e.pad_ = 0;
    e.off_A = e.off_G = e.off_M = -1;
    if (d.kind == SPNGD_BN) {
      e.off_M = place(rs_fill[r], 3 * d.g);
      e.off_dW = place(rs_fill[r], 2 * d.g);
      e.off_W = place(ag_fill[r], 2 * d.g);
    } else {
      e.off_A = place(rs_fill[r], d.a * (d.a + 1) / 2);
      e.off_G = place(rs_fill[r], d.g * (d.g + 1) / 2);
      e.off_dW = place(rs_fill[r], d.g * d.a);
      e.off_W = place(ag_fill[r], d.g * d.a);
    }
  }
  if (seg_rs) *seg_rs = std::max<int64_t>(64, *std::max_element(rs_fill.begin(), rs_fill.end()));
  if (seg_ag) *seg_ag = std::max<int64_t>(64, *std::max_element(ag_fill.begin(), ag_fill.end()));
  return SPNGD_OK;
}

int spngd_opt_create(spngd_ctx* ctx, const spngd_layer_desc* layers, int n_layers, const spngd_opt_config* cfg,
                     spngd_opt** out) {
  if (!ctx || !layers || n_layers <= 0 || !cfg || !out) return fail(SPNGD_ERR_INVALID, "spngd_opt_create: bad argument");
  if (!(cfg->lambda > 0.0)) return fail(SPNGD_ERR_NOT_POSITIVE_DEFINITE, "OptimizerConfig: lambda must be > 0");
  if (cfg->batch < 1) return fail(SPNGD_ERR_EMPTY_BATCH, "spngd_opt_create: empty per-rank batch");
  if (cfg->stale) return fail(SPNGD_ERR_INVALID, "spngd_opt_create: stale gating runs through spngd_tracker_* (not fused yet)");
  for (int i = 0; i < n_layers; ++i) {
    const auto& d = layers[i];
    if (d.kind < 0 || d.kind > 2 || d.g <= 0 || (d.kind != SPNGD_BN && (d.a <= 0 || d.hw <= 0)))
      return fail(SPNGD_ERR_SHAPE_MISMATCH, "spngd_opt_create: layer %d has an invalid shape", i);
  }
  auto* o = new spngd_opt();
  o->ctx = ctx;
  o->cfg = *cfg;
  o->world = ctx->world;
  o->rank = ctx->rank;
  SPNGD_CUDA_TRY(cudaSetDevice(ctx->device));
  int rc = build(o, layers, n_layers);
  if (rc) {
    delete o;
    return rc;
  }
  *out = o;
  return SPNGD_OK;
}

void spngd_opt_destroy(spngd_opt* opt) { delete opt; }

int spngd_opt_owner(const spngd_opt* opt, int layer) {
  if (!opt || layer < 0 || layer >= int(opt->layers.size())) return -1;
  return opt->layers[layer].owner;
}

float* spngd_opt_buffer(spngd_opt* o, int layer, int which, int64_t* ld) {
  if (!o || layer < 0 || layer >= int(o->layers.size())) return nullptr;
  LayerState& L = o->layers[layer];
  const bool mine = L.owner == o->rank;
  if (ld) *ld = 0;
  switch (which) {
    case 0: return L.act;
    case 1: return L.grad;
    case 2: return L.off_dW >= 0 ? o->rs_send + int64_t(L.owner) * o->seg_rs + L.off_dW : nullptr;
    case 3: return o->ag + int64_t(L.owner) * o->seg_ag + L.off_W;
    case 4: return mine ? L.V : nullptr;
    case 5: return L.gg;
    case 6: return L.gb;
    case 7: if (ld) *ld = L.lda; return mine ? L.Ainv : nullptr;
    case 8: if (ld) *ld = L.ldg; return mine ? L.Ginv : nullptr;
    case 9: return (mine && L.off_A >= 0) ? o->rs_recv + L.off_A : nullptr;
    case 10: return (mine && L.off_G >= 0) ? o->rs_recv + L.off_G : nullptr;
    case 11: return (mine && L.off_M >= 0) ? o->rs_recv + L.off_M : nullptr;
    case 12: if (ld) *ld = int64_t(o->world) * o->seg_ag; return o->ag;  // all weight replicas
    default: return nullptr;
  }
}

}  // extern "C"

namespace {

// The six phases of one step.  Each phase is captured once into its own CUDA
// graph; phase events are recorded between graph launches.
int issue_phase(spngd_opt* o, int phase) {
  spngd_ctx* ctx = o->ctx;
  cudaStream_t s = ctx->stream;
  int rc = SPNGD_OK;
  switch (phase) {
    case 0:  // Stages 1-3 local part: factor SYRK into the RS send buffer.
      rc = launch_repack(ctx, o->d_repack, int(o->fplan.repacks.size()), o->fplan.repack_max);
      if (rc) return rc;
      rc = launch_gemm(o->d_fprobs, o->d_fitems, int(o->fplan.items.size()), o->d_partials, ctx->d_status, s);
      ctx->launches++;
      return rc;
    case 1:  // split-K reduction + BN moments.
      rc = launch_syrk_reduce(o->d_freduce, int(o->fplan.reduce.size()), o->d_partials, s);
      ctx->launches += !o->fplan.reduce.empty();
      if (!rc) rc = launch_bn_moments(ctx, o->d_bnm, int(o->bnm.size()), o->bnm_maxc);
      return rc;
    case 2:  // Stages 2-3: ReduceScatterV of A, G/F and grads (dist.cpp:510-537).
      if (o->world > 1) rc = spngd_reduce_scatter_mean(ctx, o->rs_send, o->rs_recv, o->seg_rs);
      return rc;
    case 3: {  // Stage 4a: pi, damping, inverse (dist.cpp:539-602); size classes
               // fork onto their own streams and join.
      rc = launch_pi(ctx, o->d_pis, int(o->pis.size()));
      if (!rc) rc = launch_unpack(ctx, o->d_unpacks, int(o->unpacks.size()), o->max_n);
      if (rc) return rc;
      SPNGD_CUDA_TRY(cudaEventRecord(o->inv_fork, s));
      for (auto& c : o->inv) {
        SPNGD_CUDA_TRY(cudaStreamWaitEvent(c.stream, o->inv_fork, 0));
        ctx->stream = c.stream;
        rc = run_inverse(ctx, c.plan, c.d_probs, c.d_items, c.d_bases);
        ctx->stream = s;
        if (rc) return rc;
        SPNGD_CUDA_TRY(cudaEventRecord(c.done, c.stream));
        SPNGD_CUDA_TRY(cudaStreamWaitEvent(s, c.done, 0));
      }
      return SPNGD_OK;
    }
    case 4:  // Stage 4b: precondition + update + rescale, BN solve + update (dist.cpp:604-633).
      rc = run_precondition(ctx, o->pplan, o->d_p1, o->d_i1, o->d_p2, o->d_i2, o->d_rescale, o->d_norms);
      if (!rc)
        rc = launch_bn_update(ctx, o->d_bnu, int(o->bnu.size()), o->bnu_maxc, o->cfg.lambda, 0.0, 0.0, o->d_scal);
      return rc;
    case 5:  // Stage 5: AllGatherV of the updated weights (dist.cpp:646-663), in place.
      if (o->world > 1) rc = spngd_all_gather(ctx, o->ag + int64_t(o->rank) * o->seg_ag, o->ag, o->seg_ag);
      return rc;
  }
  return SPNGD_OK;
}

}  // namespace

extern "C" {

int spngd_opt_step(spngd_opt* o, int64_t step, double eta, double momentum) {
  if (!o) return fail(SPNGD_ERR_INVALID, "spngd_opt_step: opt is NULL");
  (void)step;
  spngd_ctx* ctx = o->ctx;
  cudaStream_t s = ctx->stream;
  // Host scalars of this step -> device (outside the graphs).  Pageable
  // source: staged before cudaMemcpyAsync returns, so no host sync.
  const float scal[2] = {float(eta), float(momentum)};
  SPNGD_CUDA_TRY(cudaMemcpyAsync(o->d_scal, scal, sizeof(scal), cudaMemcpyHostToDevice, s));
  const bool capture = o->use_graph && !o->graphs_ready;
  const int64_t l0 = ctx->launches;
  for (int ph = 0; ph < 6; ++ph) {
    SPNGD_CUDA_TRY(cudaEventRecord(o->ev[ph], s));
    if (!o->use_graph) {
      int rc = issue_phase(o, ph);
      if (rc) return rc;
      continue;
    }
    if (capture) {
      SPNGD_CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      int rc = issue_phase(o, ph);
      cudaGraph_t g = nullptr;
      cudaError_t e = cudaStreamEndCapture(s, &g);
      if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      if (e != cudaSuccess) return fail_cuda(e, "cudaStreamEndCapture");
      o->graphs[ph] = g;
      SPNGD_CUDA_TRY(cudaGraphInstantiate(&o->graph_exec[ph], g, 0));
    }
    SPNGD_CUDA_TRY(cudaGraphLaunch(o->graph_exec[ph], s));
  }
  SPNGD_CUDA_TRY(cudaEventRecord(o->ev[6], s));
  if (capture || !o->use_graph) o->launches = ctx->launches - l0;
  o->graphs_ready = o->use_graph;
  o->timed = true;
  return SPNGD_OK;
}

int spngd_opt_phase_ms(spngd_opt* o, float* out6) {
  if (!o || !out6) return fail(SPNGD_ERR_INVALID, "spngd_opt_phase_ms: bad argument");
  if (!o->timed) return fail(SPNGD_ERR_INVALID, "spngd_opt_phase_ms: no step yet");
  SPNGD_CUDA_TRY(cudaEventSynchronize(o->ev[6]));
  for (int i = 0; i < 6; ++i) SPNGD_CUDA_TRY(cudaEventElapsedTime(&out6[i], o->ev[i], o->ev[i + 1]));
  return SPNGD_OK;
}

int64_t spngd_opt_launch_count(const spngd_opt* o) { return o ? o->launches : 0; }

}  // extern "C"
