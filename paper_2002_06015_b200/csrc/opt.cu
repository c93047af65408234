// The whole SP-NGD optimizer step on one rank: Stages 2-5 of
// accumulate_microsteps (src/dist.cpp:406-675) with n = 1 micro-step.
//
//   factors + BN moments (local shard)  -> RS send buffer: a statistics region
//                                           and a gradient region, each owner-major
//   ncclReduceScatter(avg) per region    -> owner receives the shard means
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
//
// Stale gating (cfg.stale, dist.cpp:431-444 / 514-537 / 588-601): every
// statistic A:l, G:l, F:l has a StaleTracker (tracker.cu, identical on every
// rank).  A step builds, reduces (grouped ncclReduce to the owners when only
// some are due) and re-inverts only the due statistics -- both inverses of a
// layer when either factor refreshed -- while gradients, precondition, update
// and all-gather run every step.  The owner compares each fresh statistic
// with its two retained snapshots on the device (K8), the distances are
// all-reduced, and every rank's trackers advance from them at the start of
// the next step (no mid-step host sync).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <cmath>
#include <numeric>
#include <vector>

#include "bn_full.cuh"
#include "bn_reduce.cuh"
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
  // OneMC: sampled-label captures (grad_sampled, bn_g*_sampled, net.hpp:92-97)
  float* grad_s = nullptr;
  float* gg_s = nullptr;
  float* gb_s = nullptr;
  // RS offsets: off_A/G/M within the owner's statistics segment, off_dW
  // within the owner's gradient segment (floats)
  int64_t off_A = -1, off_G = -1, off_M = -1, off_dW = -1;
  // AG offsets (within the owner segment)
  int64_t off_W = -1;
  // owner-local
  float* V = nullptr;
  float* Ainv = nullptr; int64_t lda = 0;   // recursion scratch; the inverse on request
  float* Ginv = nullptr; int64_t ldg = 0;
  float *tla = nullptr, *tua = nullptr, *tlg = nullptr, *tug = nullptr;  // T = L^-1 and T^T per factor
  // BN full mode: interleaved per-sample u (B x 2c); owner: F + lambda I
  // recursion scratch / inverse on request, its factors, T u scratch (2c)
  float* u = nullptr;
  float* raw = nullptr;  // raw conv input (enable_raw_inputs); == act for 1x1 stride-1 convs
  float* dy = nullptr;   // BN backward inputs (enable_bn_inputs): dY and x_hat, B x (c*S)
  float* xh = nullptr;
  int64_t bn_S = 0;
  int64_t raw_floats = 0;
  int fa = -1, fg = -1;  // factor-plan problem indices of A and G (wgrad reuses their operands)
  float* Finv = nullptr; int64_t ldf = 0;
  float *tlf = nullptr, *tuf = nullptr, *yf = nullptr;
};

// One stale-gated statistic (A:l, G:l or F:l).
struct StatState {
  int layer = 0;
  int kind = 0;            // 0 A, 1 G, 2 F (BN 3c moments)
  int owner = 0;
  int64_t off = 0;         // within the owner's statistics segment
  int64_t count = 0;       // floats
  int64_t dim = 0;         // packed dimension n (A/G) or channels c (F)
  spngd_tracker* tr = nullptr;
  int nsnap = 0;           // retained snapshots (identical on every rank)
  float* snap[2] = {};     // owner only; snap[first] = x1, snap[first^1] = x2
  int first = 0;
};

}  // namespace

struct spngd_opt {
  spngd_ctx* ctx = nullptr;
  spngd_opt_config cfg{};
  std::vector<LayerState> layers;
  int world = 1, rank = 0;
  int64_t seg_stat = 0, seg_grad = 0, seg_ag = 0;  // per-owner padded segment sizes (floats)
  float* rs_send = nullptr;        // world * seg_stat | world * seg_grad
  float* rs_recv = nullptr;        // seg_stat | seg_grad (== rs_send when world == 1)
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
    int wave = 0;
    InversePlan plan;
    GemmProblem* d_probs = nullptr;
    GemmWorkItem* d_items = nullptr;
    BaseTask* d_bases = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;
    // stale gating: the class members and room for a re-planned subset
    std::vector<DenseMatrix> mats;
    std::vector<int> mat_layer;
    float* ws = nullptr;
    InversePlan dyn;
    GemmProblem* d_probs_dyn = nullptr;
    GemmWorkItem* d_items_dyn = nullptr;
    BaseTask* d_bases_dyn = nullptr;
  };
  std::vector<InvClass> inv;
  cudaEvent_t inv_fork = nullptr;
  // Single-GPU full steps: layers fall into waves by matrix size, largest
  // first.  Wave w's factor SYRK, reduction, pi and unpack run on the main
  // stream, then its inverse classes fork onto high-priority streams and
  // recurse while the next wave's factor SYRK fills the remaining SMs.
  struct Wave {
    std::vector<GemmWorkItem> items;
    GemmWorkItem* d_items = nullptr;
    std::vector<SyrkReduceTask> reduce;
    SyrkReduceTask* d_reduce = nullptr;
    std::vector<PiTask> pis;
    PiTask* d_pis = nullptr;
    std::vector<UnpackTask> unpacks;
    UnpackTask* d_unpacks = nullptr;
    int64_t max_n = 0;
    std::vector<OwnerReduce> owner_ops;  // world > 1: this wave's statistics -> their owners
    std::vector<SlotMeanTask> means;     // p2p_rs: this wave's owned statistics, slot means
    SlotMeanTask* d_means = nullptr;
    int64_t means_max = 0;
    cudaEvent_t ready = nullptr;         // factors of this wave reduced locally
    cudaEvent_t fork = nullptr;          // owner-side inputs of this wave's recursion ready
    // spngd_opt_step_host: this wave's captures arrive from the host on the
    // copy stream; its im2col / repack run right before its SYRK
    std::vector<RepackTask> repacks;
    RepackTask* d_repacks = nullptr;
    int64_t repack_max = 0;
    std::vector<spngd_im2col_req> i2c;
    spngd_im2col_req* d_i2c = nullptr;
    cudaEvent_t in_ready = nullptr;
    // Host-input steps, last wave: its SYRK split by layer groups that launch
    // as their captures land (the last wave holds most of the capture bytes,
    // so one launch after its last byte left ~3 ms of SYRK after the PCIe
    // stream ended).  Used when the wave has no repack / im2col.
    struct Sub {
      std::vector<GemmWorkItem> items;
      GemmWorkItem* d_items = nullptr;
      std::vector<spngd_im2col_req> i2c;  // raw-input mode: this group's device im2col
      spngd_im2col_req* d_i2c = nullptr;
      cudaEvent_t ready = nullptr;
    };
    std::vector<Sub> subs;
    bool subs_usable() const {
      static const bool off = getenv("SPNGD_NO_SUBWAVES") != nullptr;  // A/B experiments
      size_t n_i2c = 0;
      for (const auto& sb : subs) n_i2c += sb.i2c.size();
      return !off && !subs.empty() && repacks.empty() && n_i2c == i2c.size();
    }
  };
  std::vector<int> sub_of_layer;         // last wave's layer -> sub index (-1: none)
  std::vector<Wave> waves;
  cudaStream_t comm_stream = nullptr;    // world > 1: NCCL + owner-side prep of the waves
  cudaEvent_t comm_fork = nullptr, comm_done = nullptr;
  // spngd_opt_attach_peers: Stage 5 as NVLink stores into the peers' replica buffers
  bool p2p = false;
  float* peer_ag[8] = {};
  // fused reduce-scatter (no stale gating): the factor epilogues / split-K
  // reductions / BN moments write this rank's statistics straight into the
  // owner's inbox slot over NVLink; owners average the slots per wave
  bool p2p_rs = false;
  float* inbox = nullptr;            // world x seg_stat, slot q = rank q's statistics for this owner
  float* peer_inbox[8] = {};
  std::vector<SlotMeanTask> means; SlotMeanTask* d_means = nullptr; int64_t means_max = 0;
  std::vector<PeerCopyTask> pcopy; PeerCopyTask* d_pcopy = nullptr; int64_t pcopy_max = 0;
  double* d_barrier = nullptr;
  double* d_flag = nullptr;        // world > 1: status agreement before Stage 4 writes
  int* d_info = nullptr;           // 3 per layer (A, G, F): status of each owned factor's inverse
  cudaStream_t h2d_stream = nullptr;     // spngd_opt_step_host: host inputs, wave by wave
  cudaStream_t d2h_stream = nullptr;     // and the early layers' weights back
  cudaEvent_t d2h_done = nullptr;
  cudaEvent_t h2d_start = nullptr, grads_ready = nullptr;
  bool overlap_ok = false;   // no stale gating
  bool overlap_on = false;
  int inv_prio = 0;          // greatest stream priority
  cudaGraph_t graphs_ov[6] = {};
  cudaGraphExec_t graph_ov_exec[6] = {};
  bool graphs_ready_ov = false;
  float* d_scal = nullptr;         // {eta, momentum} read by the update kernels
  std::vector<SgdTask> sgd_tasks; SgdTask* d_sgd = nullptr;  // cfg.sgd: owned layers' plain update
  // cfg.bn_mode == 1 (full 2c x 2c BN blocks)
  std::vector<InterleaveTask> ilv; InterleaveTask* d_ilv = nullptr; int64_t ilv_max = 0;
  std::vector<UnpackTask> bnf_unpacks; UnpackTask* d_bnf_unpacks = nullptr; UnpackTask* d_bnf_unpacks_dyn = nullptr;
  std::vector<int> bnf_layer;               // owned BN layers in bnf_unpacks / bnf_upd order
  // raw conv inputs expanded by im2col at the start of each step
  std::vector<spngd_im2col_req> i2c; spngd_im2col_req* d_i2c = nullptr; bool raw_inputs = false;
  // spngd_opt_enable_bn_inputs: BN layers take dY / x_hat; one fused launch
  // forms the captures, the 3c moments (unless stale-gated) and the BN payload
  bool bn_inputs = false;
  BnxPlan bnx; BnxTask* d_bnx_tasks = nullptr; BnxItem* d_bnx_items = nullptr;
  double* d_bnx_slots = nullptr; int* d_bnx_cnt = nullptr;
  // cfg.wgrad: grad_payload on the device (dense GEMM over the factor operands + BN column means)
  FactorPlan wplan;                         // OneMC: the true-label grad operands (G reads grad_sampled)
  RepackTask* d_wrepack = nullptr;
  std::vector<GemmProblem> wprobs; std::vector<GemmWorkItem> witems;
  GemmProblem* d_wprobs = nullptr; GemmWorkItem* d_witems = nullptr; uint32_t wvariant = 0;
  std::vector<BnGradPayloadTask> wbn; BnGradPayloadTask* d_wbn = nullptr; int64_t wbn_maxc = 0;
  int64_t bnf_maxn = 0;
  std::vector<spngd_bn_full_update_req> bnf_upd[2];  // T u, then T^T (T u) + update
  spngd_bn_full_update_req* d_bnf_upd[2] = {};
  cudaGraph_t graphs[6] = {};
  cudaGraphExec_t graph_exec[6] = {};
  bool use_graph = true;
  bool graphs_ready = false;
  PrecondPlan pplan;
  GemmProblem* d_pp[4] = {};
  GemmWorkItem* d_pi[4] = {};
  RescaleTask* d_rescale = nullptr; double* d_norms = nullptr;
  // Wave schedule: the precondition of layers whose inverses finish before the
  // last inverse wave runs on its own stream beside that wave's recursion
  // (which leaves most SMs idle); phase 4 then covers the rest.
  // The early layers are grouped by the inverse class that finishes last for
  // them (the longest recursion among their factors' classes), one part per
  // group on its own stream, so e.g. the 2048-class layers do not wait for
  // the 4608 chain.
  struct PrePart {
    PrecondPlan plan;
    GemmProblem* d_pp[4] = {};
    GemmWorkItem* d_pi[4] = {};
    RescaleTask* d_rescale = nullptr;
    double* d_norms = nullptr;
    std::vector<int> wait;         // inverse classes (indices into inv) this part reads
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;
  };
  std::vector<PrePart> pre_early;
  PrePart pre_late;                // world 1: also inside the wave schedule (stream/done below)
  bool late_in_overlap = false;
  std::vector<SnapTask> snap; SnapTask* d_snap = nullptr; int64_t snap_max = 0;
  cudaStream_t snap_stream = nullptr;
  cudaEvent_t snap_fork = nullptr, snap_done = nullptr;
  bool pre_split = false;
  int pre_cut = 0;                 // layers of waves < pre_cut are early
  bool ov_now = false;             // the running step uses the wave schedule
  std::vector<spngd_bn_update_req> bnu; spngd_bn_update_req* d_bnu = nullptr; int64_t bnu_maxc = 0;
  float* d_damps = nullptr;
  cudaEvent_t ev[7] = {};
  // SPNGD_STEP_TRACE (ungraphed steps): labelled events of the wave schedule,
  // printed against ev[0] by spngd_opt_phase_ms (critical-path diagnosis)
  std::vector<std::pair<std::string, cudaEvent_t>> trace;
  int64_t launches = 0;
  bool timed = false;
  // ---- stale gating
  std::vector<StatState> stats;
  std::vector<int> prob_stat, reduce_stat, repack_stat, bnm_stat;  // plan entry -> statistic
  GemmWorkItem* d_fitems_dyn = nullptr; SyrkReduceTask* d_freduce_dyn = nullptr;
  RepackTask* d_repack_dyn = nullptr; spngd_bn_moments_req* d_bnm_dyn = nullptr;
  std::vector<int> pi_layer;                 // owned Kronecker layers in pis order
  PiTask* d_pis_dyn = nullptr; UnpackTask* d_unpacks_dyn = nullptr;
  StatJob* d_statreq = nullptr;
  double* d_dist = nullptr; double* h_dist = nullptr;  // 4 per statistic
  cudaEvent_t dist_ev = nullptr;
  struct Pending { int q, has1, has2; };
  std::vector<Pending> pending; int64_t pending_step = 0;
  std::vector<char> due;
  int64_t last_due = 0;
  // ---- communication ledger (CommLedger) and NCCL bytes of the last step
  std::vector<spngd_layer_desc> descs;
  std::vector<spngd_ledger_row> ledger;
  int64_t wire_stat = 0, wire_grad = 0, wire_ag = 0;

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
      if (graph_ov_exec[i]) cudaGraphExecDestroy(graph_ov_exec[i]);
      if (graphs_ov[i]) cudaGraphDestroy(graphs_ov[i]);
    }
    for (float* p : peer_ag)
      if (p) cudaIpcCloseMemHandle(p);
    for (float* p : peer_inbox)
      if (p) cudaIpcCloseMemHandle(p);
    if (pre_late.done) cudaEventDestroy(pre_late.done);
    if (pre_late.stream) cudaStreamDestroy(pre_late.stream);
    if (snap_fork) cudaEventDestroy(snap_fork);
    if (snap_done) cudaEventDestroy(snap_done);
    if (snap_stream) cudaStreamDestroy(snap_stream);
    for (auto& pp : pre_early) {
      if (pp.done) cudaEventDestroy(pp.done);
      if (pp.stream) cudaStreamDestroy(pp.stream);
    }
    if (d2h_done) cudaEventDestroy(d2h_done);
    if (d2h_stream) cudaStreamDestroy(d2h_stream);
    if (h2d_start) cudaEventDestroy(h2d_start);
    if (grads_ready) cudaEventDestroy(grads_ready);
    if (h2d_stream) cudaStreamDestroy(h2d_stream);
    for (auto& w : waves) {
      if (w.in_ready) cudaEventDestroy(w.in_ready);
      if (w.fork) cudaEventDestroy(w.fork);
      if (w.ready) cudaEventDestroy(w.ready);
      for (auto& sb : w.subs)
        if (sb.ready) cudaEventDestroy(sb.ready);
    }
    if (comm_fork) cudaEventDestroy(comm_fork);
    if (comm_done) cudaEventDestroy(comm_done);
    if (comm_stream) cudaStreamDestroy(comm_stream);
    for (auto& c : inv) {
      if (c.done) cudaEventDestroy(c.done);
      if (c.stream) cudaStreamDestroy(c.stream);
    }
    if (inv_fork) cudaEventDestroy(inv_fork);
    if (dist_ev) cudaEventDestroy(dist_ev);
    if (h_dist) cudaFreeHost(h_dist);
    for (auto& st : stats)
      if (st.tr) spngd_tracker_destroy(st.tr);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (void* p : owned) cudaFree(p);
  }
};

namespace {

double layer_cost(const spngd_layer_desc& d, bool bn_full = false) {
  if (d.kind == SPNGD_BN && bn_full) return 8.0 * double(d.g) * double(d.g) * double(d.g);  // (2c)^3 inverse
  if (d.kind == SPNGD_BN) return double(d.g);
  const double a = double(d.a), g = double(d.g);
  return a * a * a + g * g * g + 2 * g * g * a + 2 * g * a * a;
}

// Overlap waves by the larger Kronecker dimension (inverse recursion depth).
// Wave boundaries on the larger Kronecker dimension, largest first; BN layers
// (no inverse) join the last wave.  SPNGD_WAVES="3072,1536" overrides (experiments).
const std::vector<int64_t>& wave_bounds() {
  static const std::vector<int64_t> b = [] {
    std::vector<int64_t> v = {3072, 1536};
    if (const char* e = getenv("SPNGD_WAVES")) {
      v.clear();
      for (const char* p = e; *p;) {
        char* end = nullptr;
        const long long x = strtoll(p, &end, 10);
        if (end == p) break;
        v.push_back(x);
        p = *end ? end + 1 : end;
      }
    }
    return v;
  }();
  return b;
}

int wave_of(const spngd_layer_desc& d) {
  const auto& b = wave_bounds();
  if (d.kind == SPNGD_BN) return int(b.size());
  const int64_t m = std::max<int64_t>(d.a, d.g);
  int w = 0;
  while (w < int(b.size()) && m <= b[size_t(w)]) ++w;
  return w;
}

int build(spngd_opt* o, const spngd_layer_desc* descs, int n) {
  const int W = o->world;
  std::vector<spngd_layout_entry> lay(n);
  const bool bnf = o->cfg.bn_mode == 1;
  int rc0 = spngd_plan_layout_ex(descs, n, W, bnf ? SPNGD_LEDGER_BN_FULL : 0, lay.data(), &o->seg_stat, &o->seg_grad,
                                 &o->seg_ag);
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
  o->rs_send = o->alloc(size_t(W) * (o->seg_stat + o->seg_grad), true);
  o->rs_recv = (W == 1) ? o->rs_send : o->alloc(o->seg_stat + o->seg_grad, true);
  o->ag = o->alloc(size_t(W) * o->seg_ag, true);
  if (!o->rs_send || !o->rs_recv || !o->ag) return fail(SPNGD_ERR_CUDA, "opt: buffer allocation failed");

  const int64_t B = o->cfg.batch;
  std::vector<spngd_factor_req> freqs;
  std::vector<DenseMatrix> mats;
  std::vector<int> mat_layer;
  std::vector<spngd_precond_req> preqs;
  std::vector<int> preq_layer;
  std::vector<PrecondTri> ptri;
  int n_owned_kron = 0;
  for (int li = 0; li < n; ++li) {
    LayerState& L = o->layers[li];
    float* seg = o->rs_send + int64_t(L.owner) * o->seg_stat;
    auto add_stat = [&](int kind, int64_t off, int64_t count, int64_t dim) {
      StatState st;
      st.layer = li;
      st.kind = kind;
      st.owner = L.owner;
      st.off = off;
      st.count = count;
      st.dim = dim;
      o->stats.push_back(st);
      return int(o->stats.size()) - 1;
    };
    const bool one_mc = o->cfg.fisher_mode == 1;
    if (L.d.kind == SPNGD_BN) {
      const int64_t c = L.d.g;
      L.gg = o->alloc(size_t(B * c));
      L.gb = o->alloc(size_t(B * c));
      if (one_mc) {  // build_bn_block(mode = OneMC) reads the sampled pair (fisher.cpp:158-159)
        L.gg_s = o->alloc(size_t(B * c));
        L.gb_s = o->alloc(size_t(B * c));
        if (!L.gg_s || !L.gb_s) return fail(SPNGD_ERR_CUDA, "opt: capture allocation failed");
      }
      if (bnf) {  // build_bn_full: interleave, then the SYRK engine (FC layout, scale 1/B)
        L.u = o->alloc(size_t(B * 2 * c));
        if (!L.u) return fail(SPNGD_ERR_CUDA, "opt: capture allocation failed");
        o->ilv.push_back({one_mc ? L.gg_s : L.gg, one_mc ? L.gb_s : L.gb, L.u, c, 0, B});
        o->ilv_max = std::max(o->ilv_max, B * c);
        freqs.push_back({L.u, 2 * c, 1, 0, 0, B, 1.0 / double(B), seg + L.off_M});
        o->prob_stat.push_back(add_stat(2, L.off_M, (2 * c) * (2 * c + 1) / 2, 2 * c));
      } else {
        o->bnm.push_back({one_mc ? L.gg_s : L.gg, one_mc ? L.gb_s : L.gb, c, 0, B, seg + L.off_M});
        o->bnm_stat.push_back(add_stat(2, L.off_M, 3 * c, c));
        o->bnm_maxc = std::max(o->bnm_maxc, c);
      }
    } else {
      const bool conv = L.d.kind == SPNGD_CONV;
      const int64_t hw = conv ? L.d.hw : 1;
      L.act = o->alloc(size_t(B * L.d.a * hw));
      L.grad = o->alloc(size_t(B * L.d.g * hw));
      if (one_mc) L.grad_s = o->alloc(size_t(B * L.d.g * hw));  // factor_G(OneMC), fisher.cpp:127-132
      if (!L.act || !L.grad || (one_mc && !L.grad_s)) return fail(SPNGD_ERR_CUDA, "opt: capture allocation failed");
      const double nb = double(B);
      L.fa = int(freqs.size());
      freqs.push_back({L.act, L.d.a, hw, conv ? 1 : 0, 0, B, conv ? 1.0 / (nb * double(hw)) : 1.0 / nb, seg + L.off_A});
      o->prob_stat.push_back(add_stat(0, L.off_A, L.d.a * (L.d.a + 1) / 2, L.d.a));
      L.fg = int(freqs.size());
      freqs.push_back({one_mc ? L.grad_s : L.grad, L.d.g, hw, conv ? 1 : 0, 0, B, 1.0 / nb, seg + L.off_G});
      o->prob_stat.push_back(add_stat(1, L.off_G, L.d.g * (L.d.g + 1) / 2, L.d.g));
    }
  }
  // ---- owner-local state and plans
  o->d_damps = o->alloc(2 * size_t(n));
  o->d_norms = reinterpret_cast<double*>(o->alloc(2 * size_t(n)));
  o->d_info = reinterpret_cast<int*>(o->alloc(3 * size_t(n), true));
  if (!o->d_damps || !o->d_norms || !o->d_info) return fail(SPNGD_ERR_CUDA, "opt: allocation failed");
  for (int li = 0; li < n; ++li) {
    LayerState& L = o->layers[li];
    if (L.owner != o->rank) continue;
    float* wseg = o->ag + int64_t(o->rank) * o->seg_ag;
    if (L.d.kind == SPNGD_BN) {
      const int64_t c = L.d.g;
      L.V = o->alloc(size_t(2 * c), true);
      if (bnf) {  // damp_bn_full: (F + lambda I)^-1 = T^T T by the batched Cholesky (fisher.cpp:248-253)
        const int64_t d2 = 2 * c;
        L.ldf = round_up(d2, 32);
        L.Finv = o->alloc(size_t(d2 * L.ldf));
        L.tlf = o->alloc(size_t(d2 * L.ldf), true);
        L.tuf = o->alloc(size_t(d2 * L.ldf), true);
        L.yf = o->alloc(size_t(d2), true);
        if (!L.Finv || !L.tlf || !L.tuf || !L.yf || !L.V) return fail(SPNGD_ERR_CUDA, "opt: owner state allocation failed");
        o->bnf_unpacks.push_back({o->rs_recv + L.off_M, d2, nullptr, float(o->cfg.lambda), 0, L.Finv, L.ldf,
                                  o->d_info + 3 * li + 2});
        o->bnf_layer.push_back(li);
        o->bnf_maxn = std::max(o->bnf_maxn, d2);
        mats.push_back({L.Finv, L.tlf, L.tuf, L.ldf, d2, o->d_info + 3 * li + 2});
        mat_layer.push_back(li);
        // precondition_bn_full (fisher.cpp:278-296): v = T^T (T u), then the BN update
        spngd_bn_full_update_req r0{}, r1{};
        r0.finv = L.tlf; r0.ld = L.ldf; r0.grad = o->rs_recv + o->seg_stat + L.off_dW; r0.c = c;
        r0.pg_out = L.yf; r0.pb_out = L.yf + c;
        r1.finv = L.tuf; r1.ld = L.ldf; r1.grad = L.yf; r1.c = c;
        r1.gamma = wseg + L.off_W; r1.beta = wseg + L.off_W + c; r1.vgamma = L.V; r1.vbeta = L.V + c;
        o->bnf_upd[0].push_back(r0);
        o->bnf_upd[1].push_back(r1);
        continue;
      }
      spngd_bn_update_req r{};
      r.m3c = o->rs_recv + L.off_M;
      r.grad = o->rs_recv + o->seg_stat + L.off_dW;
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
    o->pi_layer.push_back(li);
    o->unpacks.push_back({o->rs_recv + L.off_A, a, dA, 0.f, 0, L.Ainv, L.lda, o->d_info + 3 * li});
    o->unpacks.push_back({o->rs_recv + L.off_G, g, dG, 0.f, 0, L.Ginv, L.ldg, o->d_info + 3 * li + 1});
    o->max_n = std::max({o->max_n, a, g});
    mats.push_back({L.Ainv, tla, tua, L.lda, a, o->d_info + 3 * li});
    mat_layer.push_back(li);
    mats.push_back({L.Ginv, tlg, tug, L.ldg, g, o->d_info + 3 * li + 1});
    mat_layer.push_back(li);
    L.tla = tla; L.tua = tua; L.tlg = tlg; L.tug = tug;
    ptri.push_back({tla, tua, tlg, tug});
    spngd_precond_req pr{};
    pr.Ginv = L.Ginv; pr.ldg = L.ldg;
    pr.Ainv = L.Ainv; pr.lda = L.lda;
    pr.dW = o->rs_recv + o->seg_stat + L.off_dW;
    pr.g = g; pr.a = a;
    pr.W = wseg + L.off_W;
    pr.V = L.V;
    pr.rescale = o->cfg.rescale;
    preqs.push_back(pr);
    preq_layer.push_back(li);
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
  if (o->cfg.wgrad) {  // grad_payload (dist.cpp:315-391) -> this rank's gradient region
    const bool one_mc = o->cfg.fisher_mode == 1;
    std::vector<spngd_factor_req> wreqs;
    std::vector<int> wl;
    for (int li = 0; li < n; ++li) {
      const LayerState& L = o->layers[li];
      if (L.d.kind == SPNGD_BN || !one_mc) continue;
      const bool conv = L.d.kind == SPNGD_CONV;
      wreqs.push_back({L.grad, L.d.g, conv ? L.d.hw : 1, conv ? 1 : 0, 0, B, 1.0, o->d_partials});
      wl.push_back(li);
    }
    if (!wreqs.empty()) {
      FactorPlan wsz;
      if ((rc = plan_factors(wreqs.data(), int(wreqs.size()), wsz))) return rc;
      float* wws = o->alloc(wsz.repack_floats);
      if ((rc = plan_factors(wreqs.data(), int(wreqs.size()), o->wplan, wws))) return rc;
      o->d_wrepack = dev_upload(o->wplan.repacks, own);
    }
    int slot = 0;
    for (int li = 0, k = 0; li < n; ++li) {
      LayerState& L = o->layers[li];
      float* dW = o->rs_send + int64_t(W) * o->seg_stat + int64_t(L.owner) * o->seg_grad + L.off_dW;
      if (L.d.kind == SPNGD_BN) {
        const float* gg = L.gg;  // grad_payload reads the true-label pair in either Fisher mode
        o->wbn.push_back({gg, L.gb, B, L.d.g, dW});
        o->wbn_maxc = std::max(o->wbn_maxc, L.d.g);
        continue;
      }
      const GemmProblem& pa = o->fplan.probs[L.fa];
      const GemmProblem& pg = one_mc ? o->wplan.probs[k++] : o->fplan.probs[L.fg];
      if (pa.K != pg.K) return fail(SPNGD_ERR_SHAPE_MISMATCH, "wgrad: layer %d operands disagree on K", li);
      // both operands must walk K in the same order (TMA3D pairs samples per stage)
      if (pa.A.mode != pg.A.mode || (pa.A.mode == OP_TMA3D && pa.A.cps != pg.A.cps))
        return fail(SPNGD_ERR_SHAPE_MISMATCH, "wgrad: layer %d operands disagree on the K layout", li);
      GemmProblem p{};
      p.A = pg.A;  // rows: output channels, K: samples x positions (conv: sum_s G_s A_s^T)
      p.B = pa.A;  // rows: c_in k^2 / d_in
      p.M = int32_t(L.d.g);
      p.N = int32_t(L.d.a);
      p.K = pa.K;
      p.mode = EPI_DENSE;
      p.alpha = float(1.0 / double(B));
      p.beta = 0.f;
      p.C = dW;
      p.ldc = L.d.a;
      plan_problem_tiles(int(o->wprobs.size()), p, false, p.K + kTileK, o->witems, nullptr, &slot, 0.0, nullptr);
      o->wprobs.push_back(p);
    }
    std::stable_sort(o->witems.begin(), o->witems.end(), [](const GemmWorkItem& x, const GemmWorkItem& y) {
      return (x.k1 - x.k0) > (y.k1 - y.k0);
    });
    o->wvariant = gemm_variant(o->wprobs.data(), int(o->wprobs.size()));
    o->d_wprobs = dev_upload(o->wprobs, own);
    o->d_witems = dev_upload(o->witems, own);
    o->d_wbn = dev_upload(o->wbn, own);
  }
  o->d_bnm = dev_upload(o->bnm, own);
  o->d_pis = dev_upload(o->pis, own);
  o->d_unpacks = dev_upload(o->unpacks, own);
  // inverse plans: one per matrix size class (owned matrices of equal n share
  // identical recursion schedules and batch into the same launches); classes
  // run concurrently on their own streams.
  o->overlap_ok = !o->cfg.stale && o->cfg.bn_mode == 0;
  o->overlap_on = o->overlap_ok && getenv("SPNGD_NO_OVERLAP") == nullptr;
  {
    int least = 0, greatest = 0;
    SPNGD_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    o->inv_prio = greatest;
  }
  {
    // class key: (wave, size); waves only matter when overlapping
    std::vector<std::pair<int, int64_t>> keys;
    auto mwave = [&](size_t m) { return o->overlap_ok ? wave_of(o->layers[mat_layer[m]].d) : 0; };
    for (size_t m = 0; m < mats.size(); ++m) keys.push_back({mwave(m), -mats[m].n});
    std::sort(keys.begin(), keys.end());  // earliest wave, then largest (critical path) first
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    for (const auto& key : keys) {
      o->inv.emplace_back();
      spngd_opt::InvClass& c = o->inv.back();
      c.wave = key.first;
      for (size_t m = 0; m < mats.size(); ++m)
        if (mwave(m) == key.first && mats[m].n == -key.second) {
          c.mats.push_back(mats[m]);
          c.mat_layer.push_back(mat_layer[m]);
        }
      InversePlan sizing;
      plan_inverse(c.mats, nullptr, sizing, false);
      c.ws = o->alloc(sizing.workspace_floats);
      plan_inverse(c.mats, c.ws, c.plan, false);
      c.d_probs = dev_upload(c.plan.probs, own);
      c.d_items = dev_upload(c.plan.items, own);
      c.d_bases = dev_upload(c.plan.bases, own);
      if (o->cfg.stale) {  // room for a re-planned subset (never larger than the full class plan)
        c.d_probs_dyn = dev_upload(c.plan.probs, own);
        c.d_items_dyn = reinterpret_cast<GemmWorkItem*>(
            o->alloc((c.plan.item_bound * sizeof(GemmWorkItem) + sizeof(float) - 1) / sizeof(float)));
        if (!c.d_items_dyn) return fail(SPNGD_ERR_CUDA, "opt: allocation failed");
        c.d_bases_dyn = dev_upload(c.plan.bases, own);
      }
      SPNGD_CUDA_TRY(cudaStreamCreateWithPriority(&c.stream, cudaStreamNonBlocking,
                                                  o->overlap_ok ? o->inv_prio : 0));
      SPNGD_CUDA_TRY(cudaEventCreateWithFlags(&c.done, cudaEventDisableTiming));
    }
    SPNGD_CUDA_TRY(cudaEventCreateWithFlags(&o->inv_fork, cudaEventDisableTiming));
  }
  o->d_scal = o->alloc(2);
  o->use_graph = getenv("SPNGD_NO_GRAPH") == nullptr;
  if (bnf) {
    o->d_ilv = dev_upload(o->ilv, own);
    o->d_bnf_unpacks = dev_upload(o->bnf_unpacks, own);
    if (o->cfg.stale) o->d_bnf_unpacks_dyn = dev_upload(o->bnf_unpacks, own);
    for (int k = 0; k < 2; ++k) o->d_bnf_upd[k] = dev_upload(o->bnf_upd[k], own);
  }
  if (o->cfg.sgd) {  // plain-gradient update over every owned layer (fisher.cpp:320-333, 348-356)
    for (int li = 0; li < n; ++li) {
      LayerState& L = o->layers[li];
      if (L.owner != o->rank) continue;
      const int64_t cnt = L.d.kind == SPNGD_BN ? 2 * L.d.g : L.d.g * L.d.a;
      o->sgd_tasks.push_back({o->ag + int64_t(o->rank) * o->seg_ag + L.off_W, L.V,
                              o->rs_recv + o->seg_stat + L.off_dW, cnt});
    }
    o->d_sgd = dev_upload(o->sgd_tasks, own);
  }
  // precondition plan
  PrecondPlan psz;
  rc = plan_precondition(preqs.data(), int(preqs.size()), 0.0, 0.0, nullptr, nullptr, psz, nullptr, ptri.data());
  if (rc) return rc;
  float* ptmp = o->alloc(psz.tmp_floats);
  rc = plan_precondition(preqs.data(), int(preqs.size()), 0.0, 0.0, ptmp, o->d_norms, o->pplan, o->d_scal,
                         ptri.data());
  if (rc) return rc;
  for (int q = 0; q < o->pplan.stages; ++q) {
    o->d_pp[q] = dev_upload(o->pplan.probs[q], own);
    o->d_pi[q] = dev_upload(o->pplan.items[q], own);
  }
  o->d_rescale = dev_upload(o->pplan.rescale, own);
  if (o->overlap_ok && !o->cfg.sgd && !o->inv.empty()) {  // early / late precondition parts
    int last = 0;
    for (const auto& c : o->inv) last = std::max(last, c.wave);
    o->pre_cut = last;
    std::vector<std::vector<int>> layer_classes(o->layers.size());
    for (size_t ci = 0; ci < o->inv.size(); ++ci)
      for (int li : o->inv[ci].mat_layer) layer_classes[size_t(li)].push_back(int(ci));
    // part key: the layer's class with the longest recursion (-1: late part)
    std::vector<int> keys;
    std::vector<int> key_of(preqs.size(), -1);
    for (size_t i = 0; i < preqs.size(); ++i) {
      const int li = preq_layer[i];
      if (wave_of(o->layers[li].d) >= last || layer_classes[size_t(li)].empty()) continue;
      int best = -1;
      for (int ci : layer_classes[size_t(li)])
        if (best < 0 || o->inv[size_t(ci)].plan.rounds.size() > o->inv[size_t(best)].plan.rounds.size()) best = ci;
      key_of[i] = best;
      if (std::find(keys.begin(), keys.end(), best) == keys.end()) keys.push_back(best);
    }
    const size_t n_late = size_t(std::count(key_of.begin(), key_of.end(), -1));
    if (!keys.empty() && n_late > 0) {
      auto build = [&](spngd_opt::PrePart& pp, int key) -> int {
        std::vector<spngd_precond_req> part;
        std::vector<PrecondTri> tri;
        for (size_t i = 0; i < preqs.size(); ++i) {
          if (key_of[i] != key) continue;
          part.push_back(preqs[i]);
          tri.push_back(ptri[i]);
          for (int ci : layer_classes[size_t(preq_layer[i])])
            if (std::find(pp.wait.begin(), pp.wait.end(), ci) == pp.wait.end()) pp.wait.push_back(ci);
        }
        PrecondPlan sz;
        int rc2 = plan_precondition(part.data(), int(part.size()), 0.0, 0.0, nullptr, nullptr, sz, nullptr, tri.data());
        if (rc2) return rc2;
        float* tmp = o->alloc(sz.tmp_floats);
        pp.d_norms = reinterpret_cast<double*>(o->alloc(2 * part.size() + 2));
        if ((rc2 = plan_precondition(part.data(), int(part.size()), 0.0, 0.0, tmp, pp.d_norms, pp.plan, o->d_scal,
                                     tri.data())))
          return rc2;
        for (int q = 0; q < pp.plan.stages; ++q) {
          pp.d_pp[q] = dev_upload(pp.plan.probs[q], own);
          pp.d_pi[q] = dev_upload(pp.plan.items[q], own);
        }
        pp.d_rescale = dev_upload(pp.plan.rescale, own);
        return SPNGD_OK;
      };
      o->pre_early.resize(keys.size());
      for (size_t k = 0; k < keys.size(); ++k) {
        spngd_opt::PrePart& pp = o->pre_early[k];
        if ((rc = build(pp, keys[k]))) return rc;
        SPNGD_CUDA_TRY(cudaStreamCreateWithFlags(&pp.stream, cudaStreamNonBlocking));
        SPNGD_CUDA_TRY(cudaEventCreateWithFlags(&pp.done, cudaEventDisableTiming));
      }
      if ((rc = build(o->pre_late, -1))) return rc;
      // One GPU: the late part runs inside the schedule too, as soon as every
      // inverse (the step's status) and the BN determinant check are done
      // (world > 1 agrees on the status with a collective in phase 4 first).
      o->pre_late.wait.clear();
      for (size_t ci = 0; ci < o->inv.size(); ++ci) o->pre_late.wait.push_back(int(ci));
      // world > 1: its stages before the update (temporaries only) still run
      // inside the schedule; the update stage and the rescale follow the
      // status agreement in phase 4
      o->late_in_overlap = o->world == 1;
      SPNGD_CUDA_TRY(cudaStreamCreateWithFlags(&o->pre_late.stream, cudaStreamNonBlocking));
      SPNGD_CUDA_TRY(cudaEventCreateWithFlags(&o->pre_late.done, cudaEventDisableTiming));
      // failure atomicity: the replica and the early layers' velocities
      const int64_t nag = int64_t(o->world) * o->seg_ag;
      o->snap.push_back({o->ag, o->alloc(size_t(nag)), nag});
      for (size_t i = 0; i < preqs.size(); ++i) {
        if (key_of[i] < 0) continue;
        const LayerState& L = o->layers[size_t(preq_layer[i])];
        const int64_t cnt = L.d.g * L.d.a;
        o->snap.push_back({L.V, o->alloc(size_t(cnt)), cnt});
      }
      for (const auto& t : o->snap) {
        if (!t.save) return fail(SPNGD_ERR_CUDA, "opt: snapshot allocation failed");
        o->snap_max = std::max(o->snap_max, t.n);
      }
      o->d_snap = dev_upload(o->snap, own);
      SPNGD_CUDA_TRY(cudaStreamCreateWithFlags(&o->snap_stream, cudaStreamNonBlocking));
      SPNGD_CUDA_TRY(cudaEventCreateWithFlags(&o->snap_fork, cudaEventDisableTiming));
      SPNGD_CUDA_TRY(cudaEventCreateWithFlags(&o->snap_done, cudaEventDisableTiming));
      o->pre_split = true;
    }
  }
  o->d_bnu = dev_upload(o->bnu, own);
  for (auto& e : o->ev) SPNGD_CUDA_TRY(cudaEventCreate(&e));
  // plan entry -> statistic maps (filtered launches: stale gating, overlap waves)
  auto stat_of_ptr = [&](const float* p) {
    for (size_t q = 0; q < o->stats.size(); ++q) {
      const StatState& st = o->stats[q];
      const float* b = o->rs_send + int64_t(st.owner) * o->seg_stat + st.off;
      if (p >= b && p < b + st.count) return int(q);
    }
    return -1;
  };
  for (const auto& t : o->fplan.reduce) o->reduce_stat.push_back(stat_of_ptr(t.packed_out));
  for (int q : o->reduce_stat)
    if (q < 0) return fail(SPNGD_ERR_INVALID, "opt: unmapped reduction task");
  if (o->overlap_ok) {
    int nw = 0;
    for (const auto& c : o->inv) nw = std::max(nw, c.wave + 1);
    for (const auto& L : o->layers) nw = std::max(nw, wave_of(L.d) + 1);
    o->waves.resize(size_t(nw));
    for (const auto& it : o->fplan.items)
      o->waves[wave_of(o->layers[o->stats[o->prob_stat[it.problem]].layer].d)].items.push_back(it);
    for (size_t i = 0; i < o->fplan.reduce.size(); ++i)
      o->waves[wave_of(o->layers[o->stats[o->reduce_stat[i]].layer].d)].reduce.push_back(o->fplan.reduce[i]);
    for (size_t k = 0; k < o->pi_layer.size(); ++k) {
      spngd_opt::Wave& wv = o->waves[wave_of(o->layers[o->pi_layer[k]].d)];
      wv.pis.push_back(o->pis[k]);
      wv.unpacks.push_back(o->unpacks[2 * k]);
      wv.unpacks.push_back(o->unpacks[2 * k + 1]);
      wv.max_n = std::max({wv.max_n, o->unpacks[2 * k].n, o->unpacks[2 * k + 1].n});
    }
    for (const StatState& st : o->stats) {
      spngd_opt::Wave& wv = o->waves[wave_of(o->layers[st.layer].d)];
      wv.owner_ops.push_back({o->rs_send + int64_t(st.owner) * o->seg_stat + st.off, o->rs_recv + st.off, st.count,
                              st.owner});
    }
    {  // world > 1: NCCL + owner prep; world 1: pi + unpack beside the next wave's SYRK
      SPNGD_CUDA_TRY(cudaStreamCreateWithPriority(&o->comm_stream, cudaStreamNonBlocking, o->inv_prio));
      SPNGD_CUDA_TRY(cudaEventCreateWithFlags(&o->comm_fork, cudaEventDisableTiming));
      SPNGD_CUDA_TRY(cudaEventCreateWithFlags(&o->comm_done, cudaEventDisableTiming));
    }
    for (const auto& t : o->fplan.repacks) {  // per-wave repacks (host-input steps)
      int q = -1;
      for (size_t f = 0; f < freqs.size(); ++f)
        if (freqs[f].x == t.src) q = o->prob_stat[f];
      if (q < 0) return fail(SPNGD_ERR_INVALID, "opt: unmapped repack task");
      spngd_opt::Wave& wv = o->waves[wave_of(o->layers[o->stats[q].layer].d)];
      wv.repacks.push_back(t);
      wv.repack_max = std::max(wv.repack_max, t.n * t.dim * t.hw);
    }
    // Host-input sub-waves of the last wave: 8 layer groups of equal SYRK work,
    // in layer order (e2e A/B: 1 / 2 / 4 / 8 groups 87.3 / 85.2 / 84.3 / 83.5 ms).
    {
      spngd_opt::Wave& wv = o->waves.back();
      o->sub_of_layer.assign(o->layers.size(), -1);
      std::vector<double> work(o->layers.size(), 0.0);
      double total = 0;
      for (const auto& it : wv.items) {
        const int li = o->stats[o->prob_stat[it.problem]].layer;
        work[size_t(li)] += double(it.k1 - it.k0);
        total += double(it.k1 - it.k0);
      }
      static const int kSubs = getenv("SPNGD_SUBWAVES") ? std::max(1, atoi(getenv("SPNGD_SUBWAVES"))) : 8;
      double acc = 0;
      for (size_t li = 0; li < o->layers.size() && total > 0; ++li) {
        if (work[li] <= 0) continue;
        o->sub_of_layer[li] = std::min(kSubs - 1, int(acc / total * kSubs));
        acc += work[li];
      }
      if (total > 0) {
        wv.subs.resize(kSubs);
        for (const auto& it : wv.items)  // wave order kept: pair items first in every sub
          wv.subs[size_t(o->sub_of_layer[size_t(o->stats[o->prob_stat[it.problem]].layer)])].items.push_back(it);
        for (auto& sb : wv.subs) {
          sb.d_items = dev_upload(sb.items, own);
          SPNGD_CUDA_TRY(cudaEventCreateWithFlags(&sb.ready, cudaEventDisableTiming));
        }
      }
    }
    for (auto& wv : o->waves) {
      wv.d_repacks = dev_upload(wv.repacks, own);
      SPNGD_CUDA_TRY(cudaEventCreateWithFlags(&wv.in_ready, cudaEventDisableTiming));
      SPNGD_CUDA_TRY(cudaEventCreateWithFlags(&wv.ready, cudaEventDisableTiming));
      wv.d_items = dev_upload(wv.items, own);
      wv.d_reduce = dev_upload(wv.reduce, own);
      wv.d_pis = dev_upload(wv.pis, own);
      wv.d_unpacks = dev_upload(wv.unpacks, own);
      SPNGD_CUDA_TRY(cudaEventCreateWithFlags(&wv.fork, cudaEventDisableTiming));
    }
  }
  if (o->cfg.stale) {
    for (const auto& t : o->fplan.repacks) {
      int q = -1;
      for (size_t f = 0; f < freqs.size(); ++f)
        if (freqs[f].x == t.src) q = o->prob_stat[f];
      o->repack_stat.push_back(q);
    }
    o->d_fitems_dyn = dev_upload(o->fplan.items, own);
    o->d_freduce_dyn = dev_upload(o->fplan.reduce, own);
    o->d_repack_dyn = dev_upload(o->fplan.repacks, own);
    o->d_bnm_dyn = dev_upload(o->bnm, own);
    o->d_pis_dyn = dev_upload(o->pis, own);
    o->d_unpacks_dyn = dev_upload(o->unpacks, own);
    std::vector<StatJob> sr(o->stats.size());
    o->d_statreq = dev_upload(sr, own);
    o->d_dist = reinterpret_cast<double*>(o->alloc(8 * o->stats.size(), true));
    SPNGD_CUDA_TRY(cudaMallocHost(&o->h_dist, 4 * sizeof(double) * o->stats.size()));
    SPNGD_CUDA_TRY(cudaEventCreateWithFlags(&o->dist_ev, cudaEventDisableTiming));
    static const char* kinds[3] = {"A", "G", "F"};
    for (auto& st : o->stats) {
      const std::string id = std::string(kinds[st.kind]) + ":" + std::to_string(st.layer);
      st.tr = spngd_tracker_create(id.c_str(), o->cfg.stale_alpha);
      if (st.owner == o->rank) {
        st.snap[0] = o->alloc(size_t(st.count));
        st.snap[1] = o->alloc(size_t(st.count));
        if (!st.snap[0] || !st.snap[1]) return fail(SPNGD_ERR_CUDA, "opt: snapshot allocation failed");
      }
    }
  }
  SPNGD_CUDA_TRY(cudaDeviceSynchronize());
  return SPNGD_OK;
}

}  // namespace

extern "C" {

int spngd_plan_layout(const spngd_layer_desc* descs, int n, int W, spngd_layout_entry* out, int64_t* seg_stat,
                      int64_t* seg_grad, int64_t* seg_ag) {
  return spngd_plan_layout_ex(descs, n, W, 0, out, seg_stat, seg_grad, seg_ag);
}

int spngd_plan_layout_ex(const spngd_layer_desc* descs, int n, int W, int flags, spngd_layout_entry* out,
                         int64_t* seg_stat, int64_t* seg_grad, int64_t* seg_ag) {
  if (!descs || !out || n <= 0 || W < 1) return fail(SPNGD_ERR_INVALID, "spngd_plan_layout: bad argument");
  const bool bn_full = (flags & SPNGD_LEDGER_BN_FULL) != 0;
  // ownership: LPT on inverse + precondition cost, deterministic tie-break
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int x, int y) { return layer_cost(descs[x], bn_full) > layer_cost(descs[y], bn_full); });
  std::vector<double> load(W, 0.0);
  for (int li : order) {
    const int r = int(std::min_element(load.begin(), load.end()) - load.begin());
    out[li].owner = r;
    load[r] += layer_cost(descs[li], bn_full);
  }
  // owner-major segment layouts (statistics, gradients, weights), 64-float
  // aligned entries, in layer order
  std::vector<int64_t> st_fill(W, 0), gr_fill(W, 0), ag_fill(W, 0);
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
      e.off_M = place(st_fill[r], bn_full ? (2 * d.g) * (2 * d.g + 1) / 2 : 3 * d.g);
      e.off_dW = place(gr_fill[r], 2 * d.g);
      e.off_W = place(ag_fill[r], 2 * d.g);
    } else {
      e.off_A = place(st_fill[r], d.a * (d.a + 1) / 2);
      e.off_G = place(st_fill[r], d.g * (d.g + 1) / 2);
      e.off_dW = place(gr_fill[r], d.g * d.a);
      e.off_W = place(ag_fill[r], d.g * d.a);
    }
  }
  if (seg_stat) *seg_stat = std::max<int64_t>(64, *std::max_element(st_fill.begin(), st_fill.end()));
  if (seg_grad) *seg_grad = std::max<int64_t>(64, *std::max_element(gr_fill.begin(), gr_fill.end()));
  if (seg_ag) *seg_ag = std::max<int64_t>(64, *std::max_element(ag_fill.begin(), ag_fill.end()));
  return SPNGD_OK;
}

int spngd_opt_create(spngd_ctx* ctx, const spngd_layer_desc* layers, int n_layers, const spngd_opt_config* cfg,
                     spngd_opt** out) {
  SPNGD_CTX_SCOPE(ctx);
  if (!ctx || !layers || n_layers <= 0 || !cfg || !out) return fail(SPNGD_ERR_INVALID, "spngd_opt_create: bad argument");
  if (!(cfg->lambda > 0.0)) return fail(SPNGD_ERR_NOT_POSITIVE_DEFINITE, "OptimizerConfig: lambda must be > 0");
  if (cfg->batch < 1) return fail(SPNGD_ERR_EMPTY_BATCH, "spngd_opt_create: empty per-rank batch");
  if (cfg->stale && !(cfg->stale_alpha > 0.0)) return fail(SPNGD_ERR_INVALID, "spngd_opt_create: stale_alpha must be > 0");
  if (cfg->fisher_mode != 0 && cfg->fisher_mode != 1) return fail(SPNGD_ERR_INVALID, "spngd_opt_create: unknown fisher_mode");
  if (cfg->sgd && cfg->stale) return fail(SPNGD_ERR_INVALID, "spngd_opt_create: sgd has no statistics to gate");
  if (cfg->bn_mode != 0 && cfg->bn_mode != 1) return fail(SPNGD_ERR_INVALID, "spngd_opt_create: unknown bn_mode");
  if (cfg->elem_size != 0 && cfg->elem_size != 2 && cfg->elem_size != 4 && cfg->elem_size != 8)
    return fail(SPNGD_ERR_INVALID, "spngd_opt_create: elem_size must be 2, 4 or 8");
  for (int i = 0; i < n_layers; ++i) {
    const auto& d = layers[i];
    if (d.kind < 0 || d.kind > 2 || d.g <= 0 || (d.kind != SPNGD_BN && (d.a <= 0 || d.hw <= 0)))
      return fail(SPNGD_ERR_SHAPE_MISMATCH, "spngd_opt_create: layer %d has an invalid shape", i);
  }
  auto* o = new spngd_opt();
  o->ctx = ctx;
  o->cfg = *cfg;
  if (o->cfg.elem_size == 0) o->cfg.elem_size = 4;
  o->descs.assign(layers, layers + n_layers);
  o->world = ctx->world;
  o->rank = ctx->rank;
  SPNGD_CUDA_TRY(cudaSetDevice(ctx->device));
  int rc = build(o, layers, n_layers);
  if (!rc) {
    o->d_flag = reinterpret_cast<double*>(o->alloc(2, true));
    if (!o->d_flag) rc = fail(SPNGD_ERR_CUDA, "spngd_opt_create: allocation failed");
  }
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
    case 2: return L.off_dW >= 0 ? o->rs_send + int64_t(o->world) * o->seg_stat + int64_t(L.owner) * o->seg_grad + L.off_dW : nullptr;
    case 3: return o->ag + int64_t(L.owner) * o->seg_ag + L.off_W;
    case 4: return mine ? L.V : nullptr;
    case 5: return L.gg;
    case 6: return L.gb;
    case 7:  // the step keeps only T = L^-1: the inverse T^T T is formed on request
      if (L.d.kind == SPNGD_BN) {
        if (!mine || !L.Finv) return nullptr;
        if (ld) *ld = L.ldf;
        const DenseMatrix m{L.Finv, L.tlf, L.tuf, L.ldf, 2 * L.d.g};
        return materialize_inverse(o->ctx, m) == SPNGD_OK ? L.Finv : nullptr;
      }
      [[fallthrough]];
    case 8: {
      const bool a = which == 7;
      if (ld) *ld = a ? L.lda : L.ldg;
      float* X = a ? L.Ainv : L.Ginv;
      if (!mine || !X) return nullptr;
      const DenseMatrix m{X, a ? L.tla : L.tlg, a ? L.tua : L.tug, a ? L.lda : L.ldg, a ? L.d.a : L.d.g};
      return materialize_inverse(o->ctx, m) == SPNGD_OK ? X : nullptr;
    }
    case 9: return (mine && L.off_A >= 0) ? o->rs_recv + L.off_A : nullptr;
    case 10: return (mine && L.off_G >= 0) ? o->rs_recv + L.off_G : nullptr;
    case 11: return (mine && L.off_M >= 0) ? o->rs_recv + L.off_M : nullptr;
    case 12: if (ld) *ld = int64_t(o->world) * o->seg_ag; return o->ag;  // all weight replicas
    case 13: return L.grad_s;
    case 14: return L.gg_s;
    case 15: return L.gb_s;
    case 16: return L.raw;
    case 17: return L.dy;
    case 18: return L.xh;
    default: return nullptr;
  }
}

}  // extern "C"

namespace {

// Stage 5 (AllGatherV of the updated weights, dist.cpp:646-663).  With peers
// attached the owners' rescale pass already stored W'' into every replica
// over NVLink; the rest (BN, unrescaled layers) goes by one peer-copy launch,
// and a one-word all-reduce orders every rank's stores before its step ends.
int issue_allgather(spngd_opt* o) {
  spngd_ctx* ctx = o->ctx;
  if (o->world == 1) return SPNGD_OK;
  if (!o->p2p) return spngd_all_gather(ctx, o->ag + int64_t(o->rank) * o->seg_ag, o->ag, o->seg_ag);
  int rc = launch_peer_copy(ctx, o->d_pcopy, int(o->pcopy.size()), o->pcopy_max);
  if (!rc) rc = comm_allreduce_sum_f64(ctx, o->d_barrier, 1);
  return rc;
}

// Raw conv inputs -> the im2col captures the GEMMs read (net.cpp:199-219);
// BN dY / x_hat -> captures, moments and payload (net.cpp:467-475,
// fisher.cpp:147-185, dist.cpp:364-371) in one launch.
int issue_inputs(spngd_opt* o) {
  int rc = launch_im2col(o->ctx, o->d_i2c, int(o->i2c.size()));
  if (!rc && o->bn_inputs)
    rc = launch_bn_backward(o->ctx, o->d_bnx_tasks, o->d_bnx_items, int64_t(o->bnx.items.size()), o->d_bnx_slots,
                            o->d_bnx_cnt);
  return rc;
}

// cfg.wgrad: this rank's shard-mean gradients from the captures (grad_payload,
// dist.cpp:315-391) into the gradient region of the send buffer.  The dense
// GEMMs read the factor plan's operands, so the factor repack must have run
// (repack = true runs it here first).
int issue_wgrad(spngd_opt* o, bool repack) {
  if (!o->cfg.wgrad) return SPNGD_OK;
  spngd_ctx* ctx = o->ctx;
  int rc = SPNGD_OK;
  if (repack) rc = launch_repack(ctx, o->d_repack, int(o->fplan.repacks.size()), o->fplan.repack_max);
  if (!rc) rc = launch_repack(ctx, o->d_wrepack, int(o->wplan.repacks.size()), o->wplan.repack_max);
  if (!rc && !o->witems.empty()) {
    rc = launch_gemm(o->d_wprobs, o->d_witems, int(o->witems.size()), o->d_partials, ctx->d_status, ctx->stream,
                     o->wvariant);
    ctx->launches++;
  }
  if (!rc) rc = launch_bn_grad_payload(ctx, o->d_wbn, int(o->wbn.size()), o->wbn_maxc);
  return rc;
}

// The six phases of one step.  Each phase is captured once into its own CUDA
// graph; phase events are recorded between graph launches.
int issue_phase(spngd_opt* o, int phase) {
  spngd_ctx* ctx = o->ctx;
  cudaStream_t s = ctx->stream;
  int rc = SPNGD_OK;
  switch (phase) {
    case 0:  // Stages 1-3 local part: factor SYRK into the RS send buffer.
      rc = issue_inputs(o);
      if (!rc) rc = launch_bn_interleave(ctx, o->d_ilv, int(o->ilv.size()), o->ilv_max);
      if (!rc) rc = launch_repack(ctx, o->d_repack, int(o->fplan.repacks.size()), o->fplan.repack_max);
      if (!rc) rc = issue_wgrad(o, false);
      if (rc) return rc;
      rc = launch_factor_gemm(ctx, o->fplan, o->d_fprobs, o->fplan.n_pair, o->d_fitems, int(o->fplan.items.size()),
                              o->d_partials, s);
      ctx->launches++;
      return rc;
    case 1:  // split-K reduction + BN moments.
      rc = launch_syrk_reduce(o->d_freduce, int(o->fplan.reduce.size()), o->d_partials, s);
      ctx->launches += !o->fplan.reduce.empty();
      if (!rc) rc = launch_bn_moments(ctx, o->d_bnm, int(o->bnm.size()), o->bnm_maxc);
      return rc;
    case 2:  // Stages 2-3: ReduceScatterV of A, G/F and grads (dist.cpp:510-537).
      if (o->world > 1) {
        if (o->p2p_rs) {  // statistics already in the owners' inboxes: barrier + slot means
          rc = comm_allreduce_sum_f64(ctx, o->d_barrier, 1);
          if (!rc) rc = launch_slot_mean(ctx, o->d_means, int(o->means.size()), o->means_max);
        } else {
          rc = spngd_reduce_scatter_mean(ctx, o->rs_send, o->rs_recv, o->seg_stat);
        }
        if (!rc)
          rc = spngd_reduce_scatter_mean(ctx, o->rs_send + int64_t(o->world) * o->seg_stat, o->rs_recv + o->seg_stat,
                                         o->seg_grad);
      }
      return rc;
    case 3: {  // Stage 4a: pi, damping, inverse (dist.cpp:539-602); size classes
               // fork onto their own streams and join.
      rc = launch_pi(ctx, o->d_pis, int(o->pis.size()));
      if (!rc) rc = launch_unpack(ctx, o->d_unpacks, int(o->unpacks.size()), o->max_n);
      if (!rc) rc = launch_unpack(ctx, o->d_bnf_unpacks, int(o->bnf_unpacks.size()), o->bnf_maxn);
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
      // No parameter is written once any inverse / BN block of any rank failed
      // (the kernels read the status word): agree on it, then check every
      // BN determinant before the first update.
      rc = agree_status(ctx, o->d_flag);
      if (!rc && !(o->ov_now && o->pre_split && o->late_in_overlap))
        rc = launch_bn_det_check(ctx, o->d_bnu, int(o->bnu.size()), o->bnu_maxc, o->cfg.lambda);
      if (!rc && o->ov_now && o->pre_split)  // undo the early parts of a failed step
        rc = launch_snapshot(ctx, o->d_snap, int(o->snap.size()), o->snap_max, true);
      if (rc) return rc;
      if (o->ov_now && o->pre_split) {  // the early parts already ran inside the wave schedule
        const spngd_opt::PrePart& pp = o->pre_late;
        if (!o->late_in_overlap)  // the stages before the update ran in the schedule
          rc = run_precondition_stages(ctx, pp.plan, pp.d_pp, pp.d_pi, pp.d_rescale, pp.d_norms,
                                       pp.plan.stages > 1 ? pp.plan.stages - 1 : 0, pp.plan.stages, true);
      } else {
        rc = run_precondition(ctx, o->pplan, o->d_pp, o->d_pi, o->d_rescale, o->d_norms);
      }
      if (!rc)
        rc = launch_bn_update(ctx, o->d_bnu, int(o->bnu.size()), o->bnu_maxc, o->cfg.lambda, 0.0, 0.0, o->d_scal);
      for (int k = 0; k < 2 && !rc; ++k)
        rc = launch_bn_full_update(ctx, o->d_bnf_upd[k], int(o->bnf_upd[k].size()), o->bnf_maxn, 0.0, 0.0, o->d_scal);
      return rc;
    case 5:  // Stage 5: AllGatherV of the updated weights (dist.cpp:646-663), in place.
      return issue_allgather(o);
  }
  return SPNGD_OK;
}

// Phases 0-3 of a full step with the inverse recursion of each wave
// overlapping the factor SYRK of the later waves.  world > 1: a communication
// stream reduces each wave's statistics to their owners as soon as the wave's
// factors are reduced locally (grouped ncclReduce(avg), the reference's
// ReduceScatterV of stage 3 split by wave, dist.cpp:510-537), runs the
// owner's pi + unpack, and forks the owner's recursion; the gradient
// reduce-scatter runs on it at the start.  The phase events 1-3 are recorded
// on the main stream after the last wave's SYRK, after its reduction + BN
// moments, and after the communication stream joins (external event nodes
// when captured), so phase 3 is what the inverse adds beyond the rest.
int issue_overlap(spngd_opt* o, bool capturing, bool host_in = false) {
  spngd_ctx* ctx = o->ctx;
  cudaStream_t s = ctx->stream;
  const bool dist = o->world > 1;
  cudaStream_t prep = o->comm_stream ? o->comm_stream : s;
  auto mark = [&](cudaEvent_t e) {
    return capturing ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal) : cudaEventRecord(e, s);
  };
  static const bool tracing = getenv("SPNGD_STEP_TRACE") != nullptr;
  auto tmark = [&](cudaStream_t st, std::string label) {
    if (!tracing || capturing) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, st);
    o->trace.emplace_back(std::move(label), e);
  };
  int rc = SPNGD_OK;
  if (!host_in) {  // host-input steps expand / repack wave by wave as the captures land
    rc = issue_inputs(o);
    if (!rc) rc = launch_repack(ctx, o->d_repack, int(o->fplan.repacks.size()), o->fplan.repack_max);
    if (!rc) rc = issue_wgrad(o, false);
    if (rc) return rc;
  }
  if (dist) {  // gradients: independent of the factors
    SPNGD_CUDA_TRY(cudaEventRecord(o->comm_fork, s));
    SPNGD_CUDA_TRY(cudaStreamWaitEvent(prep, o->comm_fork, 0));
    ctx->stream = prep;
    rc = spngd_reduce_scatter_mean(ctx, o->rs_send + int64_t(o->world) * o->seg_stat, o->rs_recv + o->seg_stat,
                                   o->seg_grad);
    ctx->stream = s;
    if (rc) return rc;
  }
  if (o->pre_split) {
    // Save what the early parts overwrite before the step is known good: one
    // short full-machine burst ahead of wave 0 (a small long-running grid or
    // copy-engine copies held SMs / HBM against the inverse chains and cost
    // 0.8-0.9 ms per step).  World > 1: peers store into this replica only
    // after a later wave barrier on prep.
    SPNGD_CUDA_TRY(cudaEventRecord(o->snap_fork, s));
    SPNGD_CUDA_TRY(cudaStreamWaitEvent(o->snap_stream, o->snap_fork, 0));
    ctx->stream = o->snap_stream;
    rc = launch_snapshot(ctx, o->d_snap, int(o->snap.size()), o->snap_max, false);
    ctx->stream = s;
    if (rc) return rc;
    SPNGD_CUDA_TRY(cudaEventRecord(o->snap_done, o->snap_stream));
    if (prep != s) SPNGD_CUDA_TRY(cudaStreamWaitEvent(prep, o->snap_done, 0));
  }
  const int nw = int(o->waves.size());
  for (int w = 0; w < nw; ++w) {
    spngd_opt::Wave& wv = o->waves[w];
    const bool last = w == nw - 1;
    const bool by_sub = host_in && last && wv.subs_usable();
    if (by_sub) {  // each layer group's SYRK as soon as its captures have landed
      for (auto& sb : wv.subs) {
        SPNGD_CUDA_TRY(cudaStreamWaitEvent(s, sb.ready, 0));
        rc = launch_im2col(ctx, sb.d_i2c, int(sb.i2c.size()));
        if (rc) return rc;
        if (sb.items.empty()) continue;
        rc = launch_factor_gemm(ctx, o->fplan, o->d_fprobs, count_pair_items(o->fplan, sb.items), sb.d_items,
                                int(sb.items.size()), o->d_partials, s);
        if (rc) return rc;
        ctx->launches++;
      }
      SPNGD_CUDA_TRY(cudaStreamWaitEvent(s, wv.in_ready, 0));  // the wave's BN inputs
    } else if (host_in) {
      SPNGD_CUDA_TRY(cudaStreamWaitEvent(s, wv.in_ready, 0));
      rc = launch_im2col(ctx, wv.d_i2c, int(wv.i2c.size()));
      if (!rc) rc = launch_repack(ctx, wv.d_repacks, int(wv.repacks.size()), wv.repack_max);
      if (rc) return rc;
    }
    if (!by_sub && !wv.items.empty()) {
      rc = launch_factor_gemm(ctx, o->fplan, o->d_fprobs, count_pair_items(o->fplan, wv.items), wv.d_items,
                              int(wv.items.size()),
                              o->d_partials, s);
      if (rc) return rc;
      ctx->launches++;
    }
    tmark(s, "wave " + std::to_string(w) + " syrk end");
    if (last) SPNGD_CUDA_TRY(mark(o->ev[1]));
    // The wave's split-K reduction and (last wave) BN moments run on the
    // high-priority prep stream: on the main stream they queued behind the
    // next wave's SYRK CTAs and the inverse streams' high-priority work.
    if (prep != s) {
      SPNGD_CUDA_TRY(cudaEventRecord(wv.ready, s));
      SPNGD_CUDA_TRY(cudaStreamWaitEvent(prep, wv.ready, 0));
    }
    ctx->stream = prep;
    rc = launch_syrk_reduce(wv.d_reduce, int(wv.reduce.size()), o->d_partials, prep);
    ctx->launches += !wv.reduce.empty();
    if (!rc && last) rc = launch_bn_moments(ctx, o->d_bnm, int(o->bnm.size()), o->bnm_maxc);
    if (rc) {
      ctx->stream = s;
      return rc;
    }
    if (last) SPNGD_CUDA_TRY(mark(o->ev[2]));  // main stream: after the last SYRK (reduction on prep)
    if (dist && o->p2p_rs) {  // every rank's wave-w statistics have landed in the inboxes after this
      rc = comm_allreduce_sum_f64(ctx, o->d_barrier, 1);
      if (!rc) rc = launch_slot_mean(ctx, wv.d_means, int(wv.means.size()), wv.means_max);
    } else if (dist) {
      rc = comm_reduce_to_owners(ctx, wv.owner_ops);
    }
    if (!rc) rc = launch_pi(ctx, wv.d_pis, int(wv.pis.size()));
    if (!rc) rc = launch_unpack(ctx, wv.d_unpacks, int(wv.unpacks.size()), wv.max_n);
    ctx->stream = s;
    if (rc) return rc;
    SPNGD_CUDA_TRY(cudaEventRecord(wv.fork, prep));
    tmark(prep, "wave " + std::to_string(w) + " reduce+pi+unpack end");
    for (auto& c : o->inv) {
      if (c.wave != w) continue;
      SPNGD_CUDA_TRY(cudaStreamWaitEvent(c.stream, wv.fork, 0));
      ctx->stream = c.stream;
      ctx->launch_prio = o->inv_prio;
      rc = run_inverse(ctx, c.plan, c.d_probs, c.d_items, c.d_bases);
      ctx->launch_prio = 0;
      ctx->stream = s;
      if (rc) return rc;
      SPNGD_CUDA_TRY(cudaEventRecord(c.done, c.stream));
      tmark(c.stream, "wave " + std::to_string(w) + " inverse class n=" +
                          std::to_string(c.mats.empty() ? 0 : c.mats[0].n) + " x" + std::to_string(c.mats.size()) +
                          " end (" + std::to_string(c.plan.rounds.size()) + " rounds)");
    }
  }
  if (prep != s) {
    SPNGD_CUDA_TRY(cudaEventRecord(o->comm_done, prep));
    SPNGD_CUDA_TRY(cudaStreamWaitEvent(s, o->comm_done, 0));
  }
  if (o->pre_split) {  // early precondition parts, each as soon as its inverse classes are done
    for (size_t k = 0; k < o->pre_early.size(); ++k) {
      const spngd_opt::PrePart& pp = o->pre_early[k];
      for (int ci : pp.wait) SPNGD_CUDA_TRY(cudaStreamWaitEvent(pp.stream, o->inv[size_t(ci)].done, 0));
      SPNGD_CUDA_TRY(cudaStreamWaitEvent(pp.stream, o->snap_done, 0));
      ctx->stream = pp.stream;
      rc = run_precondition(ctx, pp.plan, pp.d_pp, pp.d_pi, pp.d_rescale, pp.d_norms);
      ctx->stream = s;
      if (rc) return rc;
      SPNGD_CUDA_TRY(cudaEventRecord(pp.done, pp.stream));
      tmark(pp.stream, "early precondition part " + std::to_string(k) + " end");
      SPNGD_CUDA_TRY(cudaStreamWaitEvent(s, pp.done, 0));
    }
    if (o->late_in_overlap) {  // every inverse + the last wave's BN moments (its fork on prep) done
      spngd_opt::PrePart& pp = o->pre_late;
      for (int ci : pp.wait) SPNGD_CUDA_TRY(cudaStreamWaitEvent(pp.stream, o->inv[size_t(ci)].done, 0));
      SPNGD_CUDA_TRY(cudaStreamWaitEvent(pp.stream, o->waves.back().fork, 0));
      SPNGD_CUDA_TRY(cudaStreamWaitEvent(pp.stream, o->snap_done, 0));
      ctx->stream = pp.stream;
      rc = launch_bn_det_check(ctx, o->d_bnu, int(o->bnu.size()), o->bnu_maxc, o->cfg.lambda);
      if (!rc) rc = run_precondition(ctx, pp.plan, pp.d_pp, pp.d_pi, pp.d_rescale, pp.d_norms);
      ctx->stream = s;
      if (rc) return rc;
      SPNGD_CUDA_TRY(cudaEventRecord(pp.done, pp.stream));
      tmark(pp.stream, "late precondition end");
      SPNGD_CUDA_TRY(cudaStreamWaitEvent(s, pp.done, 0));
    } else if (o->pre_late.plan.stages > 1) {  // world > 1: the late part's stages before its update
      spngd_opt::PrePart& pp = o->pre_late;
      for (int ci : pp.wait) SPNGD_CUDA_TRY(cudaStreamWaitEvent(pp.stream, o->inv[size_t(ci)].done, 0));
      SPNGD_CUDA_TRY(cudaStreamWaitEvent(pp.stream, o->waves.back().fork, 0));
      ctx->stream = pp.stream;
      rc = run_precondition_stages(ctx, pp.plan, pp.d_pp, pp.d_pi, pp.d_rescale, pp.d_norms, 0, pp.plan.stages - 1,
                                   false);
      ctx->stream = s;
      if (rc) return rc;
      SPNGD_CUDA_TRY(cudaEventRecord(pp.done, pp.stream));
      tmark(pp.stream, "late precondition stages before the update end");
      SPNGD_CUDA_TRY(cudaStreamWaitEvent(s, pp.done, 0));
    }
  }
  SPNGD_CUDA_TRY(mark(o->ev[3]));
  for (auto& c : o->inv) SPNGD_CUDA_TRY(cudaStreamWaitEvent(s, c.done, 0));
  return SPNGD_OK;
}

}  // namespace

namespace {

template <typename T>
int upload_async(spngd_ctx* ctx, T* dst, const std::vector<T>& v) {
  // pageable source: staged before the call returns, so v may die right after
  if (!v.empty()) SPNGD_CUDA_TRY(cudaMemcpyAsync(dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
  return SPNGD_OK;
}

// Advances every tracker from the distances of the last refresh step
// (StaleTracker::on_refresh, stale.hpp:100-114).
int stale_apply_pending(spngd_opt* o) {
  if (o->pending.empty()) return SPNGD_OK;
  SPNGD_CUDA_TRY(cudaEventSynchronize(o->dist_ev));
  for (const auto& p : o->pending) {
    double d[4];  // the device reduction leaves weighted squares
    for (int k = 0; k < 4; ++k) d[k] = std::sqrt(std::max(o->h_dist[4 * p.q + k], 0.0));
    int64_t next = 0;
    int reason = 0;
    int rc = spngd_tracker_on_refresh(o->stats[p.q].tr, o->pending_step, p.has1, d[0], d[1], p.has2, d[2], d[3], &next,
                                      &reason);
    if (rc) return rc;
  }
  o->pending.clear();
  return SPNGD_OK;
}

// Partial refresh: the factor, reduction, RS and inverse work of the due
// statistics only (dist.cpp:510-602).
int stale_partial_phase(spngd_opt* o, int phase) {
  spngd_ctx* ctx = o->ctx;
  cudaStream_t s = ctx->stream;
  const auto& due = o->due;
  int rc = SPNGD_OK;
  switch (phase) {
    case 0: {
      std::vector<RepackTask> rp;
      for (size_t i = 0; i < o->fplan.repacks.size(); ++i)
        if (o->repack_stat[i] >= 0 && due[o->repack_stat[i]]) rp.push_back(o->fplan.repacks[i]);
      std::vector<GemmWorkItem> it;
      for (const auto& w : o->fplan.items)
        if (due[o->prob_stat[w.problem]]) it.push_back(w);
      if ((rc = upload_async(ctx, o->d_repack_dyn, rp))) return rc;
      if ((rc = upload_async(ctx, o->d_fitems_dyn, it))) return rc;
      rc = issue_inputs(o);  // every conv capture (cheap next to the refresh; wgrad needs them all)
      if (!rc) rc = launch_bn_interleave(ctx, o->d_ilv, int(o->ilv.size()), o->ilv_max);  // full BN (cheap, all layers)
      if (o->cfg.wgrad) {  // every layer's gradient is due every step: full repack + grad_payload
        if (!rc) rc = issue_wgrad(o, true);
      } else if (!rc) {
        rc = launch_repack(ctx, o->d_repack_dyn, int(rp.size()), o->fplan.repack_max);
      }
      if (!rc && !it.empty()) {
        rc = launch_factor_gemm(ctx, o->fplan, o->d_fprobs, count_pair_items(o->fplan, it), o->d_fitems_dyn,
                                int(it.size()),
                                o->d_partials, s);
        ctx->launches++;
      }
      return rc;
    }
    case 1: {
      std::vector<SyrkReduceTask> red;
      for (size_t i = 0; i < o->fplan.reduce.size(); ++i)
        if (due[o->reduce_stat[i]]) red.push_back(o->fplan.reduce[i]);
      std::vector<spngd_bn_moments_req> bm;
      for (size_t i = 0; i < o->bnm.size(); ++i)
        if (due[o->bnm_stat[i]]) bm.push_back(o->bnm[i]);
      if ((rc = upload_async(ctx, o->d_freduce_dyn, red))) return rc;
      if ((rc = upload_async(ctx, o->d_bnm_dyn, bm))) return rc;
      rc = launch_syrk_reduce(o->d_freduce_dyn, int(red.size()), o->d_partials, s);
      ctx->launches += !red.empty();
      if (!rc) rc = launch_bn_moments(ctx, o->d_bnm_dyn, int(bm.size()), o->bnm_maxc);
      return rc;
    }
    case 2: {  // gradients always; due statistics reduced to their owners
      if (o->world > 1) {
        rc = spngd_reduce_scatter_mean(ctx, o->rs_send + int64_t(o->world) * o->seg_stat, o->rs_recv + o->seg_stat,
                                       o->seg_grad);
        if (rc) return rc;
      }
      std::vector<OwnerReduce> ops;
      for (size_t q = 0; q < o->stats.size(); ++q) {
        if (!due[q]) continue;
        const StatState& st = o->stats[q];
        ops.push_back({o->rs_send + int64_t(st.owner) * o->seg_stat + st.off, o->rs_recv + st.off, st.count, st.owner});
      }
      return o->world > 1 ? comm_reduce_to_owners(ctx, ops) : SPNGD_OK;
    }
    case 3: {  // re-invert both factors of every owned layer with a refreshed A or G
               // (and every refreshed full BN block, damp_bn_full at dist.cpp:583-584)
      std::vector<char> touched(o->layers.size(), 0);
      for (size_t q = 0; q < o->stats.size(); ++q)
        if (due[q] && (o->stats[q].kind != 2 || o->cfg.bn_mode == 1)) touched[o->stats[q].layer] = 1;
      std::vector<UnpackTask> bups;
      for (size_t k = 0; k < o->bnf_layer.size(); ++k)
        if (touched[o->bnf_layer[k]]) bups.push_back(o->bnf_unpacks[k]);
      if (!bups.empty()) {
        if ((rc = upload_async(ctx, o->d_bnf_unpacks_dyn, bups))) return rc;
        if ((rc = launch_unpack(ctx, o->d_bnf_unpacks_dyn, int(bups.size()), o->bnf_maxn))) return rc;
      }
      std::vector<PiTask> pis;
      std::vector<UnpackTask> ups;
      for (size_t k = 0; k < o->pi_layer.size(); ++k)
        if (touched[o->pi_layer[k]]) {
          pis.push_back(o->pis[k]);
          ups.push_back(o->unpacks[2 * k]);
          ups.push_back(o->unpacks[2 * k + 1]);
        }
      if (pis.empty() && bups.empty()) return SPNGD_OK;
      if (!pis.empty()) {
        if ((rc = upload_async(ctx, o->d_pis_dyn, pis))) return rc;
        if ((rc = upload_async(ctx, o->d_unpacks_dyn, ups))) return rc;
        rc = launch_pi(ctx, o->d_pis_dyn, int(pis.size()));
        if (!rc) rc = launch_unpack(ctx, o->d_unpacks_dyn, int(ups.size()), o->max_n);
        if (rc) return rc;
      }
      std::vector<cudaEvent_t> joins;
      for (auto& c : o->inv) {
        std::vector<DenseMatrix> sub;
        for (size_t m = 0; m < c.mats.size(); ++m)
          if (touched[c.mat_layer[m]]) sub.push_back(c.mats[m]);
        if (sub.empty()) continue;
        plan_inverse(sub, c.ws, c.dyn, false);
        if (c.dyn.items.size() > c.plan.item_bound || c.dyn.probs.size() > c.plan.probs.size() ||
            c.dyn.bases.size() > c.plan.bases.size())
          return fail(SPNGD_ERR_INVALID, "stale re-plan exceeds the class plan's buffers");
        if ((rc = upload_async(ctx, c.d_probs_dyn, c.dyn.probs))) return rc;
        if ((rc = upload_async(ctx, c.d_items_dyn, c.dyn.items))) return rc;
        if ((rc = upload_async(ctx, c.d_bases_dyn, c.dyn.bases))) return rc;
        // the class stream forks after this class's descriptor uploads (on s)
        SPNGD_CUDA_TRY(cudaEventRecord(o->inv_fork, s));
        SPNGD_CUDA_TRY(cudaStreamWaitEvent(c.stream, o->inv_fork, 0));
        ctx->stream = c.stream;
        rc = run_inverse(ctx, c.dyn, c.d_probs_dyn, c.d_items_dyn, c.d_bases_dyn);
        ctx->stream = s;
        if (rc) return rc;
        SPNGD_CUDA_TRY(cudaEventRecord(c.done, c.stream));
        joins.push_back(c.done);
      }
      // join after every class is issued: the classes' recursions run concurrently
      for (cudaEvent_t e : joins) SPNGD_CUDA_TRY(cudaStreamWaitEvent(s, e, 0));
      return SPNGD_OK;
    }
  }
  return SPNGD_OK;
}

// The owners compare every refreshed statistic with its retained snapshots
// (similar(), stale.hpp:56-64, on the device), rotate the snapshots, and all
// ranks receive the distances for the next step's tracker update.
int stale_similarity(spngd_opt* o, int64_t step) {
  spngd_ctx* ctx = o->ctx;
  cudaStream_t s = ctx->stream;
  std::vector<StatJob> reqs;
  int64_t max_rows = 0;
  o->pending.clear();
  for (size_t q = 0; q < o->stats.size(); ++q) {
    if (!o->due[q]) continue;
    StatState& st = o->stats[q];
    o->pending.push_back({int(q), st.nsnap >= 1 ? 1 : 0, st.nsnap >= 2 ? 1 : 0});
    if (st.owner == o->rank) {
      spngd_stat_req r{};
      r.x = o->rs_recv + st.off;
      r.x1 = st.nsnap >= 1 ? st.snap[st.first] : nullptr;
      r.x2 = st.nsnap >= 2 ? st.snap[st.first ^ 1] : nullptr;
      r.n = st.dim;
      r.kind = (st.kind == 2 && o->cfg.bn_mode == 0) ? 1 : 0;  // full BN blocks are packed symmetric
      r.out4 = o->d_dist + 4 * q;
      // snapshot rotation (x2 <- x1, x1 <- x) fused into the distance pass:
      // x lands in x2's slot after the kernel has read x2 there
      reqs.push_back(StatJob{r, st.snap[st.first ^ 1]});
      max_rows = std::max(max_rows, r.kind == 0 ? r.n : (3 * r.n + 255) / 256);
      st.first ^= 1;
    }
    st.nsnap = std::min(2, st.nsnap + 1);
  }
  o->pending_step = step;
  SPNGD_CUDA_TRY(cudaMemsetAsync(o->d_dist, 0, 4 * sizeof(double) * o->stats.size(), s));
  int rc = upload_async(ctx, o->d_statreq, reqs);
  if (!rc && !reqs.empty()) rc = launch_stat_distance(ctx, o->d_statreq, int(reqs.size()), max_rows);
  if (rc) return rc;
  rc = comm_allreduce_sum_f64(ctx, o->d_dist, 4 * int64_t(o->stats.size()));
  if (rc) return rc;
  SPNGD_CUDA_TRY(cudaMemcpyAsync(o->h_dist, o->d_dist, 4 * sizeof(double) * o->stats.size(), cudaMemcpyDeviceToHost, s));
  SPNGD_CUDA_TRY(cudaEventRecord(o->dist_ev, s));
  return SPNGD_OK;
}

}  // namespace

namespace {

// One step; host_in: the inputs arrive wave by wave on the copy stream
// (spngd_opt_step_host) -- direct launches, no graphs, per-wave waits.
int step_impl(spngd_opt* o, int64_t step, double eta, double momentum, bool host_in) {
  spngd_ctx* ctx = o->ctx;
  cudaStream_t s = ctx->stream;
  // Host scalars of this step -> device (outside the graphs).  Pageable
  // source: staged before cudaMemcpyAsync returns, so no host sync.
  const float scal[2] = {float(eta), float(momentum)};
  SPNGD_CUDA_TRY(cudaMemcpyAsync(o->d_scal, scal, sizeof(scal), cudaMemcpyHostToDevice, s));
  // stale gating: which statistics refresh this step (dist.cpp:431-444)
  bool full = true, any = true;
  if (o->cfg.stale) {
    int rc = stale_apply_pending(o);
    if (rc) return rc;
    o->due.assign(o->stats.size(), 0);
    int64_t n_due = 0;
    for (size_t q = 0; q < o->stats.size(); ++q) {
      o->due[q] = char(spngd_tracker_should_refresh(o->stats[q].tr, step));
      n_due += o->due[q];
    }
    o->last_due = n_due;
    full = n_due == int64_t(o->stats.size());
    any = n_due > 0;
  }
  // Overlapped single-GPU schedule: phases 0-3 run as one unit (own graphs).
  const bool ov = o->overlap_on && full;
  {  // CommLedger rows of this step (dist.cpp:511-537, 661-662) and NCCL bytes
    const unsigned char* due = o->cfg.stale ? reinterpret_cast<const unsigned char*>(o->due.data()) : nullptr;
    const int nl = int(o->descs.size());
    const int lf = (o->cfg.sgd ? SPNGD_LEDGER_SGD : 0) | (o->cfg.bn_mode == 1 ? SPNGD_LEDGER_BN_FULL : 0);
    const int64_t nrows = spngd_ledger_step_rows(o->descs.data(), nl, o->world, step, due, o->cfg.elem_size, lf,
                                                 nullptr, 0);
    if (nrows < 0) return int(-nrows);
    const size_t at = o->ledger.size();
    o->ledger.resize(at + size_t(nrows));
    spngd_ledger_step_rows(o->descs.data(), nl, o->world, step, due, o->cfg.elem_size, lf, o->ledger.data() + at,
                           nrows);
    o->wire_stat = o->wire_grad = o->wire_ag = 0;
    if (o->world > 1) {
      const int64_t W = o->world;
      if (o->cfg.sgd) {
        o->wire_stat = 0;
      } else if (o->p2p_rs) {  // NVLink stores of the statistics owned by the other ranks
        for (const auto& st : o->stats)
          if (st.owner != o->rank) o->wire_stat += st.count * int64_t(sizeof(float));
      } else if (full && !ov) {
        o->wire_stat = W * o->seg_stat * int64_t(sizeof(float));  // one ncclReduceScatter
      } else {  // grouped ncclReduce of the due statistics to their owners
        for (size_t q = 0; q < o->stats.size(); ++q)
          if (full || o->due[q]) o->wire_stat += o->stats[q].count * int64_t(sizeof(float));
      }
      o->wire_grad = W * o->seg_grad * int64_t(sizeof(float));
      o->wire_ag = o->seg_ag * int64_t(sizeof(float));  // P2P: the owned ranges, to world-1 peers
    }
  }
  if (o->cfg.sgd) {  // Stage 3 grads RS, plain update, Stage 5 AG (dist.cpp:522-537, 604-620, 646-663)
    const int64_t l0 = ctx->launches;
    for (int ph = 0; ph < 6; ++ph) {
      SPNGD_CUDA_TRY(cudaEventRecord(o->ev[ph], s));
      int rc = SPNGD_OK;
      if (ph == 0 && o->cfg.wgrad) {
        rc = issue_inputs(o);
        if (!rc) rc = issue_wgrad(o, true);
      } else if (ph == 2 && o->world > 1)
        rc = spngd_reduce_scatter_mean(ctx, o->rs_send + int64_t(o->world) * o->seg_stat, o->rs_recv + o->seg_stat,
                                       o->seg_grad);
      else if (ph == 4) {
        rc = agree_status(ctx, o->d_flag);
        if (!rc) rc = launch_sgd_update(ctx, o->d_sgd, int(o->sgd_tasks.size()), o->d_scal);
      }
      else if (ph == 5)
        rc = issue_allgather(o);
      if (rc) return rc;
    }
    SPNGD_CUDA_TRY(cudaEventRecord(o->ev[6], s));
    o->launches = ctx->launches - l0;
    o->timed = true;
    return SPNGD_OK;
  }
  o->ov_now = ov;
  if (!o->trace.empty()) {  // keep the last step's trace only
    SPNGD_CUDA_TRY(cudaStreamSynchronize(s));
    for (auto& t : o->trace) cudaEventDestroy(t.second);
    o->trace.clear();
  }
  bool& ready = ov ? o->graphs_ready_ov : o->graphs_ready;
  const bool capture = o->use_graph && !ready && full && !host_in;
  const int64_t l0 = ctx->launches;
  for (int ph = 0; ph < 6; ++ph) {
    if (ov && ph >= 1 && ph <= 3) continue;  // inside issue_overlap
    SPNGD_CUDA_TRY(cudaEventRecord(o->ev[ph], s));
    const bool gated = ph <= 3 && !full;
    auto issue = [&](bool capturing) {
      return (ov && ph == 0) ? issue_overlap(o, capturing, host_in) : issue_phase(o, ph);
    };
    if (gated) {
      if (any || ph == 2 || (ph == 0 && o->cfg.wgrad)) {
        int rc = stale_partial_phase(o, ph);
        if (rc) return rc;
      }
    } else if (!o->use_graph || host_in || (!ready && !capture)) {
      int rc = issue(false);
      if (rc) return rc;
    } else {
      cudaGraph_t* graphs = ov ? o->graphs_ov : o->graphs;
      cudaGraphExec_t* execs = ov ? o->graph_ov_exec : o->graph_exec;
      if (capture) {
        SPNGD_CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        int rc = issue(true);
        cudaGraph_t g = nullptr;
        cudaError_t e = cudaStreamEndCapture(s, &g);
        if (rc) {
          if (g) cudaGraphDestroy(g);
          return rc;
        }
        if (e != cudaSuccess) return fail_cuda(e, "cudaStreamEndCapture");
        graphs[ph] = g;
        SPNGD_CUDA_TRY(cudaGraphInstantiateWithFlags(&execs[ph], g, cudaGraphInstantiateFlagUseNodePriority));
      }
      SPNGD_CUDA_TRY(cudaGraphLaunch(execs[ph], s));
    }
    if (ph == 3 && o->cfg.stale && any) {
      int rc = stale_similarity(o, step);
      if (rc) return rc;
    }
  }
  SPNGD_CUDA_TRY(cudaEventRecord(o->ev[6], s));
  if (capture || !o->use_graph || !full || host_in) o->launches = ctx->launches - l0;
  if (capture) ready = true;
  o->timed = true;
  return SPNGD_OK;
}

// Bytes of per-step input buffer `which` of layer L (0 if it has none).
int64_t input_floats(const spngd_opt* o, const LayerState& L, int which) {
  const int64_t B = o->cfg.batch;
  const bool bn = L.d.kind == SPNGD_BN;
  switch (which) {
    case 0: return bn ? 0 : B * L.d.a * L.d.hw;
    case 1: case 13: return bn ? 0 : B * L.d.g * L.d.hw;
    case 2: return bn ? 2 * L.d.g : L.d.g * L.d.a;
    case 5: case 6: case 14: case 15: return bn ? B * L.d.g : 0;
    case 16: return L.raw ? L.raw_floats : 0;
    case 17: case 18: return (bn && L.dy) ? B * L.d.g * L.bn_S : 0;
    default: return 0;
  }
}

}  // namespace

extern "C" {

int spngd_opt_step(spngd_opt* o, int64_t step, double eta, double momentum) {
  SPNGD_CTX_SCOPE(o ? o->ctx : nullptr);
  if (!o) return fail(SPNGD_ERR_INVALID, "spngd_opt_step: opt is NULL");
  return step_impl(o, step, eta, momentum, false);
}

int spngd_opt_step_host(spngd_opt* o, int64_t step, double eta, double momentum, const spngd_host_input* in, int n,
                        float* host_weights_out) {
  SPNGD_CTX_SCOPE(o ? o->ctx : nullptr);
  if (!o || (n > 0 && !in)) return fail(SPNGD_ERR_INVALID, "spngd_opt_step_host: null argument");
  spngd_ctx* ctx = o->ctx;
  cudaStream_t s = ctx->stream;
  struct Copy { float* dst; const void* src; int64_t bytes; int wave; int sub; };
  std::vector<Copy> copies;
  // BN dY / x_hat feed the gradient payload, which the step needs first: with
  // BN inputs the copies simply precede the step
  const bool pipelined = o->overlap_on && o->overlap_ok && !o->cfg.wgrad && !o->cfg.sgd && !o->waves.empty() &&
                         !o->bn_inputs;
  for (int i = 0; i < n; ++i) {
    if (in[i].layer < 0 || in[i].layer >= int(o->layers.size()) || !in[i].host)
      return fail(SPNGD_ERR_INVALID, "spngd_opt_step_host: bad input %d", i);
    LayerState& L = o->layers[in[i].layer];
    float* dst = spngd_opt_buffer(o, in[i].layer, in[i].which, nullptr);
    const int64_t cnt = input_floats(o, L, in[i].which);
    if (!dst || cnt <= 0) return fail(SPNGD_ERR_INVALID, "spngd_opt_step_host: layer %d has no input %d", in[i].layer,
                                      in[i].which);
    // dW first (the gradient reduce-scatter and every update need it), then
    // the captures in wave order (wave_of, largest factors first)
    const int wave = in[i].which == 2 ? -1 : (pipelined ? wave_of(L.d) : 0);
    // last wave: by sub-wave (layer group), inputs of no group (BN) last
    int sub = 0;
    if (pipelined && wave == int(o->waves.size()) - 1 && o->waves.back().subs_usable()) {
      const int g = o->sub_of_layer[size_t(in[i].layer)];
      sub = g >= 0 ? g : int(o->waves.back().subs.size());
    }
    copies.push_back({dst, in[i].host, cnt * int64_t(sizeof(float)), wave, sub});
  }
  std::stable_sort(copies.begin(), copies.end(),
                   [](const Copy& x, const Copy& y) { return x.wave != y.wave ? x.wave < y.wave : x.sub < y.sub; });
  if (!pipelined) {  // same inputs, copied before the step on its stream
    for (const Copy& c : copies) SPNGD_CUDA_TRY(cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyHostToDevice, s));
    int rc = step_impl(o, step, eta, momentum, false);
    if (rc) return rc;
  } else {
    if (!o->h2d_stream) {
      SPNGD_CUDA_TRY(cudaStreamCreateWithFlags(&o->h2d_stream, cudaStreamNonBlocking));
      SPNGD_CUDA_TRY(cudaEventCreateWithFlags(&o->h2d_start, cudaEventDisableTiming));
      SPNGD_CUDA_TRY(cudaEventCreateWithFlags(&o->grads_ready, cudaEventDisableTiming));
    }
    // the copies overwrite inputs the previous step may still read
    SPNGD_CUDA_TRY(cudaEventRecord(o->h2d_start, s));
    SPNGD_CUDA_TRY(cudaStreamWaitEvent(o->h2d_stream, o->h2d_start, 0));
    size_t i = 0;
    for (; i < copies.size() && copies[i].wave < 0; ++i)
      SPNGD_CUDA_TRY(cudaMemcpyAsync(copies[i].dst, copies[i].src, copies[i].bytes, cudaMemcpyHostToDevice,
                                     o->h2d_stream));
    SPNGD_CUDA_TRY(cudaEventRecord(o->grads_ready, o->h2d_stream));
    for (int w = 0; w < int(o->waves.size()); ++w) {
      spngd_opt::Wave& wv = o->waves[w];
      const bool by_sub = w == int(o->waves.size()) - 1 && wv.subs_usable();
      for (int k = 0; k <= (by_sub ? int(wv.subs.size()) : 0); ++k) {
        for (; i < copies.size() && copies[i].wave == w && (!by_sub || copies[i].sub == k); ++i)
          SPNGD_CUDA_TRY(cudaMemcpyAsync(copies[i].dst, copies[i].src, copies[i].bytes, cudaMemcpyHostToDevice,
                                         o->h2d_stream));
        if (by_sub && k < int(wv.subs.size())) SPNGD_CUDA_TRY(cudaEventRecord(wv.subs[size_t(k)].ready, o->h2d_stream));
      }
      SPNGD_CUDA_TRY(cudaEventRecord(wv.in_ready, o->h2d_stream));
    }
    SPNGD_CUDA_TRY(cudaStreamWaitEvent(s, o->grads_ready, 0));
    int rc = step_impl(o, step, eta, momentum, true);
    if (rc) return rc;
    if (getenv("SPNGD_STEP_TRACE")) {  // the trace's ev[0] is the step start on s
      cudaEvent_t e;
      if (cudaEventCreate(&e) == cudaSuccess) {
        cudaEventRecord(e, o->h2d_stream);
        o->trace.emplace_back("host inputs: last H2D copy landed", e);
      }
    }
  }
  if (!host_weights_out) return SPNGD_OK;
  if (pipelined && o->world == 1 && o->pre_split) {
    // One GPU: the early-preconditioned layers' weights are final when that
    // part ends (no all-gather), so they stream back while the last inverse
    // wave and phase 4 still run; the rest follows the step.
    if (!o->d2h_stream) {
      SPNGD_CUDA_TRY(cudaStreamCreateWithFlags(&o->d2h_stream, cudaStreamNonBlocking));
      SPNGD_CUDA_TRY(cudaEventCreateWithFlags(&o->d2h_done, cudaEventDisableTiming));
    }
    for (const auto& pp : o->pre_early) SPNGD_CUDA_TRY(cudaStreamWaitEvent(o->d2h_stream, pp.done, 0));
    for (const LayerState& L : o->layers) {
      const int64_t cnt = L.d.kind == SPNGD_BN ? 2 * L.d.g : L.d.g * L.d.a;
      const bool early = L.d.kind != SPNGD_BN && wave_of(L.d) < o->pre_cut;
      SPNGD_CUDA_TRY(cudaMemcpyAsync(host_weights_out + L.off_W, o->ag + L.off_W, size_t(cnt) * sizeof(float),
                                     cudaMemcpyDeviceToHost, early ? o->d2h_stream : s));
    }
    SPNGD_CUDA_TRY(cudaEventRecord(o->d2h_done, o->d2h_stream));
    SPNGD_CUDA_TRY(cudaStreamWaitEvent(s, o->d2h_done, 0));
    return SPNGD_OK;
  }
  SPNGD_CUDA_TRY(cudaMemcpyAsync(host_weights_out, o->ag, size_t(o->world) * o->seg_ag * sizeof(float),
                                 cudaMemcpyDeviceToHost, s));
  return SPNGD_OK;
}

int64_t spngd_ledger_step_rows(const spngd_layer_desc* layers, int n, int world, int64_t step,
                               const unsigned char* due, int elem_size, int flags, spngd_ledger_row* out,
                               int64_t cap) {
  if (!layers || n <= 0 || world < 1) return -int64_t(SPNGD_ERR_INVALID);
  if (elem_size == 0) elem_size = 4;
  const bool bn_full = (flags & SPNGD_LEDGER_BN_FULL) != 0;
  const bool sgd = (flags & SPNGD_LEDGER_SGD) != 0;
  // plan_statistics order (dist.cpp:256-269): per layer A, G or F
  struct Stat { int layer, kind; int64_t len; bool due; };
  std::vector<Stat> plan;
  for (int li = 0; li < n && !sgd; ++li) {
    const spngd_layer_desc& d = layers[li];
    if (d.kind == SPNGD_BN) {
      const int64_t c = d.g;
      plan.push_back({li, SPNGD_ID_F, bn_full ? (2 * c) * (2 * c + 1) / 2 : 3 * c, true});
    } else {
      plan.push_back({li, SPNGD_ID_A, d.a * (d.a + 1) / 2, true});
      plan.push_back({li, SPNGD_ID_G, d.g * (d.g + 1) / 2, true});
    }
  }
  if (due)
    for (size_t q = 0; q < plan.size(); ++q) plan[q].due = due[q] != 0;
  auto grad_len = [&](int li) { return layers[li].kind == SPNGD_BN ? 2 * layers[li].g : layers[li].g * layers[li].a; };
  int64_t count = 0;
  auto row = [&](int stage, int coll, int kind, int layer, int64_t len, bool skipped) {
    if (out && count < cap) {
      spngd_ledger_row& r = out[count];
      r.step = step;
      r.stage = stage;
      r.collective = coll;
      r.id_kind = kind;
      r.layer = layer;
      r.elements = skipped ? 0 : (world > 1 ? len : 0);  // dist.cpp:214, 231
      r.bytes = r.elements * elem_size;
      r.skipped = skipped ? 1 : 0;
      r.pad_ = 0;
    }
    ++count;
  };
  // Stage 2: RSV_A over the due A payloads, then the skips (dist.cpp:511-520)
  for (const Stat& st : plan)
    if (st.kind == SPNGD_ID_A && st.due) row(2, SPNGD_RSV_A, st.kind, st.layer, st.len, false);
  for (const Stat& st : plan)
    if (st.kind == SPNGD_ID_A && !st.due) row(2, SPNGD_RSV_A, st.kind, st.layer, 0, true);
  // Stage 3: due G/F, every grad:l, then the skips (dist.cpp:522-537)
  for (const Stat& st : plan)
    if (st.kind != SPNGD_ID_A && st.due) row(3, SPNGD_RSV_G_F_GRAD, st.kind, st.layer, st.len, false);
  for (int li = 0; li < n; ++li) row(3, SPNGD_RSV_G_F_GRAD, SPNGD_ID_GRAD, li, grad_len(li), false);
  for (const Stat& st : plan)
    if (st.kind != SPNGD_ID_A && !st.due) row(3, SPNGD_RSV_G_F_GRAD, st.kind, st.layer, 0, true);
  // Stage 5: AGV_params w:0..L-1 (dist.cpp:646-662)
  for (int li = 0; li < n; ++li) row(5, SPNGD_AGV_PARAMS, SPNGD_ID_W, li, grad_len(li), false);
  return count;
}

int64_t spngd_opt_ledger(const spngd_opt* o, spngd_ledger_row* out, int64_t cap) {
  if (!o) return -int64_t(SPNGD_ERR_INVALID);
  const int64_t n = int64_t(o->ledger.size());
  if (out)
    for (int64_t i = 0; i < std::min(n, cap); ++i) out[i] = o->ledger[size_t(i)];
  return n;
}

int spngd_opt_enable_bn_inputs(spngd_opt* o, const int64_t* spatial) {
  SPNGD_CTX_SCOPE(o ? o->ctx : nullptr);
  if (!o || !spatial) return fail(SPNGD_ERR_INVALID, "spngd_opt_enable_bn_inputs: null argument");
  if (o->bn_inputs) return fail(SPNGD_ERR_INVALID, "spngd_opt_enable_bn_inputs: already enabled");
  if (o->graphs_ready || o->graphs_ready_ov || o->timed)
    return fail(SPNGD_ERR_INVALID, "spngd_opt_enable_bn_inputs: call before the first step");
  if (o->cfg.fisher_mode != 0)
    return fail(SPNGD_ERR_INVALID, "spngd_opt_enable_bn_inputs: OneMC needs the sampled-label backward's BN capture");
  if (o->cfg.sgd) return fail(SPNGD_ERR_INVALID, "spngd_opt_enable_bn_inputs: sgd has no BN statistics");
  const int64_t B = o->cfg.batch;
  // moments fused only when every BN statistic is built every step (unit
  // blocks, no stale gating); otherwise the existing moment / SYRK paths read
  // the captures this launch writes
  const bool fuse_moments = o->cfg.bn_mode == 0 && !o->cfg.stale;
  std::vector<spngd_bn_backward_req> reqs;
  size_t k = 0;
  for (size_t li = 0; li < o->layers.size(); ++li) {
    LayerState& L = o->layers[li];
    if (L.d.kind != SPNGD_BN) continue;
    if (spatial[li] <= 0) return fail(SPNGD_ERR_SHAPE_MISMATCH, "spngd_opt_enable_bn_inputs: layer %zu: S <= 0", li);
    L.bn_S = spatial[li];
    const size_t n = size_t(B * L.d.g * L.bn_S);
    L.dy = o->alloc(n);
    L.xh = o->alloc(n);
    if (!L.dy || !L.xh) return fail(SPNGD_ERR_CUDA, "opt: BN input allocation failed");
    float* m3 = nullptr;
    if (fuse_moments) {  // the bnm entries are in layer order
      while (k < o->bnm.size() && o->bnm[k].gg != L.gg) ++k;
      if (k == o->bnm.size()) return fail(SPNGD_ERR_INVALID, "spngd_opt_enable_bn_inputs: no moment slot for layer %zu", li);
      m3 = o->bnm[k].out3c;
    }
    float* pay = spngd_opt_buffer(o, int(li), 2, nullptr);
    reqs.push_back({L.dy, L.xh, B, L.d.g, L.bn_S, L.gg, L.gb, m3, pay});
  }
  int rc = plan_bn_backward(reqs, o->bnx);
  if (rc) return rc;
  o->d_bnx_tasks = dev_upload(o->bnx.tasks, o->owned);
  o->d_bnx_items = dev_upload(o->bnx.items, o->owned);
  o->d_bnx_slots = reinterpret_cast<double*>(o->alloc(size_t(2 * std::max<int64_t>(o->bnx.slots, 1) * 5)));
  o->d_bnx_cnt = reinterpret_cast<int*>(o->alloc(size_t(std::max<int64_t>(o->bnx.channels, 1)), true));
  if (!reqs.empty() && (!o->d_bnx_tasks || !o->d_bnx_items || !o->d_bnx_slots || !o->d_bnx_cnt))
    return fail(SPNGD_ERR_CUDA, "opt: upload failed");
  if (fuse_moments) o->bnm.clear();  // the fused launch writes the moments: no separate moment kernel
  o->bn_inputs = !reqs.empty();
  return SPNGD_OK;
}

int spngd_opt_enable_raw_inputs(spngd_opt* o, const spngd_conv_geom* geoms) {
  SPNGD_CTX_SCOPE(o ? o->ctx : nullptr);
  return spngd_opt_enable_raw_inputs_ex(o, geoms, 0);
}

int spngd_opt_enable_raw_inputs_ex(spngd_opt* o, const spngd_conv_geom* geoms, int implicit) {
  SPNGD_CTX_SCOPE(o ? o->ctx : nullptr);
  if (!o || !geoms) return fail(SPNGD_ERR_INVALID, "spngd_opt_enable_raw_inputs: null argument");
  if (o->raw_inputs) return fail(SPNGD_ERR_INVALID, "spngd_opt_enable_raw_inputs: already enabled");
  if (o->graphs_ready || o->graphs_ready_ov || o->timed)
    return fail(SPNGD_ERR_INVALID, "spngd_opt_enable_raw_inputs: call before the first step");
  const int64_t B = o->cfg.batch;
  // implicit = 0: im2col_kernel expands the raw input into the capture before
  // the SYRK (TMA-fed).  implicit = 1: the A-factor SYRK
  // (and the wgrad GEMM) gather the (ch, ky, kx) x (s, oy, ox) operand straight
  // from the raw input; the capture is never materialized and its buffer is
  // released.  The gather is LSU-bound (one 4-byte cp.async per element), so
  // the explicit expansion is the default.
  bool changed = false;
  for (size_t li = 0; li < o->layers.size(); ++li) {
    LayerState& L = o->layers[li];
    if (L.d.kind != SPNGD_CONV) continue;
    const spngd_conv_geom& g = geoms[li];
    int rc = check_conv_geom(g, L.d.a, L.d.hw);
    if (rc) return rc;
    if (g.k == 1 && g.stride == 1 && g.pad == 0) {  // the raw input is already the capture layout
      L.raw = L.act;
      L.raw_floats = B * L.d.a * L.d.hw;
      continue;
    }
    L.raw_floats = B * g.c_in * g.h * g.w;
    L.raw = o->alloc(size_t(L.raw_floats));
    if (!L.raw) return fail(SPNGD_ERR_CUDA, "opt: raw input allocation failed");
    if (!implicit) {
      o->i2c.push_back({L.raw, L.act, B, g});
      if (o->overlap_ok) {
        spngd_opt::Wave& wv = o->waves[wave_of(L.d)];
        wv.i2c.push_back(o->i2c.back());
        const int sub = &wv == &o->waves.back() ? o->sub_of_layer[li] : -1;
        if (sub >= 0 && size_t(sub) < wv.subs.size()) wv.subs[size_t(sub)].i2c.push_back(o->i2c.back());
      }
      continue;
    }
    if (L.fa < 0) return fail(SPNGD_ERR_INVALID, "opt: conv layer %zu has no factor problem", li);
    float* act = L.act;
    GemmProblem& p = o->fplan.probs[size_t(L.fa)];
    const float* old_op = p.A.ptr;  // the capture, or its K-contiguous repack
    make_im2col_operand(p.A, L.raw, int(g.c_in), int(g.h), int(g.w), int(g.k), int(g.stride), int(g.pad));
    p.B = p.A;
    // the capture's repack (hw % 4 != 0) has nothing left to do
    for (auto& t : o->fplan.repacks)
      if (t.src == act) t.n = 0;
    for (auto& wv : o->waves)
      for (auto& t : wv.repacks)
        if (t.src == act) t.n = 0;
    for (auto& wp : o->wprobs)  // wgrad reads the same operand
      if (wp.B.ptr == old_op) wp.B = p.A;
    for (size_t q = 0; q < o->owned.size(); ++q)
      if (o->owned[q] == act) {
        cudaFree(act);
        o->owned.erase(o->owned.begin() + long(q));
        break;
      }
    L.act = nullptr;
    changed = true;
  }
  if (changed) {
    auto put = [&](void* d, const void* h, size_t bytes) {
      return (bytes && d) ? cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice) : cudaSuccess;
    };
    SPNGD_CUDA_TRY(put(o->d_fprobs, o->fplan.probs.data(), o->fplan.probs.size() * sizeof(GemmProblem)));
    SPNGD_CUDA_TRY(put(o->d_repack, o->fplan.repacks.data(), o->fplan.repacks.size() * sizeof(RepackTask)));
    for (auto& wv : o->waves)
      SPNGD_CUDA_TRY(put(wv.d_repacks, wv.repacks.data(), wv.repacks.size() * sizeof(RepackTask)));
    if (!o->wprobs.empty()) {
      SPNGD_CUDA_TRY(put(o->d_wprobs, o->wprobs.data(), o->wprobs.size() * sizeof(GemmProblem)));
      o->wvariant = gemm_variant(o->wprobs.data(), int(o->wprobs.size()));
    }
  }
  if (!o->i2c.empty()) {
    for (auto& wv : o->waves) {
      wv.d_i2c = dev_upload(wv.i2c, o->owned);
      for (auto& sb : wv.subs) sb.d_i2c = dev_upload(sb.i2c, o->owned);
    }
    o->d_i2c = dev_upload(o->i2c, o->owned);
    if (!o->d_i2c) return fail(SPNGD_ERR_CUDA, "opt: upload failed");
  }
  o->raw_inputs = true;
  return SPNGD_OK;
}

int spngd_opt_ipc_handle(spngd_opt* o, void* out128) {
  SPNGD_CTX_SCOPE(o ? o->ctx : nullptr);
  if (!o || !out128) return fail(SPNGD_ERR_INVALID, "spngd_opt_ipc_handle: null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
  cudaIpcMemHandle_t h[2];
  memset(h, 0, sizeof(h));
  SPNGD_CUDA_TRY(cudaIpcGetMemHandle(&h[0], o->ag));
  if (!o->cfg.stale && o->world > 1) {  // statistics inbox for the fused reduce-scatter
    if (!o->inbox) o->inbox = o->alloc(size_t(o->world) * o->seg_stat, true);
    if (!o->inbox) return fail(SPNGD_ERR_CUDA, "opt: inbox allocation failed");
    SPNGD_CUDA_TRY(cudaIpcGetMemHandle(&h[1], o->inbox));
  }
  memcpy(out128, h, sizeof(h));
  return SPNGD_OK;
}

int spngd_opt_attach_peers(spngd_opt* o, const void* handles) {
  SPNGD_CTX_SCOPE(o ? o->ctx : nullptr);
  if (!o || !handles) return fail(SPNGD_ERR_INVALID, "spngd_opt_attach_peers: null argument");
  if (o->world < 2 || o->world > kMaxPeers + 1) return fail(SPNGD_ERR_INVALID, "spngd_opt_attach_peers: world must be 2..8");
  if (o->p2p) return fail(SPNGD_ERR_INVALID, "spngd_opt_attach_peers: already attached");
  if (o->graphs_ready || o->graphs_ready_ov || o->timed)
    return fail(SPNGD_ERR_INVALID, "spngd_opt_attach_peers: call before the first step");
  const auto* hs = static_cast<const cudaIpcMemHandle_t*>(handles);  // 2 per rank: replicas, inbox
  const bool fuse_rs = o->inbox != nullptr;
  for (int q = 0; q < o->world; ++q) {
    if (q == o->rank) continue;
    void* p = nullptr;
    SPNGD_CUDA_TRY(cudaIpcOpenMemHandle(&p, hs[2 * q], cudaIpcMemLazyEnablePeerAccess));
    o->peer_ag[q] = static_cast<float*>(p);
    if (fuse_rs) {
      SPNGD_CUDA_TRY(cudaIpcOpenMemHandle(&p, hs[2 * q + 1], cudaIpcMemLazyEnablePeerAccess));
      o->peer_inbox[q] = static_cast<float*>(p);
    }
  }
  if (fuse_rs) {  // statistics producers write into the owners' inbox slots; owners average
    const float* s0 = o->rs_send;
    const float* s1 = o->rs_send + int64_t(o->world) * o->seg_stat;
    auto remap = [&](float* p) -> float* {
      if (p < s0 || p >= s1) return p;
      const int64_t d = p - s0, owner = d / o->seg_stat, off = d - owner * o->seg_stat;
      float* base = owner == o->rank ? o->inbox : o->peer_inbox[owner];
      return base + int64_t(o->rank) * o->seg_stat + off;
    };
    for (auto& p : o->fplan.probs) p.C = remap(p.C);
    for (auto& t : o->fplan.reduce) t.packed_out = remap(t.packed_out);
    for (auto& r : o->bnm) r.out3c = remap(r.out3c);
    for (auto& t : o->bnx.tasks) t.out3c = t.out3c ? remap(t.out3c) : nullptr;
    auto put = [&](void* d, const void* h, size_t bytes) {
      return (bytes && d) ? cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice) : cudaSuccess;
    };
    SPNGD_CUDA_TRY(put(o->d_fprobs, o->fplan.probs.data(), o->fplan.probs.size() * sizeof(GemmProblem)));
    SPNGD_CUDA_TRY(put(o->d_freduce, o->fplan.reduce.data(), o->fplan.reduce.size() * sizeof(SyrkReduceTask)));
    SPNGD_CUDA_TRY(put(o->d_bnm, o->bnm.data(), o->bnm.size() * sizeof(spngd_bn_moments_req)));
    SPNGD_CUDA_TRY(put(o->d_bnx_tasks, o->bnx.tasks.data(), o->bnx.tasks.size() * sizeof(BnxTask)));
    for (auto& wv : o->waves) {
      for (auto& t : wv.reduce) t.packed_out = remap(t.packed_out);
      SPNGD_CUDA_TRY(put(wv.d_reduce, wv.reduce.data(), wv.reduce.size() * sizeof(SyrkReduceTask)));
    }
    for (const StatState& st : o->stats) {
      if (st.owner != o->rank) continue;
      const SlotMeanTask t{o->inbox + st.off, o->rs_recv + st.off, o->seg_stat, st.count, o->world, 0};
      o->means.push_back(t);
      o->means_max = std::max(o->means_max, st.count);
      if (o->overlap_ok) {
        spngd_opt::Wave& wv = o->waves[wave_of(o->layers[st.layer].d)];
        wv.means.push_back(t);
        wv.means_max = std::max(wv.means_max, st.count);
      }
    }
    o->d_means = dev_upload(o->means, o->owned);
    for (auto& wv : o->waves) wv.d_means = dev_upload(wv.means, o->owned);
    o->p2p_rs = true;
  }
  auto peers_of = [&](const float* local, float** dst) {
    const int64_t off = local - o->ag;
    int k = 0;
    for (int q = 0; q < o->world; ++q)
      if (q != o->rank) dst[k++] = o->peer_ag[q] + off;
    return k;
  };
  // rescaled layers: the rescale pass stores W'' to the peers too
  std::vector<char> covered(o->layers.size(), 0);
  if (!o->cfg.sgd) {
    for (auto& t : o->pplan.rescale) {
      t.n_peers = peers_of(t.W, t.peers);
      for (size_t li = 0; li < o->layers.size(); ++li)
        if (o->ag + int64_t(o->rank) * o->seg_ag + o->layers[li].off_W == t.W) covered[li] = 1;
    }
    if (!o->pplan.rescale.empty())
      SPNGD_CUDA_TRY(cudaMemcpy(o->d_rescale, o->pplan.rescale.data(), o->pplan.rescale.size() * sizeof(RescaleTask),
                                cudaMemcpyHostToDevice));
    std::vector<spngd_opt::PrePart*> parts;
    for (auto& pp : o->pre_early) parts.push_back(&pp);
    parts.push_back(&o->pre_late);
    for (auto* ppp : parts) {
      spngd_opt::PrePart& pp = *ppp;
      for (auto& t : pp.plan.rescale) t.n_peers = peers_of(t.W, t.peers);
      if (!pp.plan.rescale.empty())
        SPNGD_CUDA_TRY(cudaMemcpy(pp.d_rescale, pp.plan.rescale.data(), pp.plan.rescale.size() * sizeof(RescaleTask),
                                  cudaMemcpyHostToDevice));
    }
  }
  for (size_t li = 0; li < o->layers.size(); ++li) {
    const LayerState& L = o->layers[li];
    if (L.owner != o->rank || covered[li]) continue;
    PeerCopyTask t{};
    t.src = o->ag + int64_t(o->rank) * o->seg_ag + L.off_W;
    t.n = L.d.kind == SPNGD_BN ? 2 * L.d.g : L.d.g * L.d.a;
    t.n_peers = peers_of(t.src, t.dst);
    o->pcopy.push_back(t);
    o->pcopy_max = std::max(o->pcopy_max, t.n);
  }
  o->d_pcopy = dev_upload(o->pcopy, o->owned);
  o->d_barrier = reinterpret_cast<double*>(o->alloc(2, true));
  if ((!o->pcopy.empty() && !o->d_pcopy) || !o->d_barrier) return fail(SPNGD_ERR_CUDA, "opt: upload failed");
  o->p2p = true;
  return SPNGD_OK;
}

int spngd_opt_ledger_clear(spngd_opt* o) {
  SPNGD_CTX_SCOPE(o ? o->ctx : nullptr);
  if (!o) return fail(SPNGD_ERR_INVALID, "spngd_opt_ledger_clear: opt is NULL");
  o->ledger.clear();
  return SPNGD_OK;
}

int spngd_opt_wire_bytes(const spngd_opt* o, int64_t* stat_bytes, int64_t* grad_bytes, int64_t* ag_bytes) {
  if (!o) return fail(SPNGD_ERR_INVALID, "spngd_opt_wire_bytes: opt is NULL");
  if (stat_bytes) *stat_bytes = o->wire_stat;
  if (grad_bytes) *grad_bytes = o->wire_grad;
  if (ag_bytes) *ag_bytes = o->wire_ag;
  return SPNGD_OK;
}

int spngd_opt_stale_info(spngd_opt* o, int layer, int which, int64_t* t_x, int64_t* delta, int64_t* refresh_count,
                         int* due_last) {
  SPNGD_CTX_SCOPE(o ? o->ctx : nullptr);
  if (!o || !o->cfg.stale) return fail(SPNGD_ERR_INVALID, "spngd_opt_stale_info: stale gating is off");
  int rc = stale_apply_pending(o);
  if (rc) return rc;
  for (size_t q = 0; q < o->stats.size(); ++q) {
    const StatState& st = o->stats[q];
    if (st.layer != layer || st.kind != which) continue;
    int64_t dp = 0;
    spngd_tracker_state(st.tr, t_x, delta, &dp, refresh_count);
    if (due_last) *due_last = o->due.empty() ? 0 : o->due[q];
    return SPNGD_OK;
  }
  return fail(SPNGD_ERR_SHAPE_MISMATCH, "spngd_opt_stale_info: layer %d has no statistic %d", layer, which);
}

int spngd_opt_set_overlap(spngd_opt* o, int on) {
  SPNGD_CTX_SCOPE(o ? o->ctx : nullptr);
  if (!o) return fail(SPNGD_ERR_INVALID, "spngd_opt_set_overlap: opt is NULL");
  if (on && !o->overlap_ok)
    return fail(SPNGD_ERR_INVALID, "spngd_opt_set_overlap: the wave schedule needs stale gating off");
  o->overlap_on = on != 0;
  return SPNGD_OK;
}

int spngd_opt_phase_ms(spngd_opt* o, float* out6) {
  SPNGD_CTX_SCOPE(o ? o->ctx : nullptr);
  if (!o || !out6) return fail(SPNGD_ERR_INVALID, "spngd_opt_phase_ms: bad argument");
  if (!o->timed) return fail(SPNGD_ERR_INVALID, "spngd_opt_phase_ms: no step yet");
  SPNGD_CUDA_TRY(cudaEventSynchronize(o->ev[6]));
  for (int i = 0; i < 6; ++i) SPNGD_CUDA_TRY(cudaEventElapsedTime(&out6[i], o->ev[i], o->ev[i + 1]));
  if (!o->trace.empty()) {
    for (auto& t : o->trace) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, o->ev[0], t.second);
      fprintf(stderr, "[step trace] %8.3f ms  %s\n", ms, t.first.c_str());
      cudaEventDestroy(t.second);
    }
    float total = 0.f;
    cudaEventElapsedTime(&total, o->ev[0], o->ev[6]);
    fprintf(stderr, "[step trace] %8.3f ms  step end\n", total);
    o->trace.clear();
  }
  return SPNGD_OK;
}

// spngd_ctx_sync plus the layer tag of a failed step (fisher.cpp:48-51
// layer_tag): the first owned factor whose inverse failed, or the first BN
// channel whose damped 2x2 block is singular.
int spngd_opt_sync(spngd_opt* o) {
  SPNGD_CTX_SCOPE(o ? o->ctx : nullptr);
  if (!o) return fail(SPNGD_ERR_INVALID, "spngd_opt_sync: opt is NULL");
  const int rc = spngd_ctx_sync(o->ctx);
  if (rc != SPNGD_ERR_NOT_POSITIVE_DEFINITE && rc != SPNGD_ERR_SINGULAR_BLOCK) return rc;
  const int n = int(o->layers.size());
  std::vector<int> info(3 * size_t(n));
  SPNGD_CUDA_TRY(cudaMemcpy(info.data(), o->d_info, sizeof(int) * info.size(), cudaMemcpyDeviceToHost));
  SPNGD_CUDA_TRY(cudaMemset(o->d_info, 0, sizeof(int) * info.size()));
  auto tag = [&](int li, char* buf, size_t cap) {
    const spngd_layer_desc& d = o->layers[li].d;
    if (d.kind == SPNGD_BN) snprintf(buf, cap, "layer %d (bn(%lld))", li, (long long)d.g);
    else snprintf(buf, cap, "layer %d (%s a=%lld g=%lld hw=%lld)", li, d.kind == SPNGD_CONV ? "conv" : "fc",
                  (long long)d.a, (long long)d.g, (long long)d.hw);
  };
  char buf[128];
  static const char* which[3] = {"A factor", "G factor", "full BN block"};
  for (int li = 0; li < n; ++li)
    for (int w = 0; w < 3; ++w)
      if (info[3 * li + w]) {
        tag(li, buf, sizeof(buf));
        return fail(info[3 * li + w], "damp_and_invert: %s: %s: Cholesky factorization failed -- non-positive pivot "
                    "or non-finite entries (no parameter was updated)", buf, which[w]);
      }
  if (rc == SPNGD_ERR_SINGULAR_BLOCK) {  // damp_bn (fisher.cpp:230-246): find the channel on the host
    for (size_t q = 0; q < o->bnu.size(); ++q) {
      const spngd_bn_update_req& r = o->bnu[q];
      std::vector<float> m(3 * size_t(r.c));
      SPNGD_CUDA_TRY(cudaMemcpy(m.data(), r.m3c, sizeof(float) * m.size(), cudaMemcpyDeviceToHost));
      for (int64_t ch = 0; ch < r.c; ++ch) {
        const double a = double(m[3 * ch]) + o->cfg.lambda, b = m[3 * ch + 1], d = double(m[3 * ch + 2]) + o->cfg.lambda;
        if (std::fabs(a * d - b * b) < 1e-30) {
          int li = -1;
          for (int k = 0; k < n; ++k)
            if (o->layers[k].owner == o->rank && o->layers[k].d.kind == SPNGD_BN && o->rs_recv + o->layers[k].off_M == r.m3c) li = k;
          tag(li < 0 ? 0 : li, buf, sizeof(buf));
          return fail(rc, "damp_bn: %s: channel %lld: inv2x2 determinant below 1e-30 (no parameter was updated)",
                      li < 0 ? "BN layer" : buf, (long long)ch);
        }
      }
    }
  }
  return rc;
}

int64_t spngd_opt_launch_count(const spngd_opt* o) { return o ? o->launches : 0; }

}  // extern "C"
