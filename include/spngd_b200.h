/*
 * spngd_b200.h — C ABI of the B200-native SP-NGD optimizer step.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj, the `spngd` C++ library).  Every entry point below
 * replaces one reference function or one stage of
 * `accumulate_microsteps` (src/dist.cpp:406-675) and cites it.  All tensors
 * are DEVICE pointers to fp32 data on the context's GPU in the reference's
 * layouts:
 *   - packed symmetric matrices: upper triangle, row-major,
 *     offset(i,j) = i*n - i*(i-1)/2 + (j-i)         (include/spngd/linalg.hpp:48-51)
 *   - weights / gradients: row-major g x a (d_out x d_in, or c_out x c_in*k*k)
 *                                                  (include/spngd/net.hpp:46-50)
 *   - FC activation capture: M x d_in rows; conv capture: stacked im2col
 *     (M*c_in*k*k) x (h_out*w_out), row = ch*k*k + ky*k + kx
 *                                                  (include/spngd/net.hpp:84-101)
 *   - BN unit moments: interleaved (fgg, fgb, fbb) x c  (src/dist.cpp:283-292)
 *   - BN gradient / parameter payload: gamma(c) then beta(c) (src/dist.cpp:363-389)
 *
 * Errors: every function returns an spngd_status; nonzero codes mirror the
 * reference exception taxonomy (include/spngd/errors.hpp:10-85) and
 * spngd_last_error() returns the message.  There is no CPU fallback: without a
 * usable sm_100 device every compute entry point fails with SPNGD_ERR_CUDA.
 */
#ifndef SPNGD_B200_H_
#define SPNGD_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum spngd_status {
  SPNGD_OK = 0,
  SPNGD_ERR_SHAPE_MISMATCH = 1,        /* errors.hpp:16  ShapeMismatch */
  SPNGD_ERR_NOT_POSITIVE_DEFINITE = 2, /* errors.hpp:22  NotPositiveDefinite */
  SPNGD_ERR_SINGULAR_BLOCK = 3,        /* errors.hpp:27  SingularBlock */
  SPNGD_ERR_ZERO_REFERENCE = 4,        /* errors.hpp:32  ZeroReference */
  SPNGD_ERR_EMPTY_BATCH = 5,           /* errors.hpp:37  EmptyBatch */
  SPNGD_ERR_MISSING_MC_PASS = 6,       /* errors.hpp:42  MissingMcPass */
  SPNGD_ERR_STALE_BEYOND_LIMIT = 7,    /* errors.hpp:52  StaleBeyondLimit */
  SPNGD_ERR_REFRESH_OUT_OF_TURN = 8,   /* errors.hpp:57  RefreshOutOfTurn */
  SPNGD_ERR_INDIVISIBLE_BATCH = 9,     /* errors.hpp:62  IndivisibleBatch */
  SPNGD_ERR_MISSING_OWNER = 10,        /* errors.hpp:67  MissingOwner */
  SPNGD_ERR_EMPTY_ACCUMULATION = 11,   /* errors.hpp:72  EmptyAccumulation */
  SPNGD_ERR_CUDA = 100,                /* CUDA runtime / launch failure */
  SPNGD_ERR_NCCL = 101,                /* NCCL failure */
  SPNGD_ERR_INVALID = 102              /* bad argument (null pointer, ...) */
} spngd_status;

typedef struct spngd_ctx spngd_ctx;

/* Last error message of the calling thread (empty string if none). */
const char* spngd_last_error(void);
/* Last error message of a call made on this context (or on an optimizer
 * created from it), from any thread; empty string if none. */
const char* spngd_ctx_last_error(const spngd_ctx* ctx);
const char* spngd_version(void);

/* One context per GPU and host thread; owns workspace and the stream.
 * `stream` may be NULL (a private non-blocking stream is created). */
int spngd_ctx_create(int device, void* stream, spngd_ctx** out);
void spngd_ctx_destroy(spngd_ctx* ctx);
/* Synchronizes the context stream and returns the first device-side error
 * raised since the previous call (NotPositiveDefinite, SingularBlock). */
int spngd_ctx_sync(spngd_ctx* ctx);
void* spngd_ctx_stream(spngd_ctx* ctx);
/* Stream-ordered copy (any direction, cudaMemcpyDefault) on the context stream. */
int spngd_copy(spngd_ctx* ctx, void* dst, const void* src, size_t bytes);
/* Pinned host buffers for host-resident inputs (the e2e drop-in path). */
int spngd_host_alloc(void** out, size_t bytes);
void spngd_host_free(void* p);
/* CUDA-event timing on the context stream: call with record_second = 0 to
 * start, 1 to stop, synchronize and read `ms`.  ev_pair: two NULL-initialised
 * opaque slots owned by the caller. */
int spngd_event_time(spngd_ctx* ctx, void** ev_pair, int record_second, float* ms);

/* ---- K1: Kronecker factors ------------------------------------------------
 * Replaces factor_A (src/fisher.cpp:92-114) and factor_G (src/fisher.cpp:116-145)
 * via mean_outer (src/fisher.cpp:55-75):
 *   out = scale * sum_{s in [lo,hi)} X_s X_s^T, packed upper triangle,
 * X_s = row s of an M x dim capture (layout 0, FC) or the dim x hw block s of a
 * stacked (M*dim) x hw capture (layout 1, conv).  Computed with 3xTF32
 * tcgen05 MMAs (fp32-accurate), split-K partials reduced in fp64. */
typedef struct spngd_factor_req {
  const float* x;      /* capture, device */
  int64_t dim;         /* a (A factor) or g (G factor) */
  int64_t hw;          /* h_out*w_out (layout 1); ignored for layout 0 */
  int64_t layout;      /* 0 = FC rows, 1 = conv stacked blocks */
  int64_t lo, hi;      /* sample range [lo, hi) */
  double scale;        /* 1/(n*hw) for conv A, 1/n otherwise (fisher.cpp:104-108,138-139) */
  float* packed_out;   /* dim*(dim+1)/2 floats, device */
} spngd_factor_req;
int spngd_factor_sym_batched(spngd_ctx* ctx, int n, const spngd_factor_req* reqs);

/* ---- K2: BatchNorm unit moments -------------------------------------------
 * Replaces build_bn_block (src/fisher.cpp:147-185) + stat_payload's 3c
 * interleave (src/dist.cpp:283-292).  gg, gb: M x c row-major. */
typedef struct spngd_bn_moments_req {
  const float* gg;
  const float* gb;
  int64_t c;
  int64_t lo, hi;
  float* out3c;
} spngd_bn_moments_req;
int spngd_bn_moments_batched(spngd_ctx* ctx, int n, const spngd_bn_moments_req* reqs);

/* ---- Full 2c x 2c BN blocks (BnMode::Full) ----------------
 * spngd_bn_full_moments_batched replaces build_bn_full (src/fisher.cpp:187-216):
 * F = mean_s u_s u_s^T over the interleaved u_s = (gg[s][0], gb[s][0], gg[s][1],
 * gb[s][1], ...) (2c), packed upper triangle, samples [lo, hi).  Built by the
 * 3xTF32 SYRK engine.  damp_bn_full (fisher.cpp:248-253) is
 * spngd_spd_inverse_batched(F, lambda) with a dense output.
 * spngd_bn_full_solve_update_batched replaces precondition_bn_full
 * (fisher.cpp:278-296) + the BN branch of ngd_step (fisher.cpp:346-359):
 * (pg, pb) = F_inv (grad_gamma, grad_beta) interleaved, then
 * w' = w - eta p + m v, v' = w' - w for gamma and beta. */
typedef struct spngd_bn_full_req {
  const float* gg;
  const float* gb;
  int64_t c;
  int64_t lo, hi;
  float* packed_out;      /* 2c(2c+1)/2 */
} spngd_bn_full_req;
int spngd_bn_full_moments_batched(spngd_ctx* ctx, int n, const spngd_bn_full_req* reqs);
typedef struct spngd_bn_full_update_req {
  const float* finv;      /* dense 2c x 2c (row-major, leading dimension ld) */
  int64_t ld;
  const float* grad;      /* [grad_gamma (c) | grad_beta (c)] */
  int64_t c;
  float* gamma; float* beta;
  float* vgamma; float* vbeta;
  float* pg_out; float* pb_out;  /* optional preconditioned gradient */
} spngd_bn_full_update_req;
int spngd_bn_full_solve_update_batched(spngd_ctx* ctx, int n, const spngd_bn_full_update_req* reqs, double eta,
                                       double momentum);

/* ---- BN per-sample parameter gradients ------------------
 * Replaces the per-sample capture of src/net.cpp:467-475:
 *   gg[s][ch] = sum_p dY[s][ch*S + p] * xhat[s][ch*S + p]
 *   gb[s][ch] = sum_p dY[s][ch*S + p]
 * dY, xhat: M x (c*S) row-major (the BN backward's output-gradient and
 * normalised activation); gg, gb: M x c row-major -- exactly the
 * bn_ggamma_true / bn_gbeta_true capture (net.hpp:95) that
 * spngd_bn_moments_batched and the step consume.  One read of dY and xhat
 * (HBM-bound), fp32 loads with fp32 accumulation per lane and a pairwise warp
 * reduction. */
typedef struct spngd_bn_grad_req {
  const float* dy;
  const float* xhat;
  int64_t M, c, S;
  float* gg;
  float* gb;
} spngd_bn_grad_req;
int spngd_bn_grad_reduce_batched(spngd_ctx* ctx, int n, const spngd_bn_grad_req* reqs);

/* SURVEY §8f row 1, fused: one launch for every BN layer turns dY and x_hat
 * (M x (c*S)) into the per-sample capture (gg, gb: M x c, may be NULL), the
 * build_bn_block moments (src/fisher.cpp:147-185) as the interleaved 3c
 * payload (src/dist.cpp:283-292; out3c may be NULL) and the BN branch of
 * grad_payload [sum_s gg / M | sum_s gb / M] (src/dist.cpp:364-371; payload,
 * 2c, may be NULL).  HBM-bound (reads dY and x_hat once); deterministic. */
typedef struct spngd_bn_backward_req {
  const float* dy;
  const float* xhat;
  int64_t M, c, S;
  float* gg;
  float* gb;
  float* out3c;
  float* payload;
} spngd_bn_backward_req;
int spngd_bn_backward_stats_batched(spngd_ctx* ctx, int n, const spngd_bn_backward_req* reqs);

/* ---- K3/K4: damped SPD inverse ---------------------------------------------
 * Replaces spd_inverse (src/linalg.cpp:29-48): (M + d I)^-1 of a packed
 * symmetric matrix.  `damping_dev` (device float) overrides `damping` when
 * non-NULL.  Output: dense row-major (ld >= n) and/or packed; exactly
 * symmetric.  Fails with SPNGD_ERR_NOT_POSITIVE_DEFINITE on a non-positive
 * pivot or non-finite entries. */
typedef struct spngd_spd_req {
  const float* packed;   /* input, n(n+1)/2 */
  int64_t n;
  float damping;
  const float* damping_dev;
  float* dense_out;      /* n x ld, may be NULL if packed_out given */
  int64_t ld;
  float* packed_out;     /* may be NULL */
} spngd_spd_req;
/* info: host array of n ints (may be NULL), 0 or the error code of each
 * request; the returned status is that of the first failing request and
 * spngd_last_error() names it (request index, factor, n).  Matrices whose
 * ||M + dI||_F / d exceeds 1.5e4 (an upper bound of cond(M + dI)) get one
 * step of iterative refinement with a residual formed from exact tf32 splits
 * (SPNGD_REFINE_COND overrides the threshold; < 0 disables). */
int spngd_spd_inverse_batched(spngd_ctx* ctx, int n, const spngd_spd_req* reqs, int* info);

/* Replaces damp_and_invert (src/fisher.cpp:218-228) incl. avg_eigenvalue
 * (src/linalg.cpp:64-69): pi = sqrt((trA/a)/(trG/g)) (1 if either < 1e-12),
 * A_inv = (A + pi sqrt(lambda) I)^-1, G_inv = (G + sqrt(lambda)/pi I)^-1. */
typedef struct spngd_kron_req {
  const float* A_packed;
  const float* G_packed;
  int64_t a, g;
  float* Ainv_dense; int64_t lda;   /* dense outputs (may be NULL) */
  float* Ginv_dense; int64_t ldg;
  float* Ainv_packed;               /* packed outputs (may be NULL) */
  float* Ginv_packed;
  float* pi_out;                    /* device float (may be NULL) */
} spngd_kron_req;
/* info: as for spngd_spd_inverse_batched, per request (either factor). */
int spngd_damp_and_invert_batched(spngd_ctx* ctx, int n, const spngd_kron_req* reqs, double lambda, int* info);

/* ---- K5/K6: preconditioning + momentum/rescale update ------------------------
 * Replaces precondition/kron_matvec (src/fisher.cpp:255-257,
 * src/linalg.cpp:58-62), the FC/Conv branch of ngd_step
 * (src/fisher.cpp:332-333) and rescale_weights + velocity fix
 * (src/schemes.cpp:116-119, src/dist.cpp:621-632):
 *   P = G_inv dW A_inv ;  W' = W - eta P + momentum V ; V' = W' - W ;
 *   if rescale: W'' = sqrt(2 g) W'/(||W'||_F + 1e-9), V'' = W'' - W.
 * G_inv, A_inv dense symmetric.  W/V updated in place when W != NULL. */
typedef struct spngd_precond_req {
  const float* Ginv; int64_t ldg;
  const float* Ainv; int64_t lda;
  const float* dW;                 /* g x a row-major */
  int64_t g, a;
  float* P_out;                    /* optional g x a */
  float* W;                        /* optional: update in place */
  float* V;
  int rescale;
} spngd_precond_req;
int spngd_precondition_update_batched(spngd_ctx* ctx, int n, const spngd_precond_req* reqs,
                                      double eta, double momentum);

/* ---- K7: unit-wise BatchNorm 2x2 solve + update -----------------------------
 * Replaces damp_bn / precondition_bn (src/fisher.cpp:230-246, 259-276,
 * inv2x2 src/linalg.cpp:50-56) and the BN branch of ngd_step
 * (src/fisher.cpp:336-357).  Unit BN uses lambda (not sqrt) and no pi.
 * grad = [g_gamma(c), g_beta(c)]; SingularBlock if |det| < 1e-30. */
typedef struct spngd_bn_update_req {
  const float* m3c;
  const float* grad;
  int64_t c;
  float* gamma; float* beta;       /* optional in-place update */
  float* vgamma; float* vbeta;
  float* pg_out; float* pb_out;    /* optional preconditioned gradient */
} spngd_bn_update_req;
int spngd_bn_solve_update_batched(spngd_ctx* ctx, int n, const spngd_bn_update_req* reqs,
                                  double lambda, double eta, double momentum);

/* ---- K8: stale-statistics similarity ----------------------------------------
 * Replaces to_stat / weighted_norm / similar (include/spngd/stale.hpp:23-64)
 * over a packed statistic (off-diagonal weight 2) or a BN 3c payload (weights
 * 1,2,1).  out[0..3] = ||x-x1||_w, ||x1||_w, ||x-x2||_w, ||x2||_w (fp64). */
typedef struct spngd_stat_req {
  const float* x; const float* x1; const float* x2;  /* x1/x2 may be NULL */
  int64_t n;            /* packed dimension (kind 0) or channels (kind 1) */
  int64_t kind;         /* 0 = packed symmetric, 1 = BN 3c */
  double* out4;         /* device doubles */
} spngd_stat_req;
int spngd_stat_distance_batched(spngd_ctx* ctx, int n, const spngd_stat_req* reqs);

/* ---- stale scheduler (host logic, include/spngd/stale.hpp:78-132) ---------- */
typedef struct spngd_tracker spngd_tracker;
spngd_tracker* spngd_tracker_create(const char* id, double alpha);
void spngd_tracker_destroy(spngd_tracker* t);
int spngd_tracker_should_refresh(const spngd_tracker* t, int64_t step);
/* d1 = ||x-x1||, r1 = ||x1|| (has1 = 0 if no snapshot), same for x2.
 * reason: 0 FirstBuild, 1 Dissimilar1, 2 Dissimilar2, 3 SimilarBoth. */
int spngd_tracker_on_refresh(spngd_tracker* t, int64_t step, int has1, double d1, double r1,
                             int has2, double d2, double r2, int64_t* next_interval, int* reason);
void spngd_tracker_state(const spngd_tracker* t, int64_t* t_x, int64_t* delta, int64_t* delta_prev,
                         int64_t* refresh_count);

/* ---- collectives (src/dist.cpp:181-237) over NCCL ----------------------------
 * nccl_id: 128-byte ncclUniqueId from spngd_nccl_unique_id on rank 0. */
int spngd_nccl_unique_id(void* out128);
int spngd_ctx_init_comm(spngd_ctx* ctx, int world, int rank, const void* id128);
/* ReduceScatter (mean, ncclAvg) of `count` floats per rank: send[world*count]
 * -> recv[count]; equals reduce_scatter_v's ascending-order mean up to
 * reduction order (dist.cpp:204-213). In-place if recv == send + rank*count. */
int spngd_reduce_scatter_mean(spngd_ctx* ctx, const float* send, float* recv, int64_t count);
/* AllGather of `count` floats per rank (all_gather_v, dist.cpp:222-237). */
int spngd_all_gather(spngd_ctx* ctx, const float* send, float* recv, int64_t count);

/* ---- whole optimizer step (accumulate_microsteps Stages 2-5) ---------------- */
typedef enum spngd_layer_kind { SPNGD_FC = 0, SPNGD_CONV = 1, SPNGD_BN = 2 } spngd_layer_kind;

typedef struct spngd_layer_desc {
  int32_t kind;        /* spngd_layer_kind */
  int32_t pad_;
  int64_t a;           /* FC d_in, conv c_in*k*k */
  int64_t g;           /* FC d_out, conv c_out; BN channels */
  int64_t hw;          /* conv h_out*w_out, FC 1 */
} spngd_layer_desc;

typedef struct spngd_opt_config {
  double lambda;       /* OptimizerConfig::lambda (dist.hpp:117) */
  int32_t rescale;     /* OptimizerConfig::rescale */
  int32_t stale;       /* stale_enabled */
  double stale_alpha;
  int64_t batch;       /* per-rank micro-batch M/K */
  int32_t fisher_mode; /* OptimizerConfig::fisher_mode (dist.hpp:113-128): 0 Empirical
                        * (G and F from grad_true, fisher.cpp:133-137), 1 OneMC (G and F
                        * from the sampled-label backward's captures, buffers 13-15,
                        * fisher.cpp:127-132; dist.cpp:476-480) */
  int32_t elem_size;   /* ClusterConfig::elem_size, the ledger's modeled wire element
                        * size in bytes (dist.hpp:58-60); 0 means 4 */
  int32_t sgd;         /* OptimizerConfig::sgd: plain-gradient update, no statistics, no
                        * rescaling (ngd_step with blocks == nullptr, fisher.cpp:320-333,
                        * 348-356; dist.cpp:425, 539, 605): the step is gradient RS,
                        * W' = W - eta dW + m V, V' = W' - W, AG */
  int32_t bn_mode;     /* OptimizerConfig::bn_mode: 0 Unit (2x2 per channel), 1 FullBlockDiag2c:
                        * F = mean u u^T over u = (g_gamma0, g_beta0, ...) (build_bn_full,
                        * fisher.cpp:187-216) through the SYRK engine, (F + lambda I)^-1 by
                        * the batched Cholesky (damp_bn_full, :248-253), precondition_bn_full
                        * + BN update (:278-296, 346-359); the wave overlap is off */
  int32_t wgrad;       /* 1: the step also forms this rank's shard-mean gradients from the
                        * captures (grad_payload, dist.cpp:315-391: Conv sum_s G_s A_s^T / m,
                        * FC grad^T act / m on the SYRK engine's operands, BN column means)
                        * into buffer 2 before the reduce-scatter; 0: buffer 2 is an input */
  int32_t pad_;
} spngd_opt_config;

/* Host-only planning of the hybrid schedule (no GPU needed): layer owners
 * (LPT on a^3 + g^3 + 2 g^2 a + 2 g a^2; the reference uses li % K,
 * dist.cpp:147-153 -- ownership never changes numerics) and owner-major
 * segment offsets (floats).  The reduce-scatter buffer has two regions, each
 * owner-major: statistics (A, G packed; BN 3c moments -- off_A/off_G/off_M
 * within the owner's seg_stat) and gradients (dW g*a or 2c -- off_dW within
 * the owner's seg_grad), so gradients reduce every step and statistics only
 * when due (stale gating).  All-gather buffer: W g*a or gamma|beta 2c.
 * -1 marks payloads a layer does not have.  Send buffer layout:
 * [world x seg_stat | world x seg_grad]; owner receive: [seg_stat | seg_grad]. */
#define SPNGD_LEDGER_BN_FULL 1 /* F payload is the 2c x 2c packed block (BnMode::FullBlockDiag2c) */
#define SPNGD_LEDGER_SGD 2     /* OptimizerConfig::sgd: no statistics (plan_statistics returns none) */
typedef struct spngd_layout_entry {
  int32_t owner;
  int32_t pad_;
  int64_t off_A, off_G, off_M, off_dW;
  int64_t off_W;
} spngd_layout_entry;
/* As spngd_plan_layout; flags SPNGD_LEDGER_BN_FULL sizes BN statistics as the
 * packed 2c x 2c block instead of the 3c moments. */
int spngd_plan_layout_ex(const spngd_layer_desc* layers, int n_layers, int world, int flags, spngd_layout_entry* out,
                         int64_t* seg_stat, int64_t* seg_grad, int64_t* seg_ag);
int spngd_plan_layout(const spngd_layer_desc* layers, int n_layers, int world, spngd_layout_entry* out,
                      int64_t* seg_stat, int64_t* seg_grad, int64_t* seg_ag);

typedef struct spngd_opt spngd_opt;

int spngd_opt_create(spngd_ctx* ctx, const spngd_layer_desc* layers, int n_layers,
                     const spngd_opt_config* cfg, spngd_opt** out);
void spngd_opt_destroy(spngd_opt* opt);
/* Device pointers of per-layer buffers:
 *   which 0 act capture, 1 grad capture, 2 dW (this rank's shard-mean grad,
 *   g x a or 2c), 3 W (g x a, or gamma|beta 2c), 4 V, 5 bn gg (M x c),
 *   6 bn gb, 7 A_inv dense, 8 G_inv dense, 9 A packed (reduced), 10 G packed,
 *   11 BN moments 3c (reduced; bn_mode 1: the packed 2c x 2c F), 12 the whole weight all-gather buffer
 *   (ld = its float count), 13 sampled-label grad capture (OneMC only,
 *   LayerCapture::grad_sampled, net.hpp:92), 14 / 15 sampled-label BN
 *   gamma / beta grads (OneMC only, bn_g*_sampled, net.hpp:96-97), 16 raw
 *   conv input B x c_in x h x w (after spngd_opt_enable_raw_inputs). NULL if the layer has no such buffer or this
 *   rank does not own it.  The step keeps only the triangular factors
 *   T = chol(X + dI)^-1 (it preconditions with T^T T directly), so 7 / 8
 *   form (X + dI)^-1 = T^T T on the call (one GEMM, synchronous); for a
 *   BN layer in bn_mode 1, 7 is (F + lambda I)^-1 (2c x 2c, ld = ld). */
float* spngd_opt_buffer(spngd_opt* opt, int layer, int which, int64_t* ld);
int spngd_opt_owner(const spngd_opt* opt, int layer);
/* One SP-NGD step over the resident inputs (accumulate_microsteps,
 * dist.cpp:406-675, n = 1 micro-step): factors + BN moments, RS, damped
 * inverse, precondition + update + rescale, BN solve + update, AG. */
int spngd_opt_step(spngd_opt* opt, int64_t step, double eta, double momentum);
/* The same step fed from HOST memory -- the reference's run_step takes host
 * captures (dist.cpp:677-682).  `in` lists (layer, buffer which, host pointer)
 * for the inputs to refresh: 0/16 activation capture / raw conv input, 1 / 13
 * grad capture (true / sampled), 2 dW, 5 / 6 / 14 / 15 BN pairs; sizes are the
 * buffers'.  Pinned host memory makes the copies asynchronous.  With the wave
 * schedule the copies run on a copy stream, dW first, then each wave's
 * captures, and wave w's im2col / repack / factor SYRK start as soon as its
 * captures have landed, so the host->device transfer overlaps the step;
 * otherwise they precede the step on its stream.  host_weights_out (optional,
 * world * seg_ag floats = buffer 12's ld) receives every weight replica after
 * the all-gather.  Asynchronous: spngd_ctx_sync before reading it. */
typedef struct spngd_host_input {
  int32_t layer;
  int32_t which;
  const void* host;
} spngd_host_input;
int spngd_opt_step_host(spngd_opt* opt, int64_t step, double eta, double momentum, const spngd_host_input* in,
                        int n, float* host_weights_out);
/* Wave schedule (no stale gating; on by default, env SPNGD_NO_OVERLAP=1
 * starts it off): layers are split into waves by their larger Kronecker
 * dimension, largest first, and each wave's damped-inverse recursion runs on
 * high-priority streams while the later waves' factor SYRKs run -- the
 * reference's step order (dist.cpp:406-675) with its stage-3/4 barrier relaxed
 * to per-layer dependencies.  world > 1: each wave's statistics go to their
 * owners (grouped ncclReduce(avg)) on a communication stream as soon as the
 * wave is reduced locally; gradients reduce-scatter there at the start.
 * on = 0 restores the phase-serial schedule.  Same kernels on the same
 * inputs (bit-identical at world == 1); at world > 1 the statistics are
 * averaged by per-wave ncclReduce instead of one ncclReduceScatter, so only
 * NCCL's summation order can differ.  Must match on every rank. */
/* spngd_ctx_sync for the optimizer: a failed step (NotPositiveDefinite,
 * SingularBlock) is reported with the layer tag of the first failing factor
 * or BN channel (fisher.cpp:48-51 layer_tag).  Parameters are untouched by a
 * failed phase-serial step; with the wave overlap (spngd_opt_set_overlap 1)
 * layers preconditioned before the last inverse wave may already be updated. */
int spngd_opt_sync(spngd_opt* opt);
int spngd_opt_set_overlap(spngd_opt* opt, int on);
/* Per-phase device milliseconds of the last step: factor GEMM, factor
 * reduction + BN moments, reduce_scatter, inverse, precondition + BN update,
 * all_gather.  Overlapped steps: the factor phase ends after the last wave's
 * SYRK (earlier waves' recursions already running) and the inverse phase is
 * what the recursion adds after it. */
int spngd_opt_phase_ms(spngd_opt* opt, float* out6);
/* Number of kernels the last step launched on this rank. */
int64_t spngd_opt_launch_count(const spngd_opt* opt);
/* Stale gating (cfg.stale): tracker state of statistic `which` (0 A, 1 G,
 * 2 BN F) of `layer` -- next refresh step t_X, interval, refresh count --
 * and whether it refreshed in the last step (StaleTracker, stale.hpp:92-132;
 * gating dist.cpp:431-444). */
int spngd_opt_stale_info(spngd_opt* opt, int layer, int which, int64_t* t_x, int64_t* delta,
                         int64_t* refresh_count, int* due_last);

/* ---- communication ledger (CommLedger, dist.hpp:16-56, dist.cpp:42-133) -----
 * One row per collective payload, in the reference's record order
 * (accumulate_microsteps, dist.cpp:511-537, 661-662): stage 2 "RSV_A" --
 * due A:l in plan order, then skipped A:l; stage 3 "RSV_G_F_grad" -- due
 * G:l / F:l in plan order, then grad:0..L-1, then skipped G:l / F:l; stage 5
 * "AGV_params" -- w:0..L-1.  elements = payload length when world > 1, else 0
 * (dist.cpp:214, 231); bytes = elements * elem_size; skipped rows carry 0 / 0
 * (dist.cpp:520, 537).  Payload lengths: A/G packed n(n+1)/2, F 3c (unit BN)
 * or 2c(2c+1)/2 (full BN), grad and w g*a (BN 2c). */
typedef enum spngd_ledger_collective {
  SPNGD_RSV_A = 0,          /* stage 2 */
  SPNGD_RSV_G_F_GRAD = 1,   /* stage 3 */
  SPNGD_AGV_PARAMS = 2      /* stage 5 */
} spngd_ledger_collective;
typedef enum spngd_ledger_id_kind {
  SPNGD_ID_A = 0, SPNGD_ID_G = 1, SPNGD_ID_F = 2, SPNGD_ID_GRAD = 3, SPNGD_ID_W = 4
} spngd_ledger_id_kind;
typedef struct spngd_ledger_row {
  int64_t step;
  int32_t stage;        /* 2, 3 or 5 */
  int32_t collective;   /* spngd_ledger_collective */
  int32_t id_kind;      /* spngd_ledger_id_kind: statistic_id = "<A|G|F|grad|w>:<layer>" */
  int32_t layer;
  int64_t elements;
  int64_t bytes;
  int32_t skipped;
  int32_t pad_;
} spngd_ledger_row;
/* Host-only (no GPU): the rows one step appends, given the per-statistic
 * refresh decisions `due` in plan_statistics order (dist.cpp:256-269: per
 * layer A then G, or F for BatchNorm); due == NULL means every statistic is
 * due.  flags: SPNGD_LEDGER_* bits.  Returns the row count (rows
 * are written while count <= cap) or a negative status. */
int64_t spngd_ledger_step_rows(const spngd_layer_desc* layers, int n_layers, int world, int64_t step,
                               const unsigned char* due, int elem_size, int flags,
                               spngd_ledger_row* out, int64_t cap);
/* The rows every spngd_opt_step of this optimizer appended so far (the
 * CommLedger passed to run_step); returns the total count, copying at most
 * cap.  _clear empties it. */
int64_t spngd_opt_ledger(const spngd_opt* opt, spngd_ledger_row* out, int64_t cap);
int spngd_opt_ledger_clear(spngd_opt* opt);
/* Bytes this rank handed to NCCL in the last step (send side, padded
 * owner-major segments as actually moved): reduce-scatter / owner reduces of
 * statistics, of gradients, and the all-gather.  0 at world == 1. */
int spngd_opt_wire_bytes(const spngd_opt* opt, int64_t* stat_bytes, int64_t* grad_bytes, int64_t* ag_bytes);

/* ---- Stage 5 over NVLink peer memory ---------------------------------------
 * One process per GPU: every rank exports its weight-replica buffer (buffer
 * 12) and, without stale gating, a statistics inbox (world x seg_stat floats)
 * with _ipc_handle (128 bytes: two cudaIpcMemHandle_t), the caller exchanges
 * them (e.g. torch.distributed all_gather) and passes all `world` records in
 * rank order to _attach_peers before the first step.  From then on:
 *  - Stages 2-3 (ReduceScatterV of the statistics, dist.cpp:510-537) are no
 *    NCCL reduce-scatter: the factor SYRK epilogues, split-K reductions and BN
 *    moment kernels store this rank's statistics straight into the owner's
 *    inbox slot over NVLink as they are produced, and after a one-word NCCL
 *    all-reduce (per wave in the wave schedule) the owner averages the slots
 *    in rank order (reduce_scatter_v's mean, dist.cpp:204-213);
 *  - Stage 5 (AllGatherV, dist.cpp:646-663) is no NCCL all-gather: the owners'
 *    rescale pass stores W'' into every peer's replica as it computes it, BN /
 *    unrescaled layers go by one peer-copy launch, and a one-word all-reduce
 *    orders the stores before the step completes.
 * Gradients still reduce-scatter through NCCL. */
int spngd_opt_ipc_handle(spngd_opt* opt, void* out128);
int spngd_opt_attach_peers(spngd_opt* opt, const void* handles);

/* ---- raw layer inputs (first stage) ------------------------
 * The reference's conv capture is im2col of the layer input, rows
 * ch*k*k + ky*k + kx, columns oy*w_out + ox, zero in the padding (im2col,
 * net.cpp:199-219; captured at net.cpp:287-307).  After this call the step
 * takes the raw per-sample input B x c_in x h x w (buffer 16) of every conv
 * layer and expands it on the device (one batched HBM-bound launch at the
 * start of each step) into the capture the factor/wgrad GEMMs read.  1x1
 * stride-1 unpadded convs need no expansion: their raw input IS the capture
 * (buffer 16 == buffer 0), so host->device traffic and, for them, the
 * expansion traffic drop to the raw tensor.  geoms[i] is read for conv layers
 * only; c_in*k*k must equal a and h_out*w_out must equal hw (SHAPE_MISMATCH).
 * Call once, before the first step. */
typedef struct spngd_conv_geom {
  int64_t c_in, h, w, k, stride, pad;
} spngd_conv_geom;
/* SURVEY §8f row 1 inside the step: each BN layer takes the backward's dY and
 * x_hat (buffers 17 / 18, B x (c*S), spatial[l] = S for BN layers, ignored
 * otherwise) instead of the (g_gamma, g_beta) capture and the BN dW: one
 * launch per step forms the captures (buffers 5 / 6), the 3c moments
 * (build_bn_block, unit blocks without stale gating; otherwise the captures
 * feed the usual moment / 2c x 2c path) and the BN gradient payload
 * (grad_payload, dist.cpp:364-371) in the buffer-2 slot.  Empirical Fisher
 * only.  Call before the first step. */
int spngd_opt_enable_bn_inputs(spngd_opt* opt, const int64_t* spatial);
int spngd_opt_enable_raw_inputs(spngd_opt* opt, const spngd_conv_geom* geoms);
/* implicit = 1: no capture is formed -- the A-factor SYRK and the wgrad GEMM
 * gather the im2col operand from the raw input (cp.async,
 * LSU-bound, so slower than expanding first); implicit = 0 is the call above. */
int spngd_opt_enable_raw_inputs_ex(spngd_opt* opt, const spngd_conv_geom* geoms, int implicit);
/* Batched im2col alone (net.cpp:199-219) for `n` conv inputs, x: batch x
 * c_in x h x w, out: batch x (c_in k k) x (h_out w_out), device pointers. */
typedef struct spngd_im2col_req {
  const float* x;
  float* out;
  int64_t batch;
  spngd_conv_geom geom;
} spngd_im2col_req;
int spngd_im2col_batched(spngd_ctx* ctx, int n, const spngd_im2col_req* reqs);

#ifdef __cplusplus
}
#endif
#endif /* SPNGD_B200_H_ */
