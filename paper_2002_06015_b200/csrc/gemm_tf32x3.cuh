// Grouped 3xTF32 tcgen05 GEMM: C[m,n] = alpha * sum_k A[m,k] B[n,k] (+ epilogue).
//
// One engine serves every dense contraction of the SP-NGD step:
//   * K1 factor construction (SYRK over captures, packed/partial epilogues),
//   * the Schur-complement recursion of the damped inverse (dense epilogues),
//   * K5 preconditioning G^-1 dW A^-1 with the fused momentum update.
// Operands are fp32 in HBM, K-major ("row r, column k") with an optional
// segmented K axis so a conv capture (M*dim) x hw is addressed in place:
//   element (r, k) = ptr[(k / seg_len) * seg_stride + r * row_stride + k % seg_len].
#pragma once

#include <cuda.h>
#include <stdint.h>

#include <vector>

namespace spngd {

enum OperandMode : int32_t {
  OP_ASYNC = 0,   // cp.async (LDGSTS) from any layout (fallback)
  OP_TMA2D = 1,   // TMA 2D box {32 k, 128 rows} of a K-contiguous matrix
  OP_TMA3D = 2,   // TMA 3D box {32 p, 128 rows, 1 segment}; K = nseg * cps * 32 (zero-padded chunks)
  OP_IM2COL = 3,  // implicit im2col of a raw conv input: row (ch, ky, kx),
                  // k = s * seg_pad + p (p < hw valid), gathered by cp.async with zero fill
};

// Geometry of an OP_IM2COL operand (the raw input x is B x c x h x w, row-major).
struct Im2colGeo {
  int32_t c, h, w, k, stride, pad;
  int32_t wo, hw;      // output width, h_out * w_out
  int32_t seg_pad;     // k-axis period per sample: the partner operand's layout (cps*32 or hw)
  int32_t pad_;
};

struct alignas(64) GemmOperand {
  CUtensorMap tmap;   // valid for OP_TMA2D / OP_TMA3D (encoded by finalize_operand)
  const float* ptr;
  int64_t row_stride;
  int64_t seg_len;
  int64_t seg_stride;
  int64_t nseg;       // number of segments (OP_TMA3D)
  int32_t rows;       // valid rows; rows >= this read as zero
  int32_t vec;        // float4 loads legal (OP_ASYNC)
  int32_t mode;       // OperandMode
  int32_t cps;        // 32-wide chunks per segment (OP_TMA3D)
  Im2colGeo geo;      // OP_IM2COL
};

// Turns `op` (the factor operand of a conv capture: TMA3D with cps chunks per
// sample, or K-contiguous after a repack) into an implicit-im2col operand over
// the raw input x with the same k order, so K, tiles and partner operands stay valid.
void make_im2col_operand(GemmOperand& op, const float* x, int c, int h, int w, int k, int stride, int pad);

enum GemmEpi : int32_t {
  EPI_PARTIAL = 0,  // raw fp32 tile -> partials[slot] (split-K)
  EPI_PACKED = 1,   // alpha*acc -> packed upper triangle (i <= j) of C (n = M)
  EPI_DENSE = 2,    // alpha*acc + beta*Cin -> C (row-major), optional mirror / transposed copy
  EPI_UPDATE = 3,   // P^T tile -> W/V momentum update (+ ||W'||^2), see precond.cu
};

enum GemmFlags : int32_t {
  FLAG_SAME_AB = 1,    // B is the same operand as A (SYRK): diagonal tiles load once
  FLAG_SYM_MIRROR = 2, // EPI_DENSE: write only i <= j and mirror to (j, i)
  FLAG_TRANS = 4,      // EPI_DENSE: also write CT[j*ldct + i]
};

struct alignas(64) GemmProblem {
  GemmOperand A, B;
  int32_t M, N, K;
  int32_t mode;
  int32_t flags;
  int32_t ktri;     // triangular operands: K range trimmed per tile (KTRI_*)
  int32_t pad_;
  float alpha, beta;
  float* C;
  int64_t ldc;
  const float* Cin;
  float* CT;
  int64_t ldct;
  // EPI_UPDATE
  float* W;
  float* V;
  float* P_out;
  double* norm2;
  float eta, momentum;
  const float* scal;   // optional device {eta, momentum}, overrides the fields above
};

enum KTri : int32_t {
  KTRI_A_LOWER = 1,  // A row i is zero for k > i      -> k < (tm+1)*128
  KTRI_A_UPPER = 2,  // A row i is zero for k < i      -> k >= tm*128
  KTRI_B_LOWER = 4,  // B row j is zero for k > j      -> k < (tn+1)*128
  KTRI_B_UPPER = 8,  // B row j is zero for k < j      -> k >= tn*128
};

struct GemmWorkItem {
  int32_t problem;
  int32_t tm, tn;
  int32_t k0, k1;
  int32_t slot;
};

// Reduction task for split-K SYRK tiles: sum partial slots, scale, pack.
struct SyrkReduceTask {
  int32_t tm, tn;
  int32_t slot0, nslots;
  int32_t n;          // matrix dimension
  int32_t stride;     // slot stride (0 or 1: consecutive; 2: the 2-CTA SYRK's interleaved sub-tiles)
  double scale;
  float* packed_out;
};

constexpr int kTileM = 128;
constexpr int kTileN = 128;
constexpr int kTileK = 32;     // fp32 elements per stage = one 128-byte swizzle row
constexpr int kStages = 4;
constexpr int kGemmThreads = 512;  // 4 A-producer, 4 B-producer, 8 drain warps (warp 8 also issues MMAs)

// Chooses the operand mode and encodes its TMA descriptor.  `K` is the true
// K extent; for OP_TMA3D the GEMM must iterate the padded K returned by
// padded_k().  allow_tma = false forces the cp.async path.
void finalize_operand(GemmOperand& op, int64_t K = -1, bool allow_tma = true);
inline int64_t padded_k(const GemmOperand& op, int64_t K) {
  return op.mode == OP_TMA3D ? op.nseg * op.cps * 32 : K;
}
size_t gemm_smem_bytes();

// Kernel variant a launch needs: bit (1 << mode) per epilogue mode in use,
// plus kVariantAsync when any operand takes the cp.async path.  Computed at
// plan time; launch_gemm runs the smallest compiled kernel that covers it.
constexpr uint32_t kVariantAsync = 0x100u;
uint32_t gemm_variant(const GemmProblem* probs, int n);

// Priority attribute of the next launch_gemm launches on this thread (0: none).
extern thread_local int g_gemm_launch_prio;

// Launch one grouped GEMM over device-resident problem/work arrays.
int launch_gemm(const GemmProblem* d_probs, const GemmWorkItem* d_items, int n_items, float* d_partials,
                int* d_status, cudaStream_t stream, uint32_t variant = 0xFu | kVariantAsync);
int launch_syrk_reduce(const SyrkReduceTask* d_tasks, int n_tasks, const float* d_partials, cudaStream_t stream);

// 2-CTA SYRK (gemm_pair.cu): 256 x 256 tiles for the large factors.  Items
// come in cluster pairs (CTA rank r: tm = 2I + r, tn = 2J, two 128x128
// sub-tiles, partial slots slot and slot + 1).
bool pair_eligible(const GemmProblem& p);
int plan_pair_tiles(int problem_index, const GemmProblem& p, int kchunk, std::vector<GemmWorkItem>& items,
                    std::vector<SyrkReduceTask>* reduce, int* next_slot, double reduce_scale, float* packed_out);
// Dense problems (EPI_DENSE incl. mirror / transposed copy, EPI_UPDATE) on the
// pair kernel: 256 x 256 tiles (upper super-tiles for symmetric results), K
// band per tile for triangular operands.
bool pair_eligible_dense(const GemmProblem& p, bool upper_only = false);
// One launch group's choice between the kernels by wave-quantized time: a pair
// CTA (128 x 256 outputs) costs ~1.45 single-kernel 128 x 128 CTAs (SYRK
// efficiency 0.62 vs 0.43 of the roofline); `rest` (ineligible problems) runs
// as a second launch in pair mode.  Small rounds keep the single kernel
// (config-5 sweep: n = 512/1024 were 9% slower on pairs, n = 4608 5% faster).
bool pair_group_wins(int64_t pair_ctas, int64_t single_ctas, int64_t rest_ctas);
// SPNGD_NO_PAIR_INV: keep the inverse recursion / refinement GEMMs on the
// 128-row kernel (A/B experiments).
inline bool no_pair_inv() {
  static const bool off = getenv("SPNGD_NO_PAIR_INV") != nullptr;
  return off;
}
int plan_pair_dense(int problem_index, const GemmProblem& p, std::vector<GemmWorkItem>& items,
                    bool upper_only = false);
int launch_syrk_pair(const GemmProblem* d_probs, const GemmWorkItem* d_items, int n_items, float* d_partials,
                     cudaStream_t stream, int* d_status = nullptr);

// Host planning helpers.
// Upper-triangle (or full) tile list for one problem with K split into chunks
// of at most `kchunk` (multiple of kTileK).  Appends to items; returns the
// number of partial slots consumed (0 if unsplit).
int plan_problem_tiles(int problem_index, const GemmProblem& p, bool upper_only, int kchunk,
                       std::vector<GemmWorkItem>& items, std::vector<SyrkReduceTask>* reduce,
                       int* next_slot, double reduce_scale, float* packed_out);

}  // namespace spngd
