// Builds INTEGRATION.md's reference-side shim (error mapping §2, function-level
// drop-in §3) against minimal stand-ins of the reference types it touches
// (errors.hpp:10-85, linalg.hpp:24-55 SymMatrix, fisher.hpp:24-31
// KroneckerBlock) and calls the library through its C ABI, the way the
// reference's own fisher.cpp / linalg.cpp bodies would after the drop-in.
//
//   shim_test --expect-no-gpu   (CPU container) the ABI loads and fails loudly:
//                               spngd_ctx_create -> spngd::Error, no fallback
//   shim_test                   (B200) test_fisher.cpp:231-249 worked example
//                               through damp_and_invert, a batch of 5 with a
//                               non-PD factor -> NotPositiveDefinite naming it
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "spngd_b200.h"

namespace spngd {
// ---- stand-ins for the reference types (errors.hpp, linalg.hpp, fisher.hpp)
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct ShapeMismatch : Error { using Error::Error; };
struct NotPositiveDefinite : Error { using Error::Error; };
struct SingularBlock : Error { using Error::Error; };
struct ZeroReference : Error { using Error::Error; };
struct EmptyBatch : Error { using Error::Error; };
struct MissingMcPass : Error { using Error::Error; };
struct StaleBeyondLimit : Error { using Error::Error; };
struct RefreshOutOfTurn : Error { using Error::Error; };
struct IndivisibleBatch : Error { using Error::Error; };
struct MissingOwner : Error { using Error::Error; };
struct EmptyAccumulation : Error { using Error::Error; };
using Index = long long;
class SymMatrix {  // packed upper triangle, row-major (linalg.hpp:48-51)
 public:
  SymMatrix() = default;
  explicit SymMatrix(Index n) : n_(n), d_(size_t(n * (n + 1) / 2), 0.0) {}
  Index dim() const { return n_; }
  Index size() const { return Index(d_.size()); }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  double& operator()(Index i, Index j) {
    if (i > j) std::swap(i, j);
    return d_[size_t(i * n_ - i * (i - 1) / 2 + (j - i))];
  }
 private:
  Index n_ = 0;
  std::vector<double> d_;
};
struct KroneckerBlock {
  SymMatrix A, G, A_inv, G_inv;
  double pi = 1.0, lambda = 0.0;
};

// ---- error mapping
namespace b200 {
inline void check(int rc) {
  if (rc == SPNGD_OK) return;
  const std::string m = spngd_last_error();
  switch (rc) {
    case SPNGD_ERR_SHAPE_MISMATCH:        throw ShapeMismatch(m);
    case SPNGD_ERR_NOT_POSITIVE_DEFINITE: throw NotPositiveDefinite(m);
    case SPNGD_ERR_SINGULAR_BLOCK:        throw SingularBlock(m);
    case SPNGD_ERR_ZERO_REFERENCE:        throw ZeroReference(m);
    case SPNGD_ERR_EMPTY_BATCH:           throw EmptyBatch(m);
    case SPNGD_ERR_MISSING_MC_PASS:       throw MissingMcPass(m);
    case SPNGD_ERR_STALE_BEYOND_LIMIT:    throw StaleBeyondLimit(m);
    case SPNGD_ERR_REFRESH_OUT_OF_TURN:   throw RefreshOutOfTurn(m);
    case SPNGD_ERR_INDIVISIBLE_BATCH:     throw IndivisibleBatch(m);
    case SPNGD_ERR_MISSING_OWNER:         throw MissingOwner(m);
    case SPNGD_ERR_EMPTY_ACCUMULATION:    throw EmptyAccumulation(m);
    default:                              throw Error(m);
  }
}
spngd_ctx* ctx() {
  static thread_local spngd_ctx* c = nullptr;
  if (!c) check(spngd_ctx_create(0, nullptr, &c));
  return c;
}
// fp64 host <-> fp32 device buffer (the §3 pattern)
class DeviceF32 {
 public:
  explicit DeviceF32(size_t n) : n_(n) {
    if (cudaMalloc(&p_, n * sizeof(float)) != cudaSuccess) throw Error("cudaMalloc");
  }
  DeviceF32(const double* src, size_t n) : DeviceF32(n) {
    std::vector<float> h(src, src + n);
    cudaMemcpy(p_, h.data(), n * sizeof(float), cudaMemcpyHostToDevice);
  }
  ~DeviceF32() { cudaFree(p_); }
  float* ptr() { return p_; }
  void copy_to(double* dst) const {
    std::vector<float> h(n_);
    cudaMemcpy(h.data(), p_, n_ * sizeof(float), cudaMemcpyDeviceToHost);
    for (size_t i = 0; i < n_; ++i) dst[i] = h[i];
  }
 private:
  float* p_ = nullptr;
  size_t n_;
};
}  // namespace b200

// ---- damp_and_invert (fisher.cpp:218-228), batched
void damp_and_invert_all(std::vector<KroneckerBlock>& blocks, double lambda) {
  std::vector<b200::DeviceF32*> keep;
  std::vector<spngd_kron_req> reqs;
  std::vector<float*> pis;
  for (auto& b : blocks) {
    auto* A = new b200::DeviceF32(b.A.data(), size_t(b.A.size()));
    auto* G = new b200::DeviceF32(b.G.data(), size_t(b.G.size()));
    auto* Ai = new b200::DeviceF32(size_t(b.A.size()));
    auto* Gi = new b200::DeviceF32(size_t(b.G.size()));
    auto* pi = new b200::DeviceF32(1);
    keep.insert(keep.end(), {A, G, Ai, Gi, pi});
    reqs.push_back({A->ptr(), G->ptr(), b.A.dim(), b.G.dim(), nullptr, 0, nullptr, 0, Ai->ptr(), Gi->ptr(), pi->ptr()});
  }
  std::vector<int> info(blocks.size());
  const int rc = spngd_damp_and_invert_batched(b200::ctx(), int(reqs.size()), reqs.data(), lambda, info.data());
  if (rc == SPNGD_OK) {
    for (size_t i = 0; i < blocks.size(); ++i) {
      auto& b = blocks[i];
      b.A_inv = SymMatrix(b.A.dim());
      keep[5 * i + 2]->copy_to(b.A_inv.data());
      b.G_inv = SymMatrix(b.G.dim());
      keep[5 * i + 3]->copy_to(b.G_inv.data());
      keep[5 * i + 4]->copy_to(&b.pi);
      b.lambda = lambda;
    }
  }
  for (auto* k : keep) delete k;
  b200::check(rc);
}
}  // namespace spngd

static int fails = 0;
#define EXPECT(c)                                                    \
  do {                                                               \
    if (!(c)) { std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); ++fails; } \
  } while (0)

int main(int argc, char** argv) {
  using namespace spngd;
  const bool no_gpu = argc > 1 && std::strcmp(argv[1], "--expect-no-gpu") == 0;
  if (no_gpu) {
    try {
      b200::ctx();
      std::printf("FAIL: context created without a GPU\n");
      return 1;
    } catch (const NotPositiveDefinite&) {
      std::printf("FAIL: wrong exception type\n");
      return 1;
    } catch (const Error& e) {  // CUDA -> spngd::Error, no CPU fallback
      std::printf("NO_GPU_OK: %s\n", e.what());
      return 0;
    }
  }
  // test_fisher.cpp:231-249: A = 4 I_2, G = I_3, lambda = 1 -> pi = 2,
  // A_inv = I/6, G_inv = (2/3) I.
  std::vector<KroneckerBlock> one(1);
  one[0].A = SymMatrix(2);
  one[0].A(0, 0) = one[0].A(1, 1) = 4.0;
  one[0].G = SymMatrix(3);
  for (int i = 0; i < 3; ++i) one[0].G(i, i) = 1.0;
  damp_and_invert_all(one, 1.0);
  EXPECT(std::fabs(one[0].pi - 2.0) < 1e-6);
  EXPECT(std::fabs(one[0].A_inv(0, 0) - 1.0 / 6.0) < 1e-6 && std::fabs(one[0].A_inv(0, 1)) < 1e-7);
  EXPECT(std::fabs(one[0].G_inv(2, 2) - 2.0 / 3.0) < 1e-6);
  // A batch of 5 with a non-PD G factor in block 3 -> NotPositiveDefinite naming it.
  std::vector<KroneckerBlock> five(5);
  for (int k = 0; k < 5; ++k) {
    five[k].A = SymMatrix(40);
    five[k].G = SymMatrix(24);
    for (int i = 0; i < 40; ++i)
      for (int j = i; j < 40; ++j) five[k].A(i, j) = (i == j ? 2.0 : 0.0) + 0.01 * std::cos(double(i * 7 + j + k));
    for (int i = 0; i < 24; ++i) five[k].G(i, i) = 1.0 + 0.1 * i;
  }
  five[3].G(5, 5) = -50.0;
  bool threw = false;
  try {
    damp_and_invert_all(five, 2.5e-4);
  } catch (const NotPositiveDefinite& e) {
    threw = true;
    const std::string m = e.what();
    EXPECT(m.find("request 3") != std::string::npos);
    EXPECT(m.find("G factor") != std::string::npos);
    std::printf("NotPositiveDefinite: %s\n", e.what());
  }
  EXPECT(threw);
  // The same batch without the bad block succeeds.
  five.erase(five.begin() + 3);
  damp_and_invert_all(five, 2.5e-4);
  EXPECT(five[0].A_inv.dim() == 40);
  std::printf(fails ? "SHIM FAIL\n" : "SHIM OK\n");
  return fails ? 1 : 0;
}
