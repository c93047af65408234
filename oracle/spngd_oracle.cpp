// SP-NGD CPU ORACLE — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
//
// A plain fp64, Eigen-free restatement of the reference's hot-path functions
// (/root/reference/proj).  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library, and only as the
// checker or as the timed CPU baseline.  The product path (the CUDA library in
// paper_2002_06015_b200/) never calls into it.
//
// The reference itself cannot be compiled here: it needs Eigen3 (absent on
// this filesystem) and git-ignored vendor headers (doctest, json, CLI11), see
// DESIGN.md "Oracle".  Parity is pinned by porting the reference's own
// known-answer and math-identity tests (tests/test_oracle_kat.py) onto this
// restatement.  Every function cites the reference file:line it follows.
//
// Conventions kept from the reference:
//  * packed symmetric storage = upper triangle, row-major,
//    offset(i,j) = i*n - i*(i-1)/2 + (j-i)            (linalg.hpp:48-51)
//  * row-major weights g x a; kron action G X A        (linalg.cpp:58-62)
//  * BN unit moments interleaved (fgg, fgb, fbb) per channel (dist.cpp:283-292)
//  * error taxonomy of errors.hpp:10-85 as integer codes (see OR_* below).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

namespace {

enum : int {
  OR_OK = 0,
  OR_SHAPE_MISMATCH = 1,        // errors.hpp:16
  OR_NOT_POSITIVE_DEFINITE = 2, // errors.hpp:22
  OR_SINGULAR_BLOCK = 3,        // errors.hpp:27
  OR_ZERO_REFERENCE = 4,        // errors.hpp:32
  OR_EMPTY_BATCH = 5,           // errors.hpp:37
};

inline int64_t packed_size(int64_t n) { return n * (n + 1) / 2; }
inline int64_t poff(int64_t n, int64_t i, int64_t j) {
  if (i > j) std::swap(i, j);
  return i * n - i * (i - 1) / 2 + (j - i);  // linalg.hpp:48-51
}

// Neumaier-compensated packed accumulator (fisher.cpp:13-33).
struct Accum {
  std::vector<double> sum, comp;
  bool on;
  Accum(int64_t n, bool c) : sum(n, 0.0), comp(c ? n : 0, 0.0), on(c) {}
  inline void add(int64_t p, double v) {
    if (!on) { sum[p] += v; return; }
    const double s = sum[p], t = s + v;
    comp[p] += (std::fabs(s) >= std::fabs(v)) ? ((s - t) + v) : ((v - t) + s);
    sum[p] = t;
  }
  double total(int64_t p) const { return on ? sum[p] + comp[p] : sum[p]; }
};

// Eigen's vectorised dot reduces in independent packet lanes; four partial
// sums restate that without SIMD intrinsics (fisher.cpp:70 `row.dot(row)`).
inline double dot4(const double* a, const double* b, int64_t n) {
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  int64_t k = 0;
  for (; k + 4 <= n; k += 4) {
    s0 += a[k] * b[k];
    s1 += a[k + 1] * b[k + 1];
    s2 += a[k + 2] * b[k + 2];
    s3 += a[k + 3] * b[k + 3];
  }
  for (; k < n; ++k) s0 += a[k] * b[k];
  return (s0 + s2) + (s1 + s3);
}

inline double dot4f(const float* a, const float* b, int64_t n) {
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  int64_t k = 0;
  for (; k + 4 <= n; k += 4) {
    s0 += double(a[k]) * b[k];
    s1 += double(a[k + 1]) * b[k + 1];
    s2 += double(a[k + 2]) * b[k + 2];
    s3 += double(a[k + 3]) * b[k + 3];
  }
  for (; k < n; ++k) s0 += double(a[k]) * b[k];
  return (s0 + s2) + (s1 + s3);
}

void unpack(const double* p, int64_t n, std::vector<double>& d) {
  d.assign(n * n, 0.0);
  int64_t q = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i; j < n; ++j) { d[i * n + j] = p[q]; d[j * n + i] = p[q]; ++q; }
}

void pack(const std::vector<double>& d, int64_t n, double* p) {
  int64_t q = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i; j < n; ++j) p[q++] = d[i * n + j];
}

// mean_outer over a stacked fp64 or fp32 capture (fisher.cpp:55-75).
template <typename T>
void mean_outer_t(const T* stacked, int64_t cols, int64_t r, int64_t lo,
                  int64_t hi, double denom, bool compensated, double* out) {
  const int64_t dim = (r == 1) ? cols : r;
  Accum acc(packed_size(dim), compensated);
  std::vector<double> row(cols);
  for (int64_t s = lo; s < hi; ++s) {
    int64_t p = 0;
    if (r == 1) {
      const T* x = stacked + s * cols;
      for (int64_t i = 0; i < dim; ++i) {
        const double xi = x[i];
        for (int64_t j = i; j < dim; ++j) acc.add(p++, xi * double(x[j]));
      }
    } else {
      const T* blk = stacked + s * r * cols;
      for (int64_t i = 0; i < dim; ++i)
        for (int64_t j = i; j < dim; ++j) {
          double d;
          if constexpr (sizeof(T) == 8)
            d = dot4(reinterpret_cast<const double*>(blk + i * cols),
                     reinterpret_cast<const double*>(blk + j * cols), cols);
          else
            d = dot4f(reinterpret_cast<const float*>(blk + i * cols),
                      reinterpret_cast<const float*>(blk + j * cols), cols);
          acc.add(p++, d);
        }
    }
  }
  const int64_t ps = packed_size(dim);
  for (int64_t q = 0; q < ps; ++q) out[q] = acc.total(q) / denom;
}

// Cholesky + solve(I) + symmetrize (linalg.cpp:29-48).  Eigen's LLT is
// restated as an unblocked lower Cholesky; solve(I) as forward then back
// substitution on the identity, exactly the two triangular solves LLT::solve
// performs.
int spd_inverse_impl(const double* packed, int64_t n, double damping, double* out) {
  if (n == 0) return OR_SHAPE_MISMATCH;
  std::vector<double> a;
  unpack(packed, n, a);
  for (int64_t i = 0; i < n; ++i) a[i * n + i] += damping;
  for (double v : a)
    if (!std::isfinite(v)) return OR_NOT_POSITIVE_DEFINITE;
  // L in the lower triangle of a (row-major), right-looking.
  for (int64_t k = 0; k < n; ++k) {
    double d = a[k * n + k];
    for (int64_t p = 0; p < k; ++p) d -= a[k * n + p] * a[k * n + p];
    if (!(d > 0.0) || !std::isfinite(d)) return OR_NOT_POSITIVE_DEFINITE;
    const double lkk = std::sqrt(d);
    a[k * n + k] = lkk;
    for (int64_t i = k + 1; i < n; ++i) {
      double s = a[i * n + k];
      const double* li = &a[i * n];
      const double* lk = &a[k * n];
      s -= dot4(li, lk, k);
      a[i * n + k] = s / lkk;
    }
  }
  // Y = L^-1 I (forward), X = L^-T Y (backward); column-by-column over the
  // identity right-hand side.
  std::vector<double> x(n * n, 0.0), col(n);
  for (int64_t c = 0; c < n; ++c) {
    for (int64_t i = 0; i < n; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int64_t p = 0; p < i; ++p) s -= a[i * n + p] * col[p];
      col[i] = s / a[i * n + i];
    }
    for (int64_t i = n - 1; i >= 0; --i) {
      double s = col[i];
      for (int64_t p = i + 1; p < n; ++p) s -= a[p * n + i] * col[p];
      col[i] = s / a[i * n + i];
    }
    for (int64_t i = 0; i < n; ++i) x[i * n + c] = col[i];
  }
  for (double v : x)
    if (!std::isfinite(v)) return OR_NOT_POSITIVE_DEFINITE;
  std::vector<double> sym(n * n);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) sym[i * n + j] = 0.5 * (x[i * n + j] + x[j * n + i]);
  pack(sym, n, out);
  return OR_OK;
}

// Cheaper equivalent used for the timed CPU baseline at ResNet scale:
// Cholesky, triangular inverse, L^-T L^-1 (n^3 flops, the convention of
// SURVEY.md §8d).  Same math, same symmetrized packed output.
int spd_inverse_fast_impl(const double* packed, int64_t n, double damping, double* out) {
  if (n == 0) return OR_SHAPE_MISMATCH;
  std::vector<double> a;
  unpack(packed, n, a);
  for (int64_t i = 0; i < n; ++i) a[i * n + i] += damping;
  for (int64_t k = 0; k < n; ++k) {
    double d = a[k * n + k] - dot4(&a[k * n], &a[k * n], k);
    if (!(d > 0.0) || !std::isfinite(d)) return OR_NOT_POSITIVE_DEFINITE;
    const double lkk = std::sqrt(d);
    a[k * n + k] = lkk;
    for (int64_t i = k + 1; i < n; ++i)
      a[i * n + k] = (a[i * n + k] - dot4(&a[i * n], &a[k * n], k)) / lkk;
  }
  // Linv stored transposed (row-major upper): ut[j*n+i] = Linv[i][j], i>=j.
  std::vector<double> ut(n * n, 0.0);
  for (int64_t j = 0; j < n; ++j) {
    ut[j * n + j] = 1.0 / a[j * n + j];
    for (int64_t i = j + 1; i < n; ++i) {
      double s = 0.0;
      for (int64_t p = j; p < i; ++p) s += a[i * n + p] * ut[j * n + p];
      ut[j * n + i] = -s / a[i * n + i];
    }
  }
  // X[i][j] = sum_{p>=max(i,j)} Linv[p][i] Linv[p][j] = dot over rows of ut.
  int64_t q = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i; j < n; ++j) {
      const double v = dot4(&ut[i * n + j], &ut[j * n + j], n - j);
      if (!std::isfinite(v)) return OR_NOT_POSITIVE_DEFINITE;
      out[q++] = v;
    }
  return OR_OK;
}

double avg_eig(const double* p, int64_t n) {  // linalg.cpp:64-69
  double t = 0.0;
  for (int64_t i = 0; i < n; ++i) t += p[poff(n, i, i)];
  return t / double(n);
}

// G X A with both factors unpacked (linalg.cpp:58-62), fp64 dense.
void kron_matvec_impl(const double* gp, const double* ap, int64_t dg, int64_t da,
                      const double* x, double* out) {
  std::vector<double> G, A, T(dg * da, 0.0);
  unpack(gp, dg, G);
  unpack(ap, da, A);
  for (int64_t i = 0; i < dg; ++i)
    for (int64_t k = 0; k < dg; ++k) {
      const double gik = G[i * dg + k];
      if (gik == 0.0) continue;
      const double* xr = x + k * da;
      double* tr = &T[i * da];
      for (int64_t j = 0; j < da; ++j) tr[j] += gik * xr[j];
    }
  for (int64_t i = 0; i < dg; ++i) {
    double* o = out + i * da;
    std::fill(o, o + da, 0.0);
    for (int64_t k = 0; k < da; ++k) {
      const double tik = T[i * da + k];
      if (tik == 0.0) continue;
      const double* ar = &A[k * da];
      for (int64_t j = 0; j < da; ++j) o[j] += tik * ar[j];
    }
  }
}

int inv2x2_impl(double a, double b, double c, double d, double* o) {  // linalg.cpp:50-56
  const double det = a * d - b * c;
  if (std::fabs(det) < 1e-30) return OR_SINGULAR_BLOCK;
  o[0] = d / det; o[1] = -b / det; o[2] = -c / det; o[3] = a / det;
  return OR_OK;
}

// splitmix64 finalizer (rng.cpp:9-14).
inline uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

}  // namespace

extern "C" {

int64_t or_packed_size(int64_t n) { return packed_size(n); }
int64_t or_packed_offset(int64_t n, int64_t i, int64_t j) { return poff(n, i, j); }

// ---- linalg (linalg.cpp) -------------------------------------------------
void or_unpack(const double* p, int64_t n, double* dense) {
  std::vector<double> d;
  unpack(p, n, d);
  std::memcpy(dense, d.data(), sizeof(double) * n * n);
}
void or_pack(const double* dense, int64_t n, double* p) {
  int64_t q = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i; j < n; ++j) p[q++] = dense[i * n + j];
}
int or_spd_inverse(const double* packed, int64_t n, double damping, double* out) {
  return spd_inverse_impl(packed, n, damping, out);
}
int or_spd_inverse_fast(const double* packed, int64_t n, double damping, double* out) {
  return spd_inverse_fast_impl(packed, n, damping, out);
}
int or_inv2x2(double a, double b, double c, double d, double* out4) {
  return inv2x2_impl(a, b, c, d, out4);
}
int or_kron_matvec(const double* gp, const double* ap, int64_t dg, int64_t da,
                   const double* x, double* out) {
  if (dg <= 0 || da <= 0) return OR_SHAPE_MISMATCH;
  kron_matvec_impl(gp, ap, dg, da, x, out);
  return OR_OK;
}
double or_avg_eigenvalue(const double* p, int64_t n) { return avg_eig(p, n); }
double or_frob_norm(const double* p, int64_t n) {  // linalg.cpp:71-80
  double acc = 0.0;
  int64_t q = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i; j < n; ++j, ++q) acc += ((i == j) ? 1.0 : 2.0) * p[q] * p[q];
  return std::sqrt(acc);
}
int or_rel_frob_distance(const double* a, const double* b, int64_t n, double* out) {
  const double ref = or_frob_norm(b, n);  // linalg.cpp:82-96
  if (ref == 0.0) return OR_ZERO_REFERENCE;
  double acc = 0.0;
  int64_t q = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i; j < n; ++j, ++q) {
      const double d = a[q] - b[q];
      acc += ((i == j) ? 1.0 : 2.0) * d * d;
    }
  *out = std::sqrt(acc) / ref;
  return OR_OK;
}

// ---- fisher (fisher.cpp) -------------------------------------------------
// stacked capture: r==1 -> M x cols rows (FC); r>1 -> (M*r) x cols (conv).
int or_mean_outer(const double* stacked, int64_t cols, int64_t r, int64_t lo,
                  int64_t hi, double denom, int compensated, double* out) {
  if (hi <= lo || lo < 0) return OR_EMPTY_BATCH;
  mean_outer_t<double>(stacked, cols, r, lo, hi, denom, compensated != 0, out);
  return OR_OK;
}
int or_mean_outer_f32(const float* stacked, int64_t cols, int64_t r, int64_t lo,
                      int64_t hi, double denom, int compensated, double* out) {
  if (hi <= lo || lo < 0) return OR_EMPTY_BATCH;
  mean_outer_t<float>(stacked, cols, r, lo, hi, denom, compensated != 0, out);
  return OR_OK;
}
// factor_A (fisher.cpp:92-114): FC denom n, conv denom n*h_out*w_out.
int or_factor_A_f32(const float* act, int64_t is_conv, int64_t a, int64_t hw,
                    int64_t lo, int64_t hi, int compensated, double* out) {
  if (hi <= lo || lo < 0) return OR_EMPTY_BATCH;
  const double n = double(hi - lo);
  if (!is_conv) mean_outer_t<float>(act, a, 1, lo, hi, n, compensated, out);
  else mean_outer_t<float>(act, hw, a, lo, hi, n * double(hw), compensated, out);
  return OR_OK;
}
// factor_G (fisher.cpp:116-145): denom n for both FC and conv.
int or_factor_G_f32(const float* grad, int64_t is_conv, int64_t g, int64_t hw,
                    int64_t lo, int64_t hi, int compensated, double* out) {
  if (hi <= lo || lo < 0) return OR_EMPTY_BATCH;
  const double n = double(hi - lo);
  if (!is_conv) mean_outer_t<float>(grad, g, 1, lo, hi, n, compensated, out);
  else mean_outer_t<float>(grad, hw, g, lo, hi, n, compensated, out);
  return OR_OK;
}
// Per-sample BN parameter gradients captured in the backward (net.cpp:467-475):
// gg[s][ch] = sum_p dY[s][ch*S+p] * xhat[s][ch*S+p], gb[s][ch] = sum_p dY[...],
// dY / xhat M x (c*S) row-major (fp32 inputs, fp64 sums), gg / gb M x c.
int or_bn_grad_reduce(const float* dy, const float* xh, int64_t M, int64_t c, int64_t S, double* gg, double* gb) {
  if (M <= 0) return 5;                   // EmptyBatch
  if (c <= 0 || S <= 0) return 1;         // ShapeMismatch
  for (int64_t s = 0; s < M; ++s)
    for (int64_t ch = 0; ch < c; ++ch) {
      const float* d = dy + (s * c + ch) * S;
      const float* x = xh + (s * c + ch) * S;
      double dot = 0.0, sum = 0.0;
      for (int64_t p = 0; p < S; ++p) {
        dot += double(d[p]) * double(x[p]);
        sum += double(d[p]);
      }
      gg[s * c + ch] = dot;
      gb[s * c + ch] = sum;
    }
  return 0;
}

// build_bn_block (fisher.cpp:147-185); gg, gb are M x c row-major.  Output is
// the interleaved 3c wire payload of dist.cpp:283-292.
int or_build_bn_block(const double* gg, const double* gb, int64_t c, int64_t lo,
                      int64_t hi, int compensated, double* out3c) {
  if (hi <= lo || lo < 0) return OR_EMPTY_BATCH;
  Accum acc(3 * c, compensated != 0);
  for (int64_t s = lo; s < hi; ++s)
    for (int64_t ch = 0; ch < c; ++ch) {
      const double g = gg[s * c + ch], b = gb[s * c + ch];
      acc.add(3 * ch + 0, g * g);
      acc.add(3 * ch + 1, g * b);
      acc.add(3 * ch + 2, b * b);
    }
  for (int64_t q = 0; q < 3 * c; ++q) out3c[q] = acc.total(q) / double(hi - lo);
  return OR_OK;
}
// build_bn_full (fisher.cpp:187-216), interleaved (gamma_i, beta_i) order.
int or_build_bn_full(const double* gg, const double* gb, int64_t c, int64_t lo,
                     int64_t hi, int compensated, double* outp) {
  if (hi <= lo || lo < 0) return OR_EMPTY_BATCH;
  const int64_t dim = 2 * c;
  Accum acc(packed_size(dim), compensated != 0);
  std::vector<double> u(dim);
  for (int64_t s = lo; s < hi; ++s) {
    for (int64_t ch = 0; ch < c; ++ch) { u[2 * ch] = gg[s * c + ch]; u[2 * ch + 1] = gb[s * c + ch]; }
    int64_t p = 0;
    for (int64_t i = 0; i < dim; ++i)
      for (int64_t j = i; j < dim; ++j) acc.add(p++, u[i] * u[j]);
  }
  for (int64_t q = 0; q < packed_size(dim); ++q) outp[q] = acc.total(q) / double(hi - lo);
  return OR_OK;
}
// damp_and_invert (fisher.cpp:218-228).
int or_damp_and_invert(const double* A, const double* G, int64_t da, int64_t dg,
                       double lambda, double* pi_out, double* Ainv, double* Ginv) {
  if (!(lambda > 0.0)) return OR_NOT_POSITIVE_DEFINITE;
  const double ea = avg_eig(A, da), eg = avg_eig(G, dg);
  const double pi = (ea < 1e-12 || eg < 1e-12) ? 1.0 : std::sqrt(ea / eg);
  const double root = std::sqrt(lambda);
  *pi_out = pi;
  int rc = spd_inverse_impl(A, da, pi * root, Ainv);
  if (rc) return rc;
  return spd_inverse_impl(G, dg, root / pi, Ginv);
}
// damp_bn (fisher.cpp:230-246): per channel inv2x2(F + lambda I).
int or_damp_bn(const double* m3c, int64_t c, double lambda, double* inv3c) {
  if (!(lambda > 0.0)) return OR_NOT_POSITIVE_DEFINITE;
  for (int64_t ch = 0; ch < c; ++ch) {
    double o[4];
    const double fgg = m3c[3 * ch], fgb = m3c[3 * ch + 1], fbb = m3c[3 * ch + 2];
    int rc = inv2x2_impl(fgg + lambda, fgb, fgb, fbb + lambda, o);
    if (rc) return rc;
    inv3c[3 * ch] = o[0]; inv3c[3 * ch + 1] = o[1]; inv3c[3 * ch + 2] = o[3];
  }
  return OR_OK;
}
// precondition_bn (fisher.cpp:259-276): recomputes the 2x2 inverse from the
// raw moments with the lambda argument.
int or_precondition_bn(const double* m3c, int64_t c, const double* gg,
                       const double* gb, double lambda, double* pg, double* pb) {
  for (int64_t ch = 0; ch < c; ++ch) {
    double o[4];
    const double fgg = m3c[3 * ch], fgb = m3c[3 * ch + 1], fbb = m3c[3 * ch + 2];
    int rc = inv2x2_impl(fgg + lambda, fgb, fgb, fbb + lambda, o);
    if (rc) return rc;
    pg[ch] = o[0] * gg[ch] + o[1] * gb[ch];
    pb[ch] = o[1] * gg[ch] + o[3] * gb[ch];
  }
  return OR_OK;
}
// precondition_bn_full (fisher.cpp:278-296).
int or_precondition_bn_full(const double* finv_p, int64_t c, const double* gg,
                            const double* gb, double* pg, double* pb) {
  const int64_t dim = 2 * c;
  std::vector<double> F;
  unpack(finv_p, dim, F);
  std::vector<double> u(dim);
  for (int64_t ch = 0; ch < c; ++ch) { u[2 * ch] = gg[ch]; u[2 * ch + 1] = gb[ch]; }
  for (int64_t ch = 0; ch < c; ++ch) {
    pg[ch] = dot4(&F[(2 * ch) * dim], u.data(), dim);
    pb[ch] = dot4(&F[(2 * ch + 1) * dim], u.data(), dim);
  }
  return OR_OK;
}
// ngd_step per-tensor update (fisher.cpp:332-333, :353-356).
void or_ngd_update(const double* p, const double* delta, const double* v, int64_t n,
                   double eta, double momentum, double* np, double* nv) {
  for (int64_t i = 0; i < n; ++i) {
    np[i] = p[i] - eta * delta[i] + momentum * v[i];
    nv[i] = np[i] - p[i];
  }
}
// rescale_weights (schemes.cpp:116-119) + velocity fix (dist.cpp:621-632).
void or_rescale(const double* w_new, const double* w_old, int64_t n, int64_t d_out,
                double* w_out, double* v_out) {
  double ss = 0.0;
  for (int64_t i = 0; i < n; ++i) ss += w_new[i] * w_new[i];
  const double target = std::sqrt(2.0 * double(d_out));
  const double s = target / (std::sqrt(ss) + 1e-9);
  for (int64_t i = 0; i < n; ++i) {
    w_out[i] = s * w_new[i];
    if (v_out) v_out[i] = w_out[i] - w_old[i];
  }
}

// ---- stale (stale.hpp:18-64) ---------------------------------------------
double or_weighted_norm(const double* x, const double* w, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += w[i] * x[i] * x[i];
  return std::sqrt(s);
}
// similar(): returns 1/0; weights taken from `ref` (stale.hpp:56-64).
int or_similar(const double* x, const double* ref, const double* w, int64_t n,
               double alpha) {
  double dn = 0.0, rn = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double d = x[i] - ref[i];
    dn += w[i] * d * d;
    rn += w[i] * ref[i] * ref[i];
  }
  dn = std::sqrt(dn); rn = std::sqrt(rn);
  if (rn == 0.0) return dn == 0.0;
  return dn / rn < alpha;
}

// ---- net capture layout (net.cpp:199-219) --------------------------------
// im2col of one sample: row = ch*k^2 + ky*k + kx, column = oy*w_out + ox.
void or_im2col(const double* x, int64_t c, int64_t h, int64_t w, int64_t k,
               int64_t stride, int64_t pad, double* out) {
  const int64_t ho = (h + 2 * pad - k) / stride + 1, wo = (w + 2 * pad - k) / stride + 1;
  for (int64_t ch = 0; ch < c; ++ch)
    for (int64_t ky = 0; ky < k; ++ky)
      for (int64_t kx = 0; kx < k; ++kx) {
        const int64_t row = ch * k * k + ky * k + kx;
        for (int64_t oy = 0; oy < ho; ++oy)
          for (int64_t ox = 0; ox < wo; ++ox) {
            const int64_t iy = oy * stride + ky - pad, ix = ox * stride + kx - pad;
            out[row * ho * wo + oy * wo + ox] =
                (iy < 0 || iy >= h || ix < 0 || ix >= w) ? 0.0 : x[(ch * h + iy) * w + ix];
          }
      }
}

// ---- rng (rng.cpp:9-83) ---------------------------------------------------
uint64_t or_rng_derive(uint64_t seed, uint64_t tag) {
  return mix64(mix64(seed) + (tag + 1) * 0x9e3779b97f4a7c15ULL);
}
// Draws n values from Rng(seed): kind 0 = uniform(), 1 = normal().
void or_rng_fill(uint64_t seed, int kind, int64_t n, double* out) {
  std::mt19937_64 e(seed);
  for (int64_t i = 0; i < n; ++i) {
    if (kind == 0) {
      out[i] = double(e() >> 11) * 0x1.0p-53;
    } else {
      const double u1 = (double(e() >> 11) + 1.0) * 0x1.0p-53;
      const double u2 = double(e() >> 11) * 0x1.0p-53;
      out[i] = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
    }
  }
}

// ---- whole-layer K-FAC step (the timed CPU baseline) ---------------------
// One Conv/FC layer of Stage 4 on one worker, composed from the restated
// primitives exactly as accumulate_microsteps does it (dist.cpp:539-633):
// factor_A, factor_G -> damp_and_invert -> precondition -> w - eta P + m v ->
// rescale.  `fast_inverse` selects the n^3 Cholesky-inverse restatement.
struct OrLayer {
  int64_t is_conv, a, g, hw, batch;
  const float* act;   // reference capture layout (net.hpp:84-101)
  const float* grad;
  const float* dW;    // g x a row-major
  const float* W;     // g x a
  const float* V;     // g x a
  double* W_out;      // g x a (may be null)
  double* V_out;
  double* Ainv_out;   // packed (may be null)
  double* Ginv_out;
  double* P_out;      // g x a preconditioned gradient (may be null)
  double seconds[4];  // factor, inverse, precondition, update
  int status;
};

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}


static void run_layer(OrLayer* L, double lambda, double eta, double momentum,
                      int rescale, int fast_inverse) {
  const int64_t a = L->a, g = L->g;
  std::vector<double> A(packed_size(a)), G(packed_size(g)), Ai(packed_size(a)), Gi(packed_size(g));
  double t0 = now_s();
  const double n = double(L->batch);
  if (!L->is_conv) {
    mean_outer_t<float>(L->act, a, 1, 0, L->batch, n, false, A.data());
    mean_outer_t<float>(L->grad, g, 1, 0, L->batch, n, false, G.data());
  } else {
    mean_outer_t<float>(L->act, L->hw, a, 0, L->batch, n * double(L->hw), false, A.data());
    mean_outer_t<float>(L->grad, L->hw, g, 0, L->batch, n, false, G.data());
  }
  double t1 = now_s();
  const double ea = avg_eig(A.data(), a), eg = avg_eig(G.data(), g);
  const double pi = (ea < 1e-12 || eg < 1e-12) ? 1.0 : std::sqrt(ea / eg);
  const double root = std::sqrt(lambda);
  auto inv = fast_inverse ? spd_inverse_fast_impl : spd_inverse_impl;
  int rc = inv(A.data(), a, pi * root, Ai.data());
  if (!rc) rc = inv(G.data(), g, root / pi, Gi.data());
  double t2 = now_s();
  L->status = rc;
  if (rc) return;
  std::vector<double> X(g * a), P(g * a);
  for (int64_t i = 0; i < g * a; ++i) X[i] = L->dW[i];
  kron_matvec_impl(Gi.data(), Ai.data(), g, a, X.data(), P.data());
  double t3 = now_s();
  std::vector<double> w(g * a), v(g * a), nw(g * a), nv(g * a);
  for (int64_t i = 0; i < g * a; ++i) { w[i] = L->W[i]; v[i] = L->V[i]; }
  or_ngd_update(w.data(), P.data(), v.data(), g * a, eta, momentum, nw.data(), nv.data());
  if (rescale) or_rescale(nw.data(), w.data(), g * a, g, nw.data(), nv.data());
  double t4 = now_s();
  if (L->W_out) std::memcpy(L->W_out, nw.data(), sizeof(double) * g * a);
  if (L->V_out) std::memcpy(L->V_out, nv.data(), sizeof(double) * g * a);
  if (L->Ainv_out) std::memcpy(L->Ainv_out, Ai.data(), sizeof(double) * Ai.size());
  if (L->Ginv_out) std::memcpy(L->Ginv_out, Gi.data(), sizeof(double) * Gi.size());
  if (L->P_out) std::memcpy(L->P_out, P.data(), sizeof(double) * g * a);
  L->seconds[0] = t1 - t0; L->seconds[1] = t2 - t1; L->seconds[2] = t3 - t2; L->seconds[3] = t4 - t3;
}

int64_t or_sizeof_layer() { return sizeof(OrLayer); }

// Runs the layers on `threads` host threads (layer-parallel, SPEC.md:285-286
// allows per-layer concurrency).  Returns the first nonzero status.
int or_kfac_layers(OrLayer* layers, int64_t n_layers, double lambda, double eta,
                   double momentum, int rescale, int fast_inverse, int threads) {
  if (threads < 1) threads = 1;
  std::vector<std::thread> pool;
  std::atomic<int64_t> next{0};
  auto worker = [&]() {
    for (;;) {
      const int64_t i = next.fetch_add(1);
      if (i >= n_layers) return;
      run_layer(&layers[i], lambda, eta, momentum, rescale, fast_inverse);
    }
  };
  if (threads == 1) worker();
  else {
    for (int t = 0; t < threads; ++t) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
  }
  for (int64_t i = 0; i < n_layers; ++i)
    if (layers[i].status) return layers[i].status;
  return OR_OK;
}

// Counter-based synthetic stream shared with the device generator
// (paper_2002_06015_b200/csrc/synth.cu): element i of stream `key` is a
// Box-Muller normal from two splitmix64 draws (rng.cpp:9-14, :36-45).
void or_synth_normal(uint64_t key, int64_t offset, int64_t n, float* out) {
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t c = uint64_t(offset + i);
    const uint64_t b1 = mix64(key ^ (2 * c)), b2 = mix64(key ^ (2 * c + 1));
    const double u1 = (double(b1 >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = double(b2 >> 11) * 0x1.0p-53;
    out[i] = float(std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2));
  }
}

}  // extern "C"
