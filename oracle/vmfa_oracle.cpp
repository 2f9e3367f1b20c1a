// =============================================================================
// vmfa_oracle.cpp — CPU fp64 ORACLE for the v-MFA hot path.
//
// TEST INFRASTRUCTURE ONLY. This file is the checker: it may be loaded by
// tests/, by __graft_entry__.smoke() and by bench.py's cpu_baseline /
// `--impl reference` legs, never by the product path
// (paper_2501_12299_b200/), which must fail loudly without its CUDA library.
//
// It is a plain-C++ restatement (no Eigen: the reference's Eigen3 dependency
// is absent from this image, so the reference library itself is unbuildable)
// of the reference's algorithm for one v-MFA EM iteration. Every function cites
// the reference file:line it follows (paths relative to /root/reference/).
// Pins: the RNG/LSE restatement is checked bit-exactly against golden vectors
// produced by compiling the reference's own Eigen-free headers
// (oracle/ref_golden.cpp -> tests/golden/rng_ref.json); the Eigen-dependent
// arithmetic is pinned by the SPEC.md known-answer examples and by dense
// covariance formulas (tests/oracle.hpp semantics) in tests/. Eigen's
// LLT/LDLT/GEMV summation orders are not reproduced bit-exactly.
//
// Layouts (the reference's in-memory layouts):
//   X      N x D float, row-major                      (dataset.hpp:13-14)
//   pi     C                                            (model.hpp:25)
//   mu     C x D row-major                              (model.hpp:26)
//   lam    C blocks of D x H column-major: (c,d,h) at c*D*H + h*D + d
//   psi    C x D row-major (the reference's `dnoise`)   (model.hpp:28)
//   U      like lam;  V  C blocks H x D col-major: (c,h,d) at c*H*D + d*H + h
//   Lmat, Sz  C blocks H x H col-major
//   K      N x C' int32 row-major, rows sorted ascending (model.hpp:90-103)
//   g      C x G int32 (-1 padded) + g_count[C]          (estep.hpp:22)
//   ret    count[N], idx[N*stride] (-1 pad), lj[N*stride] (estep.hpp:48-70)
//   Y      C blocks D x (H+1) col-major; E C blocks (H+1)^2 col-major;
//   sq     C x D row-major                                (mstep.hpp:14-22)
// =============================================================================
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <numeric>
#include <string>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

namespace orc {

using u64 = std::uint64_t;
using i64 = std::int64_t;
using i32 = std::int32_t;

constexpr double kLog2Pi = 1.8378770664093453;  // numerics.hpp:10
constexpr double kNegInf = -std::numeric_limits<double>::infinity();

// Status codes mirror the reference's exception types (errors.hpp:9-62).
enum Status : int {
  OK = 0,
  INVALID_ARGUMENT = 1,
  CHOLESKY_FAILURE = 2,
  EMPTY_KSET = 3,
  INSUFFICIENT_CANDIDATES = 4,
  SINGULAR_EC = 5,
  MAX_ITER_EXCEEDED = 6,
  TARGET_UNREACHABLE = 7,
  DEGENERATE_DATA = 8,
};

// ---------------------------------------------------------------- RNG
// Restatement of rng.hpp:9-98 (splitmix64, hash_combine, hash3, xoshiro256++
// Rng with hand-written uniform / uniform_int / Box-Muller gaussian,
// uniform_component). Pinned bit-exactly by tests/golden/rng_ref.json.
inline u64 mix_step(u64& s) {  // rng.hpp:9-14
  u64 z = (s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
inline u64 combine(u64 a, u64 b) {  // rng.hpp:16-21
  u64 s = a;
  const u64 h = mix_step(s);
  s ^= b + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
  return mix_step(s);
}
inline u64 key3(u64 a, u64 b, u64 c) { return combine(combine(a, b), c); }  // rng.hpp:23-25

struct Stream {  // rng.hpp:30-86
  u64 w[4];
  double spare = 0.0;
  bool has_spare = false;
  explicit Stream(u64 seed) {
    u64 s = seed;
    for (auto& x : w) x = mix_step(s);
  }
  static u64 rotl(u64 x, int k) { return (x << k) | (x >> (64 - k)); }
  u64 next() {
    const u64 out = rotl(w[0] + w[3], 23) + w[0];
    const u64 t = w[1] << 17;
    w[2] ^= w[0];
    w[3] ^= w[1];
    w[1] ^= w[2];
    w[0] ^= w[3];
    w[2] ^= t;
    w[3] = rotl(w[3], 45);
    return out;
  }
  double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  i64 below(i64 bound) {
    return static_cast<i64>((static_cast<unsigned __int128>(next()) *
                             static_cast<unsigned __int128>(bound)) >> 64);
  }
  double normal() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    double u1 = unit();
    while (u1 <= 0.0) u1 = unit();
    const double u2 = unit();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586 * u2;
    spare = r * std::sin(a);
    has_spare = true;
    return r * std::cos(a);
  }
};

inline int draw_component(u64 seed, u64 iteration, u64 n, int C) {  // rng.hpp:91-98
  const u64 h = key3(seed, iteration, n);
  return static_cast<int>((static_cast<unsigned __int128>(h) *
                           static_cast<unsigned __int128>(C)) >> 64);
}

// numerics.hpp:15-22 (max-shifted log-sum-exp; all -inf -> -inf)
inline double lse(const double* v, int m) {
  double mx = kNegInf;
  for (int i = 0; i < m; ++i) mx = std::max(mx, v[i]);
  if (!std::isfinite(mx)) return mx;
  double s = 0.0;
  for (int i = 0; i < m; ++i) s += std::exp(v[i] - mx);
  return mx + std::log(s);
}

// ---------------------------------------------------------------- threading
// parallel.hpp:14-34: contiguous chunks, worker w gets floor(n/T) + [w < n%T].
inline void for_chunks(i64 n, int threads, const std::function<void(int, i64, i64)>& fn) {
  if (n <= 0) return;
  if (threads > n) threads = static_cast<int>(n);
  if (threads <= 1) {
    fn(0, 0, n);
    return;
  }
  std::vector<std::thread> pool;
  const i64 base = n / threads, rem = n % threads;
  i64 b = 0;
  for (int w = 0; w < threads; ++w) {
    const i64 len = base + (w < rem ? 1 : 0);
    pool.emplace_back(fn, w, b, b + len);
    b += len;
  }
  for (auto& t : pool) t.join();
}

// ---------------------------------------------------------------- small dense fp64
// Cholesky A = R R^T (R lower, column-major n x n). Returns false on a
// non-positive / non-finite pivot (the reference's LLT info != Success).
inline bool chol(const double* A, double* R, int n) {
  std::fill(R, R + n * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double d = A[j * n + j];
    for (int k = 0; k < j; ++k) d -= R[k * n + j] * R[k * n + j];
    if (!(d > 0.0) || !std::isfinite(d)) return false;
    const double rjj = std::sqrt(d);
    R[j * n + j] = rjj;
    for (int i = j + 1; i < n; ++i) {
      double s = A[j * n + i];
      for (int k = 0; k < j; ++k) s -= R[k * n + i] * R[k * n + j];
      R[j * n + i] = s / rjj;
    }
  }
  return true;
}
// Solve (R R^T) x = b in place.
inline void chol_solve(const double* R, double* b, int n) {
  for (int i = 0; i < n; ++i) {
    double s = b[i];
    for (int k = 0; k < i; ++k) s -= R[k * n + i] * b[k];
    b[i] = s / R[i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int k = i + 1; k < n; ++k) s -= R[i * n + k] * b[k];
    b[i] = s / R[i * n + i];
  }
}

// LDL^T with diagonal pivoting as Eigen::LDLT<MatrixXd> (Lower) computes it --
// the factorisation update_params uses (mstep.cpp:129-130). Eigen is a
// third-party dependency (CMakeLists.txt:12, Eigen3 >= 3.3, not vendored);
// restated from its published ldlt_inplace<Lower>::unblocked / _solve_impl:
// left-looking, step k pivots on the largest |diagonal| of rows k.. (the
// trailing diagonal is the permuted original one), info fails only when a zero
// pivot is followed by a non-zero one or a zero pivot has a non-zero column;
// an all-zero diagonal gives D = 0. A (n x n, column-major, symmetric) is
// overwritten by L (strictly lower) and D (diagonal).
inline bool ldlt(double* A, int* perm, int n) {
  auto M = [&](int r, int c) -> double& { return A[c * n + r]; };
  std::vector<double> temp(n);
  bool ret = true, found_zero = false;
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = std::fabs(M(k, k));
    for (int j = k + 1; j < n; ++j)
      if (std::fabs(M(j, j)) > best) best = std::fabs(M(j, j)), p = j;
    perm[k] = p;
    if (p != k) {
      for (int c = 0; c < n; ++c) std::swap(M(k, c), M(p, c));
      for (int r = 0; r < n; ++r) std::swap(M(r, k), M(r, p));
    }
    for (int j = 0; j < k; ++j) temp[j] = M(j, j) * M(k, j);
    double s = 0.0;
    for (int j = 0; j < k; ++j) s += M(k, j) * temp[j];
    const double akk = M(k, k) - s;
    const bool valid = std::fabs(akk) > 0.0;
    if (k == 0 && !valid) {
      for (int j = 0; j < n; ++j) perm[j] = j;
      break;
    }
    bool col_zero = true;
    for (int i = k + 1; i < n; ++i) {
      double t = M(i, k);
      for (int j = 0; j < k; ++j) t -= M(i, j) * temp[j];
      if (valid) t /= akk;
      else col_zero = col_zero && t == 0.0;
      M(i, k) = t;
    }
    M(k, k) = akk;
    if (!valid && k + 1 < n) ret = ret && col_zero;
    if (found_zero && valid) ret = false;
    else if (!valid) found_zero = true;
  }
  return ret;
}
// x = P^T L^-T D^+ L^-1 P b, D^+_i = 1/d_i if |d_i| > DBL_MIN else 0.
inline void ldlt_solve(const double* A, const int* perm, double* b, int n) {
  for (int k = 0; k < n; ++k) std::swap(b[k], b[perm[k]]);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) b[i] -= A[j * n + i] * b[j];
  for (int i = 0; i < n; ++i) {
    const double d = A[i * n + i];
    b[i] = std::fabs(d) > std::numeric_limits<double>::min() ? b[i] / d : 0.0;
  }
  for (int i = n - 1; i >= 0; --i)
    for (int j = i + 1; j < n; ++j) b[i] -= A[i * n + j] * b[j];
  for (int k = n - 1; k >= 0; --k) std::swap(b[k], b[perm[k]]);
}

// ---------------------------------------------------------------- model
struct Caches {
  int C, D, H;
  std::vector<double> U, Lmat, V, Sz, inv_psi, logdet, log_pi;
  void alloc(int C_, int D_, int H_) {
    C = C_, D = D_, H = H_;
    U.assign((size_t)C * D * H, 0.0);
    V.assign((size_t)C * D * H, 0.0);
    Lmat.assign((size_t)C * H * H, 0.0);
    Sz.assign((size_t)C * H * H, 0.0);
    inv_psi.assign((size_t)C * D, 0.0);
    logdet.assign(C, 0.0);
    log_pi.assign(C, 0.0);
  }
};

// precompute_component, model.cpp:43-73.
inline int precompute_one(int c, int D, int H, const double* pi, const double* mu,
                          const double* lam, const double* psi, double* U, double* Lm,
                          double* V, double* Sz, double* ipsi, double* logdet,
                          double* log_pi) {
  (void)mu;
  const double* L = lam + (size_t)c * D * H;
  const double* ps = psi + (size_t)c * D;
  for (int d = 0; d < D; ++d) ipsi[d] = 1.0 / ps[d];                        // :49
  for (int h = 0; h < H; ++h)
    for (int d = 0; d < D; ++d) U[h * D + d] = ipsi[d] * L[h * D + d];     // :50
  std::vector<double> M(H * H), R(H * H);
  for (int j = 0; j < H; ++j)
    for (int i = 0; i < H; ++i) {
      double s = 0.0;
      for (int d = 0; d < D; ++d) s += L[i * D + d] * U[j * D + d];
      M[j * H + i] = s + (i == j ? 1.0 : 0.0);                              // :51-52
    }
  for (int j = 0; j < H; ++j)
    for (int i = 0; i < H; ++i) Lm[j * H + i] = 0.5 * (M[j * H + i] + M[i * H + j]);  // :53
  if (!chol(Lm, R.data(), H)) {                                             // :55-63
    for (int i = 0; i < H; ++i) Lm[i * H + i] += 1e-10;
    if (!chol(Lm, R.data(), H)) return CHOLESKY_FAILURE;
  }
  std::vector<double> b(H);
  for (int d = 0; d < D; ++d) {                                             // :64 V = L^-1 U^T
    for (int h = 0; h < H; ++h) b[h] = U[h * D + d];
    chol_solve(R.data(), b.data(), H);
    for (int h = 0; h < H; ++h) V[d * H + h] = b[h];
  }
  for (int j = 0; j < H; ++j) {                                             // :65 Sigma_z = L^-1
    for (int h = 0; h < H; ++h) b[h] = (h == j) ? 1.0 : 0.0;
    chol_solve(R.data(), b.data(), H);
    for (int h = 0; h < H; ++h) Sz[j * H + h] = b[h];
  }
  double ld = 0.0;
  for (int h = 0; h < H; ++h) ld += std::log(R[h * H + h]);
  double lp = 0.0;
  for (int d = 0; d < D; ++d) lp += std::log(ps[d]);
  *logdet = 2.0 * ld + lp;                                                  // :67-70
  *log_pi = pi[c] > 0.0 ? std::log(pi[c]) : kNegInf;                       // :71
  return OK;
}

// log_joint, model.cpp:81-95.
inline double joint(const Caches& k, int c, const double* mu_c, const float* x, double* v,
                    double* a, double* b) {
  const int D = k.D, H = k.H;
  const double* ip = k.inv_psi.data() + (size_t)c * D;
  const double* U = k.U.data() + (size_t)c * D * H;
  const double* V = k.V.data() + (size_t)c * D * H;
  double diag = 0.0;
  for (int d = 0; d < D; ++d) {
    v[d] = static_cast<double>(x[d]) - mu_c[d];
    diag += v[d] * v[d] * ip[d];
  }
  for (int h = 0; h < H; ++h) {
    double sa = 0.0;
    for (int d = 0; d < D; ++d) sa += U[h * D + d] * v[d];
    a[h] = sa;
    b[h] = 0.0;
  }
  for (int d = 0; d < D; ++d) {
    const double vd = v[d];
    for (int h = 0; h < H; ++h) b[h] += V[d * H + h] * vd;
  }
  double ab = 0.0;
  for (int h = 0; h < H; ++h) ab += a[h] * b[h];
  const double maha = diag - ab;
  return k.log_pi[c] - 0.5 * (D * kLog2Pi + k.logdet[c] + maha);
}

struct Problem {
  i64 N;
  int D, H, C, Cp, G;
  const float* X;
  const double *pi, *mu;
  const Caches* k;
};

}  // namespace orc

using namespace orc;

// =============================================================================
// C API (ctypes). Every entry returns a Status (0 = OK) unless noted.
// =============================================================================
extern "C" {

// ---- RNG pins ----------------------------------------------------------------
u64 orc_hash_combine(u64 a, u64 b) { return combine(a, b); }
u64 orc_hash3(u64 a, u64 b, u64 c) { return key3(a, b, c); }
int orc_uniform_component(u64 seed, u64 it, u64 n, int C) { return draw_component(seed, it, n, C); }
void orc_rng_u64(u64 seed, int n, u64* out) {
  Stream s(seed);
  for (int i = 0; i < n; ++i) out[i] = s.next();
}
// ops: 0 = gaussian, 1 = uniform, 2 = uniform_int(bound)
void orc_rng_ops(u64 seed, int n, const int* ops, const i64* bounds, double* out) {
  Stream s(seed);
  for (int i = 0; i < n; ++i) {
    if (ops[i] == 0) out[i] = s.normal();
    else if (ops[i] == 1) out[i] = s.unit();
    else out[i] = static_cast<double>(s.below(bounds[i]));
  }
}
double orc_log_sum_exp(const double* v, int m) { return lse(v, m); }

// ---- dataset.cpp:22-39 --------------------------------------------------------
void orc_per_dimension_variance(const float* X, i64 N, int D, double* var) {
  std::vector<double> mean(D, 0.0);
  for (i64 i = 0; i < N; ++i)
    for (int d = 0; d < D; ++d) mean[d] += static_cast<double>(X[i * D + d]);
  for (int d = 0; d < D; ++d) mean[d] /= static_cast<double>(N);
  for (int d = 0; d < D; ++d) var[d] = 0.0;
  for (i64 i = 0; i < N; ++i)
    for (int d = 0; d < D; ++d) {
      const double t = static_cast<double>(X[i * D + d]) - mean[d];
      var[d] += t * t;
    }
  for (int d = 0; d < D; ++d) var[d] /= static_cast<double>(N);
}
void orc_variance_floor(const float* X, i64 N, int D, double* floor) {
  orc_per_dimension_variance(X, N, D, floor);
  for (int d = 0; d < D; ++d) floor[d] = std::max(1e-6 * floor[d], 1e-8);
}

// ---- model.cpp:43-79 ------------------------------------------------------------
int orc_precompute(int C, int D, int H, const double* pi, const double* mu, const double* lam,
                   const double* psi, double* U, double* Lmat, double* V, double* Sz,
                   double* inv_psi, double* logdet, double* log_pi, int* failed_component) {
  for (int c = 0; c < C; ++c) {
    const int st = precompute_one(c, D, H, pi, mu, lam, psi, U + (size_t)c * D * H,
                                  Lmat + (size_t)c * H * H, V + (size_t)c * D * H,
                                  Sz + (size_t)c * H * H, inv_psi + (size_t)c * D, logdet + c,
                                  log_pi + c);
    if (st != OK) {
      if (failed_component) *failed_component = c;
      return st;
    }
  }
  return OK;
}

}  // extern "C"

namespace orc {
// Caches view over caller-owned arrays (copied: the oracle is not perf critical
// for the small parity sizes; the cpu_baseline times only the E-step body).
inline Caches make_caches(int C, int D, int H, const double* U, const double* Lmat,
                          const double* V, const double* Sz, const double* ipsi,
                          const double* logdet, const double* log_pi) {
  Caches k;
  k.C = C, k.D = D, k.H = H;
  k.U.assign(U, U + (size_t)C * D * H);
  k.V.assign(V, V + (size_t)C * D * H);
  k.Lmat.assign(Lmat, Lmat + (size_t)C * H * H);
  k.Sz.assign(Sz, Sz + (size_t)C * H * H);
  k.inv_psi.assign(ipsi, ipsi + (size_t)C * D);
  k.logdet.assign(logdet, logdet + C);
  k.log_pi.assign(log_pi, log_pi + C);
  return k;
}
}  // namespace orc

extern "C" {

double orc_log_joint(int D, int H, const double* U_c, const double* V_c, const double* ipsi_c,
                     double logdet_c, double log_pi_c, const double* mu_c, const float* x) {
  Caches k;
  k.C = 1, k.D = D, k.H = H;
  k.U.assign(U_c, U_c + (size_t)D * H);
  k.V.assign(V_c, V_c + (size_t)D * H);
  k.inv_psi.assign(ipsi_c, ipsi_c + D);
  k.logdet.assign(1, logdet_c);
  k.log_pi.assign(1, log_pi_c);
  std::vector<double> v(D), a(H), b(H);
  return joint(k, 0, mu_c, x, v.data(), a.data(), b.data());
}

// ---- variational_e_step, estep.cpp:230-336 ---------------------------------------
// K (in/out, N x Cp), g (in/out, C x G, -1 padded) + g_count (in/out),
// n_offset: global index of row 0 (a shard of a larger dataset keys its
// extra draws by the global row, estep.cpp:259-260),
// labels (out, N). Retained arrays use stride = min(Cp*G+1, C) (:238-239).
// dist_out (optional, may be null): per-component accumulator dump as
// (c, ct, sum, count) rows, capacity dist_cap; *dist_n receives the count.
int orc_estep(i64 N, int D, int H, int C, int Cp, int G, const float* X, const double* pi,
              const double* mu, const double* U, const double* Lmat, const double* V,
              const double* Sz, const double* ipsi, const double* logdet, const double* log_pi,
              i32* K, i32* g, i32* g_count, i32* labels, u64 seed, u64 iteration, int mode,
              int threads, i32* ret_count, i32* ret_idx, double* ret_lj, double* resp,
              double* F_out, u64* joints_out, i64 dist_cap, i32* dist_c, i32* dist_ct,
              double* dist_sum, i64* dist_cnt, i64* dist_n, u64 n_offset) {
  if (N < 1 || C < 1 || Cp < 1 || Cp > C || G < 1 || G > C) return INVALID_ARGUMENT;
  const Caches k = make_caches(C, D, H, U, Lmat, V, Sz, ipsi, logdet, log_pi);
  const int stride = static_cast<int>(std::min<i64>((i64)Cp * G + 1, C));  // :238-239
  const int workers = threads > 1 ? threads : 1;
  for (i64 i = 0; i < N; ++i) ret_count[i] = 0;
  for (i64 i = 0; i < N * stride; ++i) {
    ret_idx[i] = -1;
    ret_lj[i] = 0.0;
  }
  std::vector<u64> tally(workers, 0);
  std::atomic<int> err{OK};

  // Block 1 (:249-276): S(n), joints, top-C' K update.
  for_chunks(N, threads, [&](int w, i64 b, i64 e) {
    std::vector<u64> stamp(C, 0);
    u64 epoch = 0;
    std::vector<i32> space;
    std::vector<int> order;
    std::vector<double> v(D), a(H), bb(H);
    for (i64 n = b; n < e; ++n) {
      const i32 extra = draw_component(seed, iteration, n_offset + (u64)n, C);  // :259-260 (global n)
      // build_search_space_into, estep.cpp:83-101 (epoch-stamped dedup)
      ++epoch;
      space.clear();
      auto push = [&](i32 c) {
        if (stamp[c] != epoch) {
          stamp[c] = epoch;
          space.push_back(c);
        }
      };
      for (int j = 0; j < Cp; ++j) {
        const i32 c = K[n * Cp + j];
        for (int i = 0; i < g_count[c]; ++i) push(g[(i64)c * G + i]);
      }
      push(extra);
      const int m = static_cast<int>(space.size());
      ret_count[n] = m;
      i32* ids = ret_idx + n * stride;
      double* ljs = ret_lj + n * stride;
      for (int j = 0; j < m; ++j) {
        const i32 c = space[j];
        ids[j] = c;
        ljs[j] = joint(k, c, mu + (size_t)c * D, X + n * D, v.data(), a.data(), bb.data());
      }
      tally[w] += (u64)m;
      // update_k_into, estep.cpp:103-122: top-C' by (lj desc, idx asc), sorted asc.
      if (m < Cp) {
        err = INSUFFICIENT_CANDIDATES;
        return;
      }
      order.resize(m);
      std::iota(order.begin(), order.end(), 0);
      std::nth_element(order.begin(), order.begin() + (Cp - 1), order.end(), [&](int x, int y) {
        if (ljs[x] != ljs[y]) return ljs[x] > ljs[y];
        return ids[x] < ids[y];
      });
      for (int j = 0; j < Cp; ++j) K[n * Cp + j] = ids[order[j]];
      std::sort(K + n * Cp, K + n * Cp + Cp);
    }
  });
  if (err != OK) return err;
  u64 joints = 0;
  for (int w = 0; w < workers; ++w) joints += tally[w];

  auto lookup = [&](i64 n, i32 c, double* out) -> bool {  // estep.cpp:70-77
    const i32* ids = ret_idx + n * stride;
    for (int j = 0; j < ret_count[n]; ++j)
      if (ids[j] == c) {
        *out = ret_lj[n * stride + j];
        return true;
      }
    return false;
  };

  // Block 2 (:282-284): hard_partition, estep.cpp:144-173 (single-threaded).
  std::vector<std::vector<i32>> part(C);
  for (i64 n = 0; n < N; ++n) {
    i32 best = -1;
    double best_lj = kNegInf;
    for (int j = 0; j < Cp; ++j) {
      const i32 c = K[n * Cp + j];
      double lj = kNegInf;
      if (!lookup(n, c, &lj)) continue;
      if (best < 0 || lj > best_lj) {
        best = c;
        best_lj = lj;
      }
    }
    labels[n] = best;
    part[best].push_back(static_cast<i32>(n));
  }

  // Block 3 (:286-312): accumulate (kl | euclid) over retained joints, update_g.
  std::vector<std::vector<std::pair<i32, std::pair<double, i64>>>> dumps(C);
  for_chunks(C, threads, [&](int, i64 b, i64 e) {
    std::vector<double> sum(C, 0.0);
    std::vector<i64> cnt(C, 0);
    std::vector<i32> touched;
    for (i64 c = b; c < e; ++c) {
      touched.clear();
      const double log_pi_c = pi[c] > 0.0 ? std::log(pi[c]) : kNegInf;
      for (i32 n : part[c]) {
        double lc = kNegInf;
        lookup(n, (i32)c, &lc);
        const double cond_c = lc - log_pi_c;
        const i32* ids = ret_idx + (i64)n * stride;
        const double* ljs = ret_lj + (i64)n * stride;
        for (int j = 0; j < ret_count[n]; ++j) {
          const i32 ct = ids[j];
          if (ct == c || pi[ct] <= 0.0) continue;  // :301
          const double value = mode == 0 ? cond_c - (ljs[j] - std::log(pi[ct])) : -ljs[j];
          if (cnt[ct] == 0) touched.push_back(ct);
          sum[ct] += value;
          cnt[ct] += 1;
        }
      }
      // update_g, estep.cpp:204-220
      std::vector<std::pair<double, i32>> ranked;
      ranked.reserve(touched.size());
      for (i32 ct : touched) ranked.emplace_back(sum[ct] / static_cast<double>(cnt[ct]), ct);
      std::sort(ranked.begin(), ranked.end());
      std::vector<i32> out;
      out.push_back(static_cast<i32>(c));
      const int take = std::min<int>(G - 1, static_cast<int>(ranked.size()));
      for (int j = 0; j < take; ++j) out.push_back(ranked[j].second);
      std::sort(out.begin(), out.end());
      for (int i = 0; i < G; ++i) g[c * G + i] = i < (int)out.size() ? out[i] : -1;
      g_count[c] = static_cast<i32>(out.size());
      if (dist_c) {
        std::sort(touched.begin(), touched.end());
        for (i32 ct : touched) dumps[c].push_back({ct, {sum[ct], cnt[ct]}});
      }
      for (i32 ct : touched) {
        sum[ct] = 0.0;
        cnt[ct] = 0;
      }
    }
  });
  if (dist_c) {
    i64 w = 0;
    for (int c = 0; c < C; ++c)
      for (auto& e : dumps[c]) {
        if (w < dist_cap) {
          dist_c[w] = c;
          dist_ct[w] = e.first;
          dist_sum[w] = e.second.first;
          dist_cnt[w] = e.second.second;
        }
        ++w;
      }
    *dist_n = w;
  }

  // Block 4 (:314-335): responsibilities and F from retained joints.
  std::vector<double> partial(workers, 0.0);
  for_chunks(N, threads, [&](int w, i64 b, i64 e) {
    std::vector<double> kl(Cp);
    double f = 0.0;
    for (i64 n = b; n < e; ++n) {
      for (int j = 0; j < Cp; ++j) lookup(n, K[n * Cp + j], &kl[j]);
      const double l = lse(kl.data(), Cp);
      f += l;
      for (int j = 0; j < Cp; ++j) resp[n * Cp + j] = std::exp(kl[j] - l);
    }
    partial[w] = f;
  });
  double F = 0.0;
  for (int w = 0; w < workers; ++w) F += partial[w];
  *F_out = F;
  *joints_out = joints;
  return OK;
}

// ---- accumulate_suffstats, mstep.cpp:47-101 ---------------------------------------
int orc_suffstats(i64 N, int D, int H, int C, int Cp, const float* X, const double* mu,
                  const double* V, const double* Sz, const i32* K, const double* resp,
                  int threads, double* Nc, double* Y, double* E, double* sq) {
  const int H1 = H + 1;
  const int workers = threads > 1 ? threads : 1;
  struct Part {
    std::vector<double> Nc, Y, E, sq;
  };
  std::vector<Part> parts(workers);
  for (auto& p : parts) {
    p.Nc.assign(C, 0.0);
    p.Y.assign((size_t)C * D * H1, 0.0);
    p.E.assign((size_t)C * H1 * H1, 0.0);
    p.sq.assign((size_t)C * D, 0.0);
  }
  for_chunks(N, threads, [&](int w, i64 b, i64 e) {
    Part& P = parts[w];
    std::vector<double> xd(D), v(D), mz(H);
    for (i64 n = b; n < e; ++n) {
      for (int d = 0; d < D; ++d) xd[d] = static_cast<double>(X[n * D + d]);
      for (int j = 0; j < Cp; ++j) {
        const i32 c = K[n * Cp + j];
        const double q = resp[n * Cp + j];
        const double* m = mu + (size_t)c * D;
        const double* Vc = V + (size_t)c * D * H;
        for (int d = 0; d < D; ++d) v[d] = xd[d] - m[d];  // :52
        for (int h = 0; h < H; ++h) mz[h] = 0.0;
        for (int d = 0; d < D; ++d)
          for (int h = 0; h < H; ++h) mz[h] += Vc[d * H + h] * v[d];  // :53
        P.Nc[c] += q;
        double* Ec = P.E.data() + (size_t)c * H1 * H1;
        const double* S = Sz + (size_t)c * H * H;
        for (int j2 = 0; j2 < H; ++j2)
          for (int i2 = 0; i2 < H; ++i2) Ec[j2 * H1 + i2] += q * S[j2 * H + i2];  // :56
        for (int j2 = 0; j2 < H; ++j2)
          for (int i2 = 0; i2 < H; ++i2) Ec[j2 * H1 + i2] += (q * mz[i2]) * mz[j2];  // :57
        for (int h = 0; h < H; ++h) {
          Ec[H * H1 + h] += q * mz[h];  // col H
          Ec[h * H1 + H] += q * mz[h];  // row H
        }
        Ec[H * H1 + H] += q;
        double* Yc = P.Y.data() + (size_t)c * D * H1;
        for (int h = 0; h < H; ++h)
          for (int d = 0; d < D; ++d) Yc[h * D + d] += (q * xd[d]) * mz[h];  // :62
        for (int d = 0; d < D; ++d) Yc[H * D + d] += q * xd[d];
        double* sc = P.sq.data() + (size_t)c * D;
        for (int d = 0; d < D; ++d) sc[d] += q * (xd[d] * xd[d]);
      }
    }
  });
  // merge in worker order (mstep.cpp:98-99)
  std::copy(parts[0].Nc.begin(), parts[0].Nc.end(), Nc);
  std::copy(parts[0].Y.begin(), parts[0].Y.end(), Y);
  std::copy(parts[0].E.begin(), parts[0].E.end(), E);
  std::copy(parts[0].sq.begin(), parts[0].sq.end(), sq);
  for (int w = 1; w < workers; ++w) {
    for (int c = 0; c < C; ++c) Nc[c] += parts[w].Nc[c];
    for (size_t i = 0; i < parts[w].Y.size(); ++i) Y[i] += parts[w].Y[i];
    for (size_t i = 0; i < parts[w].E.size(); ++i) E[i] += parts[w].E[i];
    for (size_t i = 0; i < parts[w].sq.size(); ++i) sq[i] += parts[w].sq[i];
  }
  return OK;
}

// ---- update_params, mstep.cpp:103-162 -----------------------------------------------
// E_c A^T = Y_c^T by the LDLT restatement above (mstep.cpp:129-130); the
// jitter rule (1e-10 tr/(H+1) once on info != Success or a non-finite
// solution, else SingularEc, :131-140) is reproduced.
int orc_update_params(int C, int D, int H, i64 N, const double* Nc, const double* Y,
                      const double* E, const double* sq, const double* floor,
                      const double* pi_prev, const double* mu_prev, const double* lam_prev,
                      const double* psi_prev, double* pi, double* mu, double* lam, double* psi,
                      int* failed_component) {
  if (N <= 0) return INVALID_ARGUMENT;
  (void)pi_prev;
  const int H1 = H + 1;
  std::vector<double> Ec(H1 * H1), R(H1 * H1), At((size_t)H1 * D), b(H1);
  std::vector<int> perm(H1);
  for (int c = 0; c < C; ++c) {
    const double nc = Nc[c];
    if (nc == 0.0) {  // :119-126 freeze
      pi[c] = 0.0;
      std::copy(mu_prev + (size_t)c * D, mu_prev + (size_t)(c + 1) * D, mu + (size_t)c * D);
      std::copy(lam_prev + (size_t)c * D * H, lam_prev + (size_t)(c + 1) * D * H, lam + (size_t)c * D * H);
      std::copy(psi_prev + (size_t)c * D, psi_prev + (size_t)(c + 1) * D, psi + (size_t)c * D);
      continue;
    }
    pi[c] = nc / static_cast<double>(N);
    std::copy(E + (size_t)c * H1 * H1, E + (size_t)(c + 1) * H1 * H1, Ec.begin());
    const double* Yc = Y + (size_t)c * D * H1;
    auto solve_all = [&]() -> bool {
      R = Ec;
      if (!ldlt(R.data(), perm.data(), H1)) return false;
      for (int d = 0; d < D; ++d) {
        for (int h = 0; h < H1; ++h) b[h] = Yc[h * D + d];
        ldlt_solve(R.data(), perm.data(), b.data(), H1);
        for (int h = 0; h < H1; ++h) {
          if (!std::isfinite(b[h])) return false;
          At[(size_t)d * H1 + h] = b[h];  // At (H+1) x D stored per d
        }
      }
      return true;
    };
    if (!solve_all()) {  // :133-140
      double tr = 0.0;
      for (int i = 0; i < H1; ++i) tr += Ec[i * H1 + i];
      const double jit = 1e-10 * tr / H1;
      for (int i = 0; i < H1; ++i) Ec[i * H1 + i] += jit;
      if (!solve_all()) {
        if (failed_component) *failed_component = c;
        return SINGULAR_EC;
      }
    }
    for (int h = 0; h < H; ++h)
      for (int d = 0; d < D; ++d) lam[(size_t)c * D * H + h * D + d] = At[(size_t)d * H1 + h];  // :141
    for (int d = 0; d < D; ++d) mu[(size_t)c * D + d] = At[(size_t)d * H1 + H];  // :142
    for (int d = 0; d < D; ++d) {  // :147-153
      double fitted = 0.0;
      for (int h = 0; h < H1; ++h) fitted += Yc[h * D + d] * At[(size_t)d * H1 + h];
      psi[(size_t)c * D + d] = std::max((sq[(size_t)c * D + d] - fitted) / nc, floor[d]);
    }
  }
  double live = 0.0;
  for (int c = 0; c < C; ++c) live += pi[c];
  if (live <= 0.0) return SINGULAR_EC;  // :156-159
  for (int c = 0; c < C; ++c) pi[c] /= live;
  return OK;
}

// ---- truncated_free_energy / exact_log_likelihood, model.cpp:101-159 ------------------
int orc_truncated_F(i64 N, int D, int H, int C, int Cp, const float* X, const double* mu,
                    const double* U, const double* Lmat, const double* V, const double* Sz,
                    const double* ipsi, const double* logdet, const double* log_pi, const i32* K,
                    int threads, double* F_out, double* lj_out) {
  if (Cp < 1 || N < 1) return EMPTY_KSET;
  const Caches k = make_caches(C, D, H, U, Lmat, V, Sz, ipsi, logdet, log_pi);
  const int workers = threads > 1 ? threads : 1;
  std::vector<double> partial(workers, 0.0);
  for_chunks(N, threads, [&](int w, i64 b, i64 e) {
    std::vector<double> v(D), a(H), bb(H), lj(Cp);
    double s = 0.0;
    for (i64 n = b; n < e; ++n) {
      for (int j = 0; j < Cp; ++j) {
        const i32 c = K[n * Cp + j];
        lj[j] = joint(k, c, mu + (size_t)c * D, X + n * D, v.data(), a.data(), bb.data());
        if (lj_out) lj_out[n * Cp + j] = lj[j];
      }
      s += lse(lj.data(), Cp);
    }
    partial[w] = s;
  });
  double F = 0.0;
  for (int w = 0; w < workers; ++w) F += partial[w];
  *F_out = F;
  return OK;
}

int orc_exact_ll(i64 N, int D, int H, int C, const float* X, const double* mu, const double* U,
                 const double* Lmat, const double* V, const double* Sz, const double* ipsi,
                 const double* logdet, const double* log_pi, int threads, double* LL_out) {
  std::vector<i32> all((size_t)N * C);
  for (i64 n = 0; n < N; ++n)
    for (int c = 0; c < C; ++c) all[(size_t)n * C + c] = c;
  return orc_truncated_F(N, D, H, C, C, X, mu, U, Lmat, V, Sz, ipsi, logdet, log_pi, all.data(),
                         threads, LL_out, nullptr);
}

// ---- initialisation, seeding.cpp:123-233, trainer.cpp:32-47,107 ----------------------
// random_points_seed (seeding.cpp:123-149). count_distinct_rows (:16-32) is
// replaced by an exact hash-set count (same answer: number of distinct rows,
// capped at `needed`).
int orc_random_points_seed(const float* X, i64 N, int D, int C, u64 stream_seed, i64* seeds,
                           u64* stream_state_out) {
  if (C < 1 || C > N) return INVALID_ARGUMENT;
  struct RowHash {
    const float* X;
    int D;
    size_t operator()(i64 i) const {
      u64 h = 1469598103934665603ULL;
      const unsigned char* p = reinterpret_cast<const unsigned char*>(X + i * D);
      for (size_t b = 0; b < (size_t)D * sizeof(float); ++b) h = (h ^ p[b]) * 1099511628211ULL;
      return static_cast<size_t>(h);
    }
  };
  struct RowEq {
    const float* X;
    int D;
    bool operator()(i64 a, i64 b) const {
      for (int d = 0; d < D; ++d)
        if (!(X[a * D + d] == X[b * D + d])) return false;
      return true;
    }
  };
  {
    std::unordered_set<i64, RowHash, RowEq> distinct(16, RowHash{X, D}, RowEq{X, D});
    for (i64 i = 0; i < N && (i64)distinct.size() < C; ++i) distinct.insert(i);
    if ((i64)distinct.size() < C) return DEGENERATE_DATA;
  }
  Stream s(stream_seed);
  std::vector<std::uint8_t> used(N, 0);
  std::unordered_set<i64, RowHash, RowEq> chosen(16, RowHash{X, D}, RowEq{X, D});
  int got = 0;
  while (got < C) {  // :135-147 rejection of used rows and duplicates of chosen rows
    const i64 i = s.below(N);
    if (used[i]) continue;
    const bool dup = chosen.count(i) > 0;
    used[i] = 1;
    if (!dup) {
      chosen.insert(i);
      seeds[got++] = i;
    }
  }
  if (stream_state_out) std::memcpy(stream_state_out, s.w, sizeof(s.w));
  return OK;
}

// afkmc2_seed (seeding.cpp:60-121): AFK-MC^2 seeding, the reference's default
// InitConfig::Method (seeding.hpp:14-17). squared_distance (:34-39) in fp64
// in the device's warp order (below; Eigen's squaredNorm order is unpinned),
// distance_to_centers (:41-49), draw_from_cdf (:51-56); the proposal q and its
// cdf are built sequentially (:75-86). *dist_count receives the number of
// squared_distance calls (EvalCounter::distances).
int orc_afkmc2(const float* X, i64 N, int D, int C, int chain_length, u64 stream_seed, i64* seeds,
               u64* stream_state_out, u64* dist_count) {
  if (C < 1 || C > N || chain_length < 1) return INVALID_ARGUMENT;
  {  // count_distinct_rows (:16-32): at least C distinct rows
    std::unordered_set<std::string> distinct;
    for (i64 i = 0; i < N && (i64)distinct.size() < C; ++i)
      distinct.insert(std::string(reinterpret_cast<const char*>(X + i * D), (size_t)D * sizeof(float)));
    if ((i64)distinct.size() < C) return DEGENERATE_DATA;
  }
  u64 count = 0;
  // squared_distance's summation order (Eigen's is unpinned): 32 partials over
  // d = l, l + 32, ... (explicit fma, ascending), then the halving tree
  // v[l] += v[l + o] for o = 16, 8, 4, 2, 1 -- the device's warp order
  auto sqd = [&](i64 a, i64 b) {
    ++count;
    double v[32];
    for (int l = 0; l < 32; ++l) {
      double t = 0.0;
      for (int d = l; d < D; d += 32) {
        const double u = static_cast<double>(X[a * D + d]) - static_cast<double>(X[b * D + d]);
        t = std::fma(u, u, t);
      }
      v[l] = t;
    }
    for (int o = 16; o > 0; o >>= 1)
      for (int l = 0; l < o; ++l) v[l] = v[l] + v[l + o];
    return v[0];
  };
  std::vector<i64> centers;
  auto to_centers = [&](i64 n) {
    double best = std::numeric_limits<double>::infinity();
    for (i64 c : centers) best = std::min(best, sqd(n, c));
    return best;
  };
  Stream s(stream_seed);
  centers.push_back(s.below(N));
  std::vector<double> q(N), cdf(N);
  double sum_d2 = 0.0;
  for (i64 i = 0; i < N; ++i) {
    q[i] = sqd(i, centers[0]);
    sum_d2 += q[i];
  }
  const double uniform_part = 0.5 / static_cast<double>(N);
  for (i64 i = 0; i < N; ++i) q[i] = (sum_d2 > 0.0 ? 0.5 * q[i] / sum_d2 : 0.0) + uniform_part;
  double acc = 0.0;
  for (i64 i = 0; i < N; ++i) cdf[i] = acc += q[i];
  auto draw = [&]() {
    const double u = s.unit() * cdf.back();
    const i64 it = std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin();
    return std::min<i64>(it, N - 1);
  };
  while (static_cast<int>(centers.size()) < C) {
    i64 x = draw();
    double dx = to_centers(x);
    for (int step = 1; step < chain_length; ++step) {
      const i64 y = draw();
      const double dy = to_centers(y);
      if (dy <= 0.0) continue;
      bool accept = dx <= 0.0;
      if (!accept) accept = s.unit() < (dy * q[x]) / (dx * q[y]);
      if (accept) {
        x = y;
        dx = dy;
      }
    }
    if (dx <= 0.0) {  // :105-117 farthest point from its nearest center
      double best = -1.0;
      i64 best_i = -1;
      for (i64 i = 0; i < N; ++i) {
        const double d = to_centers(i);
        if (d > best) {
          best = d;
          best_i = i;
        }
      }
      x = best_i;
    }
    centers.push_back(x);
  }
  for (int c = 0; c < C; ++c) seeds[c] = centers[c];
  if (stream_state_out) std::memcpy(stream_state_out, s.w, sizeof(s.w));
  if (dist_count) *dist_count = count;
  return OK;
}

// init_params (seeding.cpp:151-181), continuing the same stream (trainer.cpp:36-44).
// loading_init 0: reference Lambda ~ U[0, scale); 1: BASELINE's N(0, scale^2)
// (Box-Muller from the same stream, same c->d->h order).
int orc_init_params(const float* X, i64 N, int D, int C, int H, const i64* seeds,
                    const u64* stream_state, double scale, int loading_init, const double* floor,
                    double* pi, double* mu, double* lam, double* psi) {
  std::vector<double> var(D);
  orc_per_dimension_variance(X, N, D, var.data());
  Stream s(0);
  std::memcpy(s.w, stream_state, sizeof(s.w));
  for (int c = 0; c < C; ++c) {
    pi[c] = 1.0 / C;
    for (int d = 0; d < D; ++d) {
      mu[(size_t)c * D + d] = static_cast<double>(X[seeds[c] * D + d]);
      psi[(size_t)c * D + d] = std::max(var[d], floor[d]);
    }
    for (int d = 0; d < D; ++d)
      for (int h = 0; h < H; ++h)
        lam[(size_t)c * D * H + h * D + d] = loading_init == 0 ? s.unit() * scale : s.normal() * scale;
  }
  return OK;
}

// init_varstate (seeding.cpp:207-233) with fill_distinct (:187-203) restated
// literally: a C-sized buffer holding 0..C-1 per row, the preset swap, the
// partial Fisher-Yates draws, then the first `want` entries sorted. O(N*C),
// as the reference (the product restates it over a sparse swap map in
// O(N*C'); tests/test_abi_host.py pins the two against each other and both
// against a numpy restatement over the golden stream).
int orc_init_varstate(i64 N, int C, int Cp, int G, const i64* seed_rows, int n_seeds,
                      u64 stream_seed, i32* K, i32* g, i32* g_count) {
  if (Cp < 1 || Cp > C || G < 1 || G > C) return INVALID_ARGUMENT;
  Stream s(stream_seed);
  std::vector<i32> seed_component(N, -1);  // seeding.cpp:220-223
  for (int c = 0; c < n_seeds; ++c) seed_component[seed_rows[c]] = c;
  std::vector<i32> buffer;
  auto fill = [&](int want, i32 preset, i32* out) {  // seeding.cpp:187-203
    buffer.resize(C);
    for (int i = 0; i < C; ++i) buffer[i] = i;
    int start = 0;
    if (preset >= 0) {
      std::swap(buffer[0], buffer[preset]);
      start = 1;
    }
    for (int i = start; i < want; ++i) {
      const int j = i + static_cast<int>(s.below(C - i));
      std::swap(buffer[i], buffer[j]);
    }
    std::copy(buffer.begin(), buffer.begin() + want, out);
    std::sort(out, out + want);
  };
  for (i64 n = 0; n < N; ++n) fill(Cp, seed_component[n], K + n * Cp);
  for (int c = 0; c < C; ++c) {
    fill(G, c, g + (i64)c * G);
    g_count[c] = G;
  }
  return OK;
}

}  // extern "C"
