// vmfa_host.cpp — host-only part of libvmfa_b200.so: the reference's one-time
// initialisation (trainer.cpp:32-47, 107-109; seeding.cpp:123-233;
// dataset.cpp:22-39) restated with identical draw sequences, in O(N*C')
// instead of the reference's O(N*C) buffer fill, whole-dataset or per shard.
//
// Sharded form: no rank holds all N rows.
//   floor     per_dimension_variance as two moment all-reduces over the shards
//             (vmfa_host_moments: sum x, then sum (x - global mean)^2);
//   seeds     random_points_seed's draw sequence (vmfa_seed_draws) is data-
//             independent; only the accept/reject decisions need row contents,
//             which the caller fetches for the drawn rows from their owners;
//             count_distinct_rows' DegenerateData check is a union of per-shard
//             distinct-row hashes (vmfa_host_distinct_hashes);
//   params    init_params continues the same stream after the seed draws;
//   K, g      init_varstate's stream is replayed in full (N*C' + C*G draws,
//             one next() each) while only the shard's K rows are stored.
// vmfa_host_initialize composes the same pieces over the whole dataset.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../vmfa_internal.hpp"
#include "../vmfa_rng.hpp"

namespace vmfa_b200 {
namespace {

constexpr uint64_t kSaltInit = 0x1217f01dULL;   // trainer.cpp:36
constexpr uint64_t kSaltState = 0x7a57a7e5ULL;  // trainer.cpp:107

template <class F>
void parallel_ranges(int64_t n, int threads, F&& fn) {
  if (threads < 1) threads = 1;
  if (threads > n) threads = static_cast<int>(std::max<int64_t>(n, 1));
  if (threads <= 1) {
    fn(0, int64_t{0}, n);
    return;
  }
  std::vector<std::thread> pool;
  const int64_t base = n / threads, rem = n % threads;
  int64_t b = 0;
  for (int w = 0; w < threads; ++w) {
    const int64_t len = base + (w < rem ? 1 : 0);
    pool.emplace_back([&fn, w, b, len] { fn(w, b, b + len); });
    b += len;
  }
  for (auto& t : pool) t.join();
}

int hw_threads() { return static_cast<int>(std::max(1u, std::thread::hardware_concurrency())); }

// per-dimension fp64 sums over rows in order (parallel over dimensions keeps
// each dimension's summation order): sum x (mean == nullptr) or sum (x-mean)^2
void moments(const float* X, int64_t rows, int D, const double* mean, double* out, int threads) {
  parallel_ranges(D, threads, [&](int, int64_t b, int64_t e) {
    std::vector<double> acc(e - b, 0.0);
    for (int64_t i = 0; i < rows; ++i) {
      const float* x = X + i * D;
      if (mean) {
        for (int64_t d = b; d < e; ++d) {
          const double t = static_cast<double>(x[d]) - mean[d];
          acc[d - b] += t * t;
        }
      } else {
        for (int64_t d = b; d < e; ++d) acc[d - b] += static_cast<double>(x[d]);
      }
    }
    for (int64_t d = b; d < e; ++d) out[d] = acc[d - b];
  });
}

// row bits with -0.0 read as +0.0: rows equal under the reference's float
// comparison (seeding.cpp:26, :140) have equal digests
inline uint32_t row_word(const float* x) {
  const float v = *x + 0.0f;
  uint32_t w;
  std::memcpy(&w, &v, sizeof w);
  return w;
}
inline uint64_t fnv_row(const float* x, int D) {
  uint64_t h = 1469598103934665603ULL;
  for (int d = 0; d < D; ++d) {
    const uint32_t w = row_word(x + d);
    for (int b = 0; b < 4; ++b) h = (h ^ ((w >> (8 * b)) & 0xffu)) * 1099511628211ULL;
  }
  return h;
}
struct RowHash {
  const float* X;
  int D;
  size_t operator()(int64_t i) const { return static_cast<size_t>(fnv_row(X + i * D, D)); }
};
struct RowEq {
  const float* X;
  int D;
  bool operator()(int64_t a, int64_t b) const {
    for (int d = 0; d < D; ++d)
      if (!(X[a * D + d] == X[b * D + d])) return false;
    return true;
  }
};

// fill_distinct (seeding.cpp:187-203) over a sparse swap map (unlisted
// positions hold their own index): identical output for identical draws.
struct FillDistinct {
  int C;
  std::unordered_map<int, int> over;
  int at(int p) const {
    auto it = over.find(p);
    return it == over.end() ? p : it->second;
  }
  // out == nullptr: consume the row's draws only (uniform_int is one next())
  void operator()(HostStream& rng, int want, int preset, int32_t* out) {
    const int start = preset >= 0 ? 1 : 0;
    if (!out) {
      for (int i = start; i < want; ++i) rng.next();
      return;
    }
    over.clear();
    if (preset >= 0) {
      const int a = at(0), b = at(preset);
      over[0] = b;
      over[preset] = a;
    }
    for (int i = start; i < want; ++i) {
      const int j = i + static_cast<int>(rng.uniform_int(C - i));
      const int a = at(i), b = at(j);
      over[i] = b;
      over[j] = a;
    }
    for (int i = 0; i < want; ++i) out[i] = at(i);
    std::sort(out, out + want);
  }
};

// init_params (seeding.cpp:151-181) from the stream positioned after the seed
// draws, then init_varstate (seeding.cpp:207-233) storing rows [n0, n0 + rows)
// of an N-row dataset. seed_rows_data: the C seed rows (C x D).
void init_from_seeds(HostStream& rng, int64_t N, int D, int C, int H, int Cp, int G, uint64_t seed,
                     double scale, int loading_init, const double* var, const double* floor,
                     const int64_t* seeds, const float* seed_rows_data, int64_t n0, int64_t rows, double* pi,
                     double* mu, double* lambda, double* dnoise, int32_t* K, int32_t* g, int32_t* g_count) {
  for (int c = 0; c < C; ++c) {
    pi[c] = 1.0 / C;
    for (int d = 0; d < D; ++d) {
      mu[static_cast<size_t>(c) * D + d] = static_cast<double>(seed_rows_data[static_cast<size_t>(c) * D + d]);
      dnoise[static_cast<size_t>(c) * D + d] = std::max(var[d], floor[d]);
    }
    for (int d = 0; d < D; ++d)
      for (int h = 0; h < H; ++h)
        lambda[static_cast<size_t>(c) * D * H + static_cast<size_t>(h) * D + d] =
            loading_init == 0 ? rng.uniform() * scale : rng.gaussian() * scale;
  }
  HostStream srng(key2(seed, kSaltState));
  std::unordered_map<int64_t, int32_t> seed_of;
  for (int c = 0; c < C; ++c) seed_of[seeds[c]] = c;
  FillDistinct fill{C, {}};
  for (int64_t n = 0; n < N; ++n) {
    auto it = seed_of.find(n);
    const bool mine = n >= n0 && n < n0 + rows;
    fill(srng, Cp, it == seed_of.end() ? -1 : it->second, mine ? K + (n - n0) * Cp : nullptr);
  }
  for (int c = 0; c < C; ++c) {
    fill(srng, G, c, g + static_cast<int64_t>(c) * G);
    g_count[c] = G;
  }
}

bool valid_sizes(int64_t N, int D, int C, int H, int Cp, int G) {
  return N >= 1 && D >= 1 && C >= 1 && C <= N && H >= 1 && H <= D && Cp >= 1 && Cp <= C && G >= 1 && G <= C;
}

}  // namespace
}  // namespace vmfa_b200

using namespace vmfa_b200;

// trainer.cpp:32-47 (initialize with InitConfig::Method::random_points) and
// trainer.cpp:107-109 (init_varstate) over the whole dataset.
extern "C" int vmfa_host_initialize(const float* X, int64_t N, int D, int C, int H, int Cp, int G,
                                    uint64_t seed, double scale, int loading_init, double* floor,
                                    double* pi, double* mu, double* lambda, double* dnoise,
                                    int32_t* K, int32_t* g, int32_t* g_count, int64_t* seeds) {
  if (!X || !valid_sizes(N, D, C, H, Cp, G))
    return fail(VMFA_ERR_INVALID_ARGUMENT, "vmfa_host_initialize: invalid sizes");
  const int threads = hw_threads();
  // per_dimension_variance (dataset.cpp:22-35): two fp64 passes
  std::vector<double> mean(D), var(D);
  moments(X, N, D, nullptr, mean.data(), threads);
  for (int d = 0; d < D; ++d) mean[d] /= static_cast<double>(N);
  moments(X, N, D, mean.data(), var.data(), threads);
  for (int d = 0; d < D; ++d) var[d] /= static_cast<double>(N);
  for (int d = 0; d < D; ++d) floor[d] = std::max(1e-6 * var[d], 1e-8);  // dataset.cpp:37-39

  // random_points_seed (seeding.cpp:123-149). count_distinct_rows (:16-32) is
  // an exact distinct-row count; a hash set gives the same answer.
  {
    std::unordered_set<int64_t, RowHash, RowEq> distinct(16, RowHash{X, D}, RowEq{X, D});
    for (int64_t i = 0; i < N && static_cast<int64_t>(distinct.size()) < C; ++i) distinct.insert(i);
    if (static_cast<int64_t>(distinct.size()) < C)
      return fail(VMFA_ERR_DEGENERATE_DATA, "fewer distinct rows than requested seeds");
  }
  HostStream rng(key2(seed, kSaltInit));  // trainer.cpp:36
  {
    std::vector<uint8_t> used(N, 0);
    std::unordered_set<int64_t, RowHash, RowEq> chosen(16, RowHash{X, D}, RowEq{X, D});
    int got = 0;
    while (got < C) {
      const int64_t i = rng.uniform_int(N);
      if (used[i]) continue;
      const bool dup = chosen.count(i) > 0;
      used[i] = 1;
      if (!dup) {
        chosen.insert(i);
        seeds[got++] = i;
      }
    }
  }
  std::vector<float> srows(static_cast<size_t>(C) * D);
  for (int c = 0; c < C; ++c) std::memcpy(&srows[static_cast<size_t>(c) * D], X + seeds[c] * D, sizeof(float) * D);
  init_from_seeds(rng, N, D, C, H, Cp, G, seed, scale, loading_init, var.data(), floor, seeds, srows.data(), 0, N,
                  pi, mu, lambda, dnoise, K, g, g_count);
  return VMFA_OK;
}

// ---- sharded initialisation pieces (see the file header)

extern "C" int vmfa_host_moments(const float* X, int64_t rows, int D, const double* mean, double* out,
                                 int threads) {
  if ((!X && rows > 0) || rows < 0 || D < 1 || !out)
    return fail(VMFA_ERR_INVALID_ARGUMENT, "vmfa_host_moments: bad arguments");
  moments(X, rows, D, mean, out, threads > 0 ? threads : hw_threads());
  return VMFA_OK;
}

extern "C" int vmfa_seed_draws(uint64_t seed, int64_t N, int64_t first, int64_t count, int64_t* out) {
  if (N < 1 || first < 0 || count < 0 || (!out && count > 0))
    return fail(VMFA_ERR_INVALID_ARGUMENT, "vmfa_seed_draws: bad arguments");
  HostStream rng(key2(seed, kSaltInit));
  for (int64_t k = 0; k < first; ++k) rng.next();
  for (int64_t k = 0; k < count; ++k) out[k] = rng.uniform_int(N);
  return VMFA_OK;
}

extern "C" int vmfa_host_distinct_hashes(const float* X, int64_t rows, int D, int64_t want, uint64_t* out,
                                         int64_t* n_out) {
  if ((!X && rows > 0) || rows < 0 || D < 1 || want < 0 || !n_out || (!out && want > 0))
    return fail(VMFA_ERR_INVALID_ARGUMENT, "vmfa_host_distinct_hashes: bad arguments");
  std::unordered_set<int64_t, RowHash, RowEq> distinct(16, RowHash{X, D}, RowEq{X, D});
  int64_t m = 0;
  for (int64_t i = 0; i < rows && m < want; ++i) {
    if (!distinct.insert(i).second) continue;
    // two independent 64-bit digests of the row (FNV-1a over its bytes, a
    // splitmix chain over its 32-bit words): 128 bits per distinct row
    const uint64_t h1 = fnv_row(X + i * D, D);
    uint64_t h2 = 0x243f6a8885a308d3ULL;
    for (int d = 0; d < D; ++d) h2 = key2(h2, row_word(X + i * D + d));
    out[2 * m] = h1;
    out[2 * m + 1] = h2;
    ++m;
  }
  *n_out = m;
  return VMFA_OK;
}

extern "C" int vmfa_host_init_shard(int64_t N, int D, int C, int H, int Cp, int G, uint64_t seed, double scale,
                                    int loading_init, const double* var, const double* floor,
                                    const int64_t* seeds, const float* seed_rows, int64_t seed_draws,
                                    int64_t n0, int64_t rows, double* pi, double* mu, double* lambda,
                                    double* dnoise, int32_t* K, int32_t* g, int32_t* g_count) {
  if (!valid_sizes(N, D, C, H, Cp, G) || !var || !floor || !seeds || !seed_rows || seed_draws < C || n0 < 0 ||
      rows < 0 || n0 + rows > N || !pi || !mu || !lambda || !dnoise || (!K && rows > 0) || !g || !g_count)
    return fail(VMFA_ERR_INVALID_ARGUMENT, "vmfa_host_init_shard: bad arguments");
  HostStream rng(key2(seed, kSaltInit));
  for (int64_t k = 0; k < seed_draws; ++k) rng.next();  // positioned after random_points_seed
  init_from_seeds(rng, N, D, C, H, Cp, G, seed, scale, loading_init, var, floor, seeds, seed_rows, n0, rows, pi,
                  mu, lambda, dnoise, K, g, g_count);
  return VMFA_OK;
}
