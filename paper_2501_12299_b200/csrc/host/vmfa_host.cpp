// vmfa_host.cpp — host-only part of libvmfa_b200.so:
//   * synthetic data for BASELINE.json's configs (the paper's image datasets
//     are not available; SURVEY §8(d) specifies these generators), and
//   * the reference's one-time initialisation (trainer.cpp:32-47, 107-109;
//     seeding.cpp:123-233; dataset.cpp:22-39) restated with identical draw
//     sequences, in O(N*C') instead of the reference's O(N*C) buffer fill.
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

constexpr uint64_t kSaltPi = 0x5eed91ULL;
constexpr uint64_t kSaltTruth = 0x7e0711ULL;
constexpr uint64_t kSaltRow = 0x5a3e11eULL;

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

// Separable Gaussian blur (clamped borders) of one (h x w) plane, in place.
void blur_plane(double* f, int w, int h, double sigma, std::vector<double>& tmp) {
  if (sigma <= 0.0) return;
  const int r = std::max(1, static_cast<int>(std::ceil(3.0 * sigma)));
  std::vector<double> k(2 * r + 1);
  double s = 0.0;
  for (int i = -r; i <= r; ++i) s += (k[i + r] = std::exp(-0.5 * i * i / (sigma * sigma)));
  for (double& v : k) v /= s;
  tmp.assign(static_cast<size_t>(w) * h, 0.0);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      double acc = 0.0;
      for (int i = -r; i <= r; ++i) acc += k[i + r] * f[y * w + std::clamp(x + i, 0, w - 1)];
      tmp[y * w + x] = acc;
    }
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      double acc = 0.0;
      for (int i = -r; i <= r; ++i) acc += k[i + r] * tmp[std::clamp(y + i, 0, h - 1) * w + x];
      f[y * w + x] = acc;
    }
}

// Smooth random field: blurred iid draws, standardised per field back to the
// (mean, std) of the iid draws (variance-preserving blur).
void smooth_field(HostStream& s, const vmfa_synth_spec& sp, bool uniform01, double std_t,
                  double mean_t, double* out, std::vector<double>& plane, std::vector<double>& tmp) {
  const int W = sp.img_w, Hh = sp.img_h, Ch = sp.img_c;
  const int P = W * Hh;
  for (int ch = 0; ch < Ch; ++ch) {
    plane.resize(P);
    for (int i = 0; i < P; ++i) plane[i] = uniform01 ? s.uniform() : s.gaussian();
    blur_plane(plane.data(), W, Hh, sp.blur_sigma, tmp);
    double m = 0.0, v = 0.0;
    for (int i = 0; i < P; ++i) m += plane[i];
    m /= P;
    for (int i = 0; i < P; ++i) v += (plane[i] - m) * (plane[i] - m);
    const double sd = std::sqrt(v / P);
    const double scale = sd > 0.0 ? std_t / sd : 0.0;
    for (int i = 0; i < P; ++i) out[i * Ch + ch] = mean_t + (plane[i] - m) * scale;  // channel-last
  }
}

}  // namespace
}  // namespace vmfa_b200

using namespace vmfa_b200;

extern "C" int vmfa_gen_synthetic(const vmfa_synth_spec* sp, int64_t row_begin, int64_t row_end,
                                  float* X, int32_t* labels, int threads) {
  if (!sp || !X || row_begin < 0 || row_end < row_begin || row_end > sp->n_total || sp->D < 1 ||
      sp->C_true < 1 || sp->H_true < 0)
    return fail(VMFA_ERR_INVALID_ARGUMENT, "vmfa_gen_synthetic: bad arguments");
  if (sp->kind == 1 && sp->img_w * sp->img_h * sp->img_c != sp->D)
    return fail(VMFA_ERR_INVALID_ARGUMENT, "vmfa_gen_synthetic: img_w*img_h*img_c != D");
  if (threads < 1) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  const int D = sp->D, Ct = sp->C_true, Ht = sp->H_true;

  // mixing weights: equiprobable or Dirichlet(1) = normalised Exp(1) draws
  std::vector<double> cdf(Ct);
  {
    HostStream s(key2(sp->data_seed, kSaltPi));
    double acc = 0.0;
    for (int c = 0; c < Ct; ++c) {
      const double w = sp->dirichlet ? -std::log(1.0 - s.uniform()) : 1.0;
      acc += w;
      cdf[c] = acc;
    }
  }
  // ground truth per component, each from its own keyed stream
  std::vector<float> mu(static_cast<size_t>(Ct) * D), lam(static_cast<size_t>(Ct) * D * Ht),
      sd(static_cast<size_t>(Ct) * D);
  parallel_ranges(Ct, threads, [&](int, int64_t b, int64_t e) {
    std::vector<double> field(D), plane, tmp;
    for (int64_t c = b; c < e; ++c) {
      HostStream s(key3(sp->data_seed, kSaltTruth, static_cast<uint64_t>(c)));
      float* m = mu.data() + c * D;
      float* l = lam.data() + c * D * Ht;  // [d][h]
      float* p = sd.data() + c * D;
      if (sp->kind == 0) {
        for (int d = 0; d < D; ++d) m[d] = static_cast<float>(sp->mu_std * s.gaussian());
        for (int d = 0; d < D; ++d)
          for (int h = 0; h < Ht; ++h) l[d * Ht + h] = static_cast<float>(sp->lam_std * s.gaussian());
        for (int d = 0; d < D; ++d)
          p[d] = static_cast<float>(std::sqrt(sp->psi_lo + (sp->psi_hi - sp->psi_lo) * s.uniform()));
      } else {
        smooth_field(s, *sp, true, 1.0 / std::sqrt(12.0), 0.5, field.data(), plane, tmp);
        for (int d = 0; d < D; ++d) m[d] = static_cast<float>(field[d]);
        for (int h = 0; h < Ht; ++h) {
          smooth_field(s, *sp, false, sp->lam_std, 0.0, field.data(), plane, tmp);
          for (int d = 0; d < D; ++d) l[d * Ht + h] = static_cast<float>(field[d]);
        }
        for (int d = 0; d < D; ++d) p[d] = static_cast<float>(sp->noise_std);
      }
    }
  });
  // rows: component by inverse CDF, z ~ N(0, I), eps ~ N(0, Psi)
  parallel_ranges(row_end - row_begin, threads, [&](int, int64_t b, int64_t e) {
    std::vector<double> z(std::max(Ht, 1));
    for (int64_t i = b; i < e; ++i) {
      const int64_t n = row_begin + i;
      HostStream s(key3(sp->data_seed, kSaltRow, static_cast<uint64_t>(n)));
      const double u = s.uniform() * cdf.back();
      int c = static_cast<int>(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
      c = std::min(c, Ct - 1);
      for (int h = 0; h < Ht; ++h) z[h] = s.gaussian();
      const float* m = mu.data() + static_cast<size_t>(c) * D;
      const float* l = lam.data() + static_cast<size_t>(c) * D * Ht;
      const float* p = sd.data() + static_cast<size_t>(c) * D;
      float* x = X + i * D;
      for (int d = 0; d < D; ++d) {
        double v = m[d];
        for (int h = 0; h < Ht; ++h) v += static_cast<double>(l[d * Ht + h]) * z[h];
        v += p[d] * s.gaussian();
        if (sp->kind == 1) v = std::clamp(v, 0.0, 1.0);
        x[d] = static_cast<float>(v);
      }
      if (labels) labels[i] = c;
    }
  });
  return VMFA_OK;
}

// trainer.cpp:32-47 (initialize with InitConfig::Method::random_points) and
// trainer.cpp:107-109 (init_varstate).
extern "C" int vmfa_host_initialize(const float* X, int64_t N, int D, int C, int H, int Cp, int G,
                                    uint64_t seed, double scale, int loading_init, double* floor,
                                    double* pi, double* mu, double* lambda, double* dnoise,
                                    int32_t* K, int32_t* g, int32_t* g_count, int64_t* seeds) {
  if (!X || N < 1 || D < 1 || C < 1 || C > N || H < 1 || H > D || Cp < 1 || Cp > C || G < 1 ||
      G > C)
    return fail(VMFA_ERR_INVALID_ARGUMENT, "vmfa_host_initialize: invalid sizes");
  const int threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  // per_dimension_variance (dataset.cpp:22-35): two fp64 passes, rows in order
  // per dimension (parallel over dimensions keeps each dimension's order).
  std::vector<double> var(D);
  parallel_ranges(D, threads, [&](int, int64_t b, int64_t e) {
    std::vector<double> mean(e - b, 0.0), acc(e - b, 0.0);
    for (int64_t i = 0; i < N; ++i)
      for (int64_t d = b; d < e; ++d) mean[d - b] += static_cast<double>(X[i * D + d]);
    for (int64_t d = b; d < e; ++d) mean[d - b] /= static_cast<double>(N);
    for (int64_t i = 0; i < N; ++i)
      for (int64_t d = b; d < e; ++d) {
        const double t = static_cast<double>(X[i * D + d]) - mean[d - b];
        acc[d - b] += t * t;
      }
    for (int64_t d = b; d < e; ++d) var[d] = acc[d - b] / static_cast<double>(N);
  });
  for (int d = 0; d < D; ++d) floor[d] = std::max(1e-6 * var[d], 1e-8);  // dataset.cpp:37-39

  // random_points_seed (seeding.cpp:123-149). count_distinct_rows (:16-32) is
  // an exact distinct-row count; a hash set gives the same answer.
  struct RowHash {
    const float* X;
    int D;
    size_t operator()(int64_t i) const {
      uint64_t h = 1469598103934665603ULL;
      const unsigned char* p = reinterpret_cast<const unsigned char*>(X + i * D);
      for (size_t b = 0; b < static_cast<size_t>(D) * sizeof(float); ++b) h = (h ^ p[b]) * 1099511628211ULL;
      return static_cast<size_t>(h);
    }
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
  {
    std::unordered_set<int64_t, RowHash, RowEq> distinct(16, RowHash{X, D}, RowEq{X, D});
    for (int64_t i = 0; i < N && static_cast<int64_t>(distinct.size()) < C; ++i) distinct.insert(i);
    if (static_cast<int64_t>(distinct.size()) < C)
      return fail(VMFA_ERR_DEGENERATE_DATA, "fewer distinct rows than requested seeds");
  }
  HostStream rng(key2(seed, 0x1217f01dULL));  // trainer.cpp:36
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
  // init_params (seeding.cpp:151-181), same stream
  for (int c = 0; c < C; ++c) {
    pi[c] = 1.0 / C;
    for (int d = 0; d < D; ++d) {
      mu[static_cast<size_t>(c) * D + d] = static_cast<double>(X[seeds[c] * D + d]);
      dnoise[static_cast<size_t>(c) * D + d] = std::max(var[d], floor[d]);
    }
    for (int d = 0; d < D; ++d)
      for (int h = 0; h < H; ++h)
        lambda[static_cast<size_t>(c) * D * H + static_cast<size_t>(h) * D + d] =
            loading_init == 0 ? rng.uniform() * scale : rng.gaussian() * scale;
  }
  // init_varstate (seeding.cpp:207-233): fill_distinct (:187-203) over a
  // sparse swap map (unlisted positions hold their own index).
  HostStream srng(key2(seed, 0x7a57a7e5ULL));  // trainer.cpp:107
  std::unordered_map<int64_t, int32_t> seed_of;
  for (int c = 0; c < C; ++c) seed_of[seeds[c]] = c;
  std::unordered_map<int, int> over;
  auto at = [&](int p) {
    auto it = over.find(p);
    return it == over.end() ? p : it->second;
  };
  auto fill = [&](int want, int preset, int32_t* out) {
    over.clear();
    int start = 0;
    if (preset >= 0) {
      const int a = at(0), b = at(preset);
      over[0] = b;
      over[preset] = a;
      start = 1;
    }
    for (int i = start; i < want; ++i) {
      const int j = i + static_cast<int>(srng.uniform_int(C - i));
      const int a = at(i), b = at(j);
      over[i] = b;
      over[j] = a;
    }
    for (int i = 0; i < want; ++i) out[i] = at(i);
    std::sort(out, out + want);
  };
  for (int64_t n = 0; n < N; ++n) {
    auto it = seed_of.find(n);
    fill(Cp, it == seed_of.end() ? -1 : it->second, K + n * Cp);
  }
  for (int c = 0; c < C; ++c) {
    fill(G, c, g + static_cast<int64_t>(c) * G);
    g_count[c] = G;
  }
  return VMFA_OK;
}
