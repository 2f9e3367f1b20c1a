// vmfa_synth.cpp — synthetic data for BASELINE.json's configs (the paper's
// image datasets are not available; SURVEY §8(d) specifies these generators).
// Every row draws from its own keyed stream, so any row range (a rank's
// shard, a CPU-baseline sample) is generated independently and identically.
//
// This file is benchmark INPUT infrastructure shared by both arms: it is
// compiled into libvmfa_b200.so (vmfa_gen_synthetic) and, with
// -DVMFA_SYNTH_ORACLE, into the oracle's library (orc_gen_synthetic), so the
// reference arm generates the same rows without loading the product. Both
// builds use -ffp-contract=off: the rows are bit-identical.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "vmfa_b200.h"
#include "../vmfa_rng.hpp"

#ifdef VMFA_SYNTH_ORACLE
#define VMFA_SYNTH_FN orc_gen_synthetic
#define VMFA_SYNTH_FAIL(msg) (VMFA_ERR_INVALID_ARGUMENT)
#else
#include "../vmfa_internal.hpp"
#define VMFA_SYNTH_FN vmfa_gen_synthetic
#define VMFA_SYNTH_FAIL(msg) (vmfa_b200::fail(VMFA_ERR_INVALID_ARGUMENT, msg))
#endif

namespace vmfa_b200 {
namespace {

constexpr uint64_t kSaltPi = 0x5eed91ULL;
constexpr uint64_t kSaltTruth = 0x7e0711ULL;
constexpr uint64_t kSaltRow = 0x5a3e11eULL;

template <class F>
void synth_ranges(int64_t n, int threads, F&& fn) {
  if (threads < 1) threads = 1;
  if (threads > n) threads = static_cast<int>(std::max<int64_t>(n, 1));
  if (threads <= 1) {
    fn(int64_t{0}, n);
    return;
  }
  std::vector<std::thread> pool;
  const int64_t base = n / threads, rem = n % threads;
  int64_t b = 0;
  for (int w = 0; w < threads; ++w) {
    const int64_t len = base + (w < rem ? 1 : 0);
    pool.emplace_back([&fn, b, len] { fn(b, b + len); });
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

extern "C" int VMFA_SYNTH_FN(const vmfa_synth_spec* sp, int64_t row_begin, int64_t row_end,
                                  float* X, int32_t* labels, int threads) {
  if (!sp || !X || row_begin < 0 || row_end < row_begin || row_end > sp->n_total || sp->D < 1 ||
      sp->C_true < 1 || sp->H_true < 0)
    return VMFA_SYNTH_FAIL("vmfa_gen_synthetic: bad arguments");
  if (sp->kind == 1 && sp->img_w * sp->img_h * sp->img_c != sp->D)
    return VMFA_SYNTH_FAIL("vmfa_gen_synthetic: img_w*img_h*img_c != D");
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
  synth_ranges(Ct, threads, [&](int64_t b, int64_t e) {
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
  synth_ranges(row_end - row_begin, threads, [&](int64_t b, int64_t e) {
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

