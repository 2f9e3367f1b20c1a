// vmfa_b200.hpp — C++ mirror of the reference's public API
// (/root/reference/proj/include/vmfa/*.hpp) over the C-ABI in vmfa_b200.h.
//
// Same type and function names, argument meaning and exception behaviour as
// the reference, without Eigen (the layouts are the reference's own Eigen
// layouts, stored in std::vector). A reference-side caller swaps
//   #include "vmfa/trainer.hpp"   ->   #include "vmfa_b200.hpp"
// and links libvmfa_b200.so. Device residency is kept inside a Session (one
// GPU context): the free functions take the Session in place of the
// reference's `int threads` argument, because the device owns the data and
// the caches between calls.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <chrono>
#include <cmath>
#include <limits>
#include <vector>

#include "vmfa_b200.h"

namespace vmfa_b200 {

// ---- errors (errors.hpp:9-62) ---------------------------------------------------
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CholeskyFailure : Error { using Error::Error; };
struct EmptyKSet : Error { using Error::Error; };
struct InsufficientCandidates : Error { using Error::Error; };
struct SingularEc : Error { using Error::Error; };
struct MaxIterExceeded : Error { using Error::Error; };
struct TargetUnreachable : Error { using Error::Error; };
struct DegenerateData : Error { using Error::Error; };
struct BadMagic : Error { using Error::Error; };
struct TruncatedFile : Error { using Error::Error; };
struct UnsupportedVersion : Error { using Error::Error; };
struct DeviceError : Error { using Error::Error; };  // CUDA / no device / unsupported shape

inline void check(int code) {
  if (code == VMFA_OK) return;
  const std::string msg = vmfa_last_error();
  switch (code) {
    case VMFA_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case VMFA_ERR_CHOLESKY_FAILURE: throw CholeskyFailure(msg);
    case VMFA_ERR_EMPTY_KSET: throw EmptyKSet(msg);
    case VMFA_ERR_INSUFFICIENT_CANDIDATES: throw InsufficientCandidates(msg);
    case VMFA_ERR_SINGULAR_EC: throw SingularEc(msg);
    case VMFA_ERR_MAX_ITER_EXCEEDED: throw MaxIterExceeded(msg);
    case VMFA_ERR_TARGET_UNREACHABLE: throw TargetUnreachable(msg);
    case VMFA_ERR_DEGENERATE_DATA: throw DegenerateData(msg);
    case VMFA_ERR_BAD_MAGIC: throw BadMagic(msg);
    case VMFA_ERR_TRUNCATED_FILE: throw TruncatedFile(msg);
    case VMFA_ERR_UNSUPPORTED_VERSION: throw UnsupportedVersion(msg);
    case VMFA_ERR_IO: throw Error(msg);
    default: throw DeviceError(msg);
  }
}

enum class DistanceMode { kl = VMFA_DIST_KL, euclid = VMFA_DIST_EUCLID };  // estep.hpp:12

// ---- data / model types (reference layouts) ---------------------------------------
struct Dataset {  // dataset.hpp:11-35: N x D float, row-major
  int64_t N = 0;
  int D = 0;
  std::vector<float> rows;
};

struct MfaParams {  // model.hpp:19-32
  int C = 0, D = 0, H = 0;
  std::vector<double> pi;      // C
  std::vector<double> mu;      // C x D row-major
  std::vector<double> Lambda;  // C blocks, D x H column-major
  std::vector<double> dnoise;  // C x D row-major
};

struct ComponentCaches {  // model.hpp:37-45, all C components
  std::vector<double> U, Lmat, V, Sigma_z, inv_dnoise, logdet_sigma, log_pi;
};

struct VarState {  // estep.hpp:17-29
  int C = 0, Cprime = 0, G = 0;
  std::vector<int32_t> K;        // N x C' (rows sorted ascending)
  std::vector<int32_t> g;        // C x G (rows sorted, -1 padded)
  std::vector<int32_t> g_count;  // C
  std::vector<int32_t> labels;   // N
};

struct EStepResult {  // estep.hpp:72-78
  int stride = 0;
  std::vector<int32_t> count, idx;
  std::vector<double> lj, resp;
  double free_energy = 0.0;
  uint64_t joints = 0;
};

struct SuffStats {  // mstep.hpp:14-22
  std::vector<double> Nc, Y, E, sq_sum;
};

struct EvalCounter {  // model.hpp:49-58
  uint64_t joints = 0;
  uint64_t distances = 0;
};

// ---- Session: one device context ------------------------------------------------
class Session {
 public:
  Session(const Dataset& data, int C, int H, int Cprime, int G, int device = 0,
          int64_t n_offset = 0, int64_t n_total = -1)
      : N_(data.N), D_(data.D), C_(C), H_(H), Cp_(Cprime), G_(G) {
    check(vmfa_ctx_create(&ctx_, device, C, data.D, H, Cprime, G, data.N, n_offset,
                          n_total < 0 ? n_offset + data.N : n_total, nullptr));
    check(vmfa_upload_data(ctx_, data.rows.data(), 0, data.N));
  }
  ~Session() { vmfa_ctx_destroy(ctx_); }
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;

  vmfa_ctx* handle() const { return ctx_; }
  int64_t rows() const { return N_; }
  int C() const { return C_; }
  int D() const { return D_; }
  int H() const { return H_; }
  int Cprime() const { return Cp_; }
  int G() const { return G_; }
  int stride() const { return static_cast<int>(std::min<int64_t>(int64_t{Cp_} * G_ + 1, C_)); }

  void set_floor(const std::vector<double>& floor) { check(vmfa_set_floor(ctx_, floor.data())); }
  void upload(const MfaParams& p) {
    check(vmfa_upload_params(ctx_, p.pi.data(), p.mu.data(), p.Lambda.data(), p.dnoise.data()));
  }
  void upload(const VarState& s) { check(vmfa_upload_state(ctx_, s.K.data(), s.g.data(), s.g_count.data())); }
  MfaParams download_params() const {
    MfaParams p;
    p.C = C_, p.D = D_, p.H = H_;
    p.pi.resize(C_);
    p.mu.resize(size_t(C_) * D_);
    p.Lambda.resize(size_t(C_) * D_ * H_);
    p.dnoise.resize(size_t(C_) * D_);
    check(vmfa_download_params(ctx_, p.pi.data(), p.mu.data(), p.Lambda.data(), p.dnoise.data()));
    return p;
  }
  void download(VarState& s) const {
    s.C = C_, s.Cprime = Cp_, s.G = G_;
    s.K.resize(size_t(N_) * Cp_);
    s.g.resize(size_t(C_) * G_);
    s.g_count.resize(C_);
    s.labels.resize(N_);
    check(vmfa_download_state(ctx_, s.K.data(), s.g.data(), s.g_count.data(), s.labels.data()));
  }

 private:
  vmfa_ctx* ctx_ = nullptr;
  int64_t N_;
  int D_, C_, H_, Cp_, G_;
};

// ---- the reference's free functions -------------------------------------------------
// precompute_all (model.hpp:76-78): caches of the session's parameters.
inline ComponentCaches precompute_all(Session& s, const MfaParams& params) {
  s.upload(params);  // uploads and runs precompute_all on the device
  ComponentCaches k;
  const size_t C = s.C(), D = s.D(), H = s.H();
  k.U.resize(C * D * H);
  k.V.resize(C * D * H);
  k.Lmat.resize(C * H * H);
  k.Sigma_z.resize(C * H * H);
  k.inv_dnoise.resize(C * D);
  k.logdet_sigma.resize(C);
  k.log_pi.resize(C);
  check(vmfa_download_caches(s.handle(), k.U.data(), k.Lmat.data(), k.V.data(), k.Sigma_z.data(),
                             k.inv_dnoise.data(), k.logdet_sigma.data(), k.log_pi.data()));
  return k;
}

// variational_e_step (estep.hpp:125-130): updates `state` in place.
inline EStepResult variational_e_step(Session& s, VarState& state, uint64_t seed, uint64_t iteration,
                                      DistanceMode mode, EvalCounter& counter) {
  s.upload(state);
  EStepResult r;
  check(vmfa_estep(s.handle(), seed, iteration, static_cast<int>(mode), &r.free_energy, &r.joints));
  r.stride = s.stride();
  r.count.resize(s.rows());
  r.idx.resize(size_t(s.rows()) * r.stride);
  r.lj.resize(size_t(s.rows()) * r.stride);
  r.resp.resize(size_t(s.rows()) * s.Cprime());
  check(vmfa_download_estep(s.handle(), r.count.data(), r.idx.data(), r.lj.data(), r.resp.data()));
  s.download(state);
  counter.joints += r.joints;
  return r;
}

inline SuffStats download_suffstats(Session& s) {
  SuffStats st;
  const size_t C = s.C(), D = s.D(), H1 = s.H() + 1;
  st.Nc.resize(C);
  st.Y.resize(C * D * H1);
  st.E.resize(C * H1 * H1);
  st.sq_sum.resize(C * D);
  check(vmfa_download_suffstats(s.handle(), st.Nc.data(), st.Y.data(), st.E.data(), st.sq_sum.data()));
  return st;
}

// accumulate_suffstats (mstep.hpp:27-31) of the last E-step's K and
// responsibilities, on the device.
inline SuffStats accumulate_suffstats(Session& s) {
  check(vmfa_accumulate_suffstats(s.handle()));
  return download_suffstats(s);
}

// accumulate_suffstats(params, caches, data, ksets, resp) with the caller's K
// rows (N x C') and responsibilities (N x C', aligned with K) under the
// session's parameters; the session's K becomes ksets.
inline SuffStats accumulate_suffstats(Session& s, const std::vector<int32_t>& ksets,
                                      const std::vector<double>& resp) {
  if (ksets.size() != size_t(s.rows()) * s.Cprime() || resp.size() != ksets.size())
    throw std::invalid_argument("ksets / resp sizes");
  check(vmfa_accumulate_suffstats_k(s.handle(), ksets.data(), resp.data()));
  return download_suffstats(s);
}

// update_params (mstep.hpp:39-41) from `stats`; the session keeps the result
// and its caches.
inline MfaParams update_params(Session& s, const SuffStats& stats) {
  check(vmfa_upload_suffstats(s.handle(), stats.Nc.data(), stats.Y.data(), stats.E.data(),
                              stats.sq_sum.data()));
  int failed = -1;
  check(vmfa_update_params(s.handle(), &failed));
  return s.download_params();
}

// truncated_free_energy (model.hpp:116-119) under the session's parameters
// over the caller's K rows (the session's K becomes ksets); adds N C' to the
// counter, as the reference does.
inline double truncated_free_energy(Session& s, const std::vector<int32_t>& ksets, EvalCounter& counter) {
  if (ksets.empty()) throw EmptyKSet("empty K collection");
  if (ksets.size() != size_t(s.rows()) * s.Cprime()) throw std::invalid_argument("ksets size");
  double F = 0.0;
  check(vmfa_truncated_free_energy_k(s.handle(), ksets.data(), &F));
  counter.joints += static_cast<uint64_t>(s.rows()) * s.Cprime();
  return F;
}
inline double truncated_free_energy(Session& s, const VarState& state, EvalCounter& counter) {
  return truncated_free_energy(s, state.K, counter);
}

// log_joint (model.hpp:83-86): log p(c, x) in fp64 under the session's
// parameters; counter.joints += 1 per pair. Batched: rows X (n x D).
inline std::vector<double> log_joint(Session& s, const std::vector<float>& X, const std::vector<int32_t>& comp,
                                     EvalCounter& counter) {
  if (X.size() != comp.size() * size_t(s.D())) throw std::invalid_argument("X / comp sizes");
  std::vector<double> out(comp.size());
  check(vmfa_log_joint(s.handle(), X.data(), static_cast<int64_t>(comp.size()), comp.data(), out.data()));
  counter.joints += comp.size();
  return out;
}
inline double log_joint(Session& s, int c, const float* x, EvalCounter& counter) {
  double out = 0.0;
  const int32_t cc = c;
  check(vmfa_log_joint(s.handle(), x, 1, &cc, &out));
  counter.joints += 1;
  return out;
}

// ---- the E-step's per-operation pieces (estep.hpp:82-117), batched over the
// session's rows; RetainedJoints / partition in the reference layouts
struct RetainedJoints {  // estep.hpp:48-70
  int stride = 0;
  std::vector<int32_t> count, idx;
  std::vector<double> lj;
};
// build_search_space for every row of the session's K / g: extra r_n from
// `extras` (N entries) or uniform_component(seed, iteration, n_offset + n, C)
inline RetainedJoints build_search_space(Session& s, uint64_t seed, uint64_t iteration,
                                         const std::vector<int32_t>* extras = nullptr) {
  RetainedJoints r;
  r.stride = s.stride();
  r.count.resize(s.rows());
  r.idx.resize(size_t(s.rows()) * r.stride);
  check(vmfa_build_search_space(s.handle(), seed, iteration, extras ? extras->data() : nullptr, r.count.data(),
                                r.idx.data()));
  return r;
}
// update_k for every row: top-C' by (l desc, index asc), sorted ascending
inline std::vector<int32_t> update_k(Session& s, const RetainedJoints& r) {
  std::vector<int32_t> K(size_t(s.rows()) * s.Cprime());
  check(vmfa_update_k(s.handle(), r.count.data(), r.idx.data(), r.lj.data(), K.data()));
  return K;
}
// hard_partition: labels and the partition (offsets C+1, rows ascending per cell)
inline void hard_partition(Session& s, const std::vector<int32_t>& K, const RetainedJoints& r,
                           std::vector<int32_t>& labels, std::vector<int32_t>& part_off,
                           std::vector<int32_t>& part_ent) {
  labels.resize(s.rows());
  part_off.resize(s.C() + 1);
  part_ent.resize(s.rows());
  check(vmfa_hard_partition(s.handle(), K.data(), r.count.data(), r.idx.data(), r.lj.data(), labels.data(),
                            part_off.data(), part_ent.data()));
}
struct DistanceRows {  // DistanceAccumulator (estep.hpp:34-44) as sorted rows
  std::vector<int32_t> c, ct;
  std::vector<double> sum;
  std::vector<int64_t> count;
};
inline DistanceRows accumulate_distances(Session& s, const std::vector<int32_t>& part_off,
                                         const std::vector<int32_t>& part_ent, const RetainedJoints& r,
                                         DistanceMode mode, const MfaParams& params) {
  DistanceRows d;
  int64_t n = 0;
  check(vmfa_accumulate_distances(s.handle(), static_cast<int>(mode), part_off.data(), part_ent.data(),
                                  r.count.data(), r.idx.data(), r.lj.data(), params.pi.data(), 0, nullptr, nullptr,
                                  nullptr, nullptr, &n));
  d.c.resize(n), d.ct.resize(n), d.sum.resize(n), d.count.resize(n);
  check(vmfa_accumulate_distances(s.handle(), static_cast<int>(mode), part_off.data(), part_ent.data(),
                                  r.count.data(), r.idx.data(), r.lj.data(), params.pi.data(), n, d.c.data(),
                                  d.ct.data(), d.sum.data(), d.count.data(), &n));
  return d;
}
// update_g for every component: g rows (C x G, -1 padded) and counts
inline void update_g(Session& s, const DistanceRows& d, std::vector<int32_t>& g, std::vector<int32_t>& g_count) {
  g.resize(size_t(s.C()) * s.G());
  g_count.resize(s.C());
  check(vmfa_update_g(s.handle(), static_cast<int64_t>(d.c.size()), d.c.data(), d.ct.data(), d.sum.data(),
                      d.count.data(), g.data(), g_count.data()));
}
// responsibilities_row for `rows` rows of `width` log-joints
inline std::vector<double> responsibilities(Session& s, const std::vector<double>& lj, int width) {
  std::vector<double> out(lj.size());
  check(vmfa_responsibilities(s.handle(), static_cast<int64_t>(lj.size() / width), width, lj.data(), out.data()));
  return out;
}

// exact_log_likelihood (model.hpp:108-111): sum_n log sum_c p(x_n, c) over all
// C components under the session's parameters (the NLL of trainer.cpp:49-56,
// 79-85 is -exact_log_likelihood / N); adds N C to the counter.
inline double exact_log_likelihood(Session& s, EvalCounter& counter) {
  double ll = 0.0;
  check(vmfa_exact_log_likelihood(s.handle(), &ll));
  counter.joints += static_cast<uint64_t>(s.rows()) * s.C();
  return ll;
}
inline double exact_log_likelihood(Session& s) {
  EvalCounter scratch;
  return exact_log_likelihood(s, scratch);
}

// em_full_step (mstep.hpp; mstep.cpp:164-208): full-posterior statistics of
// every (n, c) pair under the session's parameters; returns sum_n LSE_n.
inline double em_full_step(Session& s, SuffStats& stats, EvalCounter& counter) {
  double ll = 0.0;
  uint64_t j = 0;
  check(vmfa_em_full_step(s.handle(), &ll, &j));
  counter.joints += j;
  const size_t C = s.C(), D = s.D(), H1 = s.H() + 1;
  stats.Nc.resize(C);
  stats.Y.resize(C * D * H1);
  stats.E.resize(C * H1 * H1);
  stats.sq_sum.resize(C * D);
  check(vmfa_download_suffstats(s.handle(), stats.Nc.data(), stats.Y.data(), stats.E.data(),
                                stats.sq_sum.data()));
  return ll;
}

// afkmc2_seed (seeding.hpp:29-31; seeding.cpp:60-121) over the session's rows;
// `stream_state` receives the xoshiro256++ state init_params continues from.
inline std::vector<int64_t> afkmc2_seed(Session& s, int C, int chain_length, uint64_t stream_seed,
                                        uint64_t stream_state[4] = nullptr, uint64_t* distances = nullptr) {
  std::vector<int64_t> seeds(C);
  uint64_t st[4];
  check(vmfa_afkmc2_seed(s.handle(), C, chain_length, stream_seed, seeds.data(), st, distances));
  if (stream_state)
    for (int k = 0; k < 4; ++k) stream_state[k] = st[k];
  return seeds;
}

// train_vmfa's loop (trainer.cpp:111-186) with fixed warm-up / main counts.
struct IterationRecord {
  bool warmup = false;
  double F = 0.0;
  double F_estep = 0.0;
  uint64_t joint_evals = 0;
  int empty_components = 0;
};
inline std::vector<IterationRecord> train_fixed(Session& s, uint64_t seed, int warmup, int iters,
                                                DistanceMode mode = DistanceMode::kl) {
  std::vector<IterationRecord> recs;
  uint64_t it = 0, joints = 0;
  for (int w = 0; w < warmup; ++w) {
    IterationRecord r;
    uint64_t j = 0;
    check(vmfa_estep(s.handle(), seed, it++, static_cast<int>(mode), &r.F, &j));
    joints += j;
    r.warmup = true;
    r.joint_evals = joints;
    recs.push_back(r);
  }
  for (int t = 0; t < iters; ++t) {
    vmfa_iter_report rep{};
    check(vmfa_iterate(s.handle(), seed, it++, static_cast<int>(mode), &rep));
    joints += rep.joints;
    IterationRecord r;
    r.F = rep.free_energy;
    r.F_estep = rep.free_energy_estep;
    r.joint_evals = joints;
    r.empty_components = rep.empty_components;
    recs.push_back(r);
  }
  return recs;
}

// ---- on-disk containers (io.hpp:12-23) ----------------------------------------
inline void save_dataset(const Dataset& data, const std::string& path) {
  check(vmfa_save_dataset(path.c_str(), data.rows.data(), data.N, data.D));
}
inline Dataset load_dataset(const std::string& path) {
  Dataset d;
  check(vmfa_dataset_info(path.c_str(), &d.N, &d.D));
  d.rows.resize(static_cast<size_t>(d.N) * d.D);
  check(vmfa_load_dataset(path.c_str(), 0, d.N, d.D, d.rows.data()));
  return d;
}
inline void save_checkpoint(const MfaParams& p, const std::string& path) {
  check(vmfa_save_checkpoint(path.c_str(), p.C, p.D, p.H, p.pi.data(), p.mu.data(), p.Lambda.data(),
                             p.dnoise.data()));
}
inline MfaParams load_checkpoint(const std::string& path) {
  MfaParams p;
  check(vmfa_checkpoint_info(path.c_str(), &p.C, &p.D, &p.H));
  p.pi.resize(p.C);
  p.mu.resize(static_cast<size_t>(p.C) * p.D);
  p.Lambda.resize(static_cast<size_t>(p.C) * p.D * p.H);
  p.dnoise.resize(static_cast<size_t>(p.C) * p.D);
  check(vmfa_load_checkpoint(path.c_str(), p.C, p.D, p.H, p.pi.data(), p.mu.data(), p.Lambda.data(),
                             p.dnoise.data()));
  return p;
}

// check_convergence (trainer.hpp:76-80).
inline bool check_convergence(double f_prev, double f_curr, double epsilon, bool literal = false) {
  if (literal) return (f_curr - f_prev) / f_prev < epsilon;
  return std::abs(f_curr - f_prev) < epsilon * std::abs(f_prev);
}

// The TrainConfig / InitConfig fields train_vmfa's loop reads (trainer.hpp:19-37,
// seeding.hpp:18-19).
struct TrainConfig {
  uint64_t seed = 0;
  double epsilon = 1e-4;
  int max_iters = 500;
  DistanceMode distance_mode = DistanceMode::kl;
  int eval_nll_every = 0;
  bool literal_eq14 = false;
  bool halt_on_max_iters = true;
  double warmup_epsilon = 1e-4;
  int warmup_max_iters = 1000;
};
struct TrainRecord {
  int t = 0;
  bool warmup = false;
  double F = 0.0;
  uint64_t joint_evals = 0;
  double wall_ms = 0.0;
  int empty_components = 0;
  double nll_train = std::numeric_limits<double>::quiet_NaN();
};
struct TrainReport {
  std::vector<TrainRecord> iterations;
  int warmup_iterations = 0;
  int main_iterations = 0;
  bool converged = false;
  uint64_t joint_evals = 0;
  double total_wall_ms = 0.0;
  double nll_train = std::numeric_limits<double>::quiet_NaN();
};

// train_vmfa's loop (trainer.cpp:111-186) on the device after the caller's
// initialisation: convergence-gated warm-up (MaxIterExceeded at the cap),
// main iterations until check_convergence, exact NLL every eval_nll_every
// iterations (excluded from the wall time) and at the end (finalize_nll).
inline TrainReport train_vmfa(Session& s, const TrainConfig& cfg) {
  using clk = std::chrono::steady_clock;
  auto ms = [](clk::time_point a) { return std::chrono::duration<double, std::milli>(clk::now() - a).count(); };
  auto nll = [&]() { return -exact_log_likelihood(s) / static_cast<double>(s.rows()); };
  TrainReport rep;
  const auto t_start = clk::now();
  double excluded = 0.0;
  uint64_t it = 0;
  double prev = std::numeric_limits<double>::quiet_NaN();
  for (int w = 0; w < cfg.warmup_max_iters; ++w) {
    const auto t0 = clk::now();
    TrainRecord r;
    uint64_t j = 0;
    check(vmfa_estep(s.handle(), cfg.seed, it++, static_cast<int>(cfg.distance_mode), &r.F, &j));
    rep.joint_evals += j;
    r.t = ++rep.warmup_iterations;
    r.warmup = true;
    r.joint_evals = rep.joint_evals;
    r.wall_ms = ms(t0);
    rep.iterations.push_back(r);
    if (std::isfinite(prev) && check_convergence(prev, r.F, cfg.warmup_epsilon, cfg.literal_eq14)) break;
    prev = r.F;
    if (w + 1 == cfg.warmup_max_iters) throw MaxIterExceeded("warm-up did not converge");
  }
  double prev_f = std::numeric_limits<double>::quiet_NaN();
  for (int t = 1; t <= cfg.max_iters; ++t) {
    const auto t0 = clk::now();
    vmfa_iter_report ir{};
    check(vmfa_iterate(s.handle(), cfg.seed, it++, static_cast<int>(cfg.distance_mode), &ir));
    rep.joint_evals += ir.joints;
    ++rep.main_iterations;
    TrainRecord r;
    r.t = t;
    r.F = ir.free_energy;
    r.joint_evals = rep.joint_evals;
    r.wall_ms = ms(t0);
    r.empty_components = ir.empty_components;
    if (cfg.eval_nll_every > 0 && t % cfg.eval_nll_every == 0) {
      const auto t1 = clk::now();
      r.nll_train = nll();
      excluded += ms(t1);
    }
    rep.iterations.push_back(r);
    if (std::isfinite(prev_f) && check_convergence(prev_f, r.F, cfg.epsilon, cfg.literal_eq14)) {
      rep.converged = true;
      break;
    }
    prev_f = r.F;
  }
  if (!rep.converged && cfg.halt_on_max_iters)
    throw MaxIterExceeded("training did not converge within " + std::to_string(cfg.max_iters) + " iterations");
  rep.total_wall_ms = ms(t_start) - excluded;
  rep.nll_train = nll();
  return rep;
}

}  // namespace vmfa_b200
