// vmfa_capi.cu — device context and the C-ABI of libvmfa_b200.so
// (include/vmfa_b200.h). One context = one GPU's shard of the rows, the
// replicated parameters/caches, the shard's variational state and all scratch.
// Every phase is stream-ordered; host synchronisation happens only where a
// result is returned through a host pointer.

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <limits>
#include <vector>

#include "vmfa_b200.h"
#include "vmfa_internal.hpp"
#include "vmfa_rng.hpp"
#include "vmfa_kernels.cuh"

namespace vmfa_b200 {

namespace {
thread_local std::string g_err;
}
void set_error_text(const std::string& s) { g_err = s; }
const std::string& error_text() { return g_err; }

#define CU(x)                                                                                    \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess)                                                                       \
      return fail(VMFA_ERR_CUDA, "%s:%d %s -> %s", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
  } while (0)
#define TRY(x)                   \
  do {                           \
    int r_ = (x);                \
    if (r_ != VMFA_OK) return r_; \
  } while (0)

enum KernelFamily : int {
  kFamScoreAnchor = 0,
  kFamScoreExtra,
  kFamSelect,
  kFamGupdate,
  kFamStats,
  kFamUpdate,
  kFamPrecompute,
  kFamScoreTruncF,
  kFamSort,
  kFamOther,
  kFamExactLL,
  kFamFixup,
  kNumFamilies
};
const char* const kFamilyNames[kNumFamilies] = {
    "score_anchor", "score_extra", "select", "gupdate", "stats",
    "update", "precompute", "score_truncF", "csr_sort", "other", "exact_ll", "fixup_f64"};

__global__ void k_pack_scalar_u64(const unsigned long long* src, double* dst) { *dst = static_cast<double>(*src); }
__global__ void k_add_f64(const double* src, double* dst) { *dst = *src; }

}  // namespace vmfa_b200

using namespace vmfa_b200;

struct IterStatus {
  int sel;
  int empty;
  unsigned long long upd;
  unsigned long long model;
  double scal[4];
};

struct vmfa_ctx {
  int device = 0;
  Dims dm{};
  ScoreLayout L{};
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::vector<void*> allocs;
  size_t bytes = 0;

  // data
  float* X = nullptr;
  double* floor = nullptr;
  // params: two sets (current / next)
  double *pi = nullptr, *mu = nullptr, *lam = nullptr, *psi = nullptr;
  double *pi2 = nullptr, *mu2 = nullptr, *lam2 = nullptr, *psi2 = nullptr;
  // caches
  double *Lmat = nullptr, *R = nullptr, *Sz = nullptr, *logdet = nullptr, *logpi = nullptr,
         *kconst = nullptr;
  float *P = nullptr, *V32 = nullptr, *mu32 = nullptr, *WT = nullptr, *ipsi32 = nullptr;
  int Hp = 8;
  float *brec = nullptr, *srec = nullptr;  // scorer epilogue records (anchor slots / components)
  int4* jobs = nullptr;                    // scorer job table (one int4 per 128-row work item)
  int* qctr = nullptr;                     // statistics work-queue counter
  uint16_t *bimg = nullptr, *simg = nullptr;  // scorer B stage images (fp16; anchor / single)
  float *bscl = nullptr, *sscl = nullptr;     // their row scales
  float *xmax = nullptr, *mumax = nullptr;    // A-row scale bounds
  unsigned char* svimg = nullptr;             // the tcgen05 statistics kernel's V images (per precompute)
  int* svexp = nullptr;
  float* svl1 = nullptr;
  float* szbuf = nullptr;  // its zhat per K-pair (N C' x H)
  uint16_t* limg = nullptr;  // image-free anchor stages: per (anchor, group, chunk) lin / psi rows (fp16)
  bool ifree_only = false;    // the full anchor images do not fit: image-free stages everywhere
  unsigned long long* nfix = nullptr;         // scores re-evaluated in fp64 (vmfa_fixup.cu), accumulated
  long long* fix_list = nullptr;              // flagged scores of one scoring launch
  unsigned long long* fix_cnt = nullptr;      // [count, overflow]
  long long fix_cap = 0;
  int *fix_qkey = nullptr, *fix_qcnt = nullptr, *fix_qoff = nullptr, *fix_qfill = nullptr, *fix_iof = nullptr;
  int* fix_sorted = nullptr;
  unsigned long long* fix_ovf = nullptr;
  bool fix_ok = false;  // re-scoring pipeline on (warp-specialised scorer, N SL < 2^31)
  bool fix_tc = false;  // VMFA_FIX_TC=1: flagged scores pass the one-component tensor re-scoring before fp64
  double* W64 = nullptr;  // C x H x D fp64 W^T for the DMMA re-scoring (null: per-item staging)
  int scorer = 2;           // 2: warp-specialised tcgen05 (default), 1: single-role tcgen05, 0: FFMA
  bool use_tc = true;
  int score_rows = kScoreRowsTc;
  // state
  int *K = nullptr, *g = nullptr, *gcnt = nullptr, *g_new = nullptr, *gcnt_new = nullptr,
      *labels = nullptr;
  float* lablj = nullptr;
  // E-step scratch
  float* LJ = nullptr;      // N x SL
  float* LJK = nullptr;     // N x Cp
  int* rx = nullptr;
  unsigned* rkey = nullptr;
  int *ret_cnt = nullptr, *ret_idx = nullptr;
  float* ret_lj = nullptr;
  double *resp = nullptr, *lse = nullptr;
  // CSR / sort scratch
  unsigned *keys = nullptr, *keys_alt = nullptr, *keys_tmp = nullptr;
  int* sort_hist = nullptr;  // radix-sort digit histograms + scan scratch (vmfa_sort.cu)
  int* vals = nullptr;
  int *kinv_off = nullptr, *kinv_ent = nullptr, *kinv_items = nullptr;
  int *ex_off = nullptr, *ex_ent = nullptr, *ex_items = nullptr;
  int *part_off = nullptr, *part_ent = nullptr, *part_items = nullptr;
  int* stats_items = nullptr;
  int stats_rows = 256;     // K-pairs per statistics item
  int gupd_pts = 256;       // partition points per block-3 item
  double* stats_part = nullptr;
  int *cnt = nullptr, *chunks = nullptr;
  // block-3 scratch
  int gupd_grid = 0;
  long long *gt_cnt = nullptr, *gt_hi = nullptr, *gt_lo = nullptr;
  long long* xc = nullptr;  // multi-rank exchange (lazy)
  // sparse co-occurrence lists (C too large for the dense rows, or
  // VMFA_COOC=sparse): raw appended entries, their sort, the reduced list
  bool sparse = false;
  long long cl_cap = 0;
  int cl_kb = 0;
  unsigned *cl_key = nullptr, *cl_skey = nullptr, *cu_key = nullptr;
  long long *cl_cnt = nullptr, *cl_hi = nullptr, *cl_lo = nullptr;
  long long *cu_cnt = nullptr, *cu_hi = nullptr, *cu_lo = nullptr;
  int *cl_iota = nullptr, *cl_perm = nullptr, *cu_off = nullptr;
  unsigned long long* cl_n = nullptr;
  int* cl_ovf = nullptr;
  int64_t cu_n = 0;  // unique entries of the last reduction (host)
  int* cl_hist = nullptr;  // the list sort's digit histograms and scan scratch
  // stats: packed [Nc | E | Y | sq]
  double* stats = nullptr;
  size_t stats_len = 0;
  double *Nc = nullptr, *E = nullptr, *Y = nullptr, *sq = nullptr;
  // reductions / scalars / status
  double* partials = nullptr;
  double* scal = nullptr;   // [F_estep, joints, F_post, spare]
  unsigned long long* u64tmp = nullptr;
  int* st_select = nullptr;
  unsigned long long* st_model = nullptr;
  unsigned long long* st_update = nullptr;
  IterStatus* hstat = nullptr;  // pinned host readback of one iteration's statuses and scalars
  int* n_empty = nullptr;
  // exact_log_likelihood's dense pass (allocated on first use)
  int *dense_g = nullptr, *dense_gcnt = nullptr, *dense_ent = nullptr, *dense_items = nullptr,
      *dense_off = nullptr;
  int4* dense_jobs = nullptr;
  float* dense_LJ = nullptr;
  double *dense_lse = nullptr, *dense_out = nullptr;
  int64_t dense_R = 0;
  // em_full_step's full-posterior pairs of a row chunk (allocated on first use)
  double *em_resp = nullptr, *em_part = nullptr, *em_acc = nullptr;
  int *em_ent = nullptr, *em_off = nullptr, *em_items = nullptr;
  int64_t em_R = 0;
  int dense_SL = 0;
  bool kinv_for_current_K = false;
  // the anchor pass of the next E-step already ran (under the current K, g
  // and parameters) while computing the truncated free energy: LJ's anchor
  // slots are valid and the next estep_local skips block 1's anchor scoring
  bool prescored = false;
  bool lookahead = true;  // VMFA_LOOKAHEAD=0 (or vmfa_set_lookahead) scores the truncated F with its own pass
  // vmfa_upload_data_async: rows copied on a second stream; X consumers wait on x_ready
  cudaStream_t cstream = nullptr;
  cudaEvent_t x_ready = nullptr, x_free = nullptr;
  // vmfa_stage_data_async / vmfa_swap_data: a second row buffer filled on
  // cstream while the current one is in use (pipelined uploads)
  float* Xs = nullptr;
  float* xmax_s = nullptr;
  cudaEvent_t xs_ready = nullptr;
  bool xs_pending = false;
  bool x_pending = false;
  bool have_estep = false;
  // CUDA graphs of vmfa_iterate (default; VMFA_GRAPH=0 disables): one per host-side pre-state
  // (pointer parities, lookahead flags); replays restore the recorded post-state
  unsigned long long* sit = nullptr;  // (seed, E-step index) read by k_extra
  bool capturing = false;
  bool graph_off = false;
  // vmfa_iterate runs block 3 (g update) on a side stream next to the
  // statistics / update / precompute: forked after the label partition,
  // joined before the anchor images (the first reader of the new g)
  cudaStream_t gstream = nullptr;
  cudaEvent_t g_fork = nullptr, g_join = nullptr;
  double* logpi_g = nullptr;  // log pi of the E-step's parameters (precompute rewrites logpi)
  GupdArgs g_args{};
  bool g_deferred = false, g_join_pending = false;
  struct HostState {
    int *g, *gcnt, *g_new, *gcnt_new;
    double *pi, *pi2, *mu, *mu2, *lam, *lam2, *psi, *psi2;
    float *X, *xmax;  // (the staged-row double buffer swaps them)
    bool prescored, kinv, have_estep;
    int mode;
    bool lookahead;
    bool operator==(const HostState& o) const {
      return g == o.g && gcnt == o.gcnt && g_new == o.g_new && gcnt_new == o.gcnt_new && pi == o.pi &&
             pi2 == o.pi2 && mu == o.mu && mu2 == o.mu2 && lam == o.lam && lam2 == o.lam2 && psi == o.psi &&
             psi2 == o.psi2 && X == o.X && xmax == o.xmax && prescored == o.prescored && kinv == o.kinv && have_estep == o.have_estep &&
             mode == o.mode && lookahead == o.lookahead;
    }
  };
  struct GraphEntry {
    HostState pre, post;
    cudaGraphExec_t exec;
  };
  std::vector<GraphEntry> graphs;
  // dumps (parity only)
  bool dump = false;
  int *dump_c = nullptr, *dump_ct = nullptr;
  long long *dump_cnt = nullptr, *dump_hi = nullptr, *dump_lo = nullptr;
  unsigned long long* dump_n = nullptr;
  long long dump_cap = 0;
  // profiling
  bool profile = false;
  struct Ev {
    int fam;
    cudaEvent_t a, b;
    int64_t units;
  };
  std::vector<Ev> pending;
  std::vector<cudaEvent_t> ev_pool;
  double fam_ms[kNumFamilies] = {};
  int64_t fam_launches[kNumFamilies] = {};
  int64_t fam_units[kNumFamilies] = {};
  int64_t launches = 0;

  template <class T>
  int alloc(T*& p, size_t n) {
    void* q = nullptr;
    const size_t b = std::max<size_t>(n, 1) * sizeof(T);
    cudaError_t e = cudaMalloc(&q, b);
    if (e != cudaSuccess)
      return fail(VMFA_ERR_CUDA, "cudaMalloc(%zu bytes) failed: %s", b, cudaGetErrorString(e));
    allocs.push_back(q);
    bytes += b;
    p = static_cast<T*>(q);
    return VMFA_OK;
  }
  cudaEvent_t ev() {
    if (!ev_pool.empty()) {
      cudaEvent_t e = ev_pool.back();
      ev_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  // family-scoped timing: begin() returns a token, end() records
  int begin(int fam, int64_t units) {
    fam_launches[fam] += 1;
    fam_units[fam] += units;
    if (!profile) return -1;
    Ev x{fam, ev(), ev(), units};
    cudaEventRecord(x.a, stream);
    pending.push_back(x);
    return static_cast<int>(pending.size()) - 1;
  }
  void end(int tok) {
    if (tok >= 0) cudaEventRecord(pending[tok].b, stream);
  }
  void collect() {
    if (pending.empty()) return;
    cudaStreamSynchronize(stream);
    for (auto& x : pending) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, x.a, x.b);
      fam_ms[x.fam] += ms;
      ev_pool.push_back(x.a);
      ev_pool.push_back(x.b);
    }
    pending.clear();
  }
};

namespace vmfa_b200 {
namespace {

int bits_for(unsigned v) {
  int b = 1;
  while ((1ull << b) <= v) ++b;
  return b;
}

// Stable CSR of `n` keys in [0, C] (C = dropped sentinel) -> off (C+1), ent
// (indices 0..n-1 ordered by key, stable) and per-key chunk offsets for the
// persistent scoring kernels.
int csr_by_key(vmfa_ctx* x, const unsigned* keys, int64_t n, int* off, int* ent, int* items,
               int rows_per_item) {
  const int C = x->dm.C;
  cudaStream_t s = x->stream;
  const int tok = x->begin(kFamSort, n);
  CU(radix_sort_pairs(keys, nullptr, n, bits_for(static_cast<unsigned>(C)), x->keys_tmp, x->vals, x->keys_alt, ent,
                      x->sort_hist, s));
  CU(launch_offsets_sorted(x->keys_alt, n, C, off, s));
  static const bool check = [] {  // VMFA_SORT_CHECK=1: verify every CSR on the host (debugging)
    const char* v = std::getenv("VMFA_SORT_CHECK");
    return v && v[0] == '1';
  }();
  if (check && !x->capturing) {
    std::vector<unsigned> k(n), ks(n);
    std::vector<int> e(n);
    CU(cudaMemcpyAsync(k.data(), keys, 4 * n, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(ks.data(), x->keys_alt, 4 * n, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(e.data(), ent, 4 * n, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    const unsigned mask = (1u << bits_for(static_cast<unsigned>(C))) - 1u;
    for (int64_t i = 0; i < n; ++i) {
      const bool bad = e[i] < 0 || e[i] >= n || ks[i] != k[e[i]] ||
                       (i > 0 && ((ks[i - 1] & mask) > (ks[i] & mask) ||
                                  ((ks[i - 1] & mask) == (ks[i] & mask) && e[i - 1] >= e[i])));
      if (bad) {
        std::fprintf(stderr, "vmfa: csr_by_key check failed at %lld of %lld (key %u ent %d)\n",
                     static_cast<long long>(i), static_cast<long long>(n), ks[i], e[i]);
        return fail(VMFA_ERR_CUDA, "sort check failed");
      }
    }
  }
  if (items) CU(launch_items_scan(off, C, rows_per_item, 0, items, s));
  x->end(tok);
  return VMFA_OK;
}

int score_grid() { return sm_count() * 8; }
constexpr size_t kImageBudget = size_t(16) << 30;  // scorer B stage images (bytes)
constexpr size_t kImageFreeBudget = size_t(64) << 30;  // image-free stages: small + one-component images

// the compute stream waits for a pending asynchronous row upload (first X consumer)
cudaError_t wait_x(vmfa_ctx* x) {
  if (!x->x_pending) return cudaSuccess;
  x->x_pending = false;
  return cudaStreamWaitEvent(x->stream, x->x_ready, 0);
}

cudaError_t run_score(vmfa_ctx* x, int mode, const ScoreArgs& a) {
  if (cudaError_t e = wait_x(x); e != cudaSuccess) return e;
  if (x->scorer == 2) {
    if (cudaError_t e = cudaMemsetAsync(x->fix_cnt, 0, 2 * sizeof(unsigned long long), x->stream); e != cudaSuccess)
      return e;
    return launch_score_ws(mode, a,
                           WsOperands{x->xmax, x->mumax, x->mu32, x->brec, x->srec, x->bimg, x->bscl, x->simg, x->sscl,
                                      x->fix_list, x->fix_cnt, x->fix_cap, x->limg},
                           x->jobs, x->stream);
  }
  if (x->scorer == 1) return launch_score_tc(mode, a, x->WT, x->ipsi32, x->mu32, x->stream);
  return launch_score(mode, a, score_grid(), x->stream);
}

FixArgs fix_args(vmfa_ctx* x) {
  return FixArgs{x->X,       x->mu,      x->psi,         x->lam,  x->R,       x->kconst, x->fix_list, x->fix_cnt,
                 x->fix_cap, x->nfix,    x->fix_qkey,    x->fix_sorted, x->fix_qcnt, x->fix_qoff, x->fix_qfill,
                 x->fix_iof, x->fix_ovf, x->W64};
}

ScoreArgs score_args(vmfa_ctx* x) {
  ScoreArgs a{};
  a.dm = x->dm;
  a.L = x->L;
  a.X = x->X;
  a.P = x->P;
  a.kconst = x->kconst;
  a.g = x->g;
  a.gcnt = x->gcnt;
  return a;
}

// The scores the last scoring launch flagged (their terms cancel, see
// vmfa_fixup.cu): grouped by component and re-scored by the one-component
// tensor pass (rows centred on the candidate itself: no anchor expansion),
// then what is still flagged (a collapsed component's own Woodbury
// cancellation) is re-evaluated in fp64. All counts stay on the device (the
// iteration graph replays it); list overflows fall back to scanning kernels.
int rescore(vmfa_ctx* x, int mode, float* out) {
  if (!x->fix_ok) return VMFA_OK;
  const Dims& dm = x->dm;
  cudaStream_t s = x->stream;
  const int tf = x->begin(kFamFixup, 0);
  const FixArgs f = fix_args(x);
  CU(launch_fix_ovf(f, 1, s));
  if (x->fix_tc) {
    CU(launch_fix_group(dm, f, mode, x->K, x->g, x->rx, s));
    ScoreArgs a = score_args(x);
    a.off = x->fix_qoff;
    a.ent = x->fix_sorted;
    a.itemoff = x->fix_iof;
    a.out = out;
    a.list_div = mode == kModeTruncF ? dm.Cp : dm.SL;
    CU(run_score(x, kModeList, a));
    CU(launch_fix_ovf(f, 0, s));
  }
  CU(launch_fix_f64(dm, f, mode, x->K, x->g, x->rx, out, s));
  if (mode == kModeAnchor)
    CU(launch_fix_scan_anchor(dm, f, x->g, x->gcnt, x->kinv_off, x->kinv_ent, out, s));
  else if (mode == kModeExtra)
    CU(launch_fix_scan_single(dm, f, x->ex_off, x->ex_ent, dm.SL, dm.Cp * dm.G, out, s));
  else
    CU(launch_fix_scan_single(dm, f, x->kinv_off, x->kinv_ent, 0, dm.Cp, out, s));
  x->end(tf);
  return VMFA_OK;
}

int run_precompute(vmfa_ctx* x, int* failed, bool sync = true) {
  cudaStream_t s = x->stream;
  CU(cudaMemsetAsync(x->st_model, 0xff, sizeof(unsigned long long), s));
  PrecompArgs a{};
  a.dm = x->dm;
  a.L = x->L;
  a.pi = x->pi;
  a.mu = x->mu;
  a.lam = x->lam;
  a.psi = x->psi;
  a.Lmat = x->Lmat;
  a.R = x->R;
  a.Sz = x->Sz;
  a.logdet = x->logdet;
  a.logpi = x->logpi;
  a.kconst = x->kconst;
  a.P = x->scorer == 0 ? x->P : nullptr;  // (the FFMA scorer's packed rows)
  a.V32 = x->V32;
  a.mu32 = x->mu32;
  a.WT = x->WT;
  a.ipsi32 = x->ipsi32;
  a.Hp = x->Hp;
  a.status = x->st_model;
  a.W64 = x->W64;
  const int tok = x->begin(kFamPrecompute, x->dm.C);
  CU(launch_precompute(a, s));
  if (x->scorer == 2) {
    CU(launch_ws_images(x->dm, 1, x->WT, x->mu32, x->ipsi32, x->g, x->gcnt, x->simg, x->sscl, s));
    CU(launch_ws_records(x->dm, 1, x->WT, x->mu32, x->ipsi32, x->kconst, x->g, x->gcnt, x->sscl, x->srec, s, 0,
                         x->logpi, x->logdet));
    CU(launch_rowmax(x->dm.C, x->dm.D, x->mu32, x->mumax, s));
  }
  if (x->svimg) CU(launch_stats_vimg(x->dm, x->V32, x->svimg, x->svexp, x->svl1, s));
  x->end(tok);
  if (!sync) return VMFA_OK;  // the caller checks st_model later
  unsigned long long st = 0;
  CU(cudaMemcpyAsync(&st, x->st_model, sizeof st, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (st != ~0ull) {
    const int comp = static_cast<int>(st >> 8), code = static_cast<int>(st & 0xff);
    if (failed) *failed = comp;
    return fail(code, "L_c not positive definite for component %d", comp);
  }
  return VMFA_OK;
}

int ensure_kinv_current(vmfa_ctx* x) {
  if (x->kinv_for_current_K) return VMFA_OK;
  const Dims& dm = x->dm;
  TRY(csr_by_key(x, reinterpret_cast<const unsigned*>(x->K), dm.N * dm.Cp, x->kinv_off, x->kinv_ent, x->kinv_items,
                 x->score_rows));
  x->kinv_for_current_K = true;
  return VMFA_OK;
}

// Block 1's anchor pass: log-joints of every (n, c in U_{a in K(n)} g_a) into
// the LJ slots, under the current K, g and parameters.
int score_anchors(vmfa_ctx* x) {
  const Dims& dm = x->dm;
  cudaStream_t s = x->stream;
  TRY(ensure_kinv_current(x));
  if (x->scorer == 2) {
    const int tok = x->begin(kFamOther, dm.C);
    CU(launch_ws_images(dm, 0, x->WT, x->mu32, x->ipsi32, x->g, x->gcnt, x->bimg, x->bscl, s, x->sscl, x->brec,
                        x->limg));
    CU(launch_ws_records(dm, 0, x->WT, x->mu32, x->ipsi32, x->kconst, x->g, x->gcnt, x->bscl, x->brec, s, 1,
                         x->logpi, x->logdet));
    x->end(tok);
  }
  ScoreArgs a = score_args(x);
  a.off = x->kinv_off;
  a.ent = x->kinv_ent;
  a.itemoff = x->kinv_items;
  a.out = x->LJ;
  const int tok = x->begin(kFamScoreAnchor, dm.N * dm.Cp);
  CU(run_score(x, kModeAnchor, a));
  x->end(tok);
  TRY(rescore(x, kModeAnchor, x->LJ));
  return VMFA_OK;
}

// Sparse co-occurrence lists: every block-3 item appends its exact partial
// table (items of up to 512 points, all of them adding into the list). Set up
// at creation with VMFA_COOC=sparse, else on the first multi-rank E-step of a
// context without the dense rows. Capacity N (S - 1) entries (a random
// initial state gives nearly distinct candidates), bounded by 16 GB at 60 B
// per entry; overflow is reported, never silent.
int enable_lists(vmfa_ctx* x) {
  if (x->sparse) return VMFA_OK;
  const Dims& dm = x->dm;
  const int64_t N = dm.N;
  const int64_t bal = std::max<int64_t>(128, N / (4 * sm_count()));
  x->cl_kb = bits_for(static_cast<unsigned>(dm.C));
  if (2 * x->cl_kb > 32) return fail(VMFA_ERR_UNSUPPORTED, "sparse co-occurrence keys need C < 65536");
  const int64_t budget = (int64_t{16} << 30) / 60;
  x->cl_cap = std::max<int64_t>(int64_t{1} << 20, std::min<int64_t>(N * (dm.stride - 1), budget));
  const size_t L = static_cast<size_t>(x->cl_cap);
  int r = VMFA_OK;
  auto A = [&](auto*& p, size_t n) {
    if (r == VMFA_OK) r = x->alloc(p, n);
  };
  A(x->cl_key, L);
  A(x->cl_skey, L);
  A(x->cu_key, L);
  A(x->cl_cnt, L);
  A(x->cl_hi, L);
  A(x->cl_lo, L);
  A(x->cu_cnt, L);
  A(x->cu_hi, L);
  A(x->cu_lo, L);
  A(x->cl_iota, L);
  A(x->cl_perm, L);
  A(x->cu_off, static_cast<size_t>(dm.C) + 1);
  A(x->cl_n, 1);
  A(x->cl_ovf, 1);
  A(x->cl_hist, static_cast<size_t>(sort_hist_ints(x->cl_cap)));
  if (r != VMFA_OK) return r;
  x->gupd_pts = static_cast<int>(std::min<int64_t>(bal, 512));
  x->sparse = true;
  return VMFA_OK;
}

// Sparse co-occurrence: reduce the n raw entries in cl_* (sorted by key,
// exact sums per unique key) into cu_* and the per-component offsets cu_off.
int cooc_reduce(vmfa_ctx* x, int64_t n) {
  cudaStream_t s = x->stream;
  if (n > x->cl_cap) return fail(VMFA_ERR_UNSUPPORTED, "co-occurrence list of %lld entries exceeds its capacity %lld",
                                 static_cast<long long>(n), static_cast<long long>(x->cl_cap));
  // (cu_key and cl_iota are free until the reduction: the sort's scratch)
  CU(radix_sort_pairs(x->cl_key, nullptr, n, 2 * x->cl_kb, x->cu_key, x->cl_iota, x->cl_skey, x->cl_perm, x->cl_hist, s));
  CoocArgs a{};
  a.dm = x->dm;
  a.kb = x->cl_kb;
  a.key = x->cl_skey;
  a.perm = x->cl_perm;
  a.cnt = x->cl_cnt;
  a.hi = x->cl_hi;
  a.lo = x->cl_lo;
  a.n = static_cast<int>(n);
  a.head = x->cl_iota;  // reused: heads, then their inclusive scan
  a.u_key = x->cu_key;
  a.u_cnt = x->cu_cnt;
  a.u_hi = x->cu_hi;
  a.u_lo = x->cu_lo;
  a.u_off = x->cu_off;
  CU(launch_cooc_heads(a, s));
  if (n > 0) CU(scan_i32(x->cl_iota, x->cl_iota, n, true, x->cl_hist, s));
  for (long long* q : {x->cu_cnt, x->cu_hi, x->cu_lo})
    CU(cudaMemsetAsync(q, 0, static_cast<size_t>(std::max<int64_t>(n, 1)) * sizeof(long long), s));
  CU(launch_cooc_sums(a, s));
  int un = 0;
  if (n > 0) CU(cudaMemcpyAsync(&un, x->cl_iota + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  x->cu_n = un;
  return VMFA_OK;
}
CoocArgs cooc_args(vmfa_ctx* x) {
  CoocArgs a{};
  a.dm = x->dm;
  a.kb = x->cl_kb;
  a.u_key = x->cu_key;
  a.u_cnt = x->cu_cnt;
  a.u_hi = x->cu_hi;
  a.u_lo = x->cu_lo;
  a.u_off = x->cu_off;
  return a;
}
// entries appended by the last k_gupdate (host read; overflow is an error)
int cooc_count(vmfa_ctx* x, int64_t* n) {
  unsigned long long c = 0;
  int ovf = 0;
  CU(cudaMemcpyAsync(&c, x->cl_n, sizeof c, cudaMemcpyDeviceToHost, x->stream));
  CU(cudaMemcpyAsync(&ovf, x->cl_ovf, sizeof ovf, cudaMemcpyDeviceToHost, x->stream));
  CU(cudaStreamSynchronize(x->stream));
  if (ovf || static_cast<long long>(c) > x->cl_cap)
    return fail(VMFA_ERR_UNSUPPORTED, "co-occurrence list overflow (%llu entries, capacity %lld)", c,
                static_cast<long long>(x->cl_cap));
  *n = static_cast<int64_t>(c);
  return VMFA_OK;
}

// E-step blocks 1, 2, 4 and the local part of block 3.
int estep_local(vmfa_ctx* x, uint64_t seed, uint64_t it, int mode, bool exchange, bool defer_g = false) {
  const Dims& dm = x->dm;
  cudaStream_t s = x->stream;
  CU(cudaMemsetAsync(x->st_select, 0, sizeof(int), s));
  const bool prescored = x->prescored;
  x->prescored = false;
  // anchor blocks: inverted K (stable counting sort by component)
  if (!prescored) TRY(ensure_kinv_current(x));
  // extras not already covered by U g_a
  {
    const int tok = x->begin(kFamOther, dm.N);
    if (!x->capturing) {  // (a captured iteration gets them from vmfa_iterate, outside the graph)
      const unsigned long long sit[2] = {seed, it};
      CU(cudaMemcpyAsync(x->sit, sit, sizeof sit, cudaMemcpyHostToDevice, s));  // pageable: staged
    }
    CU(launch_extra(dm, x->K, x->g, x->gcnt, x->sit, x->rx, x->rkey, s));
    x->end(tok);
  }
  TRY(csr_by_key(x, x->rkey, dm.N, x->ex_off, x->ex_ent, x->ex_items, x->score_rows));
  // block 1: scoring (the anchor pass unless it ran ahead with the last F)
  if (!prescored) TRY(score_anchors(x));
  {
    ScoreArgs a = score_args(x);
    a.out = x->LJ;
    a.off = x->ex_off;
    a.ent = x->ex_ent;
    a.itemoff = x->ex_items;
    const int tok2 = x->begin(kFamScoreExtra, dm.N);
    CU(run_score(x, kModeExtra, a));
    x->end(tok2);
    TRY(rescore(x, kModeExtra, x->LJ));
  }
  // selection, labels, block 4
  {
    SelectArgs a{};
    a.dm = dm;
    a.K = x->K;
    a.g = x->g;
    a.gcnt = x->gcnt;
    a.rx = x->rx;
    a.LJ = x->LJ;
    a.labels = x->labels;
    a.lablj = x->lablj;
    a.resp = x->resp;
    a.ret_cnt = x->ret_cnt;
    a.ret_idx = x->ret_idx;
    a.ret_lj = x->ret_lj;
    a.lse = x->lse;
    a.status = x->st_select;
    const int tok = x->begin(kFamSelect, dm.N);
    CU(launch_select(a, s));
    x->end(tok);
  }
  x->kinv_for_current_K = false;
  // block 2: partition by label (stable => ascending n per component)
  TRY(csr_by_key(x, reinterpret_cast<const unsigned*>(x->labels), dm.N, x->part_off, x->part_ent, nullptr, 1));
  CU(launch_items_scan(x->part_off, dm.C, x->gupd_pts, 1, x->part_items, s));
  // block 3 (local accumulation; selection unless exchanging)
  CU(launch_logpi(x->pi, dm.C, x->logpi_g, s));
  {
    GupdArgs a{};
    a.dm = dm;
    a.mode = mode;
    a.part_off = x->part_off;
    a.part_ent = x->part_ent;
    a.ret_cnt = x->ret_cnt;
    a.ret_idx = x->ret_idx;
    a.ret_lj = x->ret_lj;
    a.lablj = x->lablj;
    a.logpi = x->logpi_g;
    a.g_new = x->g_new;
    a.gcnt_new = x->gcnt_new;
    a.gt_cnt = x->gt_cnt;
    a.gt_hi = x->gt_hi;
    a.gt_lo = x->gt_lo;
    a.itemoff = x->part_items;
    a.pts_per_item = x->gupd_pts;
    a.exchange = exchange ? 1 : 0;
    // (a dense shared-memory table holds every key for C <= kGupdDenseMax)
    a.force_rows = ((x->xc && dm.C - 1 > kGupdCap / 2 && dm.C > kGupdDenseMax) || x->sparse) ? 1 : 0;
    a.xc = x->xc;
    if (x->sparse) {
      a.list = 1;
      a.cl_key = x->cl_key;
      a.cl_cnt = x->cl_cnt;
      a.cl_hi = x->cl_hi;
      a.cl_lo = x->cl_lo;
      a.cl_n = x->cl_n;
      a.cl_cap = x->cl_cap;
      a.cl_kb = x->cl_kb;
      a.cl_ovf = x->cl_ovf;
      CU(cudaMemsetAsync(x->cl_n, 0, sizeof(unsigned long long), s));
      CU(cudaMemsetAsync(x->cl_ovf, 0, sizeof(int), s));
    }
    a.dump = x->dump ? 1 : 0;
    if (x->dump) {
      CU(cudaMemsetAsync(x->dump_n, 0, sizeof(unsigned long long), s));
      a.dump_c = x->dump_c;
      a.dump_ct = x->dump_ct;
      a.dump_cnt = x->dump_cnt;
      a.dump_hi = x->dump_hi;
      a.dump_lo = x->dump_lo;
      a.dump_n = x->dump_n;
      a.dump_cap = x->dump_cap;
    }
    // (vmfa_iterate: launched by launch_deferred_gupdate on the side stream)
    x->g_deferred = defer_g && !exchange && !x->sparse && !x->dump && !x->profile;
    if (x->g_deferred) x->g_args = a;
    const int tok = x->g_deferred ? -1 : x->begin(kFamGupdate, dm.N);
    if (!x->g_deferred) CU(launch_gupdate(a, x->gupd_grid, s));
    if (!x->g_deferred && !exchange && x->xc)
      CU(launch_gselect_dense(dm, x->xc, x->part_items, a.force_rows, x->g_new, x->gcnt_new, s));
    if (x->sparse) {
      // the rank-local list reduced by key (sent as it is in exchange mode);
      // single context: every component's g from it
      int64_t n = 0;
      TRY(cooc_count(x, &n));
      TRY(cooc_reduce(x, n));
      if (!exchange) CU(launch_cooc_select(cooc_args(x), 0, dm.C, 0, x->g_new, x->gcnt_new, s));
    }
    if (!x->g_deferred) x->end(tok);
  }
  // scalars: F_estep = sum lse, joints = sum ret_cnt
  CU(launch_sum_f64(x->lse, dm.N, x->partials, x->scal + 0, s));
  CU(launch_sum_i32(x->ret_cnt, dm.N, x->u64tmp, s));
  k_pack_scalar_u64<<<1, 1, 0, s>>>(x->u64tmp, x->scal + 1);
  CU(cudaGetLastError());
  x->have_estep = true;
  return VMFA_OK;
}

int estep_finish(vmfa_ctx* x, bool exchange, bool sync = true) {
  const Dims& dm = x->dm;
  cudaStream_t s = x->stream;
  if (exchange && !x->sparse) {
    const int tok = x->begin(kFamGupdate, dm.C);
    CU(launch_gselect_dense(dm, x->xc, x->part_items, 1, x->g_new, x->gcnt_new, s));
    x->end(tok);
  }
  std::swap(x->g, x->g_new);
  std::swap(x->gcnt, x->gcnt_new);
  if (!sync) return VMFA_OK;  // the caller checks st_select later
  int flag = 0;
  CU(cudaMemcpyAsync(&flag, x->st_select, sizeof(int), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (flag) return fail(VMFA_ERR_INSUFFICIENT_CANDIDATES, "search space smaller than C'");
  return VMFA_OK;
}

// Block 3 of a deferred E-step (estep_local with defer_g) on the side stream:
// it depends on the selection and the label partition only, so it runs next
// to the K inversion, the statistics, update_params and precompute;
// join_gupdate orders it before the first
// reader of the new g (the anchor images of the next scoring pass).
int launch_deferred_gupdate(vmfa_ctx* x) {
  if (!x->g_deferred) return VMFA_OK;
  x->g_deferred = false;
  const GupdArgs& a = x->g_args;
  CU(cudaEventRecord(x->g_fork, x->stream));
  CU(cudaStreamWaitEvent(x->gstream, x->g_fork, 0));
  CU(launch_gupdate(a, x->gupd_grid, x->gstream));
  if (x->xc) CU(launch_gselect_dense(x->dm, x->xc, x->part_items, a.force_rows, a.g_new, a.gcnt_new, x->gstream));
  CU(cudaEventRecord(x->g_join, x->gstream));
  x->g_join_pending = true;
  return VMFA_OK;
}
int join_gupdate(vmfa_ctx* x) {
  if (!x->g_join_pending) return VMFA_OK;
  x->g_join_pending = false;
  CU(cudaStreamWaitEvent(x->stream, x->g_join, 0));
  return VMFA_OK;
}

int stats_local(vmfa_ctx* x) {
  if (!x->have_estep) return fail(VMFA_ERR_INVALID_ARGUMENT, "accumulate_suffstats needs a preceding E-step (responsibilities)");
  TRY(ensure_kinv_current(x));
  CU(wait_x(x));
  StatsArgs a{};
  a.dm = x->dm;
  a.X = x->X;
  a.resp = x->resp;
  a.off = x->kinv_off;
  a.ent = x->kinv_ent;
  a.V32 = x->V32;
  a.mu32 = x->mu32;
  a.Sz = x->Sz;
  a.Nc = x->Nc;
  a.E = x->E;
  a.Y = x->Y;
  a.sq = x->sq;
  a.qctr = x->qctr;
  a.xmax = x->xmax;  // (the tcgen05 kernel's row scales; null without the warp-specialised scorer)
  a.mumax = x->mumax;
  a.vimg = x->svimg;
  a.vexp = x->svexp;
  a.vl1 = x->svl1;
  a.zbuf = x->szbuf;
  const int tok = x->begin(kFamStats, x->dm.N * x->dm.Cp);
  CU(launch_items_scan(x->kinv_off, x->dm.C, x->stats_rows, 0, x->stats_items, x->stream));
  CU(launch_stats(a, x->stats_items, x->stats_rows, x->stats_part, x->stream));
  x->end(tok);
  return VMFA_OK;
}

// update_params into the "next" buffers; status in st_update (~0 = success)
int launch_update_params(vmfa_ctx* x) {
  x->prescored = false;  // parameters change
  const Dims& dm = x->dm;
  cudaStream_t s = x->stream;
  CU(cudaMemsetAsync(x->st_update, 0xff, sizeof(unsigned long long), s));
  UpdateArgs a{};
  a.dm = dm;
  a.Nc = x->Nc;
  a.E = x->E;
  a.Y = x->Y;
  a.sq = x->sq;
  a.floor = x->floor;
  a.mu_prev = x->mu;
  a.lam_prev = x->lam;
  a.psi_prev = x->psi;
  a.pi = x->pi2;
  a.mu = x->mu2;
  a.lam = x->lam2;
  a.psi = x->psi2;
  a.status = x->st_update;
  const int tok = x->begin(kFamUpdate, dm.C);
  CU(launch_update(a, s));
  CU(launch_renorm(dm, x->pi2, x->st_update, s));
  x->end(tok);
  return VMFA_OK;
}
void swap_params(vmfa_ctx* x) {
  std::swap(x->pi, x->pi2);
  std::swap(x->mu, x->mu2);
  std::swap(x->lam, x->lam2);
  std::swap(x->psi, x->psi2);
}
int update_status(unsigned long long st, int* failed) {
  const int comp = static_cast<int>(st >> 8), code = static_cast<int>(st & 0xff);
  if (failed) *failed = comp == 0xffffff ? -1 : comp;
  return fail(code, comp == 0xffffff ? "all components empty after update" : "E_c singular for component %d", comp);
}

int update_and_precompute(vmfa_ctx* x, int* failed) {
  x->prescored = false;  // parameters change
  const Dims& dm = x->dm;
  cudaStream_t s = x->stream;
  CU(cudaMemsetAsync(x->st_model, 0xff, sizeof(unsigned long long), s));
  UpdateArgs a{};
  a.dm = dm;
  a.Nc = x->Nc;
  a.E = x->E;
  a.Y = x->Y;
  a.sq = x->sq;
  a.floor = x->floor;
  a.mu_prev = x->mu;
  a.lam_prev = x->lam;
  a.psi_prev = x->psi;
  a.pi = x->pi2;
  a.mu = x->mu2;
  a.lam = x->lam2;
  a.psi = x->psi2;
  a.status = x->st_model;
  const int tok = x->begin(kFamUpdate, dm.C);
  CU(launch_update(a, s));
  CU(launch_renorm(dm, x->pi2, x->st_model, s));
  x->end(tok);
  unsigned long long st = 0;
  CU(cudaMemcpyAsync(&st, x->st_model, sizeof st, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (st != ~0ull) {
    const int comp = static_cast<int>(st >> 8), code = static_cast<int>(st & 0xff);
    if (failed) *failed = comp == 0xffffff ? -1 : comp;
    return fail(code, comp == 0xffffff ? "all components empty after update"
                                       : "E_c singular for component %d", comp);
  }
  std::swap(x->pi, x->pi2);
  std::swap(x->mu, x->mu2);
  std::swap(x->lam, x->lam2);
  std::swap(x->psi, x->psi2);
  return run_precompute(x, failed);
}

// truncated_free_energy (model.cpp:150-159) under the current parameters.
// lookahead: run the next E-step's anchor pass now (it needs exactly these K,
// g and parameters, and scores every (n, c in K(n)) -- anchor c scores itself
// with the one-component arithmetic) and read F from its self slots; the next
// estep_local then skips that pass. Otherwise one-component jobs over K.
int free_energy_local(vmfa_ctx* x, bool lookahead) {
  const Dims& dm = x->dm;
  cudaStream_t s = x->stream;
  if (lookahead) {
    TRY(score_anchors(x));
    const int tok = x->begin(kFamScoreTruncF, dm.N * dm.Cp);
    CU(launch_self_slots(dm, x->K, x->g, x->gcnt, x->LJ, x->LJK, s));
    CU(launch_lse_rows(x->LJK, dm.N, dm.Cp, x->lse, s));
    x->end(tok);
    x->prescored = true;
  } else {
    TRY(ensure_kinv_current(x));
    ScoreArgs a = score_args(x);
    a.off = x->kinv_off;
    a.ent = x->kinv_ent;
    a.itemoff = x->kinv_items;
    a.out = x->LJK;
    const int tok = x->begin(kFamScoreTruncF, dm.N * dm.Cp);
    CU(run_score(x, kModeTruncF, a));
    TRY(rescore(x, kModeTruncF, x->LJK));
    CU(launch_lse_rows(x->LJK, dm.N, dm.Cp, x->lse, s));
    x->end(tok);
  }
  CU(launch_sum_f64(x->lse, dm.N, x->partials, x->scal + 2, s));
  return VMFA_OK;
}

int read_scalars(vmfa_ctx* x, double out[4]) {
  CU(cudaMemcpyAsync(out, x->scal, 4 * sizeof(double), cudaMemcpyDeviceToHost, x->stream));
  CU(cudaStreamSynchronize(x->stream));
  return VMFA_OK;
}

int check_ctx(const vmfa_ctx* x) {
  if (!x) return fail(VMFA_ERR_INVALID_ARGUMENT, "null context");
  return VMFA_OK;
}

}  // namespace
}  // namespace vmfa_b200

// ============================================================================ C-ABI
constexpr int kStatsMaxRowsHost = 1024;  // K-pairs per statistics item (kernels: kStatsMaxRows)

// ---- dense pass helpers (exact_log_likelihood, em_full_step)
// rows per dense chunk (<= 1 GiB of log-joints) and the dense buffers
int ensure_dense(vmfa_ctx* x, int64_t* Rout) {
  const Dims& dm = x->dm;
  const int C = dm.C, G = dm.G;
  const int nb = (C + G - 1) / G;
  const int SL = nb * G;
  int64_t R = std::max<int64_t>(128, (int64_t(1) << 30) / (4 * static_cast<int64_t>(SL)));
  R = std::min<int64_t>(R, (std::numeric_limits<int>::max() - nb) / nb);  // flat entries n * nb + b
  R = std::min<int64_t>(R, dm.N);
  if (!x->dense_g) {
    TRY(x->alloc(x->dense_g, static_cast<size_t>(C) * G));
    TRY(x->alloc(x->dense_gcnt, C));
    TRY(x->alloc(x->dense_items, C + 1));
    TRY(x->alloc(x->dense_off, C + 1));
    TRY(x->alloc(x->dense_ent, static_cast<size_t>(nb) * R));
    TRY(x->alloc(x->dense_jobs, static_cast<size_t>(dense_jobs(nb, static_cast<int>(R)))));
    TRY(x->alloc(x->dense_LJ, static_cast<size_t>(R) * SL));
    TRY(x->alloc(x->dense_lse, dm.N));
    TRY(x->alloc(x->dense_out, 1));
    x->dense_R = R;
    x->dense_SL = SL;
  }
  *Rout = std::min<int64_t>(R, x->dense_R);
  return VMFA_OK;
}
// pseudo-anchor blocks of G components and their scorer images
int dense_prepare(vmfa_ctx* x) {
  const Dims& dm = x->dm;
  cudaStream_t s = x->stream;
  CU(launch_dense_groups(dm.C, dm.G, x->dense_g, x->dense_gcnt, s));
  if (x->scorer == 2) {
    CU(launch_ws_images(dm, 0, x->WT, x->mu32, x->ipsi32, x->dense_g, x->dense_gcnt, x->bimg, x->bscl, s,
                        x->sscl, nullptr, x->ifree_only ? x->limg : nullptr));
    CU(launch_ws_records(dm, 0, x->WT, x->mu32, x->ipsi32, x->kconst, x->dense_g, x->dense_gcnt, x->bscl, x->brec,
                         s, 0, x->logpi, x->logdet));
  }
  return VMFA_OK;
}
// log-joints of rows [r0, r0 + Rc) against every component into dense_LJ
// (row stride dense_SL, slot c = component c) and their LSE into dense_lse
int dense_chunk(vmfa_ctx* x, int64_t r0, int Rc) {
  const Dims& dm = x->dm;
  const int C = dm.C, G = dm.G, D = dm.D;
  const int nb = (C + G - 1) / G;
  const int SL = x->dense_SL;
  cudaStream_t s = x->stream;
  const bool ws = x->scorer == 2;
  {
    CU(launch_dense_chunk(C, G, nb, Rc, x->dense_ent, x->dense_jobs, x->dense_items, s));
    Dims dd = dm;
    dd.N = Rc;
    dd.Cp = nb;
    dd.SL = SL;
    ScoreArgs a = score_args(x);
    a.dm = dd;
    a.X = x->X + r0 * D;
    a.off = nullptr;
    a.ent = x->dense_ent;
    a.itemoff = x->dense_items;
    a.g = x->dense_g;
    a.gcnt = x->dense_gcnt;
    a.out = x->dense_LJ;
    CU(wait_x(x));
    if (ws) {
      WsOperands op{x->xmax + r0, x->mumax, x->mu32, x->brec, x->srec, x->bimg, x->bscl, x->simg, x->sscl};
      if (x->ifree_only) op.limg = x->limg;
      CU(launch_score_ws(kModeAnchor, a, op, x->dense_jobs, s, false));
    } else {  // single-role scorers (shapes the warp-specialised one does not take): CSR items
      CU(launch_dense_csr(C, G, Rc, x->score_rows, x->dense_off, x->dense_items, s));
      a.off = x->dense_off;
      CU(run_score(x, kModeAnchor, a));
    }
    CU(launch_lse_dense(x->dense_LJ, Rc, SL, C, x->dense_lse + r0, s));
  }
  return VMFA_OK;
}

extern "C" {

int vmfa_abi_version(void) { return VMFA_ABI_VERSION; }
const char* vmfa_last_error(void) { return error_text().c_str(); }

int vmfa_device_available(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) {
    cudaGetLastError();
    return 0;
  }
  cudaDeviceProp p{};
  if (cudaGetDeviceProperties(&p, 0) != cudaSuccess) return 0;
  return p.major == 10 ? 1 : 0;
}

int vmfa_ctx_create(vmfa_ctx** out, int device, int C, int D, int H, int Cp, int G, int64_t n_local,
                    int64_t n_offset, int64_t n_total, void* stream) {
  if (!out) return fail(VMFA_ERR_INVALID_ARGUMENT, "out is null");
  *out = nullptr;
  if (C < 1 || D < 1 || H < 1 || H > D || Cp < 1 || Cp > C || G < 1 || G > C || n_local < 1 ||
      n_offset < 0 || n_total < n_offset + n_local)
    return fail(VMFA_ERR_INVALID_ARGUMENT, "invalid sizes (C=%d D=%d H=%d C'=%d G=%d N=%lld)", C, D, H, Cp, G,
                static_cast<long long>(n_local));
  if (H + 1 > 65) return fail(VMFA_ERR_UNSUPPORTED, "H > 64 not supported by this build");
  if (Cp > 8 || Cp * G + 1 > 256) return fail(VMFA_ERR_UNSUPPORTED, "C' <= 8 and C'G+1 <= 256 required");
  // the g-selection kernels hold the G-1 picks and the output row in fixed
  // 64-entry arrays (k_gupdate, k_gselect_dense, k_cooc_select)
  if (G > 64) return fail(VMFA_ERR_UNSUPPORTED, "G <= 64 required by this build");
  if (n_local * Cp >= (int64_t{1} << 31)) return fail(VMFA_ERR_UNSUPPORTED, "shard too large (N*C' >= 2^31)");
  if (!vmfa_device_available()) return fail(VMFA_ERR_NO_DEVICE, "no sm_100 CUDA device visible");
  CU(cudaSetDevice(device));
  auto* x = new vmfa_ctx();
  x->device = device;
  Dims& dm = x->dm;
  dm.C = C, dm.D = D, dm.H = H, dm.Cp = Cp, dm.G = G;
  dm.SL = Cp * G + 1;
  dm.stride = static_cast<int>(std::min<int64_t>(static_cast<int64_t>(Cp) * G + 1, C));
  dm.N = n_local, dm.n0 = n_offset, dm.Ntot = n_total;
  x->L = score_layout(H);
  x->Hp = ws_hp(H);
  {
    const char* la = std::getenv("VMFA_LOOKAHEAD");
    x->lookahead = !(la && la[0] == '0');
    const char* sc = std::getenv("VMFA_SCORER");
    const std::string v = sc ? sc : "ws";
    x->scorer = v == "ffma" ? 0 : (v == "tc" ? 1 : 2);
    if (x->scorer == 2 && !score_ws_supported(x->dm)) x->scorer = 1;
    // the warp-specialised scorer streams prebuilt B stage images: fall back
    // to the single-role tensor scorer when they exceed the memory budget
    if (x->scorer == 2 &&
        static_cast<size_t>(ws_image_halves(x->dm, 0) + ws_image_halves(x->dm, 1)) * 2 > kImageBudget) {
      // ... unless the image-free anchor stages fit (small per-anchor lin / psi
      // images + the one-component images; config 5: ~50 GB instead of ~200)
      const size_t free_bytes =
          static_cast<size_t>(ws_small_image_halves(x->dm) + ws_image_halves(x->dm, 1)) * 2;
      if (ws_image_free_ok(x->dm) && free_bytes <= kImageFreeBudget) x->ifree_only = true;
      else x->scorer = 1;
    }
    // VMFA_IMAGE_FREE=2: the image-free route as if the full images did not fit (tests)
    if (x->scorer == 2 && ws_image_free_ok(x->dm) && std::getenv("VMFA_IMAGE_FREE") &&
        std::getenv("VMFA_IMAGE_FREE")[0] == '2')
      x->ifree_only = true;
    if (x->scorer == 1 && !score_tc_supported(x->dm)) x->scorer = 0;
    if (x->scorer == 0 && static_cast<size_t>(D) * kXsStride * sizeof(float) > 200 * 1024) {
      const size_t dmax = 200 * 1024 / (kXsStride * sizeof(float));
      delete x;
      return fail(VMFA_ERR_UNSUPPORTED, "D > %zu not supported by the FFMA scoring tile", dmax);
    }
    x->use_tc = x->scorer != 0;
    x->score_rows = x->use_tc ? kScoreRowsTc : kScoreRows;
  }
  if (stream) {
    x->stream = static_cast<cudaStream_t>(stream);
  } else {
    if (cudaStreamCreateWithFlags(&x->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete x;
      return fail(VMFA_ERR_CUDA, "cudaStreamCreate failed");
    }
    x->own_stream = true;
  }
  if (cudaStreamCreateWithFlags(&x->gstream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&x->g_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&x->g_join, cudaEventDisableTiming) != cudaSuccess) {
    vmfa_ctx_destroy(x);
    return fail(VMFA_ERR_CUDA, "side stream creation failed");
  }
  const size_t N = static_cast<size_t>(n_local), Cs = static_cast<size_t>(C);
  const size_t H1 = static_cast<size_t>(H) + 1;
  int r = VMFA_OK;
  auto A = [&](auto*& p, size_t n) {
    if (r == VMFA_OK) r = x->alloc(p, n);
  };
  const char* cooc_env = std::getenv("VMFA_COOC");
  const bool force_sparse = cooc_env && std::string(cooc_env) == "sparse";
  // dense C x C co-occurrence rows (24 C^2 B): one context up to C ~ 18 900;
  // a shard of a multi-rank run only up to C = 4096 (the rows are the
  // all-reduce payload: 0.4 GB at C = 4096), beyond that the owner-routed
  // sparse lists
  const bool sharded = n_total > n_local;
  const bool dense_rows = !force_sparse && 3.0 * Cs * Cs * sizeof(long long) <= 8.0 * (1ull << 30) &&
                          (!sharded || C <= 4096);
  A(x->X, N * D);
  A(x->floor, D);
  for (double** p : {&x->pi, &x->pi2}) A(*p, Cs);
  for (double** p : {&x->mu, &x->mu2, &x->psi, &x->psi2}) A(*p, Cs * D);
  for (double** p : {&x->lam, &x->lam2}) A(*p, Cs * D * H);
  A(x->Lmat, Cs * H * H);
  A(x->R, Cs * H * H);
  A(x->Sz, Cs * H * H);
  A(x->logdet, Cs);
  A(x->logpi, Cs);
  A(x->logpi_g, Cs);
  A(x->kconst, Cs);
  A(x->P, Cs * D * x->L.HP);
  A(x->V32, Cs * D * H);
  A(x->mu32, Cs * D);
  A(x->WT, Cs * x->Hp * D);
  if (x->scorer == 2) {
    // items <= sum_c ceil(rows_c / 128); the re-scoring lists hold <= fix_cap
    // entries: every slot of the anchor pass up to 2^26 (16 B per entry), so
    // that the scanning fallback (vmfa_fixup.cu, list overflow) stays rare --
    // config 2 flags ~1e6 scores per pass
    x->fix_cap = std::max<long long>(1 << 20, std::min<long long>(static_cast<long long>(N) * dm.SL, 1LL << 26));
    A(x->jobs, static_cast<size_t>(x->fix_cap) / 128 + Cs + 2);
    // image-free anchor stages: required when the full anchor images exceed
    // the budget (ifree_only: no bimg at all), else opt-in (VMFA_IMAGE_FREE=1);
    // the loader then assembles every stage from 3 + 2 G bulk copies, which
    // measured slower at config 3 (anchor pass 7.84 -> 9.66 ms) than one copy
    // of the prebuilt image
    if (!x->ifree_only) A(x->bimg, ws_image_halves(dm, 0));
    if (x->ifree_only ||
        (ws_image_free_ok(dm) && std::getenv("VMFA_IMAGE_FREE") && std::getenv("VMFA_IMAGE_FREE")[0] == '1'))
      A(x->limg, ws_small_image_halves(dm));
    A(x->simg, ws_image_halves(dm, 1));
    A(x->bscl, ws_scale_floats(dm, 0));
    A(x->brec, ws_record_floats(dm, 0));
    A(x->srec, ws_record_floats(dm, 1));
    A(x->sscl, ws_scale_floats(dm, 1));
    A(x->xmax, N);
    A(x->mumax, Cs);
  }
  A(x->ipsi32, Cs * D);
  A(x->nfix, 2);
  A(x->fix_cnt, 2);
  A(x->fix_ovf, 2);
  x->fix_ok = x->scorer == 2 && static_cast<int64_t>(N) * dm.SL < (int64_t{1} << 31);
  if (const char* v = std::getenv("VMFA_FIX_TC")) x->fix_tc = v[0] != '0';
  if (x->fix_ok && fix_dmma_ok(D, dm.H) && static_cast<int64_t>(Cs) * dm.H * D * 8 <= (int64_t{4} << 30))
    A(x->W64, static_cast<size_t>(Cs) * dm.H * D);
  A(x->fix_list, static_cast<size_t>(x->fix_cap));
  A(x->fix_sorted, static_cast<size_t>(x->fix_cap));
  A(x->fix_qkey, static_cast<size_t>(x->fix_cap));
  A(x->fix_qcnt, Cs);
  A(x->fix_qoff, Cs + 1);
  A(x->fix_qfill, Cs);
  A(x->fix_iof, Cs + 1);
  if (r == VMFA_OK) cudaMemsetAsync(x->nfix, 0, 2 * sizeof(unsigned long long), x->stream);
  A(x->K, N * Cp);
  // g and its counts contiguous ([C*G | C] int32), so the sparse exchange can
  // all-reduce a rank's selected rows as one buffer (VMFA_XCHG_G)
  A(x->g, Cs * G + Cs);
  A(x->g_new, Cs * G + Cs);
  if (r == VMFA_OK) {
    x->gcnt = x->g + Cs * G;
    x->gcnt_new = x->g_new + Cs * G;
  }
  A(x->labels, N);
  A(x->lablj, N);
  A(x->LJ, N * dm.SL);
  A(x->LJK, N * Cp);
  A(x->rx, N);
  A(x->rkey, N);
  A(x->ret_cnt, N);
  A(x->ret_idx, N * dm.stride);
  A(x->ret_lj, N * dm.stride);
  A(x->resp, N * Cp);
  A(x->lse, N);
  A(x->keys_alt, N * Cp);
  A(x->keys_tmp, N * Cp);
  A(x->vals, N * Cp);
  A(x->sort_hist, static_cast<size_t>(sort_hist_ints(static_cast<int64_t>(N * Cp))));
  A(x->kinv_off, Cs + 1);
  A(x->kinv_ent, N * Cp);
  A(x->kinv_items, Cs + 1);
  A(x->ex_off, Cs + 1);
  A(x->ex_ent, N);
  A(x->ex_items, Cs + 1);
  A(x->part_off, Cs + 1);
  A(x->part_ent, N);
  A(x->part_items, Cs + 1);
  A(x->sit, 2);
  A(x->stats_items, Cs + 1);
  A(x->qctr, 2);
  {
    const int64_t pairs = static_cast<int64_t>(N) * Cp;
    const int64_t target = (pairs + sm_count() * 8 - 1) / (sm_count() * 8);
    const int64_t cap = stats_rows_cap(dm);
    x->stats_rows = static_cast<int>(std::min<int64_t>(cap, std::max<int64_t>(256, (target + 31) / 32 * 32)));
    if (const char* v = std::getenv("VMFA_STATS_ROWS"))  // experiments: K-pairs per statistics item
      x->stats_rows = static_cast<int>(std::min<int64_t>(cap, std::max<int64_t>(32, std::atoll(v) / 32 * 32)));
    if (x->scorer == 2 && stats_use_tc(dm)) {  // the tcgen05 statistics kernel
      x->stats_rows = stats_tc_rows();
      A(x->svimg, static_cast<size_t>(stats_tc_image_bytes(dm)));
      A(x->svexp, Cs * 16);
      A(x->svl1, Cs * 16);
      A(x->szbuf, static_cast<size_t>(pairs) * H);
    }
    const int64_t max_items = C + (pairs + x->stats_rows - 1) / x->stats_rows;
    A(x->stats_part, static_cast<size_t>(max_items) * stats_part_stride(dm));
    const int64_t bal = std::max<int64_t>(128, static_cast<int64_t>(N) / (4 * sm_count()));
    // large C (with the dense rows): every item adds into the rows through a
    // small hash (k_gupdate force_rows); items of up to 512 points
    const int64_t capb = (C - 1 <= kGupdCap / 2 || C <= kGupdDenseMax) ? (int64_t{1} << 30) : 512;
    x->gupd_pts = static_cast<int>(std::min(bal, capb));
  }
  // dense C x C rows (count, fixed-point hi, lo) for split components and the
  // multi-rank exchange; without it (very large C) components are not split.
  if (dense_rows) {
    A(x->xc, 3 * Cs * Cs);
    if (r == VMFA_OK) cudaMemsetAsync(x->xc, 0, 3 * Cs * Cs * sizeof(long long), x->stream);
  } else {
    // single context without the dense rows: components are not split (the
    // per-CTA global tables below take the keys a shared-memory hash cannot);
    // the sparse lists are set up for the multi-rank exchange (enable_lists)
    x->gupd_pts = 1 << 30;
  }
  A(x->cnt, Cs + 1);
  A(x->chunks, Cs + 1);
  x->gupd_grid = sm_count() * 4;
  // per-CTA dense fallback tables: only needed without the dense C x C rows
  const size_t gt_n = dense_rows ? 1 : static_cast<size_t>(x->gupd_grid) * Cs;
  A(x->gt_cnt, gt_n);
  A(x->gt_hi, gt_n);
  A(x->gt_lo, gt_n);
  x->stats_len = Cs + Cs * H1 * H1 + Cs * H1 * D + Cs * D;
  A(x->stats, x->stats_len);
  A(x->partials, 512);
  A(x->scal, 4);
  A(x->u64tmp, 1);
  A(x->st_select, 1);
  A(x->st_model, 1);
  A(x->st_update, 1);
  A(x->n_empty, 1);
  if (r == VMFA_OK && cudaMallocHost(&x->hstat, sizeof(IterStatus)) != cudaSuccess)
    r = fail(VMFA_ERR_CUDA, "cudaMallocHost failed");
  if (r != VMFA_OK) {
    vmfa_ctx_destroy(x);
    return r;
  }
  x->Nc = x->stats;
  x->E = x->Nc + Cs;
  x->Y = x->E + Cs * H1 * H1;
  x->sq = x->Y + Cs * H1 * D;
  if (force_sparse && r == VMFA_OK) r = enable_lists(x);
  if (r != VMFA_OK) {
    vmfa_ctx_destroy(x);
    return r;
  }
  cudaMemsetAsync(x->scal, 0, 4 * sizeof(double), x->stream);
  cudaMemsetAsync(x->labels, 0, N * sizeof(int), x->stream);
  if (cudaStreamSynchronize(x->stream) != cudaSuccess) {
    vmfa_ctx_destroy(x);
    return fail(VMFA_ERR_CUDA, "context initialisation failed");
  }
  *out = x;
  return VMFA_OK;
}

int vmfa_ctx_destroy(vmfa_ctx* x) {
  if (!x) return VMFA_OK;
  cudaSetDevice(x->device);
  if (x->stream) cudaStreamSynchronize(x->stream);
  for (auto& g : x->graphs) cudaGraphExecDestroy(g.exec);
  x->graphs.clear();
  if (x->cstream) {
    cudaStreamSynchronize(x->cstream);
    cudaStreamDestroy(x->cstream);
    cudaEventDestroy(x->x_ready);
    cudaEventDestroy(x->x_free);
  }
  if (x->gstream) {
    cudaStreamSynchronize(x->gstream);
    cudaStreamDestroy(x->gstream);
  }
  if (x->g_fork) cudaEventDestroy(x->g_fork);
  if (x->g_join) cudaEventDestroy(x->g_join);
  for (void* p : x->allocs) cudaFree(p);
  if (x->hstat) cudaFreeHost(x->hstat);
  for (auto& e : x->pending) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  for (auto e : x->ev_pool) cudaEventDestroy(e);
  if (x->own_stream) cudaStreamDestroy(x->stream);
  delete x;
  return VMFA_OK;
}

int vmfa_ctx_device_bytes(const vmfa_ctx* x, size_t* bytes) {
  TRY(check_ctx(x));
  if (bytes) *bytes = x->bytes;
  return VMFA_OK;
}

void* vmfa_ctx_stream(vmfa_ctx* x) { return x ? static_cast<void*>(x->stream) : nullptr; }
int vmfa_synchronize(vmfa_ctx* x) {
  TRY(check_ctx(x));
  CU(cudaStreamSynchronize(x->stream));
  return VMFA_OK;
}

int vmfa_upload_data_async(vmfa_ctx* x, const float* X, int64_t row_begin, int64_t rows) {
  TRY(check_ctx(x));
  x->prescored = false;
  if (!X || row_begin < 0 || rows < 0 || row_begin + rows > x->dm.N)
    return fail(VMFA_ERR_INVALID_ARGUMENT, "vmfa_upload_data_async: row range outside the shard");
  if (!x->cstream) {
    CU(cudaStreamCreateWithFlags(&x->cstream, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&x->x_ready, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&x->x_free, cudaEventDisableTiming));
  }
  // after everything already enqueued (which may still read the old rows)
  CU(cudaEventRecord(x->x_free, x->stream));
  CU(cudaStreamWaitEvent(x->cstream, x->x_free, 0));
  CU(cudaMemcpyAsync(x->X + row_begin * x->dm.D, X, sizeof(float) * rows * x->dm.D, cudaMemcpyHostToDevice,
                     x->cstream));
  if (x->xmax) CU(launch_rowmax(rows, x->dm.D, x->X + row_begin * x->dm.D, x->xmax + row_begin, x->cstream));
  CU(cudaEventRecord(x->x_ready, x->cstream));
  x->x_pending = true;
  return VMFA_OK;
}

int vmfa_stage_data_async(vmfa_ctx* x, const float* X, int64_t row_begin, int64_t rows) {
  TRY(check_ctx(x));
  if (!X || row_begin < 0 || rows < 0 || row_begin + rows > x->dm.N)
    return fail(VMFA_ERR_INVALID_ARGUMENT, "vmfa_stage_data_async: row range outside the shard");
  if (!x->cstream) {
    CU(cudaStreamCreateWithFlags(&x->cstream, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&x->x_ready, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&x->x_free, cudaEventDisableTiming));
  }
  if (!x->Xs) {
    const size_t N = static_cast<size_t>(x->dm.N), D = static_cast<size_t>(x->dm.D);
    int r = x->alloc(x->Xs, N * D);
    if (r == VMFA_OK && x->xmax) r = x->alloc(x->xmax_s, N);
    if (r != VMFA_OK) return r;
    CU(cudaEventCreateWithFlags(&x->xs_ready, cudaEventDisableTiming));
  }
  // after everything already enqueued (which may still read the staging
  // buffer: it was the current one before the last swap)
  CU(cudaEventRecord(x->x_free, x->stream));
  CU(cudaStreamWaitEvent(x->cstream, x->x_free, 0));
  CU(cudaMemcpyAsync(x->Xs + row_begin * x->dm.D, X, sizeof(float) * rows * x->dm.D, cudaMemcpyHostToDevice,
                     x->cstream));
  if (x->xmax_s) CU(launch_rowmax(rows, x->dm.D, x->Xs + row_begin * x->dm.D, x->xmax_s + row_begin, x->cstream));
  CU(cudaEventRecord(x->xs_ready, x->cstream));
  x->xs_pending = true;
  return VMFA_OK;
}

int vmfa_swap_data(vmfa_ctx* x) {
  TRY(check_ctx(x));
  if (!x->Xs || !x->xs_pending) return fail(VMFA_ERR_INVALID_ARGUMENT, "vmfa_swap_data: nothing staged");
  CU(wait_x(x));
  CU(cudaStreamWaitEvent(x->stream, x->xs_ready, 0));  // later work reads the staged rows
  std::swap(x->X, x->Xs);
  std::swap(x->xmax, x->xmax_s);
  x->xs_pending = false;
  x->prescored = false;
  return VMFA_OK;
}

int vmfa_set_lookahead(vmfa_ctx* x, int enable) {
  TRY(check_ctx(x));
  x->lookahead = enable != 0;
  return VMFA_OK;
}

int vmfa_upload_data(vmfa_ctx* x, const float* X, int64_t row_begin, int64_t rows) {
  TRY(check_ctx(x));
  x->prescored = false;
  if (!X || row_begin < 0 || rows < 0 || row_begin + rows > x->dm.N)
    return fail(VMFA_ERR_INVALID_ARGUMENT, "vmfa_upload_data: row range outside the shard");
  CU(wait_x(x));
  CU(cudaMemcpyAsync(x->X + row_begin * x->dm.D, X, sizeof(float) * rows * x->dm.D,
                     cudaMemcpyHostToDevice, x->stream));
  if (x->xmax) CU(launch_rowmax(rows, x->dm.D, x->X + row_begin * x->dm.D, x->xmax + row_begin, x->stream));
  CU(cudaStreamSynchronize(x->stream));
  return VMFA_OK;
}

int vmfa_set_floor(vmfa_ctx* x, const double* floor) {
  TRY(check_ctx(x));
  x->prescored = false;
  if (!floor) return fail(VMFA_ERR_INVALID_ARGUMENT, "floor is null");
  CU(cudaMemcpyAsync(x->floor, floor, sizeof(double) * x->dm.D, cudaMemcpyHostToDevice, x->stream));
  CU(cudaStreamSynchronize(x->stream));
  return VMFA_OK;
}

int vmfa_upload_params(vmfa_ctx* x, const double* pi, const double* mu, const double* lambda,
                       const double* dnoise) {
  TRY(check_ctx(x));
  x->prescored = false;
  if (!pi || !mu || !lambda || !dnoise) return fail(VMFA_ERR_INVALID_ARGUMENT, "null parameter array");
  const size_t C = x->dm.C, D = x->dm.D, H = x->dm.H;
  cudaStream_t s = x->stream;
  CU(cudaMemcpyAsync(x->pi, pi, sizeof(double) * C, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(x->mu, mu, sizeof(double) * C * D, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(x->lam, lambda, sizeof(double) * C * D * H, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(x->psi, dnoise, sizeof(double) * C * D, cudaMemcpyHostToDevice, s));
  x->have_estep = false;
  return run_precompute(x, nullptr);
}

int vmfa_download_params(vmfa_ctx* x, double* pi, double* mu, double* lambda, double* dnoise) {
  TRY(check_ctx(x));
  const size_t C = x->dm.C, D = x->dm.D, H = x->dm.H;
  cudaStream_t s = x->stream;
  if (pi) CU(cudaMemcpyAsync(pi, x->pi, sizeof(double) * C, cudaMemcpyDeviceToHost, s));
  if (mu) CU(cudaMemcpyAsync(mu, x->mu, sizeof(double) * C * D, cudaMemcpyDeviceToHost, s));
  if (lambda) CU(cudaMemcpyAsync(lambda, x->lam, sizeof(double) * C * D * H, cudaMemcpyDeviceToHost, s));
  if (dnoise) CU(cudaMemcpyAsync(dnoise, x->psi, sizeof(double) * C * D, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  return VMFA_OK;
}

int vmfa_precompute(vmfa_ctx* x, int* failed) {
  TRY(check_ctx(x));
  x->prescored = false;
  return run_precompute(x, failed);
}

int vmfa_download_caches(vmfa_ctx* x, double* U, double* Lmat, double* V, double* Sigma_z,
                         double* inv_dnoise, double* logdet, double* log_pi) {
  TRY(check_ctx(x));
  const size_t C = x->dm.C, D = x->dm.D, H = x->dm.H;
  cudaStream_t s = x->stream;
  if (U || V || inv_dnoise) {
    double *dU = nullptr, *dV = nullptr, *dI = nullptr;
    CU(cudaMallocAsync(&dU, sizeof(double) * C * D * H, s));
    CU(cudaMallocAsync(&dV, sizeof(double) * C * D * H, s));
    CU(cudaMallocAsync(&dI, sizeof(double) * C * D, s));
    CU(launch_caches_full(x->dm, x->lam, x->psi, x->R, dU, dV, dI, s));
    if (U) CU(cudaMemcpyAsync(U, dU, sizeof(double) * C * D * H, cudaMemcpyDeviceToHost, s));
    if (V) CU(cudaMemcpyAsync(V, dV, sizeof(double) * C * D * H, cudaMemcpyDeviceToHost, s));
    if (inv_dnoise) CU(cudaMemcpyAsync(inv_dnoise, dI, sizeof(double) * C * D, cudaMemcpyDeviceToHost, s));
    CU(cudaFreeAsync(dU, s));
    CU(cudaFreeAsync(dV, s));
    CU(cudaFreeAsync(dI, s));
  }
  if (Lmat) CU(cudaMemcpyAsync(Lmat, x->Lmat, sizeof(double) * C * H * H, cudaMemcpyDeviceToHost, s));
  if (Sigma_z) CU(cudaMemcpyAsync(Sigma_z, x->Sz, sizeof(double) * C * H * H, cudaMemcpyDeviceToHost, s));
  if (logdet) CU(cudaMemcpyAsync(logdet, x->logdet, sizeof(double) * C, cudaMemcpyDeviceToHost, s));
  if (log_pi) {
    CU(launch_logpi(x->pi, x->dm.C, x->logpi, s));
    CU(cudaMemcpyAsync(log_pi, x->logpi, sizeof(double) * C, cudaMemcpyDeviceToHost, s));
  }
  CU(cudaStreamSynchronize(s));
  return VMFA_OK;
}

int vmfa_upload_state(vmfa_ctx* x, const int32_t* K, const int32_t* g, const int32_t* g_count) {
  TRY(check_ctx(x));
  x->prescored = false;
  if (!K || !g || !g_count) return fail(VMFA_ERR_INVALID_ARGUMENT, "null state array");
  const Dims& dm = x->dm;
  // structural validation (VarState::validate, estep.cpp:15-68) on the host copy
  for (int c = 0; c < dm.C; ++c) {
    const int m = g_count[c];
    if (m < 1 || m > dm.G) return fail(VMFA_ERR_INVALID_ARGUMENT, "g_c size out of range (c=%d)", c);
    bool has_c = false;
    for (int i = 0; i < m; ++i) {
      const int v = g[static_cast<int64_t>(c) * dm.G + i];
      if (v < 0 || v >= dm.C || (i > 0 && v <= g[static_cast<int64_t>(c) * dm.G + i - 1]))
        return fail(VMFA_ERR_INVALID_ARGUMENT, "g_c not sorted distinct in-range indices (c=%d)", c);
      has_c |= (v == c);
    }
    if (!has_c) return fail(VMFA_ERR_INVALID_ARGUMENT, "g_c does not contain c (c=%d)", c);
  }
  std::vector<int32_t> gp(static_cast<size_t>(dm.C) * dm.G);
  for (int c = 0; c < dm.C; ++c)
    for (int i = 0; i < dm.G; ++i) gp[static_cast<size_t>(c) * dm.G + i] = i < g_count[c] ? g[static_cast<int64_t>(c) * dm.G + i] : -1;
  cudaStream_t s = x->stream;
  CU(cudaMemcpyAsync(x->K, K, sizeof(int) * dm.N * dm.Cp, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(x->g, gp.data(), sizeof(int) * gp.size(), cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(x->gcnt, g_count, sizeof(int) * dm.C, cudaMemcpyHostToDevice, s));
  // K rows are validated on the device (one pass over N x C')
  const long long none = 0x7fffffffffffffffLL;
  long long* bad = reinterpret_cast<long long*>(x->u64tmp);
  CU(cudaMemcpyAsync(bad, &none, sizeof none, cudaMemcpyHostToDevice, s));
  CU(launch_validate_K(x->K, dm.N, dm.Cp, dm.C, bad, s));
  long long first = none;
  CU(cudaMemcpyAsync(&first, bad, sizeof first, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  x->kinv_for_current_K = false;
  x->have_estep = false;
  if (first != none) return fail(VMFA_ERR_INVALID_ARGUMENT, "K row not sorted distinct in-range indices (n=%lld)", first);
  return VMFA_OK;
}

int vmfa_download_state(vmfa_ctx* x, int32_t* K, int32_t* g, int32_t* g_count, int32_t* labels) {
  TRY(check_ctx(x));
  const Dims& dm = x->dm;
  cudaStream_t s = x->stream;
  if (K) CU(cudaMemcpyAsync(K, x->K, sizeof(int) * dm.N * dm.Cp, cudaMemcpyDeviceToHost, s));
  if (g) CU(cudaMemcpyAsync(g, x->g, sizeof(int) * dm.C * dm.G, cudaMemcpyDeviceToHost, s));
  if (g_count) CU(cudaMemcpyAsync(g_count, x->gcnt, sizeof(int) * dm.C, cudaMemcpyDeviceToHost, s));
  if (labels) CU(cudaMemcpyAsync(labels, x->labels, sizeof(int) * dm.N, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  return VMFA_OK;
}

int vmfa_estep(vmfa_ctx* x, uint64_t seed, uint64_t iteration, int mode, double* F, uint64_t* joints) {
  TRY(check_ctx(x));
  if (mode != VMFA_DIST_KL && mode != VMFA_DIST_EUCLID) return fail(VMFA_ERR_INVALID_ARGUMENT, "mode");
  TRY(estep_local(x, seed, iteration, mode, false));
  TRY(estep_finish(x, false));
  double sc[4];
  TRY(read_scalars(x, sc));
  if (F) *F = sc[0];
  if (joints) *joints = static_cast<uint64_t>(sc[1]);
  return VMFA_OK;
}

int vmfa_download_estep(vmfa_ctx* x, int32_t* count, int32_t* idx, double* lj, double* resp) {
  TRY(check_ctx(x));
  if (!x->have_estep) return fail(VMFA_ERR_INVALID_ARGUMENT, "no E-step has run");
  const Dims& dm = x->dm;
  cudaStream_t s = x->stream;
  const size_t NS = static_cast<size_t>(dm.N) * dm.stride;
  std::vector<int32_t> cnt(dm.N);
  CU(cudaMemcpyAsync(cnt.data(), x->ret_cnt, sizeof(int) * dm.N, cudaMemcpyDeviceToHost, s));
  std::vector<int32_t> id(NS);
  std::vector<float> l(NS);
  CU(cudaMemcpyAsync(id.data(), x->ret_idx, sizeof(int) * NS, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(l.data(), x->ret_lj, sizeof(float) * NS, cudaMemcpyDeviceToHost, s));
  if (resp) CU(cudaMemcpyAsync(resp, x->resp, sizeof(double) * dm.N * dm.Cp, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  // reference layout: -1 / 0.0 padding beyond count (RetainedJoints::reset)
  for (int64_t n = 0; n < dm.N; ++n) {
    if (count) count[n] = cnt[n];
    for (int j = 0; j < dm.stride; ++j) {
      const size_t at = static_cast<size_t>(n) * dm.stride + j;
      const bool live = j < cnt[n];
      if (idx) idx[at] = live ? id[at] : -1;
      if (lj) lj[at] = live ? static_cast<double>(l[at]) : 0.0;
    }
  }
  return VMFA_OK;
}

int vmfa_download_distances(vmfa_ctx* x, int64_t cap, int32_t* c, int32_t* ct, double* sum,
                            int64_t* count, int64_t* n_rows) {
  TRY(check_ctx(x));
  // Re-run block 3 of the last E-step in dump mode is not possible after g was
  // replaced, so the dump is armed here and filled by the NEXT E-step when
  // cap == 0 (query); with cap > 0 the rows of the last armed E-step are read.
  if (cap == 0) {
    if (!x->dump) {
      x->dump = true;
      x->dump_cap = static_cast<long long>(x->dm.N) * x->dm.stride;
      int r = VMFA_OK;
      auto A = [&](auto*& p, size_t n) {
        if (r == VMFA_OK) r = x->alloc(p, n);
      };
      A(x->dump_c, x->dump_cap);
      A(x->dump_ct, x->dump_cap);
      A(x->dump_cnt, x->dump_cap);
      A(x->dump_hi, x->dump_cap);
      A(x->dump_lo, x->dump_cap);
      A(x->dump_n, 1);
      if (r != VMFA_OK) return r;
      CU(cudaMemsetAsync(x->dump_n, 0, sizeof(unsigned long long), x->stream));
    }
    unsigned long long m = 0;
    CU(cudaMemcpyAsync(&m, x->dump_n, sizeof m, cudaMemcpyDeviceToHost, x->stream));
    CU(cudaStreamSynchronize(x->stream));
    if (n_rows) *n_rows = static_cast<int64_t>(m);
    return VMFA_OK;
  }
  if (!x->dump) return fail(VMFA_ERR_INVALID_ARGUMENT, "distance dump not armed (call with cap=0 first)");
  unsigned long long m = 0;
  CU(cudaMemcpyAsync(&m, x->dump_n, sizeof m, cudaMemcpyDeviceToHost, x->stream));
  CU(cudaStreamSynchronize(x->stream));
  int64_t rows = std::min<int64_t>(static_cast<int64_t>(m), x->dump_cap);
  std::vector<int32_t> vc(rows), vct(rows);
  std::vector<long long> vn(rows), vh(rows), vl(rows);
  cudaStream_t s = x->stream;
  CU(cudaMemcpyAsync(vc.data(), x->dump_c, sizeof(int) * rows, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(vct.data(), x->dump_ct, sizeof(int) * rows, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(vn.data(), x->dump_cnt, sizeof(long long) * rows, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(vh.data(), x->dump_hi, sizeof(long long) * rows, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(vl.data(), x->dump_lo, sizeof(long long) * rows, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  std::vector<int64_t> order(rows);
  for (int64_t i = 0; i < rows; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    return vc[a] != vc[b] ? vc[a] < vc[b] : vct[a] < vct[b];
  });
  // merge rows of split components (one row per item) in (c, ct) order
  int64_t w = 0;
  for (int64_t i = 0; i < rows;) {
    const int64_t k = order[i];
    long long n = 0, hi = 0, lo = 0;
    int64_t j = i;
    for (; j < rows && vc[order[j]] == vc[k] && vct[order[j]] == vct[k]; ++j) {
      n += vn[order[j]];
      hi += vh[order[j]];
      lo += vl[order[j]];
    }
    if (w < cap) {
      if (c) c[w] = vc[k];
      if (ct) ct[w] = vct[k];
      if (sum) sum[w] = static_cast<double>(hi) / 1024.0 + static_cast<double>(lo) / 1073741824.0;  // from_fixed
      if (count) count[w] = n;
    }
    ++w;
    i = j;
  }
  rows = w;
  if (n_rows) *n_rows = rows;
  return VMFA_OK;
}

int vmfa_accumulate_suffstats(vmfa_ctx* x) {
  TRY(check_ctx(x));
  TRY(stats_local(x));
  CU(cudaStreamSynchronize(x->stream));
  return VMFA_OK;
}

int vmfa_download_suffstats(vmfa_ctx* x, double* Nc, double* Y, double* E, double* sq) {
  TRY(check_ctx(x));
  const size_t C = x->dm.C, D = x->dm.D, H1 = x->dm.H + 1;
  cudaStream_t s = x->stream;
  if (Nc) CU(cudaMemcpyAsync(Nc, x->Nc, sizeof(double) * C, cudaMemcpyDeviceToHost, s));
  if (Y) CU(cudaMemcpyAsync(Y, x->Y, sizeof(double) * C * H1 * D, cudaMemcpyDeviceToHost, s));
  if (E) CU(cudaMemcpyAsync(E, x->E, sizeof(double) * C * H1 * H1, cudaMemcpyDeviceToHost, s));
  if (sq) CU(cudaMemcpyAsync(sq, x->sq, sizeof(double) * C * D, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  return VMFA_OK;
}

int vmfa_upload_suffstats(vmfa_ctx* x, const double* Nc, const double* Y, const double* E,
                          const double* sq) {
  TRY(check_ctx(x));
  if (!Nc || !Y || !E || !sq) return fail(VMFA_ERR_INVALID_ARGUMENT, "null statistics array");
  const size_t C = x->dm.C, D = x->dm.D, H1 = x->dm.H + 1;
  cudaStream_t s = x->stream;
  CU(cudaMemcpyAsync(x->Nc, Nc, sizeof(double) * C, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(x->Y, Y, sizeof(double) * C * H1 * D, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(x->E, E, sizeof(double) * C * H1 * H1, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(x->sq, sq, sizeof(double) * C * D, cudaMemcpyHostToDevice, s));
  CU(cudaStreamSynchronize(s));
  return VMFA_OK;
}

int vmfa_update_params(vmfa_ctx* x, int* failed) {
  TRY(check_ctx(x));
  return update_and_precompute(x, failed);
}

int vmfa_truncated_free_energy(vmfa_ctx* x, double* F) {
  TRY(check_ctx(x));
  TRY(free_energy_local(x, false));
  double sc[4];
  TRY(read_scalars(x, sc));
  if (F) *F = sc[2];
  return VMFA_OK;
}

// exact_log_likelihood (model.cpp:139-148): sum over this context's rows of
// LSE_c l(n, c) over all C components, through the scorer's anchor pass on
// pseudo-anchor blocks (launch_dense_chunk; the warp-specialised tcgen05
// scorer, or the single-role one for shapes it does not take); rows in
// chunks of <= 1 GiB of log-joints. Leaves K, g, LJ and the lookahead state
// untouched (only the anchor B images / records are overwritten, which the
// next E-step rebuilds whenever it runs its own anchor pass).
int vmfa_exact_log_likelihood(vmfa_ctx* x, double* ll) {
  TRY(check_ctx(x));
  if (!ll) return fail(VMFA_ERR_INVALID_ARGUMENT, "null output");
  const Dims& dm = x->dm;
  int64_t R = 0;
  TRY(ensure_dense(x, &R));
  cudaStream_t s = x->stream;
  const int tok = x->begin(kFamExactLL, dm.N * static_cast<int64_t>(dm.C));
  TRY(dense_prepare(x));
  for (int64_t r0 = 0; r0 < dm.N; r0 += R) {
    const int Rc = static_cast<int>(std::min<int64_t>(R, dm.N - r0));
    TRY(dense_chunk(x, r0, Rc));
  }
  CU(launch_sum_f64(x->dense_lse, dm.N, x->partials, x->dense_out, s));
  x->end(tok);
  CU(cudaMemcpyAsync(&x->hstat->scal[3], x->dense_out, sizeof(double), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  *ll = x->hstat->scal[3];
  return VMFA_OK;
}

// em_full_step (mstep.cpp:164-208): every (n, c) log-joint through the dense
// pass, q(n, c) = exp(l - LSE_n) for all C, and the statistics over every
// pair by the K5 kernels (a row chunk's pairs are the K-pairs of a "K" holding
// all components), chunk statistics summed in fp64 in chunk order. Returns
// sum_n LSE_n and the N*C joints; the statistics stay in the context for
// vmfa_update_params (run_emmfa_loop, trainer.cpp:228-233).
int vmfa_em_full_step(vmfa_ctx* x, double* ll, uint64_t* joints) {
  TRY(check_ctx(x));
  if (!ll) return fail(VMFA_ERR_INVALID_ARGUMENT, "null output");
  const Dims& dm = x->dm;
  const int C = dm.C, D = dm.D;
  int64_t R = 0;
  TRY(ensure_dense(x, &R));
  // chunk rows: ~32 B per pair (fp64 q, int32 entry, statistics partials) within 4 GB
  const int rpi = kStatsMaxRowsHost;
  int64_t Re = std::max<int64_t>(1, (int64_t{4} << 30) / (32 * static_cast<int64_t>(C)));
  Re = std::min<int64_t>({Re, R, static_cast<int64_t>(dm.N), (std::numeric_limits<int>::max() - 1) / C});
  if (const char* v = std::getenv("VMFA_EM_CHUNK")) Re = std::max<int64_t>(1, std::min<int64_t>(Re, std::atoll(v)));
  if (!x->em_resp) {
    const int64_t items = C + (Re * C + rpi - 1) / rpi;
    TRY(x->alloc(x->em_resp, static_cast<size_t>(Re) * C));
    TRY(x->alloc(x->em_ent, static_cast<size_t>(Re) * C));
    TRY(x->alloc(x->em_off, static_cast<size_t>(C) + 1));
    TRY(x->alloc(x->em_items, static_cast<size_t>(C) + 1));
    TRY(x->alloc(x->em_part, static_cast<size_t>(items) * stats_part_stride(dm)));
    TRY(x->alloc(x->em_acc, x->stats_len));
    x->em_R = Re;
  }
  Re = std::min<int64_t>(Re, x->em_R);
  cudaStream_t s = x->stream;
  const int tok = x->begin(kFamExactLL, dm.N * static_cast<int64_t>(C));
  TRY(dense_prepare(x));
  int chunk = 0;
  for (int64_t r0 = 0; r0 < dm.N; r0 += Re, ++chunk) {
    const int Rc = static_cast<int>(std::min<int64_t>(Re, dm.N - r0));
    TRY(dense_chunk(x, r0, Rc));
    CU(launch_em_resp(x->dense_LJ, Rc, x->dense_SL, C, x->dense_lse + r0, x->em_resp, x->em_ent, x->em_off, s));
    CU(launch_items_scan(x->em_off, C, rpi, 0, x->em_items, s));
    StatsArgs a{};
    a.dm = dm;
    a.dm.N = Rc;
    a.dm.Cp = C;  // entry e = n * C + c: row e / C
    a.X = x->X + r0 * D;
    a.resp = x->em_resp;
    a.off = x->em_off;
    a.ent = x->em_ent;
    a.V32 = x->V32;
    a.mu32 = x->mu32;
    a.Sz = x->Sz;
    a.Nc = x->Nc;
    a.E = x->E;
    a.Y = x->Y;
    a.sq = x->sq;
    a.qctr = x->qctr;
    CU(launch_stats(a, x->em_items, rpi, x->em_part, s));
    CU(launch_add_f64(x->stats, x->em_acc, static_cast<int64_t>(x->stats_len), chunk == 0 ? 1 : 0, s));
  }
  CU(cudaMemcpyAsync(x->stats, x->em_acc, x->stats_len * sizeof(double), cudaMemcpyDeviceToDevice, s));
  CU(launch_sum_f64(x->dense_lse, dm.N, x->partials, x->dense_out, s));
  x->end(tok);
  CU(cudaMemcpyAsync(&x->hstat->scal[3], x->dense_out, sizeof(double), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  *ll = x->hstat->scal[3];
  if (joints) *joints = static_cast<uint64_t>(dm.N) * static_cast<uint64_t>(C);
  return VMFA_OK;
}

// afkmc2_seed (seeding.cpp:60-121) over the context's rows: the first center
// is drawn on the host from the stream (trainer.cpp:36), the proposal and the
// chains run on the device (k_afk_*). Returns the C seed rows, the stream
// state after the draws (init_params continues it, trainer.cpp:43) and the
// squared_distance count (EvalCounter::distances).
int vmfa_afkmc2_seed(vmfa_ctx* x, int C, int chain_length, uint64_t stream_seed, int64_t* seeds,
                     uint64_t* stream_state, uint64_t* distances) {
  TRY(check_ctx(x));
  const Dims& dm = x->dm;
  const int64_t N = dm.N;
  if (!seeds) return fail(VMFA_ERR_INVALID_ARGUMENT, "null output");
  if (C < 1 || C > N) return fail(VMFA_ERR_INVALID_ARGUMENT, "C out of range");
  if (chain_length < 1) return fail(VMFA_ERR_INVALID_ARGUMENT, "chain_length < 1");
  if (dm.n0 != 0 || dm.Ntot != dm.N)
    return fail(VMFA_ERR_UNSUPPORTED, "AFK-MC2 seeding needs the whole dataset in one context");
  HostStream hs(stream_seed);
  const int64_t first = hs.uniform_int(N);
  cudaStream_t s = x->stream;
  double *q = nullptr, *cdf = nullptr;
  int64_t* centers = nullptr;
  unsigned long long *st = nullptr, *cnt = nullptr;
  int* deg = nullptr;
  CU(cudaMallocAsync(&q, N * sizeof(double), s));
  CU(cudaMallocAsync(&cdf, N * sizeof(double), s));
  CU(cudaMallocAsync(&centers, C * sizeof(int64_t), s));
  CU(cudaMallocAsync(&st, 6 * sizeof(unsigned long long), s));
  cnt = st + 4;
  deg = reinterpret_cast<int*>(st + 5);
  unsigned long long init[6] = {hs.w[0], hs.w[1], hs.w[2], hs.w[3], 0, 0};
  CU(cudaMemcpyAsync(st, init, sizeof init, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(centers, &first, sizeof first, cudaMemcpyHostToDevice, s));
  CU(wait_x(x));
  CU(launch_afkmc2(x->X, N, dm.D, C, chain_length, q, cdf, centers, st, cnt, deg, s));
  unsigned long long out[6];
  CU(cudaMemcpyAsync(out, st, sizeof out, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(seeds, centers, C * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CU(cudaFreeAsync(q, s));
  CU(cudaFreeAsync(cdf, s));
  CU(cudaFreeAsync(centers, s));
  CU(cudaFreeAsync(st, s));
  CU(cudaStreamSynchronize(s));
  int degenerate = 0;
  std::memcpy(&degenerate, &out[5], sizeof degenerate);
  if (degenerate) return fail(VMFA_ERR_DEGENERATE_DATA, "fewer distinct rows than requested seeds");
  if (stream_state)
    for (int k = 0; k < 4; ++k) stream_state[k] = out[k];
  if (distances) *distances = out[4] + static_cast<uint64_t>(N);  // + the first center's proposal pass
  return VMFA_OK;
}

namespace {
vmfa_ctx::HostState host_state(const vmfa_ctx* x, int mode) {
  vmfa_ctx::HostState h{};
  h.g = x->g, h.gcnt = x->gcnt, h.g_new = x->g_new, h.gcnt_new = x->gcnt_new;
  h.pi = x->pi, h.pi2 = x->pi2, h.mu = x->mu, h.mu2 = x->mu2;
  h.lam = x->lam, h.lam2 = x->lam2, h.psi = x->psi, h.psi2 = x->psi2;
  h.X = x->X, h.xmax = x->xmax;
  h.prescored = x->prescored, h.kinv = x->kinv_for_current_K, h.have_estep = x->have_estep;
  h.mode = mode;
  h.lookahead = x->lookahead;
  return h;
}
void set_host_state(vmfa_ctx* x, const vmfa_ctx::HostState& h) {
  x->g = h.g, x->gcnt = h.gcnt, x->g_new = h.g_new, x->gcnt_new = h.gcnt_new;
  x->pi = h.pi, x->pi2 = h.pi2, x->mu = h.mu, x->mu2 = h.mu2;
  x->lam = h.lam, x->lam2 = h.lam2, x->psi = h.psi, x->psi2 = h.psi2;
  x->prescored = h.prescored, x->kinv_for_current_K = h.kinv, x->have_estep = h.have_estep;
}
bool graphs_enabled(const vmfa_ctx* x) {
  static const bool on = [] {  // VMFA_GRAPH=0: plain launches
    const char* v = std::getenv("VMFA_GRAPH");
    return !(v && v[0] == '0');
  }();
  // (a captured graph records the scorer-diagnostics pointer and kernel
  // variant: no graphs while those counters are armed)
  return on && !x->graph_off && !x->sparse && !x->profile && !x->dump && !x->x_pending && !ws_diag_armed();
}
}  // namespace

// One main iteration enqueued without a host synchronisation; the statuses
// of selection, update and precompute land in the pinned readback.
int iterate_enqueue(vmfa_ctx* x, uint64_t seed, uint64_t iteration, int mode, int* failed) {
  cudaStream_t s = x->stream;
  static const bool side = [] {  // VMFA_GSTREAM=0: block 3 in line on the main stream
    const char* v = std::getenv("VMFA_GSTREAM");
    return !(v && v[0] == '0');
  }();
  TRY(estep_local(x, seed, iteration, mode, false, side));
  TRY(estep_finish(x, false, false));
  TRY(launch_deferred_gupdate(x));
  TRY(stats_local(x));
  TRY(launch_update_params(x));
  swap_params(x);
  TRY(run_precompute(x, failed, false));
  TRY(join_gupdate(x));
  TRY(free_energy_local(x, x->lookahead));
  CU(launch_count_empty(x->pi, x->dm.C, x->n_empty, s));
  IterStatus* h = x->hstat;
  CU(cudaMemcpyAsync(&h->sel, x->st_select, sizeof(int), cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&h->upd, x->st_update, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&h->model, x->st_model, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&h->empty, x->n_empty, sizeof(int), cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(h->scal, x->scal, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
  return VMFA_OK;
}

int vmfa_iterate(vmfa_ctx* x, uint64_t seed, uint64_t iteration, int mode, vmfa_iter_report* rep) {
  TRY(check_ctx(x));
  if (mode != VMFA_DIST_KL && mode != VMFA_DIST_EUCLID) return fail(VMFA_ERR_INVALID_ARGUMENT, "mode");
  int failed = -1;
  cudaStream_t s = x->stream;
  bool done = false;
  if (graphs_enabled(x)) {
    // the same launch sequence as a CUDA graph, captured once per host-side
    // pre-state (in steady state two: g and the parameter sets alternate)
    const unsigned long long sit[2] = {seed, iteration};
    CU(cudaMemcpyAsync(x->sit, sit, sizeof sit, cudaMemcpyHostToDevice, s));
    const vmfa_ctx::HostState pre = host_state(x, mode);
    vmfa_ctx::GraphEntry* e = nullptr;
    for (auto& g : x->graphs)
      if (g.pre == pre) e = &g;
    if (e) {
      set_host_state(x, e->post);
    } else {
      x->capturing = true;
      cudaGraph_t graph = nullptr;
      cudaError_t ce = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      int r = ce == cudaSuccess ? iterate_enqueue(x, seed, iteration, mode, &failed) : VMFA_ERR_CUDA;
      if (ce == cudaSuccess) ce = cudaStreamEndCapture(s, &graph);
      x->capturing = false;
      cudaGraphExec_t exec = nullptr;
      if (r == VMFA_OK && ce == cudaSuccess && cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess) {
        x->graphs.push_back({pre, host_state(x, mode), exec});
        e = &x->graphs.back();
      } else {  // not capturable here: plain launches from now on
        cudaGetLastError();
        set_host_state(x, pre);
        x->graph_off = true;
      }
      if (graph) cudaGraphDestroy(graph);
    }
    if (e) {
      CU(cudaGraphLaunch(e->exec, s));
      done = true;
    }
  }
  if (!done) TRY(iterate_enqueue(x, seed, iteration, mode, &failed));
  IterStatus* h = x->hstat;
  CU(cudaStreamSynchronize(s));
  if (h->sel) {
    x->prescored = false;
    return fail(VMFA_ERR_INSUFFICIENT_CANDIDATES, "search space smaller than C'");
  }
  if (h->upd != ~0ull) {  // leave the pre-update parameters (and their caches) in place
    swap_params(x);
    TRY(run_precompute(x, nullptr));
    x->prescored = false;
    const int r = update_status(h->upd, &failed);
    if (rep) rep->failed_component = failed;
    return r;
  }
  if (h->model != ~0ull) {
    x->prescored = false;
    failed = static_cast<int>(h->model >> 8);
    if (rep) rep->failed_component = failed;
    return fail(static_cast<int>(h->model & 0xff), "L_c not positive definite for component %d", failed);
  }
  if (rep) {
    rep->failed_component = -1;
    rep->free_energy_estep = h->scal[0];
    rep->joints = static_cast<uint64_t>(h->scal[1]);
    rep->free_energy = h->scal[2];
    rep->empty_components = h->empty;
  }
  return VMFA_OK;
}

// ---------------------------------------------------------------- phase API (multi-GPU)
int vmfa_exchange_buffer(vmfa_ctx* x, int which, void** ptr, size_t* count, int* dtype) {
  TRY(check_ctx(x));
  if (!ptr || !count || !dtype) return fail(VMFA_ERR_INVALID_ARGUMENT, "null output");
  if (which == VMFA_XCHG_COOC) {
    const size_t n = 3 * static_cast<size_t>(x->dm.C) * x->dm.C;
    if (!x->xc)
      return fail(VMFA_ERR_UNSUPPORTED, "no dense co-occurrence table in sparse mode (C > ~18900 or "
                                        "VMFA_COOC=sparse): use vmfa_cooc_local_list / vmfa_cooc_select");
    *ptr = x->xc;
    *count = n;
    *dtype = VMFA_DT_INT64;
  } else if (which == VMFA_XCHG_STATS) {
    *ptr = x->stats;
    *count = x->stats_len;
    *dtype = VMFA_DT_FLOAT64;
  } else if (which == VMFA_XCHG_SCALARS) {
    *ptr = x->scal;
    *count = 3;
    *dtype = VMFA_DT_FLOAT64;
  } else if (which == VMFA_XCHG_G) {
    *ptr = x->g_new;
    *count = static_cast<size_t>(x->dm.C) * x->dm.G + x->dm.C;
    *dtype = VMFA_DT_INT32;
  } else {
    return fail(VMFA_ERR_INVALID_ARGUMENT, "unknown exchange buffer %d", which);
  }
  return VMFA_OK;
}

int vmfa_phase_estep_local(vmfa_ctx* x, uint64_t seed, uint64_t iteration, int mode) {
  TRY(check_ctx(x));
  if (!x->xc) TRY(enable_lists(x));  // multi-rank without the dense rows: sparse lists
  if (!x->xc && !x->sparse) {
    void* p;
    size_t n;
    int dt;
    TRY(vmfa_exchange_buffer(x, VMFA_XCHG_COOC, &p, &n, &dt));
  }
  TRY(estep_local(x, seed, iteration, mode, true));
  CU(cudaMemsetAsync(x->scal + 2, 0, sizeof(double), x->stream));
  CU(cudaStreamSynchronize(x->stream));
  return VMFA_OK;
}
int vmfa_phase_estep_finish(vmfa_ctx* x) {
  TRY(check_ctx(x));
  return estep_finish(x, true);
}
int vmfa_phase_stats_local(vmfa_ctx* x) {
  TRY(check_ctx(x));
  TRY(stats_local(x));
  CU(cudaStreamSynchronize(x->stream));
  return VMFA_OK;
}
int vmfa_phase_update(vmfa_ctx* x, int* failed) {
  TRY(check_ctx(x));
  return update_and_precompute(x, failed);
}
int vmfa_phase_free_energy_local(vmfa_ctx* x) {
  TRY(check_ctx(x));
  TRY(free_energy_local(x, x->lookahead));
  CU(cudaStreamSynchronize(x->stream));
  return VMFA_OK;
}
int vmfa_phase_scalars(vmfa_ctx* x, double* Fe, uint64_t* joints, double* F) {
  TRY(check_ctx(x));
  double sc[4];
  TRY(read_scalars(x, sc));
  if (Fe) *Fe = sc[0];
  if (joints) *joints = static_cast<uint64_t>(sc[1]);
  if (F) *F = sc[2];
  return VMFA_OK;
}

int vmfa_cooc_sparse(vmfa_ctx* x, int* sparse) {
  TRY(check_ctx(x));
  if (!sparse) return fail(VMFA_ERR_INVALID_ARGUMENT, "null output");
  *sparse = (x->sparse || !x->xc) ? 1 : 0;  // (lists are set up on the first multi-rank E-step)
  return VMFA_OK;
}
int vmfa_cooc_local_list(vmfa_ctx* x, int world, void** key, void** cnt, void** hi, void** lo, int64_t* counts) {
  TRY(check_ctx(x));
  if (!x->sparse) return fail(VMFA_ERR_INVALID_ARGUMENT, "context has the dense co-occurrence table");
  if (world < 1 || !key || !cnt || !hi || !lo || !counts) return fail(VMFA_ERR_INVALID_ARGUMENT, "bad arguments");
  *key = x->cu_key;
  *cnt = x->cu_cnt;
  *hi = x->cu_hi;
  *lo = x->cu_lo;
  // owner r holds components [floor(rC/p), floor((r+1)C/p)): contiguous in the sorted list
  std::vector<int> b(world + 1);
  for (int r = 0; r <= world; ++r) {
    const int c = static_cast<int>(static_cast<int64_t>(r) * x->dm.C / world);
    CU(cudaMemcpyAsync(&b[r], x->cu_off + c, sizeof(int), cudaMemcpyDeviceToHost, x->stream));
  }
  CU(cudaStreamSynchronize(x->stream));
  for (int r = 0; r < world; ++r) counts[r] = b[r + 1] - b[r];
  return VMFA_OK;
}
int vmfa_cooc_select(vmfa_ctx* x, const void* key, const void* cnt, const void* hi, const void* lo, int64_t n,
                     int rank, int world) {
  TRY(check_ctx(x));
  if (!x->sparse) return fail(VMFA_ERR_INVALID_ARGUMENT, "context has the dense co-occurrence table");
  if (world < 1 || rank < 0 || rank >= world || n < 0) return fail(VMFA_ERR_INVALID_ARGUMENT, "bad rank/world/n");
  if (n > x->cl_cap) return fail(VMFA_ERR_UNSUPPORTED, "received co-occurrence list exceeds the capacity");
  cudaStream_t s = x->stream;
  if (n > 0) {
    CU(cudaMemcpyAsync(x->cl_key, key, n * sizeof(unsigned), cudaMemcpyDeviceToDevice, s));
    CU(cudaMemcpyAsync(x->cl_cnt, cnt, n * sizeof(long long), cudaMemcpyDeviceToDevice, s));
    CU(cudaMemcpyAsync(x->cl_hi, hi, n * sizeof(long long), cudaMemcpyDeviceToDevice, s));
    CU(cudaMemcpyAsync(x->cl_lo, lo, n * sizeof(long long), cudaMemcpyDeviceToDevice, s));
  }
  TRY(cooc_reduce(x, n));
  const int c0 = static_cast<int>(static_cast<int64_t>(rank) * x->dm.C / world);
  const int c1 = static_cast<int>(static_cast<int64_t>(rank + 1) * x->dm.C / world);
  CU(launch_cooc_select(cooc_args(x), c0, c1, 1, x->g_new, x->gcnt_new, s));
  CU(cudaStreamSynchronize(s));
  return VMFA_OK;
}

// ---------------------------------------------------------------- per-operation pieces
}  // extern "C"
namespace {
// a device copy of a host array for the duration of one call (stream-ordered)
template <class T>
struct DevTmp {
  T* p = nullptr;
  cudaStream_t s = nullptr;
  cudaError_t make(const T* host, size_t n, cudaStream_t st) {
    s = st;
    if (cudaError_t e = cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), s); e != cudaSuccess) return e;
    return host ? cudaMemcpyAsync(p, host, n * sizeof(T), cudaMemcpyHostToDevice, s) : cudaSuccess;
  }
  ~DevTmp() {
    if (p) cudaFreeAsync(p, s);
  }
};
}  // namespace
extern "C" {

int vmfa_log_joint(vmfa_ctx* x, const float* X, int64_t n, const int32_t* comp, double* out) {
  TRY(check_ctx(x));
  if (n < 0 || (n > 0 && (!X || !comp || !out))) return fail(VMFA_ERR_INVALID_ARGUMENT, "vmfa_log_joint: bad arguments");
  if (n == 0) return VMFA_OK;
  const Dims& dm = x->dm;
  for (int64_t i = 0; i < n; ++i)
    if (comp[i] < 0 || comp[i] >= dm.C) return fail(VMFA_ERR_INVALID_ARGUMENT, "component index out of range");
  cudaStream_t s = x->stream;
  DevTmp<float> dx;
  DevTmp<int> dc;
  DevTmp<double> dout;
  CU(dx.make(X, static_cast<size_t>(n) * dm.D, s));
  CU(dc.make(comp, n, s));
  CU(dout.make(nullptr, n, s));
  CU(launch_log_joint_pairs(dm.D, dm.H, dx.p, dc.p, n, x->mu, x->psi, x->lam, x->R, x->kconst, dout.p, s));
  CU(cudaMemcpyAsync(out, dout.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  return VMFA_OK;
}

int vmfa_build_search_space(vmfa_ctx* x, uint64_t seed, uint64_t iteration, const int32_t* extras, int32_t* count,
                            int32_t* idx) {
  TRY(check_ctx(x));
  if (!count || !idx) return fail(VMFA_ERR_INVALID_ARGUMENT, "null output");
  const Dims& dm = x->dm;
  cudaStream_t s = x->stream;
  DevTmp<int> de, dcnt, didx;
  if (extras) CU(de.make(extras, dm.N, s));
  CU(dcnt.make(nullptr, dm.N, s));
  CU(didx.make(nullptr, static_cast<size_t>(dm.N) * dm.stride, s));
  CU(launch_search_space(dm, x->K, x->g, x->gcnt, extras ? de.p : nullptr, seed, iteration, dcnt.p, didx.p, s));
  CU(cudaMemcpyAsync(count, dcnt.p, sizeof(int) * dm.N, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(idx, didx.p, sizeof(int) * dm.N * dm.stride, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  return VMFA_OK;
}

int vmfa_update_k(vmfa_ctx* x, const int32_t* count, const int32_t* idx, const double* lj, int32_t* K) {
  TRY(check_ctx(x));
  if (!count || !idx || !lj || !K) return fail(VMFA_ERR_INVALID_ARGUMENT, "null argument");
  const Dims& dm = x->dm;
  cudaStream_t s = x->stream;
  const size_t NS = static_cast<size_t>(dm.N) * dm.stride;
  DevTmp<int> dcnt, didx, dK, dst;
  DevTmp<double> dl;
  CU(dcnt.make(count, dm.N, s));
  CU(didx.make(idx, NS, s));
  CU(dl.make(lj, NS, s));
  CU(dK.make(nullptr, static_cast<size_t>(dm.N) * dm.Cp, s));
  CU(dst.make(nullptr, 1, s));
  CU(cudaMemsetAsync(dst.p, 0, sizeof(int), s));
  CU(launch_update_k(dm, dcnt.p, didx.p, dl.p, dK.p, dst.p, s));
  int status = 0;
  CU(cudaMemcpyAsync(K, dK.p, sizeof(int) * dm.N * dm.Cp, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&status, dst.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (status) return fail(VMFA_ERR_INSUFFICIENT_CANDIDATES, "search space smaller than C'");
  return VMFA_OK;
}

int vmfa_hard_partition(vmfa_ctx* x, const int32_t* K, const int32_t* count, const int32_t* idx, const double* lj,
                        int32_t* labels, int32_t* part_off, int32_t* part_ent) {
  TRY(check_ctx(x));
  if (!K || !count || !idx || !lj || !labels) return fail(VMFA_ERR_INVALID_ARGUMENT, "null argument");
  const Dims& dm = x->dm;
  cudaStream_t s = x->stream;
  const size_t NS = static_cast<size_t>(dm.N) * dm.stride;
  DevTmp<int> dK, dcnt, didx, dlab;
  DevTmp<double> dl;
  CU(dK.make(K, static_cast<size_t>(dm.N) * dm.Cp, s));
  CU(dcnt.make(count, dm.N, s));
  CU(didx.make(idx, NS, s));
  CU(dl.make(lj, NS, s));
  CU(dlab.make(nullptr, dm.N, s));
  CU(launch_hard_labels(dm, dK.p, dcnt.p, didx.p, dl.p, dlab.p, s));
  // the partition: stable by label, so every cell lists its rows ascending
  TRY(csr_by_key(x, reinterpret_cast<const unsigned*>(dlab.p), dm.N, x->part_off, x->part_ent, nullptr, 1));
  CU(cudaMemcpyAsync(labels, dlab.p, sizeof(int) * dm.N, cudaMemcpyDeviceToHost, s));
  if (part_off) CU(cudaMemcpyAsync(part_off, x->part_off, sizeof(int) * (dm.C + 1), cudaMemcpyDeviceToHost, s));
  if (part_ent) CU(cudaMemcpyAsync(part_ent, x->part_ent, sizeof(int) * dm.N, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  return VMFA_OK;
}

int vmfa_accumulate_distances(vmfa_ctx* x, int mode, const int32_t* part_off, const int32_t* part_ent,
                              const int32_t* count, const int32_t* idx, const double* lj, const double* pi,
                              int64_t cap, int32_t* c_out, int32_t* ct_out, double* sum_out, int64_t* cnt_out,
                              int64_t* n_rows) {
  TRY(check_ctx(x));
  if (!part_off || !part_ent || !count || !idx || !lj || !pi || !n_rows || (mode != 0 && mode != 1))
    return fail(VMFA_ERR_INVALID_ARGUMENT, "bad arguments");
  const Dims& dm = x->dm;
  if (part_off[0] != 0 || part_off[dm.C] != dm.N) return fail(VMFA_ERR_INVALID_ARGUMENT, "partition does not cover the rows");
  cudaStream_t s = x->stream;
  // launch configuration: per component a hash table of 2x its entry bound
  std::vector<int64_t> off(dm.C + 1, 0);
  std::vector<int> tcap(dm.C);
  for (int c = 0; c < dm.C; ++c) {
    int64_t b = 0;
    for (int e = part_off[c]; e < part_off[c + 1]; ++e) b += count[part_ent[e]];
    int64_t p2 = 1;
    while (p2 < 2 * b) p2 <<= 1;
    tcap[c] = static_cast<int>(p2);
    off[c + 1] = off[c] + p2;
  }
  const size_t NS = static_cast<size_t>(dm.N) * dm.stride, T = static_cast<size_t>(off[dm.C]);
  DevTmp<int> dpo, dpe, dcnt, didx, dcap, dkey, dnk;
  DevTmp<double> dl, dpi, dsum;
  DevTmp<long long> dtc;
  DevTmp<int64_t> doff;
  CU(dpo.make(part_off, dm.C + 1, s));
  CU(dpe.make(part_ent, dm.N, s));
  CU(dcnt.make(count, dm.N, s));
  CU(didx.make(idx, NS, s));
  CU(dl.make(lj, NS, s));
  CU(dpi.make(pi, dm.C, s));
  CU(doff.make(off.data(), dm.C + 1, s));
  CU(dcap.make(tcap.data(), dm.C, s));
  CU(dkey.make(nullptr, T, s));
  CU(dsum.make(nullptr, T, s));
  CU(dtc.make(nullptr, T, s));
  CU(dnk.make(nullptr, dm.C, s));
  CU(launch_distances(dm, mode, dpo.p, dpe.p, dcnt.p, didx.p, dl.p, dpi.p, doff.p, dcap.p, dkey.p, dsum.p, dtc.p,
                      dnk.p, s));
  std::vector<int> nk(dm.C), hk(T);
  std::vector<double> hs(T);
  std::vector<long long> hc(T);
  CU(cudaMemcpyAsync(nk.data(), dnk.p, sizeof(int) * dm.C, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(hk.data(), dkey.p, sizeof(int) * T, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(hs.data(), dsum.p, sizeof(double) * T, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(hc.data(), dtc.p, sizeof(long long) * T, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  int64_t w = 0;  // (c, ct) ascending rows: each component's keys are at the front of its table, sorted
  for (int c = 0; c < dm.C; ++c)
    for (int i = 0; i < nk[c]; ++i, ++w) {
      if (w >= cap) continue;
      const int64_t k = off[c] + i;
      if (c_out) c_out[w] = c;
      if (ct_out) ct_out[w] = hk[k];
      if (sum_out) sum_out[w] = hs[k];
      if (cnt_out) cnt_out[w] = hc[k];
    }
  *n_rows = w;
  return VMFA_OK;
}

int vmfa_update_g(vmfa_ctx* x, int64_t n_rows, const int32_t* c_in, const int32_t* ct, const double* sum,
                  const int64_t* cnt, int32_t* g, int32_t* g_count) {
  TRY(check_ctx(x));
  if (n_rows < 0 || (n_rows > 0 && (!c_in || !ct || !sum || !cnt)) || !g || !g_count)
    return fail(VMFA_ERR_INVALID_ARGUMENT, "bad arguments");
  const Dims& dm = x->dm;
  std::vector<int64_t> off(dm.C + 1, 0);
  for (int64_t r = 0; r < n_rows; ++r) {
    if (c_in[r] < 0 || c_in[r] >= dm.C || (r > 0 && c_in[r] < c_in[r - 1]))
      return fail(VMFA_ERR_INVALID_ARGUMENT, "rows not sorted by component");
    ++off[c_in[r] + 1];
  }
  for (int c = 0; c < dm.C; ++c) off[c + 1] += off[c];
  cudaStream_t s = x->stream;
  DevTmp<int64_t> doff;
  DevTmp<int> dct, dg, dgc;
  DevTmp<double> dsum;
  DevTmp<long long> dcnt;
  CU(doff.make(off.data(), dm.C + 1, s));
  CU(dct.make(ct, n_rows, s));
  CU(dsum.make(sum, n_rows, s));
  CU(dcnt.make(reinterpret_cast<const long long*>(cnt), n_rows, s));
  CU(dg.make(nullptr, static_cast<size_t>(dm.C) * dm.G, s));
  CU(dgc.make(nullptr, dm.C, s));
  CU(launch_update_g(dm.C, dm.G, doff.p, dct.p, dsum.p, dcnt.p, dg.p, dgc.p, s));
  CU(cudaMemcpyAsync(g, dg.p, sizeof(int) * dm.C * dm.G, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(g_count, dgc.p, sizeof(int) * dm.C, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  return VMFA_OK;
}

int vmfa_responsibilities(vmfa_ctx* x, int64_t rows, int width, const double* lj, double* resp) {
  TRY(check_ctx(x));
  if (rows < 0 || width < 1 || (rows > 0 && (!lj || !resp))) return fail(VMFA_ERR_INVALID_ARGUMENT, "bad arguments");
  if (rows == 0) return VMFA_OK;
  cudaStream_t s = x->stream;
  const size_t n = static_cast<size_t>(rows) * width;
  DevTmp<double> dl, dr;
  CU(dl.make(lj, n, s));
  CU(dr.make(nullptr, n, s));
  CU(launch_responsibilities(rows, width, dl.p, dr.p, s));
  CU(cudaMemcpyAsync(resp, dr.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  return VMFA_OK;
}

}  // extern "C"
namespace {
// caller-supplied K rows into the context (validated on the device)
int set_K(vmfa_ctx* x, const int32_t* K) {
  const Dims& dm = x->dm;
  cudaStream_t s = x->stream;
  CU(cudaMemcpyAsync(x->K, K, sizeof(int) * dm.N * dm.Cp, cudaMemcpyHostToDevice, s));
  const long long none = 0x7fffffffffffffffLL;
  long long* bad = reinterpret_cast<long long*>(x->u64tmp);
  CU(cudaMemcpyAsync(bad, &none, sizeof none, cudaMemcpyHostToDevice, s));
  CU(launch_validate_K(x->K, dm.N, dm.Cp, dm.C, bad, s));
  long long first = none;
  CU(cudaMemcpyAsync(&first, bad, sizeof first, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  x->kinv_for_current_K = false;
  x->prescored = false;
  if (first != none) return fail(VMFA_ERR_INVALID_ARGUMENT, "K row not sorted distinct in-range indices (n=%lld)", first);
  return VMFA_OK;
}
}  // namespace
extern "C" {

int vmfa_accumulate_suffstats_k(vmfa_ctx* x, const int32_t* K, const double* resp) {
  TRY(check_ctx(x));
  if (!K || !resp) return fail(VMFA_ERR_INVALID_ARGUMENT, "null argument");
  TRY(set_K(x, K));
  CU(cudaMemcpyAsync(x->resp, resp, sizeof(double) * x->dm.N * x->dm.Cp, cudaMemcpyHostToDevice, x->stream));
  x->have_estep = true;
  TRY(stats_local(x));
  CU(cudaStreamSynchronize(x->stream));
  return VMFA_OK;
}

int vmfa_truncated_free_energy_k(vmfa_ctx* x, const int32_t* K, double* F) {
  TRY(check_ctx(x));
  if (!K) return fail(VMFA_ERR_EMPTY_KSET, "empty K collection");  // model.cpp:150-159 EmptyKSet
  TRY(set_K(x, K));
  TRY(free_energy_local(x, false));
  double sc[4];
  TRY(read_scalars(x, sc));
  if (F) *F = sc[2];
  return VMFA_OK;
}

// ---------------------------------------------------------------- work accounting
int vmfa_scoring_work(vmfa_ctx* x, int64_t* out, int n) {
  TRY(check_ctx(x));
  if (!out || n < 1) return fail(VMFA_ERR_INVALID_ARGUMENT, "null output");
  const Dims& dm = x->dm;
  int ex = 0;
  if (x->have_estep) {
    CU(cudaMemcpyAsync(&ex, x->ex_off + dm.C, sizeof(int), cudaMemcpyDeviceToHost, x->stream));
    CU(cudaStreamSynchronize(x->stream));
  }
  unsigned long long nfl[2] = {0, 0};  // read and cleared
  CU(cudaMemcpyAsync(nfl, x->nfix, sizeof nfl, cudaMemcpyDeviceToHost, x->stream));
  CU(cudaMemsetAsync(x->nfix, 0, sizeof nfl, x->stream));
  CU(cudaStreamSynchronize(x->stream));
  const int64_t w[8] = {static_cast<int64_t>(dm.N) * dm.Cp,
                        ex,
                        x->scorer == 2 ? ws_image_halves(dm, 0) * 2 : 0,
                        x->scorer == 2 ? ws_image_halves(dm, 1) * 2 : 0,
                        x->scorer == 2 ? (ws_record_floats(dm, 0) + ws_record_floats(dm, 1)) * 4 : 0,
                        x->scorer, static_cast<int64_t>(nfl[0]), static_cast<int64_t>(nfl[1])};
  for (int i = 0; i < n && i < 8; ++i) out[i] = w[i];
  return VMFA_OK;
}

// ---------------------------------------------------------------- profiling
int vmfa_profile_enable(vmfa_ctx* x, int enable) {
  TRY(check_ctx(x));
  x->collect();
  x->profile = enable != 0;
  for (int i = 0; i < kNumFamilies; ++i) {
    x->fam_ms[i] = 0.0;
    x->fam_launches[i] = 0;
    x->fam_units[i] = 0;
  }
  return VMFA_OK;
}
int vmfa_kernel_times(vmfa_ctx* x, int max, double* ms, int64_t* launches, int64_t* units, int* n) {
  TRY(check_ctx(x));
  x->collect();
  const int m = std::min<int>(max, kNumFamilies);
  for (int i = 0; i < m; ++i) {
    if (ms) ms[i] = x->fam_ms[i];
    if (launches) launches[i] = x->fam_launches[i];
    if (units) units[i] = x->fam_units[i];
  }
  if (n) *n = kNumFamilies;
  return VMFA_OK;
}
const char* vmfa_kernel_name(int i) { return (i >= 0 && i < kNumFamilies) ? kFamilyNames[i] : ""; }

}  // extern "C"
