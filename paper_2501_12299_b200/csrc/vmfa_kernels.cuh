// vmfa_kernels.cuh — device kernels of the v-MFA hot path (sm_100a) and their
// argument blocks. See DESIGN.md for the data layout in HBM and the roofline of
// each kernel. Reference correspondences:
//   k_extra        uniform_component + the union test of
//                  build_search_space_into (rng.hpp:91-98, estep.cpp:83-101)
//   k_score_*      log_joint over anchor blocks (model.cpp:81-95)
//   k_select       update_k_into + hard_partition label + block 4
//                  (estep.cpp:103-122, :144-173, :314-335)
//   k_gupdate      block 3 + update_g (estep.cpp:286-312, :204-220)
//   k_stats        accumulate_point / accumulate_suffstats (mstep.cpp:47-101)
//   k_update       update_params (mstep.cpp:103-162)
//   k_precompute   precompute_component (model.cpp:43-73)
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

namespace vmfa_b200 {

constexpr int kScoreRows = 64;      // rows (points) per scoring item
constexpr int kScoreThreads = 128;  // 4 warps; each warp scores one component x 64 rows
constexpr int kXsStride = kScoreRows + 2;  // transposed x tile stride (floats)
constexpr int kStatsThreads = 256;
constexpr int kGupdCap = 8192;      // smem hash capacity of the block-3 accumulator (24 B per entry)
constexpr int kGupdThreads = 512;
constexpr int kGupdDenseMax = 11000;  // C up to which the g-update table is a dense shared-memory row (20 B each)
constexpr int kGupdRowsCap = 2048;  // hash of an item that adds into the dense rows (overflow goes to xc)

// Packed fp32 scoring parameters of one component (precompute output):
// per dimension d a row of HP floats: [W_0 .. W_{Hc-1}, mu_d, 1/psi_d, 0, 0]
// where W = U R^{-T} (so (U^T v).(V v) = |W^T v|^2), Hc = H rounded up to the
// h-chunk. HP = Hc + 4 keeps every row 16-byte aligned.
struct ScoreLayout {
  int hc;   // h-chunk (4, 8 or 16)
  int Hc;   // H rounded up to a multiple of hc
  int HP;   // floats per dimension row
};
inline ScoreLayout score_layout(int H) {
  ScoreLayout L;
  L.hc = H <= 4 ? 4 : (H <= 8 ? 8 : 16);
  L.Hc = (H + L.hc - 1) / L.hc * L.hc;
  L.HP = L.Hc + 4;
  return L;
}

struct Dims {
  int C, D, H, Cp, G;
  int SL;      // candidate slots per point = Cp*G + 1
  int stride;  // retained stride = min(Cp*G+1, C)
  int64_t N;   // rows of this context
  int64_t n0;  // global row offset
  int64_t Ntot;
};

// scoring modes
// kModeList: one-component re-scoring of listed output indices (the scores
// the anchor / extra / truncated-F passes flagged, grouped by component);
// entry = output index, row = entry / ScoreArgs.list_div
enum ScoreMode : int { kModeAnchor = 0, kModeExtra = 1, kModeTruncF = 2, kModeList = 3 };

struct ScoreArgs {
  Dims dm;
  ScoreLayout L;
  const float* X;
  const float* P;         // packed params, C x D x HP
  const double* kconst;   // log pi - 0.5 (D log 2pi + log|Sigma|), -inf if frozen
  const int* off;         // CSR offsets by component (C+1)
  const int* ent;         // CSR entries (flat K index n*Cp+j, or row n for extras)
  const int* itemoff;     // exclusive scan of per-component chunk counts (C+1)
  const int* g;           // neighbourhoods C x G
  const int* gcnt;
  float* out;             // LJ slots (N x SL) or LJK (N x Cp)
  int list_div = 1;       // kModeList: row = entry / list_div (SL or C')
};

struct SelectArgs {
  Dims dm;
  int* K;                 // in: old K (search space); out: new K
  const int* g;
  const int* gcnt;
  const int* rx;          // extra candidate per row
  const float* LJ;        // N x SL slots
  int* labels;
  float* lablj;           // log-joint of the label
  double* resp;           // N x Cp
  int* ret_cnt;
  int* ret_idx;           // N x stride
  float* ret_lj;          // N x stride
  double* lse;            // per-row log-sum-exp over new K (block-4 F terms)
  int* status;            // [0]: InsufficientCandidates flag
};

struct GupdArgs {
  Dims dm;
  int mode;               // 0 kl, 1 euclid
  const int* part_off;    // partition by label (C+1)
  const int* part_ent;
  const int* ret_cnt;
  const int* ret_idx;
  const float* ret_lj;
  const float* lablj;
  const double* logpi;    // fp64 log pi (-inf when pi == 0)
  int* g_new;
  int* gcnt_new;
  // global fallback tables (per CTA slice of C entries) for components whose
  // key bound exceeds the shared-memory hash
  long long* gt_cnt;
  long long* gt_hi;
  long long* gt_lo;
  // exchange (multi-rank) / dump modes
  const int* itemoff;     // items over the partition: chunks of pts_per_item points
  int pts_per_item;
  int exchange;           // 1: write dense C x C rows to xc_* instead of selecting
  int force_rows;         // 1: every item adds into the dense rows (large C); small hash, overflow -> xc
  long long* xc;          // 3*C*C int64: [cnt | hi | lo]
  int dump;               // 1: append (c, ct, cnt, hi, lo) rows to dump arrays
  int* dump_c;
  int* dump_ct;
  long long* dump_cnt;
  long long* dump_hi;
  long long* dump_lo;
  unsigned long long* dump_n;
  long long dump_cap;
  // sparse co-occurrence list (large C; SURVEY §8(e) sparse variant): every
  // item appends its exact (c, c~) partial sums; key = c << cl_kb | c~
  int list;
  unsigned* cl_key;
  long long* cl_cnt;
  long long* cl_hi;
  long long* cl_lo;
  unsigned long long* cl_n;
  long long cl_cap;
  int cl_kb;
  int* cl_ovf;
};

// reduced (unique-key) co-occurrence list and its selection
struct CoocArgs {
  Dims dm;
  int kb;                    // key = c << kb | c~
  const unsigned* key;       // sorted keys (n)
  const int* perm;           // sorted position -> source entry
  const long long* cnt;      // source entries (n)
  const long long* hi;
  const long long* lo;
  int n;
  int* head;                 // scratch (n): segment heads, then inclusive scan
  unsigned* u_key;           // unique keys (<= n)
  long long* u_cnt;
  long long* u_hi;
  long long* u_lo;
  int* u_off;                // C + 1: unique entries of component c
};

struct StatsArgs {
  Dims dm;
  const float* X;
  const double* resp;     // N x Cp
  const int* off;         // CSR by component over new K
  const int* ent;
  const float* V32;       // C x D x H  (V^T rows: mz = V (x - mu))
  const float* mu32;      // C x D
  const double* Sz;       // C x H x H
  double* Nc;
  double* E;              // C x (H+1)^2 col-major
  double* Y;              // C x (H+1) x D  (D x (H+1) col-major)
  double* sq;             // C x D
  int* qctr;              // work-queue counter (zeroed per pass; nullptr: static item order)
  const float* xmax = nullptr;   // per-row max |x| and per-component max |mu32| (the tcgen05
  const float* mumax = nullptr;  // kernel's row scales; nullptr: the mma.sync / FFMA kernels)
  const void* vimg = nullptr;    // its GEMM i B images (launch_stats_vimg, per precompute)
  const int* vexp = nullptr;
  const float* vl1 = nullptr;
  float* zbuf = nullptr;         // the tcgen05 kernel's zhat per K-pair (>= pairs x H floats)
};
// the tcgen05 statistics kernel takes the pass (opt-in: VMFA_STATS=tc)
bool stats_use_tc(const Dims& dm);
int stats_rows_cap(const Dims& dm);

struct UpdateArgs {
  Dims dm;
  const double* Nc;
  const double* E;
  const double* Y;
  const double* sq;
  const double* floor;
  const double* mu_prev;
  const double* lam_prev;
  const double* psi_prev;
  double* pi;
  double* mu;
  double* lam;
  double* psi;
  unsigned long long* status;  // min over (c << 8 | code)
};

struct PrecompArgs {
  Dims dm;
  ScoreLayout L;
  const double* pi;
  const double* mu;
  const double* lam;
  const double* psi;
  double* Lmat;           // C x H x H
  double* R;              // C x H x H (row-major lower Cholesky factor of Lmat)
  double* Sz;             // C x H x H
  double* logdet;
  double* logpi;
  double* kconst;
  float* P;               // packed scoring params
  float* V32;             // C x D x H
  float* mu32;            // C x D
  float* WT;              // C x Hp x D  K-major W rows (tensor-core scorer)
  float* ipsi32;          // C x D
  int Hp;                 // H padded to {4, 8, 16, 32, 64}
  unsigned long long* status;
  double* W64;            // C x H x D fp64 W^T = R^-1 Lambda^T Psi^-1 (fp64 re-scoring), or null
};

// launchers (return cudaError_t of the launch)
// vmfa_sort.cu: stable LSD radix sort of (key, value) pairs over 8-bit
// digits (vals null: value = input index; keys < 2^bits), the result in
// (kout, vout); ktmp / vtmp scratch of n entries; hist: sort_hist_ints(n)
// ints. scan_i32: int32 prefix sum (in == out allowed), tmp: scan_tmp_ints(n).
int64_t sort_hist_ints(int64_t n);
int64_t scan_tmp_ints(int64_t n);
cudaError_t radix_sort_pairs(const unsigned* keys, const int* vals, int64_t n, int bits, unsigned* ktmp, int* vtmp,
                             unsigned* kout, int* vout, int* hist, cudaStream_t s);
cudaError_t scan_i32(const int* in, int* out, int64_t n, bool inclusive, int* tmp, cudaStream_t s);
cudaError_t launch_iota(int* v, int64_t n, cudaStream_t s);
cudaError_t launch_fill_i32(int* v, int64_t n, int value, cudaStream_t s);
cudaError_t launch_keys_from_i32(const int* src, unsigned* keys, int64_t n, cudaStream_t s);
cudaError_t launch_hist(const unsigned* keys, int64_t n, int C, int* cnt, cudaStream_t s);
cudaError_t launch_chunks(const int* cnt, int C, int rows, int* chunks, cudaStream_t s);
cudaError_t launch_offsets_sorted(const unsigned* sorted, int64_t n, int C, int* off, cudaStream_t s);
cudaError_t launch_items_scan(const int* off, int C, int rows, int min1, int* items, cudaStream_t s);
cudaError_t launch_extra(const Dims& dm, const int* K, const int* g, const int* gcnt,
                         const unsigned long long* sit, int* rx, unsigned* rkey, cudaStream_t s);
cudaError_t launch_score(int mode, const ScoreArgs& a, int grid, cudaStream_t s);
cudaError_t launch_select(const SelectArgs& a, cudaStream_t s);
cudaError_t launch_gupdate(const GupdArgs& a, int grid, cudaStream_t s);
// sparse co-occurrence: heads of the sorted keys, (after an inclusive scan of
// the heads) exact per-key sums and per-component offsets, and g selection
// for components [c0, c1) (rows outside are zeroed when zero_others)
cudaError_t launch_cooc_heads(const CoocArgs& a, cudaStream_t s);
cudaError_t launch_cooc_sums(const CoocArgs& a, cudaStream_t s);
cudaError_t launch_cooc_select(const CoocArgs& a, int c0, int c1, int zero_others, int* g_new, int* gcnt_new,
                               cudaStream_t s);
cudaError_t launch_gselect_dense(const Dims& dm, long long* xc, const int* itemoff, int all,
                                 int* g_new, int* gcnt_new, cudaStream_t s);
cudaError_t launch_chunks_from_off(const int* off, int C, int rows, int min1, int* chunks,
                                   cudaStream_t s);
cudaError_t launch_stats(const StatsArgs& a, const int* itemoff, int rows_per_item, double* part,
                         cudaStream_t s);
int64_t stats_part_stride(const Dims& dm);
cudaError_t launch_update(const UpdateArgs& a, cudaStream_t s);
cudaError_t launch_renorm(const Dims& dm, double* pi, unsigned long long* status, cudaStream_t s);
cudaError_t launch_precompute(const PrecompArgs& a, cudaStream_t s);
cudaError_t launch_caches_full(const Dims& dm, const double* lam, const double* psi,
                               const double* R, double* U, double* V, double* ipsi,
                               cudaStream_t s);
cudaError_t launch_lse_rows(const float* LJK, int64_t N, int Cp, double* lse, cudaStream_t s);
cudaError_t launch_self_slots(const Dims& dm, const int* K, const int* g, const int* gcnt, const float* LJ,
                              float* LJK, cudaStream_t s);
cudaError_t launch_sum_f64(const double* v, int64_t n, double* partials, double* out,
                           cudaStream_t s);
cudaError_t launch_sum_i32(const int* v, int64_t n, unsigned long long* out, cudaStream_t s);
cudaError_t launch_count_empty(const double* pi, int C, int* out, cudaStream_t s);
cudaError_t launch_validate_K(const int* K, int64_t N, int Cp, int C, long long* bad, cudaStream_t s);
cudaError_t launch_logpi(const double* pi, int C, double* logpi, cudaStream_t s);

int sm_count();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and size:
// the call costs host time on every launch and opened gaps between queued
// kernels in the plain-launch (profiling) path
cudaError_t ensure_dyn_smem(const void* kern, size_t bytes);
// tensor-core scorer (vmfa_score_tc.cu)
bool score_tc_supported(const Dims& dm);
cudaError_t launch_score_tc(int mode, const ScoreArgs& s, const float* WT, const float* ipsi32,
                            const float* mu32, cudaStream_t st);
constexpr int kScoreRowsTc = 128;
// warp-specialised tensor-core scorer (vmfa_score_ws.cu)
int ws_hp(int H);  // W rows per component in WT (H padded to 8, 16, 32, 64)
bool score_ws_supported(const Dims& dm);
int ws_groups(const Dims& dm);
// operands of the scorer beyond ScoreArgs
struct WsOperands {
  const float* xmax;   // per row max |x| (N)
  const float* mumax;  // per component max |mu32| (C)
  const float* mu32;
  const float* brec;   // per (anchor, slot) epilogue records (per E-step)
  const float* srec;   // per component records (per precompute)
  const void* bimg;    // anchor-job B stage images (fp16 hi/lo), rebuilt per E-step
  const float* bscl;   // their row scales
  const void* simg;    // one-component B stage images (extra / truncated F), per precompute
  const float* sscl;
  long long* fix_list = nullptr;           // flagged scores: output indices (vmfa_fixup.cu)
  unsigned long long* fix_cnt = nullptr;   // [0] count, [1] overflow
  long long fix_cap = 0;
  const void* limg = nullptr;  // image-free anchor stages: lin / psi images (bimg unused)
};
// fp64 re-evaluation of the scores the tensor-core scorer flagged (vmfa_fixup.cu)
struct FixArgs {
  const float* X;
  const double* mu;
  const double* psi;
  const double* lam;
  const double* R;
  const double* kconst;
  const long long* list;         // flagged output indices appended by the scorer
  unsigned long long* cnt;       // [0] entries appended, [1] overflow (list full: scan instead)
  long long cap;                 // list capacity
  unsigned long long* nfix;      // scores re-evaluated (accumulated)
  int* qkey;                     // grouping scratch: component per entry (cap)
  int* sorted;                   // entries grouped by component (cap)
  int* qcnt;                     // per component (C), offsets (C+1), fill cursors (C)
  int* qoff;
  int* qfill;
  int* iof;                      // work-item offsets per component (C+1)
  unsigned long long* ovf;       // [1]: a list overflowed (the scan kernels run)
  const double* W64;             // C x H x D fp64 W^T from the precompute (DMMA re-scoring), or null
};
// the fp64 tensor-core (DMMA) re-scoring applies: H a multiple of 8 up to 32,
// D a multiple of 16, W^T of one component fits in shared memory
bool fix_dmma_ok(int D, int H);
cudaError_t launch_fix_ovf(const FixArgs& f, int first, cudaStream_t s);
cudaError_t launch_fix_group(const Dims& dm, const FixArgs& f, int mode, const int* K, const int* g, const int* rx,
                             cudaStream_t s);
cudaError_t launch_fix_f64(const Dims& dm, const FixArgs& f, int mode, const int* K, const int* g, const int* rx,
                           float* out, cudaStream_t s);
cudaError_t launch_fix_scan_anchor(const Dims& dm, const FixArgs& f, const int* g, const int* gcnt,
                                   const int* kinv_off, const int* kinv_ent, float* LJ, cudaStream_t s);
cudaError_t launch_fix_scan_single(const Dims& dm, const FixArgs& f, const int* off, const int* ent, int extra_stride,
                                   int extra_col, float* out, cudaStream_t s);
// the statistics on tcgen05 (vmfa_stats_tc.cu): H <= 16, D % 4 == 0, D <= 832;
// items of stats_tc_rows() K-pairs
bool stats_tc_ok(const Dims& dm);
int stats_tc_rows();
int64_t stats_tc_image_bytes(const Dims& dm);
cudaError_t launch_stats_vimg(const Dims& dm, const float* V32, void* img, int* vexp, float* vl1, cudaStream_t s);
cudaError_t launch_stats_tc(const StatsArgs& a, const float* xmax, const float* mumax, const int* itemoff, int nh1,
                            double* part, int64_t part_stride, cudaStream_t s);
// per-operation E-step pieces and log_joint (vmfa_ops.cu)
cudaError_t launch_log_joint_pairs(int D, int H, const float* X, const int* comp, int64_t n, const double* mu,
                                   const double* psi, const double* lam, const double* R, const double* kconst,
                                   double* out, cudaStream_t s);
cudaError_t launch_search_space(const Dims& dm, const int* K, const int* g, const int* gcnt, const int* extras,
                                uint64_t seed, uint64_t it, int* count, int* idx, cudaStream_t s);
cudaError_t launch_update_k(const Dims& dm, const int* count, const int* idx, const double* lj, int* Kout,
                            int* status, cudaStream_t s);
cudaError_t launch_hard_labels(const Dims& dm, const int* K, const int* count, const int* idx, const double* lj,
                               int* labels, cudaStream_t s);
cudaError_t launch_responsibilities(int64_t rows, int width, const double* lj, double* resp, cudaStream_t s);
cudaError_t launch_distances(const Dims& dm, int mode, const int* part_off, const int* part_ent, const int* count,
                             const int* idx, const double* lj, const double* pi, const int64_t* tab_off,
                             const int* tab_cap, int* key, double* sum, long long* cnt, int* nkeys, cudaStream_t s);
cudaError_t launch_update_g(int C, int G, const int64_t* row_off, const int* ct, const double* sum,
                            const long long* cnt, int* g, int* gcnt, cudaStream_t s);
// true while vmfa_diag_scorer_cycles has the scorer counters armed
bool ws_diag_armed();
cudaError_t launch_score_ws(int mode, const ScoreArgs& s, const WsOperands& op, int4* jobs, cudaStream_t st,
                            bool build_jobs = true);
// dense all-pairs pass (exact_log_likelihood): pseudo-anchor groups, per-chunk
// entries / row-tile-major jobs / item total, and the per-row LSE over C slots
cudaError_t launch_dense_groups(int C, int G, int* g, int* gcnt, cudaStream_t s);
cudaError_t launch_dense_chunk(int C, int G, int nb, int R, int* ent, int4* jobs, int* itemoff, cudaStream_t s);
cudaError_t launch_dense_csr(int C, int G, int R, int rows, int* off, int* itemoff, cudaStream_t s);
int64_t dense_jobs(int nb, int R);
cudaError_t launch_em_resp(const float* LJ, int64_t R, int SL, int C, const double* lse, double* resp, int* ent,
                           int* off, cudaStream_t s);
cudaError_t launch_add_f64(const double* a, double* acc, int64_t n, int first, cudaStream_t s);
cudaError_t launch_afkmc2(const float* X, int64_t N, int D, int C, int m, double* q, double* cdf, int64_t* centers,
                          unsigned long long* state, unsigned long long* count, int* degenerate, cudaStream_t s);
cudaError_t launch_lse_dense(const float* LJ, int64_t R, int SL, int C, double* lse, cudaStream_t s);
int64_t ws_record_floats(const Dims& dm, int single);
cudaError_t launch_ws_records(const Dims& dm, int single, const float* WT, const float* mu32, const float* ipsi32,
                              const double* kconst, const int* g, const int* gcnt, const float* scl, float* rec,
                              cudaStream_t s, int fused = 0, const double* logpi = nullptr,
                              const double* logdet = nullptr);
// B stage images (single != 0: one component per job), sizes in halves / floats
int64_t ws_image_halves(const Dims& dm, int single);
int64_t ws_scale_floats(const Dims& dm, int single);
cudaError_t launch_ws_images(const Dims& dm, int single, const float* WT, const float* mu32, const float* ipsi32,
                             const int* g, const int* gcnt, void* img, float* bscl, cudaStream_t s,
                             const float* sscl = nullptr, float* rec = nullptr, void* limg = nullptr);
int64_t ws_small_image_halves(const Dims& dm);
bool ws_image_free_ok(const Dims& dm);
// per-row max |value| of an N x D fp32 matrix (A-row scale bounds)
cudaError_t launch_rowmax(int64_t N, int D, const float* X, float* xmax, cudaStream_t s);

}  // namespace vmfa_b200
