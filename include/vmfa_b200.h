/*
 * vmfa_b200.h — C-ABI of the B200-native v-MFA hot path (libvmfa_b200.so).
 *
 * This is the drop-in boundary for the reference's public C++ API in
 * /root/reference/proj/include/vmfa/ (SURVEY.md §8(b)). The reference is a
 * C++20 library with Eigen types in its signatures; this ABI carries the same
 * data as plain pointers + sizes in the reference's own memory layouts
 * over an opaque device context, so the C++ façade in
 * include/vmfa_b200.hpp (reference names and semantics) and any FFI
 * (ctypes/cgo/JNI) can bind it. No torch or CUDA types appear here; streams
 * are passed as void*.
 *
 * Layouts (identical to the reference's):
 *   X       N x D float32 row-major                        (dataset.hpp:13-14)
 *   pi      C float64                                       (model.hpp:25)
 *   mu      C x D float64 row-major                         (model.hpp:26)
 *   lambda  C blocks, each D x H column-major (d,h) at h*D+d (model.hpp:27)
 *   dnoise  C x D float64 row-major (Psi, variances)        (model.hpp:28)
 *   K       N x C' int32 row-major, rows sorted ascending   (model.hpp:90-103)
 *   g       C x G int32 row-major, rows sorted, -1 padded, plus g_count[C]
 *                                                           (estep.hpp:22)
 *   labels  N int32                                         (estep.hpp:24)
 *   retained: count[N], idx[N*stride] (-1 pad), lj[N*stride] float64 with
 *            stride = min(C'*G+1, C)                        (estep.hpp:48-70)
 *   resp    N x C' float64, aligned with K rows             (estep.hpp:74)
 *   caches: U C x (D x H col-major), Lmat/Sigma_z C x (H x H col-major),
 *           V C x (H x D col-major), inv_dnoise C x D, logdet C, log_pi C
 *                                                           (model.hpp:37-45)
 *   stats:  Nc C, Y C x (D x (H+1) col-major), E C x ((H+1)^2 col-major),
 *           sq_sum C x D                                    (mstep.hpp:14-22)
 *
 * Error model: every entry returns a vmfa_status; codes map 1:1 onto the
 * reference's exception types (errors.hpp:9-62) plus std::invalid_argument.
 * vmfa_last_error() returns a thread-local message for the last failure.
 * Calls are stream-ordered on the context's stream and synchronous unless the
 * name ends in _async; results returned through host pointers are complete on
 * return.
 */
#ifndef VMFA_B200_H_
#define VMFA_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VMFA_ABI_VERSION 1

typedef enum vmfa_status {
  VMFA_OK = 0,
  VMFA_ERR_INVALID_ARGUMENT = 1,       /* std::invalid_argument            */
  VMFA_ERR_CHOLESKY_FAILURE = 2,       /* vmfa::CholeskyFailure errors.hpp:16 */
  VMFA_ERR_EMPTY_KSET = 3,             /* vmfa::EmptyKSet        errors.hpp:21 */
  VMFA_ERR_INSUFFICIENT_CANDIDATES = 4,/* vmfa::InsufficientCandidates :26 */
  VMFA_ERR_SINGULAR_EC = 5,            /* vmfa::SingularEc       errors.hpp:31 */
  VMFA_ERR_MAX_ITER_EXCEEDED = 6,      /* vmfa::MaxIterExceeded  errors.hpp:36 */
  VMFA_ERR_TARGET_UNREACHABLE = 7,     /* vmfa::TargetUnreachable errors.hpp:41 */
  VMFA_ERR_DEGENERATE_DATA = 8,        /* vmfa::DegenerateData   errors.hpp:46 */
  VMFA_ERR_BAD_MAGIC = 9,              /* vmfa::BadMagic         errors.hpp:51 */
  VMFA_ERR_TRUNCATED_FILE = 10,        /* vmfa::TruncatedFile    errors.hpp:56 */
  VMFA_ERR_UNSUPPORTED_VERSION = 11,   /* vmfa::UnsupportedVersion errors.hpp:61 */
  VMFA_ERR_IO = 12,                    /* vmfa::Error (errors.hpp:9): cannot open / write, invalid header sizes */
  VMFA_ERR_CUDA = 100,                 /* CUDA runtime failure (no reference twin) */
  VMFA_ERR_NO_DEVICE = 101,            /* no usable sm_100 device          */
  VMFA_ERR_UNSUPPORTED = 102           /* shape/feature outside this build */
} vmfa_status;

typedef enum vmfa_distance_mode {
  VMFA_DIST_KL = 0,     /* DistanceMode::kl     estep.hpp:12 */
  VMFA_DIST_EUCLID = 1  /* DistanceMode::euclid estep.hpp:12 */
} vmfa_distance_mode;

typedef struct vmfa_ctx vmfa_ctx;

/* ------------------------------------------------------------------ misc */
int vmfa_abi_version(void);
const char* vmfa_last_error(void);
/* 1 if a CUDA device of compute capability 10.x is visible, else 0. */
int vmfa_device_available(void);

/* ------------------------------------------------------------------ context
 * A context owns one GPU's shard of the data (rows [n_offset, n_offset+n_local)
 * of an n_total-row dataset), replicated parameters and caches, the variational
 * state of its rows, and all scratch. The global row index n_offset+n keys the
 * per-point random extra candidate (rng.hpp:91-98, estep.cpp:259-260), so a
 * sharded run draws exactly the candidates of the unsharded one.
 * stream: a cudaStream_t (NULL = create a private non-blocking stream).    */
int vmfa_ctx_create(vmfa_ctx** out, int device, int C, int D, int H, int Cprime, int G,
                    int64_t n_local, int64_t n_offset, int64_t n_total, void* stream);
int vmfa_ctx_destroy(vmfa_ctx* ctx);
/* Device bytes held by the context (data + state + params + scratch). */
int vmfa_ctx_device_bytes(const vmfa_ctx* ctx, size_t* bytes);

/* ------------------------------------------------------------------ data
 * Dataset rows (dataset.hpp:11-35). rows may be a sub-range of the shard:
 * local rows [row_begin, row_begin+rows). Host memory may be pageable or
 * pinned.                                                                   */
int vmfa_upload_data(vmfa_ctx* ctx, const float* X, int64_t row_begin, int64_t rows);
/* The same, asynchronous: the rows are copied on a second stream while the
 * context keeps working (parameter / state uploads, the E-step's CSR and image
 * builds); the first kernel that reads X waits for the copy. X must stay
 * valid and unchanged until the next call that synchronises the context
 * (iterate, any download, ...). Page-locked X gives a truly asynchronous copy. */
int vmfa_upload_data_async(vmfa_ctx* ctx, const float* X, int64_t row_begin, int64_t rows);
/* Pipelined uploads (a second device row buffer): vmfa_stage_data_async
 * copies rows into the staging buffer on the copy stream, after the work
 * already enqueued that may still read it; vmfa_swap_data makes the staged
 * rows current (later work waits for their copy) and the previous rows the
 * staging buffer. A training / serving loop stages the next batch while the
 * current one is processed. X stays valid until the next synchronising call. */
int vmfa_stage_data_async(vmfa_ctx* ctx, const float* X, int64_t row_begin, int64_t rows);
int vmfa_swap_data(vmfa_ctx* ctx);
/* Lookahead (default on, env VMFA_LOOKAHEAD=0 turns it off): the truncated
 * free energy after the M-step is read from the next E-step's anchor pass,
 * which that E-step then skips. Off: F gets its own one-component pass (same
 * value) -- cheaper when the caller re-uploads data or state every iteration. */
int vmfa_set_lookahead(vmfa_ctx* ctx, int enable);
/* Variance floor max(1e-8, 1e-6 var_d) (dataset.cpp:37-39), computed by the
 * caller over ALL n_total rows (global).                  */
int vmfa_set_floor(vmfa_ctx* ctx, const double* floor);

/* ------------------------------------------------------------------ params / caches */
/* MfaParams (model.hpp:19-32). Upload also runs precompute_all.            */
int vmfa_upload_params(vmfa_ctx* ctx, const double* pi, const double* mu, const double* lambda,
                       const double* dnoise);
int vmfa_download_params(vmfa_ctx* ctx, double* pi, double* mu, double* lambda, double* dnoise);
/* precompute_all (model.cpp:75-79) on the device. On CholeskyFailure the
 * failing component index is written to *failed (may be NULL).             */
int vmfa_precompute(vmfa_ctx* ctx, int* failed);
/* ComponentCache for all C components (model.hpp:37-45); any pointer may be
 * NULL to skip that field.                                                  */
int vmfa_download_caches(vmfa_ctx* ctx, double* U, double* Lmat, double* V, double* Sigma_z,
                         double* inv_dnoise, double* logdet, double* log_pi);

/* ------------------------------------------------------------------ variational state */
/* VarState (estep.hpp:17-29): K rows (sorted), g rows (sorted, -1 padded).  */
int vmfa_upload_state(vmfa_ctx* ctx, const int32_t* K, const int32_t* g, const int32_t* g_count);
int vmfa_download_state(vmfa_ctx* ctx, int32_t* K, int32_t* g, int32_t* g_count, int32_t* labels);

/* ------------------------------------------------------------------ the hot path */
/* variational_e_step (estep.hpp:125-130, estep.cpp:230-336): blocks 1-4 at the
 * current parameters. Updates K, labels, partition and g in place; returns the
 * block-4 free energy (sum over this context's rows) and the joint count
 * sum_n |S(n)| of this context's rows. On a multi-context (multi-GPU) run use
 * the phase API below instead so g is computed from all ranks' rows.        */
int vmfa_estep(vmfa_ctx* ctx, uint64_t seed, uint64_t iteration, int mode, double* free_energy,
               uint64_t* joints);
/* EStepResult pieces for parity (estep.hpp:72-78): retained joints (stride =
 * min(C'G+1, C)) and responsibilities of the last E-step. NULL skips.       */
int vmfa_download_estep(vmfa_ctx* ctx, int32_t* count, int32_t* idx, double* lj, double* resp);
/* Block-3 accumulator of the last E-step (DistanceAccumulator, estep.hpp:34-44)
 * as (c, ctilde, sum, count) rows in (c, ctilde) ascending order. Pass cap=0
 * to query the row count in *n_rows.                                        */
int vmfa_download_distances(vmfa_ctx* ctx, int64_t cap, int32_t* c, int32_t* ct, double* sum,
                            int64_t* count, int64_t* n_rows);

/* accumulate_suffstats (mstep.hpp:27-31) with the pre-update caches and the
 * last E-step's K/resp, into the context's statistics buffer.               */
int vmfa_accumulate_suffstats(vmfa_ctx* ctx);
int vmfa_download_suffstats(vmfa_ctx* ctx, double* Nc, double* Y, double* E, double* sq_sum);
int vmfa_upload_suffstats(vmfa_ctx* ctx, const double* Nc, const double* Y, const double* E,
                          const double* sq_sum);
/* update_params (mstep.hpp:39-41, mstep.cpp:103-162) from the statistics
 * buffer, then precompute_all. *failed receives the failing component.      */
int vmfa_update_params(vmfa_ctx* ctx, int* failed);
/* truncated_free_energy (model.hpp:116-119) over this context's rows under
 * the current parameters and K.                                             */
int vmfa_truncated_free_energy(vmfa_ctx* ctx, double* free_energy);
/* exact_log_likelihood (model.hpp:108-111) over this context's rows.        */
int vmfa_exact_log_likelihood(vmfa_ctx* ctx, double* log_likelihood);
/* em_full_step (mstep.cpp:164-208, used by run_emmfa_loop trainer.cpp:228):
 * every (n, c) log-joint (the dense pass above), q(n, c) = exp(l - LSE_n)
 * over all C, and the sufficient statistics over every pair; returns
 * sum_n LSE_n and N*C joints. The statistics stay in the context
 * (vmfa_download_suffstats / vmfa_update_params follow).                   */
int vmfa_em_full_step(vmfa_ctx* ctx, double* log_likelihood, uint64_t* joints);
/* afkmc2_seed (seeding.cpp:60-121; the reference's default InitConfig
 * method): C seed rows of this context's data (the whole dataset), the
 * xoshiro256++ stream state after the draws (init_params continues it,
 * trainer.cpp:36-44) and the squared-distance count (EvalCounter::distances).
 * DegenerateData when fewer than C distinct rows exist.                    */
int vmfa_afkmc2_seed(vmfa_ctx* ctx, int C, int chain_length, uint64_t stream_seed, int64_t* seeds,
                     uint64_t* stream_state, uint64_t* distances);

/* ---- reference entry points with caller-supplied state (mstep.hpp:27-31,
 * model.hpp:116-119). Both replace the context's K with `K` (N x C', rows
 * sorted, validated like vmfa_upload_state).
 * accumulate_suffstats(params, caches, data, ksets, resp): statistics of the
 * given K rows and responsibilities (N x C' fp64, aligned with K) under the
 * context's (pre-update) parameters, into the statistics buffer -- e.g. the
 * per-cluster FA fit of kmeans.cpp:195-210 (C = C' = 1, K = 0, resp = 1).  */
int vmfa_accumulate_suffstats_k(vmfa_ctx* ctx, const int32_t* K, const double* resp);
/* truncated_free_energy(params, caches, data, ksets): sum_n LSE over the
 * given K rows under the context's parameters (EmptyKSet for K == NULL).   */
int vmfa_truncated_free_energy_k(vmfa_ctx* ctx, const int32_t* K, double* free_energy);

/* ---- log_joint (model.hpp:83-86, model.cpp:81-95), batched: out[i] =
 * log p(c_i, x_i) for n rows X (n x D, host) and components comp[i], in fp64
 * under the context's parameters (the reference's EvalCounter adds n).     */
int vmfa_log_joint(vmfa_ctx* ctx, const float* X, int64_t n, const int32_t* comp, double* out);

/* ---- the E-step's per-operation pieces (estep.hpp:82-117), each batched
 * over the context's N rows (stride = min(C'G+1, C)); host arrays in the
 * reference layouts (RetainedJoints: count N, idx / lj N x stride).
 *   build_search_space (estep.cpp:126-133): S(n) of the context's K and g
 *     with extra r_n = extras[n], or (extras == NULL) uniform_component(seed,
 *     iteration, n_offset + n, C) (rng.hpp:91-98), insertion order, -1 pad;
 *   update_k (estep.cpp:135-142): top-C' of each row by (l desc, index asc),
 *     sorted ascending; InsufficientCandidates if count < C';
 *   hard_partition (estep.cpp:144-173): labels and the partition as offsets
 *     (C+1) and rows (N, ascending within each component);
 *   accumulate_distances (estep.cpp:175-202): block 3's accumulator as rows
 *     (c, ct, sum, count) in (c, ct) order (fp64 sums in the reference's
 *     per-key order); pass cap = 0 to query the row count in *n_rows;
 *   update_g (estep.cpp:204-220): g rows (C x G, -1 padded) + counts from
 *     accumulator rows;
 *   responsibilities_row (estep.cpp:222-228): rows x width softmax.        */
int vmfa_build_search_space(vmfa_ctx* ctx, uint64_t seed, uint64_t iteration, const int32_t* extras,
                            int32_t* count, int32_t* idx);
int vmfa_update_k(vmfa_ctx* ctx, const int32_t* count, const int32_t* idx, const double* lj, int32_t* K);
int vmfa_hard_partition(vmfa_ctx* ctx, const int32_t* K, const int32_t* count, const int32_t* idx,
                        const double* lj, int32_t* labels, int32_t* part_off, int32_t* part_ent);
int vmfa_accumulate_distances(vmfa_ctx* ctx, int mode, const int32_t* part_off, const int32_t* part_ent,
                              const int32_t* count, const int32_t* idx, const double* lj, const double* pi,
                              int64_t cap, int32_t* c, int32_t* ct, double* sum, int64_t* count_out,
                              int64_t* n_rows);
int vmfa_update_g(vmfa_ctx* ctx, int64_t n_rows, const int32_t* c, const int32_t* ct, const double* sum,
                  const int64_t* count, int32_t* g, int32_t* g_count);
int vmfa_responsibilities(vmfa_ctx* ctx, int64_t rows, int width, const double* lj, double* resp);

/* One main-loop iteration of train_vmfa (trainer.cpp:149-160): E-step,
 * statistics, update, precompute, post-M-step truncated free energy.
 * Single-context only (use the phase API for multi-GPU).                    */
typedef struct vmfa_iter_report {
  double free_energy_estep; /* block-4 F(K_new, Theta_old), estep.cpp:316-334 */
  double free_energy;       /* F(K_new, Theta_new), trainer.cpp:158-160      */
  uint64_t joints;          /* sum_n |S(n)|                                  */
  int32_t empty_components; /* pi == 0 count, trainer.cpp:27-29              */
  int32_t failed_component; /* component of a CholeskyFailure/SingularEc     */
} vmfa_iter_report;
int vmfa_iterate(vmfa_ctx* ctx, uint64_t seed, uint64_t iteration, int mode,
                 vmfa_iter_report* report);

/* ------------------------------------------------------------------ multi-GPU phase API
 * Data-parallel over points: each rank runs the phases on its
 * shard and sums the exchange buffers across ranks between phases (NCCL
 * all-reduce over NVLink; the caller owns the communicator). Exchange buffers
 * are device pointers in the context:
 *   VMFA_XCHG_COOC   int64 buffer: dense C x C co-occurrence accumulator
 *                    (count, fixed-point sum hi, lo) — exact integer sums, so
 *                    g is bit-identical for every rank count.
 *   VMFA_XCHG_STATS  float64 buffer: [Nc | E | Y | sq_sum] packed.
 *   VMFA_XCHG_SCALARS float64 buffer: [F_estep, joints, F_post] partials.
 * Sequence per main iteration:
 *   vmfa_phase_estep_local -> allreduce(COOC) -> vmfa_phase_estep_finish ->
 *   vmfa_phase_stats_local -> allreduce(STATS) -> vmfa_phase_update ->
 *   vmfa_phase_free_energy_local -> allreduce(SCALARS).                    */
typedef enum vmfa_exchange {
  VMFA_XCHG_COOC = 0,
  VMFA_XCHG_STATS = 1,
  VMFA_XCHG_SCALARS = 2,
  VMFA_XCHG_G = 3
} vmfa_exchange;
typedef enum vmfa_dtype { VMFA_DT_INT64 = 0, VMFA_DT_FLOAT64 = 1, VMFA_DT_INT32 = 2 } vmfa_dtype;
int vmfa_exchange_buffer(vmfa_ctx* ctx, int which, void** device_ptr, size_t* count, int* dtype);
int vmfa_phase_estep_local(vmfa_ctx* ctx, uint64_t seed, uint64_t iteration, int mode);
int vmfa_phase_estep_finish(vmfa_ctx* ctx);
int vmfa_phase_stats_local(vmfa_ctx* ctx);
int vmfa_phase_update(vmfa_ctx* ctx, int* failed);
int vmfa_phase_free_energy_local(vmfa_ctx* ctx);
/* Reads the (reduced) scalars buffer: F_estep, joints, F_post.             */
int vmfa_phase_scalars(vmfa_ctx* ctx, double* free_energy_estep, uint64_t* joints,
                       double* free_energy);
/* Sparse co-occurrence exchange (SURVEY §8(e) sparse variant; used when C is
 * too large for the dense table: C > 4096 in a sharded context (C > ~18900
 * in a single one), or with VMFA_COOC=sparse at
 * context creation). In place of allreduce(COOC):
 *   vmfa_phase_estep_local   (each rank reduces its (c, c~) list by key)
 *   vmfa_cooc_local_list     (device arrays key u32 = c << b | c~, cnt/hi/lo
 *                             int64, sorted by key; counts[r] = entries owned
 *                             by rank r = components [rC/p, (r+1)C/p), which
 *                             are contiguous)
 *   all-to-all of the four arrays with those counts (NCCL send/recv)
 *   vmfa_cooc_select         (the received lists, concatenated: reduced by key
 *                             and g_c selected for this rank's components into
 *                             the VMFA_XCHG_G buffer, other rows zero)
 *   allreduce(G, int32 sum) -> vmfa_phase_estep_finish.
 * The per-key sums are exact integers, so g is bit-identical to the dense
 * path for every rank count. Replaces estep.cpp:286-312's accumulator +
 * update_g (estep.cpp:204-220) across ranks.                              */
int vmfa_cooc_sparse(vmfa_ctx* ctx, int* sparse);
int vmfa_cooc_local_list(vmfa_ctx* ctx, int world, void** key, void** cnt, void** hi, void** lo,
                         int64_t* counts);
int vmfa_cooc_select(vmfa_ctx* ctx, const void* key, const void* cnt, const void* hi, const void* lo,
                     int64_t n, int rank, int world);

/* ------------------------------------------------------------------ timing / profiling */
/* Records CUDA events around the scoring kernels of subsequent calls;
 * vmfa_kernel_times returns accumulated milliseconds and launch counts per
 * kernel family since the last reset (names in vmfa_kernel_name).          */
int vmfa_profile_enable(vmfa_ctx* ctx, int enable);
int vmfa_kernel_times(vmfa_ctx* ctx, int max, double* ms, int64_t* launches, int64_t* units,
                      int* n);
const char* vmfa_kernel_name(int i);
/* Diagnostics: per-role cycle counters of the warp-specialised scorer summed
 * over CTAs since the last read (producer: wait-accumulator, job sync, wait
 * stage, build; MMA: wait-accumulator, wait stage, issue; epilogue: wait,
 * work). enable=1 arms (or keeps) the counters; out (n entries) reads and
 * clears them; enable=0 disarms.                                            */
int vmfa_diag_scorer_cycles(int enable, unsigned long long* out, int n);

/* Diagnostic: the K1 inversion's device radix sort (vmfa_sort.cu) on n host
 * keys < 2^bits, run `reps` times; keys_out / vals_out get the stably sorted
 * keys and their input indices. Returns the number of repetitions whose
 * output differed from the first (0), or -1 on a CUDA error.              */
int vmfa_diag_radix_sort(const uint32_t* keys, int64_t n, int bits, uint32_t* keys_out, int32_t* vals_out, int reps);

/* Work accounting of the candidate-scoring launches (the anchor pass and the
 * extras of one E-step) for roofline figures: out[0] anchor row visits
 * (N*C'), out[1] extra row visits of the last E-step (rows whose r_n is not
 * in the union of their anchors' g), out[2] / out[3] bytes of the anchor /
 * one-component B stage images, out[4] bytes of the epilogue records,
 * out[5] the scorer (2 warp-specialised tcgen05, 1 single-role tcgen05, 0
 * FFMA), out[6] scores re-evaluated in fp64 since the last call (the
 * scorer flags scores whose terms cancel, vmfa_fixup.cu), out[7] flagged
 * scores re-scored by the one-component tensor pass since the last call
 * (out[6] is what that pass still flagged). n: entries wanted (<= 8).       */
int vmfa_scoring_work(vmfa_ctx* ctx, int64_t* out, int n);

/* Stream of the context (a cudaStream_t) for callers that order their own
 * work (e.g. NCCL) against it.                                              */
void* vmfa_ctx_stream(vmfa_ctx* ctx);
int vmfa_synchronize(vmfa_ctx* ctx);

/* ------------------------------------------------------------------ host-side helpers
 * Host-only (no GPU needed): synthetic data for BASELINE.json's configs and
 * the reference's initialisation (trainer.cpp:32-47, 107-109), restated
 * with identical draw sequences.                                            */
typedef struct vmfa_synth_spec {
  int kind;            /* 0: Gaussian MFA (configs 1,2,4); 1: image-like fields (3,5) */
  int64_t n_total;     /* N                                                   */
  int D;               /* data dimension                                      */
  int C_true;          /* ground-truth components                             */
  int H_true;          /* ground-truth latent dimension                        */
  int dirichlet;       /* 1: pi ~ Dirichlet(1); 0: equiprobable               */
  double mu_std;       /* kind 0: mu ~ N(0, mu_std^2 I)                       */
  double lam_std;      /* kind 0: Lambda ~ N(0, lam_std^2); kind 1: field std  */
  double psi_lo, psi_hi; /* kind 0: Psi ~ U[psi_lo, psi_hi]                   */
  double noise_std;    /* kind 1: isotropic noise std                         */
  int img_w, img_h, img_c; /* kind 1: field geometry (D = w*h*c)             */
  double blur_sigma;   /* kind 1: Gaussian blur sigma in pixels               */
  uint64_t data_seed;
} vmfa_synth_spec;
/* Fills rows [row_begin, row_end) of X (row-major, (row_end-row_begin) x D);
 * labels (nullable) receives the true component per row. Each row draws from
 * its own keyed stream, so shards can be generated independently.          */
int vmfa_gen_synthetic(const vmfa_synth_spec* spec, int64_t row_begin, int64_t row_end,
                       float* X, int32_t* labels, int threads);

/* Initialisation (random-points seeding): floor (D), params, K (N x C'),
 * g (C x G) + g_count. loading_init 0 = reference U[0, scale) (seeding.cpp:
 * 175-176); 1 = BASELINE's N(0, scale^2) from the same stream. The caller's X
 * is the FULL dataset (N x D).                                              */
int vmfa_host_initialize(const float* X, int64_t N, int D, int C, int H, int Cprime, int G,
                         uint64_t seed, double scale, int loading_init, double* floor,
                         double* pi, double* mu, double* lambda, double* dnoise, int32_t* K,
                         int32_t* g, int32_t* g_count, int64_t* seeds);

/* Sharded initialisation: the same result as
 * vmfa_host_initialize without any rank holding all N rows. Protocol (the
 * caller owns the collectives; paper_2501_12299_b200/sharded.py runs it over
 * torch.distributed):
 *   1. variance (dataset.cpp:22-35): vmfa_host_moments(shard, mean=NULL) ->
 *      all-reduce -> mean = sum/N; vmfa_host_moments(shard, mean) -> all-reduce
 *      -> var = sum/N; floor = max(1e-6 var, 1e-8) (dataset.cpp:37-39);
 *   2. count_distinct_rows (seeding.cpp:16-32): vmfa_host_distinct_hashes on
 *      each shard (up to C distinct rows, 128-bit digests) -> all-gather ->
 *      fewer than C distinct digests = DegenerateData;
 *   3. random_points_seed (seeding.cpp:123-149): the draw sequence
 *      vmfa_seed_draws(seed, N, first, count) is data independent; the owners
 *      of the drawn rows contribute their contents (an exact integer-sum
 *      all-reduce of the bit patterns) and every rank applies the reference's
 *      used / duplicate rejection in draw order, counting the draws consumed;
 *   4. vmfa_host_init_shard: init_params (seeding.cpp:151-181) continuing the
 *      init stream after seed_draws draws, and init_varstate (seeding.cpp:
 *      207-233) replaying its whole stream but storing only K rows
 *      [n0, n0+rows).                                                        */
/* per-dimension fp64 sums over the rows in order: sum x (mean == NULL) or
 * sum (x - mean)^2. threads <= 0: all hardware threads.                     */
int vmfa_host_moments(const float* X, int64_t rows, int D, const double* mean, double* out, int threads);
/* draws [first, first+count) of the init stream Rng(hash_combine(seed,
 * 0x1217f01d)) (trainer.cpp:36) as uniform_int(N) (rng.hpp:55-60)          */
int vmfa_seed_draws(uint64_t seed, int64_t N, int64_t first, int64_t count, int64_t* out);
/* up to `want` distinct rows of X, in row order: two 64-bit digests each
 * (out: 2*want u64), *n_out = rows digested                                  */
int vmfa_host_distinct_hashes(const float* X, int64_t rows, int D, int64_t want, uint64_t* out,
                              int64_t* n_out);
/* var, floor: D; seeds: C global row indices; seed_rows: their contents
 * (C x D); seed_draws: draws random_points_seed consumed. Outputs as
 * vmfa_host_initialize, with K holding rows [n0, n0 + rows) only.            */
int vmfa_host_init_shard(int64_t N, int D, int C, int H, int Cprime, int G, uint64_t seed, double scale,
                         int loading_init, const double* var, const double* floor, const int64_t* seeds,
                         const float* seed_rows, int64_t seed_draws, int64_t n0, int64_t rows, double* pi,
                         double* mu, double* lambda, double* dnoise, int32_t* K, int32_t* g,
                         int32_t* g_count);

/* ---- on-disk containers, host only, no device needed ----
 * MFAD dataset (io.hpp:12-16, io.cpp:91-125): "MFAD", u32 version 1, u64 N,
 * u32 D, u8 dtype 0 (f32), 7 reserved bytes, N x D f32 row-major, little-endian.
 * Loads take a row range so each rank reads only its shard.                 */
int vmfa_save_dataset(const char* path, const float* X, int64_t N, int D);
int vmfa_dataset_info(const char* path, int64_t* N, int* D);
int vmfa_load_dataset(const char* path, int64_t row_begin, int64_t rows, int D, float* X);
/* MFAM checkpoint (io.hpp:18-23, io.cpp:127-179): "MFAM", u32 version 1, u32 C,
 * D, H, then pi, mu, Lambda (row-major D x H per component in the file; this
 * ABI's column-major blocks in memory), dnoise as f64. Save validates like
 * MfaParams::validate (model.cpp:14-41).                                      */
int vmfa_save_checkpoint(const char* path, int C, int D, int H, const double* pi, const double* mu,
                         const double* lambda, const double* dnoise);
int vmfa_checkpoint_info(const char* path, int* C, int* D, int* H);
int vmfa_load_checkpoint(const char* path, int C, int D, int H, double* pi, double* mu, double* lambda,
                         double* dnoise);
/* MFAK variational-state sidecar (this project, for exact resume): "MFAK",
 * u32 version 1, u64 N, u32 C', u32 C, u32 G, then K (i32 N x C'), g (i32
 * C x G), g_count (i32 C).                                                    */
int vmfa_save_state(const char* path, int64_t N, int Cprime, int C, int G, const int32_t* K,
                    const int32_t* g, const int32_t* g_count);
int vmfa_state_info(const char* path, int64_t* N, int* Cprime, int* C, int* G);
int vmfa_load_state(const char* path, int64_t row_begin, int64_t rows, int Cprime, int C, int G,
                    int32_t* K, int32_t* g, int32_t* g_count);

#ifdef __cplusplus
}
#endif
#endif /* VMFA_B200_H_ */
