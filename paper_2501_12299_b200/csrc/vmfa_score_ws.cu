// vmfa_score_ws.cu — warp-specialised tcgen05 scorer of the candidate
// log-joints (log_joint, model.cpp:81-95) over anchor blocks.
//
// Same mathematics as vmfa_score_tc.cu (rows centred on the anchor mean,
// 3xTF32 split products, fp32 accumulation in TMEM):
//   GEMM1  [v]   (128 x D) x [ -2 psi_q^-1 delta_q (16 rows) | W_q (Hp rows per q) ]
//   GEMM2  [v^2] (128 x D) x [ psi_q^-1 (16 rows) ]
// with delta_q = mu_q - mu_a, and per-(anchor, q) constants b = W_q^T delta_q,
// m = sum psi_q^-1 delta_q^2 precomputed once per E-step (k_anchor_consts):
//   y_q = acc_W - b,   diag_q = acc_psi + acc_lin + m,
//   l = kconst_q - 0.5 (diag_q - |y_q|^2).
// Roles (13 warps):
//   warps 0-7  producers: gather + centre + split the 128 rows of each K
//              chunk (A tiles), build the lin / psi^-1 B rows, and bulk-copy
//              the per-component pre-split, pre-swizzled W blocks
//              (cp.async.bulk, mbarrier transaction count);
//   warp  8    MMA issuer: tcgen05.mma.kind::tf32 from smem descriptors,
//              tcgen05.commit to the stage's empty barrier;
//   warps 9-12 epilogue: tcgen05.ld of a finished accumulator (TMEM double
//              buffered), log-joint assembly, scatter to the candidate slots.
#include <algorithm>
#include <cstdint>

#include "vmfa_b200.h"
#include "vmfa_kernels.cuh"

namespace vmfa_b200 {
namespace {

constexpr int kRows = 128;
constexpr int kKC = 32;               // K chunk: 32 tf32 = one 128-byte swizzle row
constexpr int kTileA = kRows * 128;   // 16 KB
constexpr int kProdWarps = 8;
constexpr int kMmaWarp = 8;
constexpr int kEpiWarp0 = 9;
constexpr int kLoadWarp = 13;         // B-loader warp
constexpr int kThreads = (kLoadWarp + 1) * 32;
constexpr int kMaxNB = 8;             // B ring stages (smem)
constexpr int kAhead = 5;             // producer row prefetch depth (chunks, cp.async ring)
constexpr int kProdThreads = kProdWarps * 32;
constexpr uint32_t kXRingBytes = (kAhead + 1) * 4 * kProdThreads * 16;
constexpr int kMaxD = 1024;
constexpr int kNL = 16;               // lin rows / psi rows per group (qg <= 16)

struct WsArgs {
  Dims dm;
  int mode;
  int Hp;            // W rows per component (>= 8)
  int qg;            // components per job (group)
  int N1max;         // 16 + round16(qg * Hp)
  int nbstage;        // B ring depth
  int nacc;          // accumulator buffers in TMEM (2 when they fit beside the A stages)
  uint32_t tmem_cols;
  uint32_t TB;       // TMEM columns per accumulator buffer
  uint32_t stage_bytes;
  const float* X;
  const float* WTS;  // [C][nchunk][2][Hp][32] pre-split, pre-swizzled W blocks
  const float* mu32;
  const float* ipsi32;
  const double* kconst;
  const float* acst; // [C][G][Hp + 1] : b (Hp) then m, anchor mode only
  const float* img;  // B stage images [C][groups][nchunk][stage] (nullptr: per-block copies)
  const float* lblk; // anchor mode: [C][ngroups][nchunk][4][16][32] lin hi|lo, psi hi|lo tiles
  const float* cblk; // single mode: [C][nchunk][4][16][32] (lin = 0, psi row 0)
  int ngroups;
  const int4* jobs;  // per item {component, first CSR row, rows, components}
  const int* itemoff;
  const int* ent;
  const int* g;
  const int* gcnt;
  float* out;
  unsigned long long* prof;  // optional per-role cycle counters (nullptr: off)
  int dbg;                   // diagnostics only: bit0 skip x loads, bit1 skip B copies
};

// per-role cycle accounting (debug builds of the pipeline; prof == nullptr in production)
enum ProfSite { kPWaitTE, kPSync, kPWaitEmpty, kPBuild, kMWaitTE, kMWaitFull, kMIssue, kEWait, kEWork, kPSplit, kPStore, kNumSites };
struct Prof {
  unsigned long long acc[kNumSites];
  unsigned long long t;
  __device__ void start() { t = clock64(); }
  __device__ void lap(int site) {
    const unsigned long long now = clock64();
    acc[site] += now - t;
    t = now;
  }
};

// timeline trace of CTA 0 (diagnostics): slot = 16 + 4 * event_index + kind
constexpr int kTraceEvents = 512;
__device__ __forceinline__ void trace(unsigned long long* prof, int idx, int kind) {
  if (prof && blockIdx.x == 0 && idx < kTraceEvents) prof[16 + 8 * idx + kind] = clock64();
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void split(float x, uint32_t& hi, uint32_t& lo) {
  hi = to_tf32(x);
  lo = to_tf32(x - __uint_as_float(hi));
}
// hi = x rounded to tf32 (nearest, ties away: +half an ulp of tf32 on the
// magnitude bits, then truncate), lo = x - hi exactly (the tensor core reads
// its top 19 bits); two integer ops instead of the emulated cvt.rna.tf32.
__device__ __forceinline__ void split_fast(float x, uint32_t& hi, uint32_t& lo) {
  hi = (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
  lo = __float_as_uint(x - __uint_as_float(hi));
}
__device__ __forceinline__ void st4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
__device__ __forceinline__ uint32_t swz(int r, int j) {
  return static_cast<uint32_t>(((r >> 3) << 10) + ((r & 7) << 7) + (((j ^ (r & 7)) & 7) << 4));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
__device__ __forceinline__ uint32_t idesc(int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(kRows >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t id, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(id), "r"(accum));
}
// A operand from TMEM (lane = row, one tf32 per 32-bit column), B from smem
__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t id,
                                            uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(id), "r"(accum));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// Waits for the phase with the given parity; a wait longer than ~10 s of SM
// clocks traps (a pipeline bug then fails the launch instead of hanging the GPU).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  long long t0 = 0;
  for (uint32_t spin = 0;; ++spin) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    if ((spin & 1023u) == 0) {
      const long long now = clock64();
      if (spin == 0) t0 = now;
      else if (now - t0 > 20000000000LL) __trap();
    }
  }
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_copy(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int W>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float* v) {
  static_assert(W == 8 || W == 16, "width");
  uint32_t r[16];
  if constexpr (W == 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "r"(taddr));
  } else {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
        "%12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < W; ++i) v[i] = __uint_as_float(r[i]);
}

template <int W>
__device__ __forceinline__ void tmem_ld_nowait(uint32_t taddr, float* v) {
  static_assert(W == 8 || W == 16, "width");
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  if constexpr (W == 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "r"(taddr));
  } else {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
        "%12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
  }
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// pin registers written by tcgen05.ld after the wait: the empty volatile asm
// keeps their consumers from being scheduled above tcgen05.wait::ld
template <int N>
__device__ __forceinline__ void pin_regs(float* v) {
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("" : "+f"(v[i]));
}

// Job table: one int4 {component, first CSR row, rows, components to score}
// per work item (built per launch by k_build_jobs), so every role decodes a
// job with one 16-byte load instead of a binary search over the item offsets.
__global__ void k_build_jobs(int C, int mode, int G, const int* off, const int* itemoff, const int* gcnt,
                             int4* jobs) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    const int i0 = itemoff[c], i1 = itemoff[c + 1];
    const int r0 = off[c], r1 = off[c + 1];
    const int nc = mode == kModeAnchor ? gcnt[c] : 1;
    (void)G;
    for (int it = i0; it < i1; ++it) {
      const int row0 = r0 + (it - i0) * kRows;
      jobs[it] = make_int4(c, row0, min(kRows, r1 - row0), nc);
    }
  }
}

__device__ __forceinline__ int4 load_job(const int4* jobs, int item) { return __ldg(jobs + item); }

// Walk of the (item, component group) sequence every role follows.
struct Walk {
  int item, g0;
  int4 J;  // {c, row0, nrows, ncomp}
  __device__ bool valid(int total) const { return item < total; }
  __device__ void advance(const int4* jobs, int qg, int total) {
    g0 += qg;
    if (g0 >= J.w) {
      g0 = 0;
      item += gridDim.x;
      if (item < total) J = load_job(jobs, item);
    }
  }
};
__device__ __forceinline__ Walk walk_begin(const int4* jobs, int total) {
  Walk w{static_cast<int>(blockIdx.x), 0, make_int4(0, 0, 0, 0)};
  if (w.item < total) w.J = load_job(jobs, w.item);
  return w;
}

// x-row index of the producer's row `ar` in job J (-1: padding row)
__device__ __forceinline__ int job_row(const WsArgs& a, const int4& J, int ar) {
  if (ar >= J.z) return -1;
  const int e = __ldg(a.ent + J.y + ar);
  return a.mode == kModeExtra ? e : e / a.dm.Cp;
}

template <int HP, bool PROF>
__global__ void __launch_bounds__(kThreads, 1) k_score_ws(WsArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  __shared__ uint64_t s_afull[2], s_aempty[2], s_tfull[2], s_tempty[2];
  __shared__ uint64_t s_bfull[kMaxNB], s_bempty[kMaxNB];
  __shared__ uint64_t s_mufull[2], s_muempty[2];
  __shared__ __align__(16) float s_mu[2][kMaxD + 8];
  __shared__ int s_muoff[2];
  __shared__ uint32_t s_tmem;
  const Dims dm = a.dm;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = (smem_u32(smem_dyn) + 1023u) & ~1023u;
  const int nchunk = (dm.D + kKC - 1) / kKC;
  const int total = __ldg(a.itemoff + dm.C);
  const int NB = a.nbstage;
  unsigned long long* tp = PROF && a.mode == kModeAnchor ? a.prof : nullptr;  // timeline trace

  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_afull[i], kProdWarps);
      mbar_init(&s_aempty[i], 1);
      mbar_init(&s_tfull[i], 1);
      mbar_init(&s_tempty[i], 4);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_mufull[i], 1);
      mbar_init(&s_muempty[i], kProdWarps);
    }
    for (int i = 0; i < NB; ++i) {
      mbar_init(&s_bfull[i], 1);
      mbar_init(&s_bempty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(a.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (uint32_t i = tid * 16; i < a.stage_bytes * NB; i += kThreads * 16) st4(sbase + i, 0, 0, 0, 0);
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = s_tmem;
  // B stage map (offsets from a 1024-aligned stage base)
  const uint32_t offB1 = 0;                          // B1 hi, then B1 lo (N1max rows each)
  const uint32_t offB2 = offB1 + 2 * a.N1max * 128;  // B2 hi, then B2 lo (16 rows each)
  // TMEM map: accumulators [0, nacc*TB), then the two A stages of 128 columns
  const uint32_t colA = a.nacc * a.TB;

  if (warp < kProdWarps) {
    // ============================================================ A producers
    // thread = (row ar of the 128-row block, K half ah of each 32-wide chunk).
    // Each thread streams its own 64-byte row pieces into a private shared-
    // memory ring with cp.async, `ahead` chunks in advance and across job
    // borders (no registers held, no cross-thread sync: cp.async groups are
    // per thread); the anchor mean arrives in shared memory from the loader.
    const int ar = 32 * (warp & 3) + lane, ah = warp >> 2;
    const int ahead = min(kAhead, nchunk);  // prefetch stays within the next job
    const uint32_t xbase = sbase + NB * a.stage_bytes;  // X ring: (kAhead+1) x [4][256] x 16 B
    Prof pf{};
    if (PROF) pf.start();
    Walk w = walk_begin(a.jobs, total);
    Walk wn = w;
    wn.advance(a.jobs, a.qg, total);
    int n_cur = w.valid(total) ? job_row(a, w.J, ar) : -1;
    int n_nxt = wn.valid(total) ? job_row(a, wn.J, ar) : -1;
    const bool vec = (dm.D & 3) == 0;
    auto issue_x = [&](int n, int ch, uint32_t unit) {
      const uint32_t slot = xbase + (unit % (kAhead + 1)) * (4 * kProdThreads * 16);
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int d = ch * kKC + 16 * ah + 4 * jj;
        const uint32_t dst = slot + (jj * kProdThreads + tid) * 16;
        const float* src = a.X + (int64_t)(n < 0 ? 0 : n) * dm.D + d;
        if (n < 0 || d >= dm.D || (PROF && (a.dbg & 1))) {
          st4(dst, 0, 0, 0, 0);
        } else if (vec) {
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
        } else {
          for (int k = 0; k < 4; ++k) {
            if (d + k < dm.D) asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst + 4 * k), "l"(src + k) : "memory");
            else asm volatile("st.shared.b32 [%0], %1;" ::"r"(dst + 4 * k), "r"(0u) : "memory");
          }
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto wait_x = [&]() {  // all but the newest `ahead` groups landed
      switch (ahead) {
        case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
        case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
        case 3: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
        case 4: asm volatile("cp.async.wait_group 4;" ::: "memory"); break;
        default: asm volatile("cp.async.wait_group 5;" ::: "memory"); break;
      }
    };
    uint32_t sc = 0;  // flat chunk (unit) counter
    if (w.valid(total))
      for (int k = 0; k < ahead; ++k) issue_x(n_cur, k, static_cast<uint32_t>(k));
    int jb = 0;
    while (w.valid(total)) {
      const int mslot = jb & 1;
      mbar_wait(&s_mufull[mslot], (jb >> 1) & 1);
      const float* mu_s = s_mu[mslot] + s_muoff[mslot];
      for (int ch = 0; ch < nchunk; ++ch, ++sc) {
        {  // prefetch unit sc + ahead (this job or the next)
          const int c2 = ch + ahead;
          if (c2 < nchunk) issue_x(n_cur, c2, sc + ahead);
          else issue_x(wn.valid(total) ? n_nxt : -1, c2 - nchunk, sc + ahead);
        }
        wait_x();
        const int s = static_cast<int>(sc & 1u);
        const uint32_t use = sc >> 1;
        const int d0 = ch * kKC;
        const uint32_t slot = xbase + (sc % (kAhead + 1)) * (4 * kProdThreads * 16);
        // v = x - mu_a and v^2, split hi (round to tf32) / lo (exact residual)
        uint32_t vh[16], vl[16], qh[16], ql[16];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int d = d0 + 16 * ah + 4 * jj;
          float xv[4];
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(xv[0]), "=f"(xv[1]), "=f"(xv[2]), "=f"(xv[3])
                       : "r"(slot + (jj * kProdThreads + tid) * 16)
                       : "memory");
          float v[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) v[k] = d + k < dm.D ? xv[k] - mu_s[d + k] : 0.f;
          if (n_cur < 0) v[0] = v[1] = v[2] = v[3] = 0.f;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            split_fast(v[k], vh[4 * jj + k], vl[4 * jj + k]);
            split_fast(v[k] * v[k], qh[4 * jj + k], ql[4 * jj + k]);
          }
        }
        if (PROF) pf.lap(kPSplit);
        if (use >= 1) mbar_wait(&s_aempty[s], (use - 1) & 1u);
        if (PROF) pf.lap(kPWaitEmpty);
        if (tid == 32) trace(tp, static_cast<int>(sc), 0);
        const uint32_t ta = tmem + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + colA + s * 128 + 16 * ah;
        tmem_st16(ta, vh);
        tmem_st16(ta + 32, vl);
        tmem_st16(ta + 64, qh);
        tmem_st16(ta + 96, ql);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_afull[s]);
        if (tid == 32) trace(tp, static_cast<int>(sc), 1);
        if (PROF) pf.lap(kPStore);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_muempty[mslot]);  // done with this job's mean
      ++jb;
      // next job
      w = wn;
      if (!w.valid(total)) break;
      wn.advance(a.jobs, a.qg, total);
      n_cur = n_nxt;
      n_nxt = wn.valid(total) ? job_row(a, wn.J, ar) : -1;
      if (PROF) pf.lap(kPSync);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    if (PROF && a.prof && lane == 0) {
      atomicAdd(a.prof + kPSync, pf.acc[kPSync]);
      atomicAdd(a.prof + kPWaitEmpty, pf.acc[kPWaitEmpty]);
      atomicAdd(a.prof + kPSplit, pf.acc[kPSplit]);
      atomicAdd(a.prof + kPStore, pf.acc[kPStore]);
    }
  } else if (warp == kLoadWarp) {
    // ============================================================ B loader
    // one thread fills an NB-deep shared-memory ring with the B operands,
    // running ahead of the MMA across job borders: one bulk copy of the
    // prebuilt stage image per chunk (few large copies keep many bytes in
    // flight; small copies are serialised by the copy engine), else per-block
    // copies of the pre-split W blocks and lin/psi tiles
    if (lane == 0) {
      uint32_t bc = 0;
      int jb = 0;
      for (Walk w = walk_begin(a.jobs, total); w.valid(total); w.advance(a.jobs, a.qg, total), ++jb) {
        const int c = w.J.x;
        const int nq = min(a.qg, w.J.w - w.g0);
        const int grp = w.g0 / a.qg;
        {  // the job's centring mean mu_a -> s_mu[jb & 1] (16-byte aligned window)
          const int m = jb & 1;
          if (jb >= 2) mbar_wait(&s_muempty[m], ((jb >> 1) - 1) & 1);
          const int64_t f0 = (int64_t)c * dm.D, fa = f0 & ~int64_t{3};
          const uint32_t bytes = static_cast<uint32_t>(((f0 - fa + dm.D + 3) & ~int64_t{3}) * 4);
          s_muoff[m] = static_cast<int>(f0 - fa);
          mbar_arrive_expect_tx(&s_mufull[m], bytes);
          bulk_copy(smem_u32(s_mu[m]), a.mu32 + fa, bytes, &s_mufull[m]);
        }
        int comp[kNL];
        if (!a.img)
          for (int qi = 0; qi < nq; ++qi)
            comp[qi] = a.mode == kModeAnchor ? __ldg(a.g + (int64_t)c * dm.G + w.g0 + qi) : c;
        for (int ch = 0; ch < nchunk; ++ch, ++bc) {
          const int s = static_cast<int>(bc % NB);
          const uint32_t use = bc / NB;
          if (use >= 1) mbar_wait(&s_bempty[s], (use - 1) & 1u);
          trace(tp, static_cast<int>(bc), 5);
          const uint32_t st = sbase + s * a.stage_bytes;
          if (a.img) {
            const int ng = a.mode == kModeAnchor ? a.ngroups : 1;
            const float* src = a.img + (((int64_t)c * ng + grp) * nchunk + ch) * (a.stage_bytes / 4);
            mbar_arrive_expect_tx(&s_bfull[s], a.stage_bytes);
            bulk_copy(st, src, a.stage_bytes, &s_bfull[s]);
          } else {
            const uint32_t blk = HP * 128;
            mbar_arrive_expect_tx(&s_bfull[s], 2 * nq * blk + 4 * kNL * 128);
            for (int qi = 0; qi < nq; ++qi) {
              const float* src = a.WTS + ((int64_t)comp[qi] * nchunk + ch) * 2 * HP * 32;
              const uint32_t row = kNL + qi * HP;
              bulk_copy(st + offB1 + row * 128, src, blk, &s_bfull[s]);
              bulk_copy(st + offB1 + a.N1max * 128 + row * 128, src + HP * 32, blk, &s_bfull[s]);
            }
            const float* lb = (a.mode == kModeAnchor
                                   ? a.lblk + ((int64_t)c * a.ngroups + grp) * nchunk * 4 * kNL * 32
                                   : a.cblk + (int64_t)c * nchunk * 4 * kNL * 32) +
                              (int64_t)ch * 4 * kNL * 32;
            bulk_copy(st + offB1, lb, kNL * 128, &s_bfull[s]);                             // lin hi
            bulk_copy(st + offB1 + a.N1max * 128, lb + kNL * 32, kNL * 128, &s_bfull[s]);  // lin lo
            bulk_copy(st + offB2, lb + 2 * kNL * 32, kNL * 128, &s_bfull[s]);              // psi hi
            bulk_copy(st + offB2 + kNL * 128, lb + 3 * kNL * 32, kNL * 128, &s_bfull[s]);  // psi lo
          }
          trace(tp, static_cast<int>(bc), 6);
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ============================================================ MMA issuer
    uint32_t sc = 0, bc = 0;
    int jb = 0;
    Prof pf{};
    if (PROF) pf.start();
    for (Walk w = walk_begin(a.jobs, total); w.valid(total); w.advance(a.jobs, a.qg, total), ++jb) {
      const int b = a.nacc == 2 ? (jb & 1) : 0;
      const int use_b = a.nacc == 2 ? (jb >> 1) : jb;
      const int nq = min(a.qg, w.J.w - w.g0);
      const int N1 = kNL + ((nq * HP + 15) / 16) * 16;
      const uint32_t acc1 = tmem + b * a.TB, acc2 = acc1 + N1;
      if (use_b >= 1) mbar_wait(&s_tempty[b], (use_b - 1) & 1);
      fence_after();
      if (PROF) pf.lap(kMWaitTE);
      for (int ch = 0; ch < nchunk; ++ch, ++sc, ++bc) {
        const int s = static_cast<int>(sc & 1u);
        const int sb = static_cast<int>(bc % NB);
        mbar_wait(&s_afull[s], (sc >> 1) & 1u);
        if (lane == 0) trace(tp, static_cast<int>(sc), 4);
        mbar_wait(&s_bfull[sb], (bc / NB) & 1u);
        fence_after();
        if (PROF) pf.lap(kMWaitFull);
        if (lane == 0) trace(tp, static_cast<int>(sc), 2);
        if (lane == 0) {
          const uint32_t st = sbase + sb * a.stage_bytes;
          const uint32_t id1 = idesc(N1), id2 = idesc(kNL);
          const uint32_t tA = tmem + colA + s * 128;  // v hi | v lo | v^2 hi | v^2 lo
          const uint32_t Av[3] = {tA, tA, tA + 32};
          const uint32_t Aq[3] = {tA + 64, tA + 64, tA + 96};
          const uint32_t B1[3] = {st + offB1, st + offB1 + a.N1max * 128, st + offB1};
          const uint32_t B2[3] = {st + offB2, st + offB2 + kNL * 128, st + offB2};
#pragma unroll
          for (int p = 0; p < ((PROF && (a.dbg & 4)) ? 0 : 3); ++p) {
#pragma unroll
            for (int k = 0; k < kKC / 8; ++k) {
              const uint32_t acc = (ch > 0 || p > 0 || k > 0) ? 1u : 0u;
              mma_tf32_ts(acc1, Av[p] + k * 8, sdesc(B1[p] + k * 32), id1, acc);
              mma_tf32_ts(acc2, Aq[p] + k * 8, sdesc(B2[p] + k * 32), id2, acc);
            }
          }
          commit(&s_aempty[s]);
          commit(&s_bempty[sb]);
          if (ch == nchunk - 1) commit(&s_tfull[b]);
        }
        __syncwarp();
        if (PROF) pf.lap(kMIssue);
        if (lane == 0) trace(tp, static_cast<int>(sc), 3);
      }
    }
    if (PROF && a.prof && lane == 0)
      for (int i = kMWaitTE; i <= kMIssue; ++i) atomicAdd(a.prof + i, pf.acc[i]);
  } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {
    // ============================================================ epilogue
    constexpr int kEpiBatch = HP >= 32 ? 1 : 32 / HP;  // components per tcgen05.ld batch
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    int jb = 0;
    Prof pf{};
    if (PROF) pf.start();
    for (Walk w = walk_begin(a.jobs, total); w.valid(total); w.advance(a.jobs, a.qg, total), ++jb) {
      const int b = a.nacc == 2 ? (jb & 1) : 0;
      const int use_b = a.nacc == 2 ? (jb >> 1) : jb;
      const int c = w.J.x;
      const int nq = min(a.qg, w.J.w - w.g0);
      const int e = r < w.J.z ? __ldg(a.ent + w.J.y + r) : -1;
      mbar_wait(&s_tfull[b], use_b & 1);
      fence_after();
      if (PROF) pf.lap(kEWait);
      const int N1 = kNL + ((nq * HP + 15) / 16) * 16;
      const uint32_t trow = tmem + b * a.TB + (static_cast<uint32_t>(quad * 32) << 16);
      float lin[16], d2[16];
      tmem_ld_nowait<16>(trow, lin);
      tmem_ld_nowait<16>(trow + N1, d2);
      tmem_wait_ld();
      pin_regs<16>(lin);
      pin_regs<16>(d2);
      for (int q0 = 0; q0 < nq; q0 += kEpiBatch) {
        const int nb = min(kEpiBatch, nq - q0);
        float y[kEpiBatch][HP];
#pragma unroll
        for (int qi = 0; qi < kEpiBatch; ++qi) {
          if (qi < nb) {
#pragma unroll
            for (int h0 = 0; h0 < HP; h0 += 16) {
              if constexpr (HP >= 16) tmem_ld_nowait<16>(trow + kNL + (q0 + qi) * HP + h0, y[qi] + h0);
              else tmem_ld_nowait<8>(trow + kNL + (q0 + qi) * HP + h0, y[qi] + h0);
            }
          }
        }
        tmem_wait_ld();
        pin_regs<kEpiBatch * HP>(&y[0][0]);
#pragma unroll
        for (int qi = 0; qi < kEpiBatch; ++qi) {
          if (qi >= nb) break;
          const int slot = w.g0 + q0 + qi;
          const int q = a.mode == kModeAnchor ? __ldg(a.g + (int64_t)c * dm.G + slot) : c;
          float m = 0.f;
          float yy = 0.f;
          if (a.mode == kModeAnchor) {
            const float* cst = a.acst + ((int64_t)c * dm.G + slot) * (HP + 1);
#pragma unroll
            for (int h = 0; h < HP; ++h) {
              const float t = y[qi][h] - __ldg(cst + h);
              yy = fmaf(t, t, yy);
            }
            m = __ldg(cst + HP);
          } else {
#pragma unroll
            for (int h = 0; h < HP; ++h) yy = fmaf(y[qi][h], y[qi][h], yy);
          }
          float linq = 0.f, d2q = 0.f;
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (i == q0 + qi) {
              linq = lin[i];
              d2q = d2[i];
            }
          const double diag = static_cast<double>(d2q) + static_cast<double>(linq) + static_cast<double>(m);
          const float lj = static_cast<float>(__ldg(a.kconst + q) - 0.5 * (diag - static_cast<double>(yy)));
          if (e >= 0) {
            if (a.mode == kModeAnchor) {
              const int n = e / dm.Cp, j = e - n * dm.Cp;
              a.out[(int64_t)n * dm.SL + j * dm.G + slot] = lj;
            } else if (a.mode == kModeExtra) {
              a.out[(int64_t)e * dm.SL + dm.Cp * dm.G] = lj;
            } else {
              a.out[e] = lj;
            }
          }
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_tempty[b]);
      if (PROF) pf.lap(kEWork);
    }
    if (PROF && a.prof && lane == 0)
      for (int i = kEWait; i <= kEWork; ++i) atomicAdd(a.prof + i, pf.acc[i]);
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols));
}

// Per-(anchor, slot) constants: b = W_q^T (mu_q - mu_a), m = sum psi_q^-1 (mu_q - mu_a)^2
// (fp32 operands of the scorer, fp64 accumulation). One warp per (anchor, slot).
__global__ void __launch_bounds__(256) k_anchor_consts(Dims dm, int Hp, const float* WT, const float* mu32,
                                                      const float* ipsi32, const int* g, const int* gcnt,
                                                      float* acst) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = gw; w < (int64_t)dm.C * dm.G; w += nw) {
    const int c = static_cast<int>(w / dm.G), i = static_cast<int>(w - (int64_t)c * dm.G);
    float* out = acst + w * (Hp + 1);
    if (i >= gcnt[c]) continue;
    const int q = g[(int64_t)c * dm.G + i];
    const float* mq = mu32 + (int64_t)q * dm.D;
    const float* ma = mu32 + (int64_t)c * dm.D;
    const float* ip = ipsi32 + (int64_t)q * dm.D;
    double m = 0.0;
    for (int d = lane; d < dm.D; d += 32) {
      const double dl = static_cast<double>(mq[d]) - static_cast<double>(ma[d]);
      const float dlf = mq[d] - ma[d];  // same fp32 rounding as the scorer's operands
      m += static_cast<double>(ip[d]) * static_cast<double>(dlf) * static_cast<double>(dlf);
      (void)dl;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
    for (int h = 0; h < Hp; ++h) {
      const float* wr = WT + ((int64_t)q * Hp + h) * dm.D;
      double s = 0.0;
      for (int d = lane; d < dm.D; d += 32) s += static_cast<double>(wr[d]) * static_cast<double>(mq[d] - ma[d]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) out[h] = static_cast<float>(s);
    }
    if (lane == 0) out[Hp] = static_cast<float>(m);
  }
}

// Pre-split, pre-swizzled W blocks: WTS[q][chunk][hi|lo][Hp rows][32] so that a
// block lands verbatim in a 128B-swizzled K-major tile at any 8-row boundary.
__global__ void k_build_wts(Dims dm, int Hp, const float* WT, float* WTS) {
  const int nchunk = (dm.D + kKC - 1) / kKC;
  const int64_t total = (int64_t)dm.C * nchunk * Hp * kKC;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int e = static_cast<int>(i % kKC);
    int64_t t = i / kKC;
    const int h = static_cast<int>(t % Hp);
    t /= Hp;
    const int ch = static_cast<int>(t % nchunk);
    const int q = static_cast<int>(t / nchunk);
    const int d = ch * kKC + e;
    const float w = d < dm.D ? WT[((int64_t)q * Hp + h) * dm.D + d] : 0.f;
    uint32_t hi, lo;
    split(w, hi, lo);
    const int j = e >> 2;
    const int pos = h * 32 + (((j ^ (h & 7)) & 7) << 2) + (e & 3);
    float* blk = WTS + ((int64_t)q * nchunk + ch) * 2 * Hp * 32;
    blk[pos] = __uint_as_float(hi);
    blk[Hp * 32 + pos] = __uint_as_float(lo);
  }
}

// Anchor-dependent B blocks, once per E-step (g and the parameters are fixed
// during the E-step): for anchor a, component group grp, K chunk ch, the 16-row
// tiles [lin hi | lin lo | psi hi | psi lo] with lin_q = -2 psi_q^-1 (mu_q - mu_a),
// pre-split and pre-swizzled exactly as the smem B tiles. single != 0 builds
// the one-component blocks (q = a, lin = 0) of the extra / truncated-F passes.
__global__ void k_build_blocks(Dims dm, int qg, int ngroups, int single, const float* mu32,
                               const float* ipsi32, const int* g, const int* gcnt, float* blk) {
  const int nchunk = (dm.D + kKC - 1) / kKC;
  const int ng = single ? 1 : ngroups;
  const int64_t total = (int64_t)dm.C * ng * nchunk * kNL * kKC;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int e = static_cast<int>(i % kKC);
    int64_t t = i / kKC;
    const int qi = static_cast<int>(t % kNL);
    t /= kNL;
    const int ch = static_cast<int>(t % nchunk);
    t /= nchunk;
    const int grp = static_cast<int>(t % ng);
    const int a = static_cast<int>(t / ng);
    const int d = ch * kKC + e;
    int q = -1;
    if (single) {
      if (qi == 0) q = a;
    } else {
      const int slot = grp * qg + qi;
      if (qi < qg && slot < gcnt[a]) q = g[(int64_t)a * dm.G + slot];
    }
    float lin = 0.f, ip = 0.f;
    if (q >= 0 && d < dm.D) {
      ip = ipsi32[(int64_t)q * dm.D + d];
      lin = single ? 0.f : -2.f * ip * (mu32[(int64_t)q * dm.D + d] - mu32[(int64_t)a * dm.D + d]);
    }
    uint32_t lh, ll, ph, pl;
    split(lin, lh, ll);
    split(ip, ph, pl);
    const int j = e >> 2;
    const int pos = qi * 32 + (((j ^ (qi & 7)) & 7) << 2) + (e & 3);
    float* b = blk + (((int64_t)a * ng + grp) * nchunk + ch) * 4 * kNL * 32;
    b[pos] = __uint_as_float(lh);
    b[kNL * 32 + pos] = __uint_as_float(ll);
    b[2 * kNL * 32 + pos] = __uint_as_float(ph);
    b[3 * kNL * 32 + pos] = __uint_as_float(pl);
  }
}

// B stage images: for anchor a, component group grp and K chunk ch, the exact
// shared-memory stage the MMA reads -- [B1 hi | B1 lo] (N1max rows: 16 lin
// rows, then Hp W rows per component of the group) and [B2 hi | B2 lo] (16
// psi^-1 rows) -- pre-split into tf32 hi/lo and 128B-swizzled, so the loader
// moves a whole stage with one bulk copy. single != 0: one component (q = a),
// lin = 0 (extra candidates, truncated F).
__global__ void __launch_bounds__(256) k_build_images(Dims dm, int Hp, int qg, int ngroups, int N1max, int single,
                                                      const float* WT, const float* mu32, const float* ipsi32,
                                                      const int* g, const int* gcnt, float* img) {
  // one CTA per stage image (a, grp, ch); 32-bit index math inside a stage
  const int nchunk = (dm.D + kKC - 1) / kKC;
  const int ng = single ? 1 : ngroups;
  const int sf = 2 * 32 * (N1max + kNL);  // floats per stage
  const int nstages = dm.C * ng * nchunk;
  __shared__ int s_q[kNL];
  __shared__ int s_nq;
  for (int sid = blockIdx.x; sid < nstages; sid += gridDim.x) {
    const int ch = sid % nchunk;
    const int grp = (sid / nchunk) % ng;
    const int a = sid / (nchunk * ng);
    __syncthreads();
    if (threadIdx.x == 0) s_nq = single ? 1 : min(qg, gcnt[a] - grp * qg);
    if (threadIdx.x < kNL)
      s_q[threadIdx.x] = single ? a : (threadIdx.x < min(qg, gcnt[a] - grp * qg) ? g[(int64_t)a * dm.G + grp * qg + threadIdx.x] : 0);
    __syncthreads();
    const int nq = s_nq;
    float* out = img + (int64_t)sid * sf;
    for (int f = threadIdx.x; f < sf; f += blockDim.x) {
      // region: 0 B1 hi, 1 B1 lo (N1max rows each), 2 B2 hi, 3 B2 lo (16 rows each)
      int reg, loc;
      if (f < 2 * N1max * 32) reg = f / (N1max * 32), loc = f - reg * N1max * 32;
      else reg = 2 + (f - 2 * N1max * 32) / (kNL * 32), loc = (f - 2 * N1max * 32) - (reg - 2) * kNL * 32;
      const int r = loc >> 5, pos = loc & 31;
      const int e = ((((pos >> 2) ^ (r & 7)) & 7) << 2) | (pos & 3);  // un-swizzled column
      const int d = ch * kKC + e;
      float v = 0.f;
      if (d < dm.D) {
        if (reg < 2) {
          if (r < kNL) {
            if (!single && r < nq) {
              const int q = s_q[r];
              v = -2.f * __ldg(ipsi32 + (int64_t)q * dm.D + d) *
                  (__ldg(mu32 + (int64_t)q * dm.D + d) - __ldg(mu32 + (int64_t)a * dm.D + d));
            }
          } else {
            const int qi = (r - kNL) / Hp, h = (r - kNL) - qi * Hp;
            if (qi < nq) v = __ldg(WT + ((int64_t)s_q[qi] * Hp + h) * dm.D + d);
          }
        } else if (r < nq) {
          v = __ldg(ipsi32 + (int64_t)s_q[r] * dm.D + d);
        }
      }
      uint32_t hi, lo;
      split(v, hi, lo);
      out[f] = __uint_as_float((reg & 1) ? lo : hi);
    }
  }
}

}  // namespace

int64_t ws_image_floats(const Dims& dm, int single) {
  const int Hp = ws_hp(dm.H);
  const int qg = single ? 1 : std::max(1, std::min(std::min(dm.G, kNL), (256 - kNL) / Hp));
  const int N1max = kNL + ((qg * Hp + 15) / 16) * 16;
  const int nchunk = (dm.D + kKC - 1) / kKC;
  const int ng = single ? 1 : ws_groups(dm);
  return (int64_t)dm.C * ng * nchunk * 2 * 32 * (N1max + kNL);
}

cudaError_t launch_ws_images(const Dims& dm, int single, const float* WT, const float* mu32, const float* ipsi32,
                             const int* g, const int* gcnt, float* img, cudaStream_t s) {
  const int Hp = ws_hp(dm.H);
  const int qg = single ? 1 : std::max(1, std::min(std::min(dm.G, kNL), (256 - kNL) / Hp));
  const int N1max = kNL + ((qg * Hp + 15) / 16) * 16;
  k_build_images<<<sm_count() * 8, 256, 0, s>>>(dm, Hp, qg, ws_groups(dm), N1max, single, WT, mu32, ipsi32, g,
                                                 gcnt, img);
  return cudaGetLastError();
}

int ws_groups(const Dims& dm) {
  const int Hp = ws_hp(dm.H);
  const int qg = std::max(1, std::min(std::min(dm.G, kNL), (256 - kNL) / Hp));
  return (dm.G + qg - 1) / qg;
}

cudaError_t launch_ws_blocks(const Dims& dm, int single, const float* mu32, const float* ipsi32,
                             const int* g, const int* gcnt, float* blk, cudaStream_t s) {
  const int Hp = ws_hp(dm.H);
  const int qg = std::max(1, std::min(std::min(dm.G, kNL), (256 - kNL) / Hp));
  k_build_blocks<<<sm_count() * 8, 256, 0, s>>>(dm, qg, ws_groups(dm), single, mu32, ipsi32, g, gcnt, blk);
  return cudaGetLastError();
}

bool score_ws_supported(const Dims& dm) { return dm.D <= kMaxD && dm.H <= 64 && dm.G <= 64; }

int ws_hp(int H) { return H <= 8 ? 8 : H <= 16 ? 16 : H <= 32 ? 32 : 64; }

cudaError_t launch_ws_prep(const Dims& dm, const float* WT, float* WTS, cudaStream_t s) {
  const int Hp = ws_hp(dm.H);
  k_build_wts<<<sm_count() * 8, 256, 0, s>>>(dm, Hp, WT, WTS);
  return cudaGetLastError();
}

cudaError_t launch_anchor_consts(const Dims& dm, const float* WT, const float* mu32, const float* ipsi32,
                                 const int* g, const int* gcnt, float* acst, cudaStream_t s) {
  const int Hp = ws_hp(dm.H);
  k_anchor_consts<<<sm_count() * 8, 256, 0, s>>>(dm, Hp, WT, mu32, ipsi32, g, gcnt, acst);
  return cudaGetLastError();
}

unsigned long long* g_ws_prof = nullptr;  // set by vmfa_diag_scorer_cycles
int g_ws_dbg = 0;                          // diagnostics flags (enable >> 1)
constexpr int kProfWords = 16 + 8 * kTraceEvents;

cudaError_t launch_score_ws(int mode, const ScoreArgs& s, const float* WTS, const float* mu32,
                            const float* ipsi32, const float* acst, const float* lblk, const float* cblk,
                            const float* img, int4* jobs, cudaStream_t st) {
  WsArgs a{};
  a.dm = s.dm;
  a.mode = mode;
  a.Hp = ws_hp(s.dm.H);
  const int ncomp_max = mode == kModeAnchor ? s.dm.G : 1;
  a.qg = std::max(1, std::min(std::min(ncomp_max, kNL), (256 - kNL) / a.Hp));
  a.N1max = kNL + ((a.qg * a.Hp + 15) / 16) * 16;
  const int cols = a.N1max + kNL;
  a.TB = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : 256;
  a.nacc = (2 * a.TB + 2 * 128 <= 512) ? 2 : 1;  // A stages use 2 x 128 TMEM columns
  const uint32_t need = a.nacc * a.TB + 2 * 128;
  a.tmem_cols = need <= 256 ? 256 : 512;
  a.stage_bytes = static_cast<uint32_t>(2 * 128 * (a.N1max + kNL));
  // B ring: as deep as ~200 KB of shared memory allows
  // shared memory: B ring (as deep as fits, >= 2) + the producers' X ring
  a.nbstage = std::max(2, std::min(kMaxNB, static_cast<int>((200u * 1024u - kXRingBytes) / a.stage_bytes)));
  const size_t dyn = static_cast<size_t>(a.nbstage) * a.stage_bytes + kXRingBytes + 1024;
  a.X = s.X;
  a.WTS = WTS;
  a.mu32 = mu32;
  a.ipsi32 = ipsi32;
  a.kconst = s.kconst;
  a.acst = acst;
  a.lblk = lblk;
  a.cblk = cblk;
  a.img = img;
  a.ngroups = ws_groups(s.dm);
  a.jobs = jobs;
  a.itemoff = s.itemoff;
  a.ent = s.ent;
  a.g = s.g;
  a.gcnt = s.gcnt;
  a.out = s.out;
  a.prof = g_ws_prof;
  a.dbg = g_ws_prof ? g_ws_dbg : 0;
  k_build_jobs<<<(s.dm.C + 255) / 256, 256, 0, st>>>(s.dm.C, mode, s.dm.G, s.off, s.itemoff, s.gcnt, jobs);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn));
    kern<<<sm_count(), kThreads, dyn, st>>>(a);
  };
  const bool prof = g_ws_prof != nullptr;
  switch (a.Hp) {
    case 8: prof ? go(k_score_ws<8, true>) : go(k_score_ws<8, false>); break;
    case 16: prof ? go(k_score_ws<16, true>) : go(k_score_ws<16, false>); break;
    case 32: prof ? go(k_score_ws<32, true>) : go(k_score_ws<32, false>); break;
    default: prof ? go(k_score_ws<64, true>) : go(k_score_ws<64, false>); break;
  }
  return cudaGetLastError();
}

}  // namespace vmfa_b200

// Diagnostics: per-role cycle counters of the warp-specialised scorer.
extern "C" int vmfa_diag_scorer_cycles(int enable, unsigned long long* out, int n) {
  using namespace vmfa_b200;
  g_ws_dbg = enable >> 1;
  if (enable && !g_ws_prof) {
    if (cudaMalloc(&g_ws_prof, sizeof(unsigned long long) * kProfWords) != cudaSuccess) return VMFA_ERR_CUDA;
    cudaMemset(g_ws_prof, 0, sizeof(unsigned long long) * kProfWords);
  }
  if (out && g_ws_prof) {
    cudaDeviceSynchronize();
    cudaMemcpy(out, g_ws_prof, sizeof(unsigned long long) * (n < kProfWords ? n : kProfWords), cudaMemcpyDeviceToHost);
    cudaMemset(g_ws_prof, 0, sizeof(unsigned long long) * kProfWords);
  }
  if (!enable && g_ws_prof) {
    cudaFree(g_ws_prof);
    g_ws_prof = nullptr;
  }
  return VMFA_OK;
}
