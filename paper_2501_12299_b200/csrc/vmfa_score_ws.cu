// vmfa_score_ws.cu — warp-specialised tcgen05 scorer of the candidate
// log-joints (log_joint, model.cpp:81-95) over anchor blocks.
//
// For anchor a, the rows n with a in K(n) need every component q in g_a, so a
// job is a dense block: 128 rows x the components of g_a. Rows are centred on
// the anchor mean (v = x - mu_a) and three products share the A operands:
//   GEMM1  [v]   (128 x D) x [ -2 psi_q^-1 delta_q (16 rows) | W_q (Hp rows per q) ]
//   GEMM2  [v^2] (128 x D) x [ psi_q^-1 (16 rows) ]
// with delta_q = mu_q - mu_a, and per-(anchor, q) constants b = W_q^T delta_q,
// m = sum psi_q^-1 delta_q^2 precomputed once per E-step (k_build_records):
//   y_q = acc_W - b,   diag_q = acc_psi + acc_lin + m,
//   l = kconst_q - 0.5 (diag_q - |y_q|^2).
//
// Arithmetic: 3xFP16 on tcgen05.mma.kind::f16 with fp32 accumulation in TMEM.
// Every operand row is scaled by a power of two so its largest element is
// ~2^14 (A rows by a bound on |x_n - mu_a|, B rows by their max over D; the
// scales are undone exactly in the epilogue), then split x = hi + lo into two
// fp16 values (22 significant bits, the same as 3xTF32); hi*hi + hi*lo + lo*hi
// drops only lo*lo. K = 16 per instruction (twice tf32's K = 8) halves the
// instruction count, and fp16 operands halve the B bytes.
//
// Roles (22 warps, one CTA per SM, persistent over the job table):
//   warps 0-15 A producers: each thread streams its own pieces of a row into
//              a shared ring of row chunks (bulk copies) ahead, centres / scales /
//              splits them and stores the A operands into TMEM (tcgen05.st);
//   warp 16    MMA issuer (one thread): TS-form tcgen05.mma, A from TMEM, B
//              from shared memory, commits to the stage / accumulator barriers;
//   warps 17-20 epilogue: stage the job's per-slot records in shared memory,
//              tcgen05.ld a finished accumulator (double buffered), assemble
//              the log-joints, scatter them to the candidate slots;
//   warp 21    loader (one thread): per job the anchor mean into s_mu, per
//              chunk one bulk copy of the prebuilt B stage image into an
//              NB-deep ring (few large copies keep many bytes in flight).
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include <cuda.h>  // CUtensorMap (the encoder is fetched through cudaGetDriverEntryPoint)
#include <cuda_fp16.h>

#include "vmfa_b200.h"
#include "vmfa_kernels.cuh"

namespace vmfa_b200 {
namespace {

constexpr int kRows = 128;
constexpr int kKC = 64;               // K chunk: 64 fp16 = one 128-byte swizzle row
constexpr int kProdWarps = 16;        // 4 per TMEM lane quadrant (row gathers scale with issuing warps)
constexpr int kProdThreads = kProdWarps * 32;
constexpr int kKSplit = kProdWarps / 4;       // K slices of a chunk per row
constexpr int kElem = 64 / kKSplit;           // x values per producer thread per chunk
constexpr int kMmaWarp = kProdWarps;
constexpr int kEpiWarp0 = kProdWarps + 1;
constexpr int kLoadWarp = kProdWarps + 5;
constexpr int kThreads = (kLoadWarp + 1) * 32;
constexpr int kMaxNB = 8;             // B ring stages (smem)
constexpr int kMaxXSlots = 4;         // X ring slots (row chunks); prefetch depth = slots - 1
constexpr int kXSeg = kElem / 4;      // 16-byte pieces per thread per chunk
constexpr int kMaxCps = 2;             // K chunks per X-ring slot, at most
// floats per row of a slot holding `cps` chunks (padded: conflict-free LDS.128)
// (cps * 64 + 8 floats: a 4-row gather4 group is 4 * 544 bytes, a multiple of
// 128; the 32-byte row skew leaves 2-way conflicts on the producers' LDS.128)
__host__ __device__ constexpr int x_row(int cps) { return cps * kKC + 8; }
__host__ __device__ constexpr uint32_t x_slot_bytes(int cps) { return kRows * x_row(cps) * 4; }
constexpr int kMaxD = 1024;
constexpr int kNL = 16;               // lin rows / psi rows per group (qg <= 16)
constexpr int kTargetExp = 14;        // operands scaled to |value| <= 2^14
__host__ __device__ constexpr int rec_stride(int Hp) { return 8 + 2 * Hp; }  // floats per epilogue record
// a score whose terms B exceed kCancel M, M a lower bound of the log-joint's
// term magnitude (_helpers.lj_term_scale), is re-evaluated in fp64: the
// ~1e-6 B error of the fp32-accurate terms then stays below 1e-4 M
constexpr float kCancel = 32.f;
// components per anchor job: the accumulator [16 lin | qg*Hp W | 16 psi] must
// fit one 256-column TMEM buffer
__host__ __device__ constexpr int qg_max(int Hp) { return (256 - 2 * kNL) / Hp < kNL ? (256 - 2 * kNL) / Hp : kNL; }

struct WsArgs {
  Dims dm;
  int mode;
  // image-free anchor stages (Hp % 8 == 0): per (anchor, group, chunk) a
  // small image [lin hi | lin lo | psi hi | psi lo] (16 lines each) and the
  // W rows of every component copied from its one-component image
  const __half* limg;
  const __half* simg1;
  int N1max1;
  int Hp;            // W rows per component (>= 8)
  int qg;            // components per job (group)
  int N1max;         // 16 + round16(qg * Hp)
  int nbstage;       // B ring depth
  int xslots;        // X ring slots (2..kMaxXSlots)
  int cps;           // K chunks per X-ring slot (one bulk copy per row and slot)
  int gather;        // 1: rows arrive by tile::gather4 (4 rows per TMA operation)
  int nacc;          // accumulator buffers in TMEM (2 when they fit beside the A stages)
  uint32_t tmem_cols;
  uint32_t TB;       // TMEM columns per accumulator buffer
  uint32_t stage_bytes;
  const float* X;
  const float* xmax;   // per row max |x| (A-row scale bound)
  const float* mumax;  // per component max |mu32|
  const float* mu32;
  const float* rec;    // epilogue records [C][G or 1][rec_stride(Hp)]
  const __half* img;   // B stage images [C][groups][nchunk][stage]
  int ngroups;
  const int4* jobs;    // per item {component, first CSR row, rows, components}
  const int* itemoff;
  const int* ent;
  const int* g;
  const int* gcnt;
  float* out;
  int list_div;              // kModeList: row = entry / list_div
  long long* fix_list;       // flagged scores (output indices), nullptr: flags only
  unsigned long long* fix_cnt;
  long long fix_cap;
  unsigned long long* prof;  // optional per-role cycle counters (nullptr: off)
  int dbg;                   // diagnostics only: bit0 skip x loads, bit2 skip MMAs
};

// per-role cycle accounting (diagnostic instantiation only)
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

// timeline trace of CTA 0 (diagnostics): slot = 16 + 8 * event_index + kind
constexpr int kTraceEvents = 512;
__device__ __forceinline__ void trace(unsigned long long* prof, int idx, int kind) {
  if (prof && blockIdx.x == 0 && idx < kTraceEvents) prof[16 + 8 * idx + kind] = clock64();
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// Power-of-two exponent k with |value| * 2^k <= 2^14 for |value| <= bound.
__device__ __forceinline__ int scale_exp(float bound) {
  if (!(bound > 0.f)) return 0;
  const uint32_t b = __float_as_uint(bound);
  int e = static_cast<int>((b >> 23) & 0xffu) - 127;  // bound in [2^e, 2^(e+1))
  if ((b & 0x7fffffu) != 0u) e += 1;                  // bound <= 2^e
  if (((b >> 23) & 0xffu) == 0u) e = -126;            // denormal bound
  return max(-100, min(100, kTargetExp - e));
}
__device__ __forceinline__ float exp2i(int k) { return __uint_as_float(static_cast<uint32_t>(k + 127) << 23); }
// hi = fp16(x), lo = fp16(x - hi) for two values, packed (element 0 in the low half)
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x0, x1);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
__device__ __forceinline__ void st4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
// K-major, 128-byte-swizzled smem operand descriptor (8-row groups 1 KB apart)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
// kind::f16 instruction descriptor: fp32 accumulate, fp16 A and B, K-major, M = 128
__device__ __forceinline__ uint32_t idesc(int N) {
  return (1u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(kRows >> 4) << 24);
}
// A operand from TMEM (lane = row, two fp16 per 32-bit column), B from smem
__device__ __forceinline__ void mma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t id,
                                           uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(id), "r"(accum));
}
template <int W>
__device__ __forceinline__ void tmem_st(uint32_t taddr, const uint32_t* v) {
  static_assert(W == 8 || W == 16, "width");
  if constexpr (W == 16) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
        "%12, %13, %14, %15, %16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
  } else {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
  }
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
// four rows (r0..r3) x box-width columns from col of a 2-D tensor map into
// consecutive smem rows (sm_100a tile::gather4)
__device__ __forceinline__ void gather4(uint32_t dst, const CUtensorMap* map, int col, int r0, int r1, int r2, int r3,
                                        uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

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
__global__ void k_build_jobs(int C, int mode, const int* off, const int* itemoff, const int* gcnt, int4* jobs) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    const int i0 = itemoff[c], i1 = itemoff[c + 1];
    const int r0 = off[c], r1 = off[c + 1];
    const int nc = mode == kModeAnchor ? gcnt[c] : 1;
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

// x-row index of row `r` of job J (-1: padding row)
__device__ __forceinline__ int job_row(const WsArgs& a, const int4& J, int r) {
  if (r >= J.z) return -1;
  const int e = __ldg(a.ent + J.y + r);
  return a.mode == kModeExtra ? e : e / (a.mode == kModeList ? a.list_div : a.dm.Cp);
}
// A-row scale exponent of row n centred on component c (same in producer and epilogue)
__device__ __forceinline__ int row_exp(const WsArgs& a, int n, int c) {
  return n < 0 ? 0 : scale_exp(__ldg(a.xmax + n) + __ldg(a.mumax + c));
}

template <int HP, bool PROF>
__global__ void __launch_bounds__(kThreads, 1) k_score_ws(WsArgs a, const __grid_constant__ CUtensorMap xmap) {
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  __shared__ uint64_t s_afull[2], s_aempty[2], s_tfull[2], s_tempty[2];
  __shared__ uint64_t s_bfull[kMaxNB], s_bempty[kMaxNB];
  __shared__ uint64_t s_mufull[2], s_muempty[2];
  __shared__ uint64_t s_xfull[kMaxXSlots][4], s_xempty[kMaxXSlots][4];  // X ring, per lane quadrant
  __shared__ __align__(16) float s_mu[2][kMaxD + 8];
  __shared__ int s_muoff[2];
  __shared__ __align__(16) float s_rec[4 * qg_max(HP) * rec_stride(HP)];  // epilogue records, per warp
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
      mbar_init(&s_mufull[i], 1);
      mbar_init(&s_muempty[i], kProdWarps);
    }
    for (int i = 0; i < NB; ++i) {
      mbar_init(&s_bfull[i], 1);
      mbar_init(&s_bempty[i], 1);
    }
    for (int i = 0; i < kMaxXSlots; ++i)
      for (int q = 0; q < 4; ++q) {
        mbar_init(&s_xfull[i][q], 1);
        mbar_init(&s_xempty[i][q], kKSplit);
      }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(a.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = s_tmem;
  // B stage map (offsets from a 1024-aligned stage base): B1 hi | B1 lo (N1max
  // rows each) | B2 hi | B2 lo (16 rows each), 128-byte rows
  const uint32_t offB1 = 0;
  const uint32_t offB2 = offB1 + 2 * a.N1max * 128;
  // TMEM map: accumulators [0, nacc*TB), then the two A stages of 128 columns
  const uint32_t colA = a.nacc * a.TB;

  if (warp < kProdWarps) {
    // ============================================================ A producers
    // thread = (row ar of the 128-row block, K slice ah of each 64-wide chunk).
    // Rows arrive in a shared-memory ring of row chunks (64 floats per row,
    // padded rows) slots - 1 chunks ahead and across job borders: in each TMEM
    // lane quadrant the slice-0 warp issues one bulk copy per row (32 lanes in
    // parallel keep many copies in flight), and the quadrant's four warps
    // release the slot after reading it. Then v = (x - mu_a) 2^k and
    // q = v^2 2^-14 are split into fp16 hi / lo pairs and stored to TMEM.
    const int ar = 32 * (warp & 3) + lane, ah = warp >> 2;  // row, K slice
    const int quad = warp & 3;
    const int XS = a.xslots;
    const int CPS = a.cps;
    const int XR = x_row(CPS);
    const uint32_t SLOT = x_slot_bytes(CPS);
    const int nslot = (nchunk + CPS - 1) / CPS;  // X-ring slots per job
    const int ahead = min(XS - 1, nslot);
    const uint32_t xbase = sbase + NB * a.stage_bytes;
    Prof pf{};
    if (PROF) pf.start();
    Walk w = walk_begin(a.jobs, total);
    Walk wn = w;
    wn.advance(a.jobs, a.qg, total);
    int n_cur = w.valid(total) ? job_row(a, w.J, ar) : -1;
    int n_nxt = wn.valid(total) ? job_row(a, wn.J, ar) : -1;
    // issue unit `unit` (slot p = chunks [p*CPS, (p+1)*CPS) of row n) of this
    // quadrant (slice-0 warps only): one bulk copy per row covers CPS chunks
    // (the SM accepts a bulk copy only every ~26 cycles, tools/micro/bulk_issue.cu)
    // (slot index and use count are carried incrementally: the runtime
    // divisions by XS / CPS per chunk were ~10 % of the kernel's stall samples)
    auto issue_x = [&](int n, int p, int sl, uint32_t use) {
      if (use >= 1) mbar_wait(&s_xempty[sl][quad], (use - 1) & 1u);
      const int d0 = p * CPS * kKC;
      const bool valid = n >= 0 && d0 < dm.D && !(PROF && (a.dbg & 1));
      const unsigned vm = __ballot_sync(0xffffffffu, valid);
      if (a.gather) {
        // lane g < 8 moves the quadrant's rows 4g..4g+3 with one gather4 (the
        // full box width; padding rows repeat a valid row of the group)
        int rr[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) rr[k] = __shfl_sync(0xffffffffu, n, (4 * lane + k) & 31);
        const unsigned gm = lane < 8 ? (vm >> (4 * lane)) & 0xfu : 0u;
        const unsigned ops = __ballot_sync(0xffffffffu, gm != 0u);
        if (lane == 0)
          mbar_arrive_expect_tx(&s_xfull[sl][quad], static_cast<uint32_t>(__popc(ops)) * 4u * XR * 4u);
        __syncwarp();
        if (gm != 0u) {
          const int any = rr[__ffs(gm) - 1];
#pragma unroll
          for (int k = 0; k < 4; ++k) rr[k] = ((gm >> k) & 1u) ? rr[k] : any;
          gather4(xbase + sl * SLOT + (32 * quad + 4 * lane) * (XR * 4), &xmap, d0, rr[0], rr[1], rr[2], rr[3],
                  &s_xfull[sl][quad]);
        }
      } else {
        const uint32_t bytes = static_cast<uint32_t>(min(CPS * kKC, dm.D - d0)) * 4u;
        if (lane == 0) mbar_arrive_expect_tx(&s_xfull[sl][quad], static_cast<uint32_t>(__popc(vm)) * bytes);
        __syncwarp();
        if (valid)
          bulk_copy(xbase + sl * SLOT + ar * (XR * 4), a.X + (int64_t)n * dm.D + d0, bytes, &s_xfull[sl][quad]);
      }
    };
    uint32_t sc = 0;  // flat chunk counter (A stages)
    uint32_t su = 0;  // flat X-ring slot counter
    int xs = 0;
    if (w.valid(total) && ah == 0)
      for (int k = 0; k < ahead; ++k) issue_x(n_cur, k, k, 0u);
    uint32_t sdiv = 0;  // su / XS (xs = su % XS)
    int jb = 0;
    while (w.valid(total)) {
      const int mslot = jb & 1;
      const float sA = exp2i(row_exp(a, n_cur, w.J.x));
      mbar_wait(&s_mufull[mslot], (jb >> 1) & 1);
      const float* mu_s = s_mu[mslot] + s_muoff[mslot];
      for (int ch = 0; ch < nchunk; ++ch, ++sc) {
        const int within = CPS == 1 ? 0 : (ch & (CPS - 1));  // CPS is 1 or 2
        if (within == 0) {
          if (ah == 0) {  // prefetch slot su + ahead (this job or the next)
            const int p2 = (CPS == 1 ? ch : ch >> 1) + ahead;
            int sl = xs + ahead;
            uint32_t use = sdiv;
            if (sl >= XS) sl -= XS, use += 1u;
            if (p2 < nslot) issue_x(n_cur, p2, sl, use);
            else issue_x(wn.valid(total) ? n_nxt : -1, p2 - nslot, sl, use);
          }
          mbar_wait(&s_xfull[xs][quad], sdiv & 1u);
        }
        if (PROF) pf.lap(kPBuild);  // (waiting for the row pieces)
        const int s = static_cast<int>(sc & 1u);
        const uint32_t use = sc >> 1;
        const int d0 = ch * kKC + kElem * ah;
        const uint32_t xrow = xbase + xs * SLOT + ar * (XR * 4) + (within * kKC + kElem * ah) * 4;
        uint32_t vh[kElem / 2], vl[kElem / 2], qh[kElem / 2], ql[kElem / 2];
        // (a live row's slice inside D -- nearly every call -- skips the per-element bounds selects)
        auto build = [&](auto fullc) {
          constexpr bool kFullSlice = decltype(fullc)::value;
#pragma unroll
          for (int jj = 0; jj < kXSeg; ++jj) {
            const int d = d0 + 4 * jj;
            float xv[4];
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(xv[0]), "=f"(xv[1]), "=f"(xv[2]), "=f"(xv[3])
                         : "r"(xrow + jj * 16)
                         : "memory");
            const float4 m4 = *reinterpret_cast<const float4*>(mu_s + d);  // (D % 4 == 0: aligned window)
            const float mv[4] = {m4.x, m4.y, m4.z, m4.w};
            float v[4], q[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if constexpr (kFullSlice) v[k] = (xv[k] - mv[k]) * sA;
              else v[k] = (d + k < dm.D && n_cur >= 0) ? (xv[k] - mv[k]) * sA : 0.f;
              q[k] = (v[k] * v[k]) * exp2i(-kTargetExp);
            }
            split2(v[0], v[1], vh[2 * jj], vl[2 * jj]);
            split2(v[2], v[3], vh[2 * jj + 1], vl[2 * jj + 1]);
            split2(q[0], q[1], qh[2 * jj], ql[2 * jj]);
            split2(q[2], q[3], qh[2 * jj + 1], ql[2 * jj + 1]);
          }
        };
        if (n_cur >= 0 && d0 + kElem <= dm.D) build(std::true_type{});
        else build(std::false_type{});
        if (within == CPS - 1 || ch == nchunk - 1) {  // this warp is done with the row slot
          __syncwarp();
          if (lane == 0) mbar_arrive(&s_xempty[xs][quad]);
          ++su;
          if (++xs == XS) xs = 0, ++sdiv;
        }
        if (PROF) pf.lap(kPSplit);
        if (use >= 1) mbar_wait(&s_aempty[s], (use - 1) & 1u);
        if (PROF) pf.lap(kPWaitEmpty);
        if (tid == 32) trace(tp, static_cast<int>(sc), 0);
        // operand columns: v hi | v lo | q hi | q lo (32 each); this thread's K slice
        const uint32_t ta =
            tmem + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + colA + s * 128 + (kElem / 2) * ah;
        tmem_st<kElem / 2>(ta, vh);
        tmem_st<kElem / 2>(ta + 32, vl);
        tmem_st<kElem / 2>(ta + 64, qh);
        tmem_st<kElem / 2>(ta + 96, ql);
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
      w = wn;
      if (!w.valid(total)) break;
      wn.advance(a.jobs, a.qg, total);
      n_cur = n_nxt;
      n_nxt = wn.valid(total) ? job_row(a, wn.J, ar) : -1;
      if (PROF) pf.lap(kPSync);
    }
    // drain: the slots issued beyond the last chunk (nothing is read from them)
    if (ah == 0 && su > 0)
      for (uint32_t u = su; u < su + static_cast<uint32_t>(ahead); ++u)
        mbar_wait(&s_xfull[u % XS][quad], (u / XS) & 1u);
    if (PROF && a.prof && lane == 0) {
      atomicAdd(a.prof + kPSync, pf.acc[kPSync]);
      atomicAdd(a.prof + kPBuild, pf.acc[kPBuild]);
      atomicAdd(a.prof + kPWaitEmpty, pf.acc[kPWaitEmpty]);
      atomicAdd(a.prof + kPSplit, pf.acc[kPSplit]);
      atomicAdd(a.prof + kPStore, pf.acc[kPStore]);
    }
  } else if (warp == kLoadWarp) {
    // ============================================================ loader
    if (lane == 0) {
      uint32_t bc = 0, luse = 0;
      int ls = 0;
      int jb = 0;
      for (Walk w = walk_begin(a.jobs, total); w.valid(total); w.advance(a.jobs, a.qg, total), ++jb) {
        const int c = w.J.x;
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
        const int ng = a.mode == kModeAnchor ? a.ngroups : 1;
        const __half* src0 = a.img + ((int64_t)c * ng + grp) * nchunk * (a.stage_bytes / 2);
        const bool ifree = a.mode == kModeAnchor && a.limg != nullptr;
        const int nq = min(a.qg, w.J.w - w.g0);
        const uint32_t wb = HP * 128;                 // one plane of a component's W rows
        const uint32_t s1 = 2 * 128 * (a.N1max1 + kNL);  // one-component stage bytes
        for (int ch = 0; ch < nchunk; ++ch, ++bc, ls = ls + 1 == NB ? (++luse, 0) : ls + 1) {
          const int s = ls;  // bc % NB, and luse = bc / NB, carried incrementally
          const uint32_t use = luse;
          if (use >= 1) mbar_wait(&s_bempty[s], (use - 1) & 1u);
          trace(tp, static_cast<int>(bc), 5);
          const uint32_t dst = sbase + s * a.stage_bytes;
          if (!ifree) {
            mbar_arrive_expect_tx(&s_bfull[s], a.stage_bytes);
            bulk_copy(dst, src0 + (int64_t)ch * (a.stage_bytes / 2), a.stage_bytes, &s_bfull[s]);
          } else {
            // stage = [B1 hi: lin 16 | W of q_0..q_nq-1 | B1 lo: same | B2 hi | B2 lo]
            const __half* li = a.limg + (((int64_t)c * ng + grp) * nchunk + ch) * (4 * kNL * 64);
            const uint32_t lo1 = a.N1max * 128;  // B1 lo plane offset (bytes)
            mbar_arrive_expect_tx(&s_bfull[s], 4u * kNL * 128u + 2u * wb * static_cast<uint32_t>(nq));
            bulk_copy(dst, li, kNL * 128, &s_bfull[s]);                          // lin hi
            bulk_copy(dst + lo1, li + kNL * 64, kNL * 128, &s_bfull[s]);         // lin lo
            bulk_copy(dst + 2 * lo1, li + 2 * kNL * 64, 2 * kNL * 128, &s_bfull[s]);  // psi hi | psi lo
            for (int qi = 0; qi < nq; ++qi) {
              const int q = __ldg(a.g + (int64_t)c * dm.G + w.g0 + qi);
              const __half* sq = a.simg1 + ((int64_t)q * nchunk + ch) * (s1 / 2);
              const uint32_t o = (kNL + qi * HP) * 128;
              bulk_copy(dst + o, sq + kNL * 64, wb, &s_bfull[s]);                              // W hi
              bulk_copy(dst + lo1 + o, sq + (a.N1max1 + kNL) * 64, wb, &s_bfull[s]);           // W lo
            }
          }
          trace(tp, static_cast<int>(bc), 6);
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ============================================================ MMA issuer
    uint32_t sc = 0, bc = 0;
    int sb = 0;        // bc % NB and the parity of bc / NB, carried incrementally
    uint32_t bph = 0;
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
      for (int ch = 0; ch < nchunk; ++ch, ++sc, ++bc, sb = sb + 1 == NB ? (bph ^= 1u, 0) : sb + 1) {
        const int s = static_cast<int>(sc & 1u);
        mbar_wait(&s_afull[s], (sc >> 1) & 1u);
        if (lane == 0) trace(tp, static_cast<int>(sc), 4);
        mbar_wait(&s_bfull[sb], bph);
        fence_after();
        if (PROF) pf.lap(kMWaitFull);
        if (lane == 0) trace(tp, static_cast<int>(sc), 2);
        if (lane == 0) {
          const uint32_t st = sbase + sb * a.stage_bytes;
          const uint32_t id1 = idesc(N1), id2 = idesc(kNL);
          const uint32_t tA = tmem + colA + s * 128;  // v hi | v lo | q hi | q lo
          const uint32_t Av[3] = {tA, tA, tA + 32};
          const uint32_t Aq[3] = {tA + 64, tA + 64, tA + 96};
          const uint32_t B1[3] = {st + offB1, st + offB1 + a.N1max * 128, st + offB1};
          const uint32_t B2[3] = {st + offB2, st + offB2 + kNL * 128, st + offB2};
#pragma unroll
          for (int p = 0; p < ((PROF && (a.dbg & 4)) ? 0 : 3); ++p) {
#pragma unroll
            for (int k = 0; k < kKC / 16; ++k) {
              const uint32_t acc = (ch > 0 || p > 0 || k > 0) ? 1u : 0u;
              mma_f16_ts(acc1, Av[p] + k * 8, sdesc(B1[p] + k * 32), id1, acc);
              mma_f16_ts(acc2, Aq[p] + k * 8, sdesc(B2[p] + k * 32), id2, acc);
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
    // Each warp stages the job's per-slot records in its own shared-memory
    // block (vector loads, before waiting for the accumulator), then reads
    // them as broadcasts while assembling its 32 rows.
    constexpr int kEpiBatch = HP >= 16 ? 1 : 16 / HP;  // components per tcgen05.ld batch
    constexpr int R = rec_stride(HP);
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    float* srec = s_rec + quad * (qg_max(HP) * R);
    int jb = 0;
    Prof pf{};
    if (PROF) pf.start();
    for (Walk w = walk_begin(a.jobs, total); w.valid(total); w.advance(a.jobs, a.qg, total), ++jb) {
      const int b = a.nacc == 2 ? (jb & 1) : 0;
      const int use_b = a.nacc == 2 ? (jb >> 1) : jb;
      const int c = w.J.x;
      const int nq = min(a.qg, w.J.w - w.g0);
      const int e = r < w.J.z ? __ldg(a.ent + w.J.y + r) : -1;
      const int n = e < 0 ? -1 : (a.mode == kModeExtra ? e : e / (a.mode == kModeList ? a.list_div : dm.Cp));
      {
        const float4* src = reinterpret_cast<const float4*>(
            a.rec + ((int64_t)c * (a.mode == kModeAnchor ? dm.G : 1) + w.g0) * R);
        __syncwarp();
        for (int i = lane; i < nq * R / 4; i += 32) reinterpret_cast<float4*>(srec)[i] = __ldg(src + i);
        __syncwarp();
      }
      const int kA = row_exp(a, n, c);
      const float invA = exp2i(-kA), invQ = exp2i(kTargetExp - 2 * kA);
      mbar_wait(&s_tfull[b], use_b & 1);
      fence_after();
      if (PROF) pf.lap(kEWait);
      const int N1 = kNL + ((nq * HP + 15) / 16) * 16;
      const uint32_t trow = tmem + b * a.TB + (static_cast<uint32_t>(quad * 32) << 16);
      float lin[16], d2[16];
      if constexpr (HP != 16) {  // (HP == 16: loaded after the W columns, see below)
        tmem_ld_nowait<16>(trow, lin);
        tmem_ld_nowait<16>(trow + N1, d2);
        tmem_wait_ld();
        pin_regs<16>(lin);
        pin_regs<16>(d2);
      }
      int64_t obase = 0;
      if (e >= 0) {
        if (a.mode == kModeAnchor) {
          const int nn = e / dm.Cp, j = e - nn * dm.Cp;
          obase = (int64_t)nn * dm.SL + j * dm.G + w.g0;
        } else if (a.mode == kModeExtra) {
          obase = (int64_t)e * dm.SL + dm.Cp * dm.G;
        } else {
          obase = e;
        }
      }
      // one component's log-joint from |y|^2 (yy), its lin / psi accumulators and record.
      // Cancellation check: the fp32-accurate terms carry ~1e-6 of their
      // magnitude B = sum u^2/psi + |lin| + m + 2 sum |t|(|y| + |b|); when B
      // exceeds kCancel M (M <= the log-joint's term magnitude) the result
      // could miss the 1e-4 bar, so the
      // slot is flagged in the lowest mantissa bit of its score (every other
      // score has that bit cleared: 1 ulp) and vmfa_fixup.cu re-evaluates it
      // in fp64.
      auto finish = [&](int qi, float yy, float ey) {
        const float* rc = srec + qi * R;
        float linq = 0.f, d2q = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (i == qi) {
            linq = lin[i];
            d2q = d2[i];
          }
        linq *= invA * rc[3];
        d2q *= invQ * rc[4];
        const double kc = static_cast<double>(rc[1]) + static_cast<double>(rc[5]);
        const double diag = static_cast<double>(d2q) + static_cast<double>(linq) + static_cast<double>(rc[2]);
        const double Q = diag - static_cast<double>(yy);
        float lj = static_cast<float>(kc - 0.5 * Q);
        // the test's scale (_helpers.lj_term_scale) is >= max(0.92 D, |kconst| - |log pi|, |Q| / 2)
        const float B = fabsf(d2q) + fabsf(linq) + fabsf(rc[2]) + 2.f * ey + yy;
        // M: a lower bound of that term scale; rc[6] + |Q| / 2 is the scale itself
        const float M = fmaxf(fmaxf(fmaxf(0.9f * static_cast<float>(dm.D), fabsf(static_cast<float>(kc)) - 20.f),
                                    0.5f * fabsf(static_cast<float>(Q))),
                              rc[6] + 0.5f * fabsf(static_cast<float>(Q)));
        const bool flag = B > kCancel * M;
        unsigned bits = __float_as_uint(lj);
        if (isfinite(lj)) bits = flag ? (bits | 1u) : (bits & ~1u);
        lj = __uint_as_float(bits);
        if (e >= 0) {
          const int64_t o = obase + (a.mode == kModeAnchor ? qi : 0);
          a.out[o] = lj;
          if (flag && a.fix_list && isfinite(lj)) {
            const unsigned long long pos = atomicAdd(a.fix_cnt, 1ull);
            if (static_cast<long long>(pos) < a.fix_cap) a.fix_list[pos] = o;
            else a.fix_cnt[1] = 1ull;
          }
        }
      };
      if constexpr (HP == 16) {
        // The accumulator is held only while its columns are read: |y|^2 and
        // the error sum of every component first (two registers each), then
        // the lin / psi columns; the buffer is released before the fp64
        // assembly, flags and stores (with one accumulator buffer -- 192
        // columns at config 3 -- the next job's MMAs wait for this release)
        constexpr int QMAX = qg_max(HP);
        float yyv[QMAX], eyv[QMAX];
#pragma unroll
        for (int q0 = 0; q0 < QMAX; q0 += kEpiBatch) {
          if (q0 >= nq) break;
          const int nb = min(kEpiBatch, nq - q0);
          float y[kEpiBatch][HP];
#pragma unroll
          for (int qi = 0; qi < kEpiBatch; ++qi)
            if (qi < nb) tmem_ld_nowait<HP>(trow + kNL + (q0 + qi) * HP, y[qi]);
          tmem_wait_ld();
          pin_regs<kEpiBatch * HP>(&y[0][0]);
#pragma unroll
          for (int qi = 0; qi < kEpiBatch; ++qi) {
            if (q0 + qi >= QMAX) break;
            float yy = 0.f, ey = 0.f;
            if (qi < nb) {
              const float* rc = srec + (q0 + qi) * R;
#pragma unroll
              for (int h = 0; h < HP; ++h) {
                const float ys = y[qi][h] * (invA * rc[8 + HP + h]);
                const float t = ys - rc[8 + h];
                yy = fmaf(t, t, yy);
                ey = fmaf(fabsf(t), fabsf(ys) + fabsf(rc[8 + h]), ey);
              }
            }
            yyv[q0 + qi] = yy;
            eyv[q0 + qi] = ey;
          }
        }
        tmem_ld_nowait<16>(trow, lin);
        tmem_ld_nowait<16>(trow + N1, d2);
        tmem_wait_ld();
        pin_regs<16>(lin);
        pin_regs<16>(d2);
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_tempty[b]);
        if (PROF) pf.lap(kEWork);
#pragma unroll
        for (int qi = 0; qi < QMAX; ++qi) {
          if (qi >= nq) break;
          finish(qi, yyv[qi], eyv[qi]);
        }
        continue;
      } else if constexpr (HP < 16) {  // two accumulator buffers fit: the epilogue overlaps the next job as it is
        for (int q0 = 0; q0 < nq; q0 += kEpiBatch) {
          const int nb = min(kEpiBatch, nq - q0);
          float y[kEpiBatch][HP];
#pragma unroll
          for (int qi = 0; qi < kEpiBatch; ++qi)
            if (qi < nb) tmem_ld_nowait<HP>(trow + kNL + (q0 + qi) * HP, y[qi]);
          tmem_wait_ld();
          pin_regs<kEpiBatch * HP>(&y[0][0]);
#pragma unroll
          for (int qi = 0; qi < kEpiBatch; ++qi) {
            if (qi >= nb) break;
            const float* rc = srec + (q0 + qi) * R;
            float yy = 0.f, ey = 0.f;
#pragma unroll
            for (int h = 0; h < HP; ++h) {
              const float ys = y[qi][h] * (invA * rc[8 + HP + h]);
              const float t = ys - rc[8 + h];
              yy = fmaf(t, t, yy);
              ey = fmaf(fabsf(t), fabsf(ys) + fabsf(rc[8 + h]), ey);
            }
            finish(q0 + qi, yy, ey);
          }
        }
      } else {  // wide factors: 16 columns at a time
        for (int qi = 0; qi < nq; ++qi) {
          const float* rc = srec + qi * R;
          float yy = 0.f, ey = 0.f;
          for (int h0 = 0; h0 < HP; h0 += 16) {
            float y[16];
            tmem_ld_nowait<16>(trow + kNL + qi * HP + h0, y);
            tmem_wait_ld();
            pin_regs<16>(y);
#pragma unroll
            for (int h = 0; h < 16; ++h) {
              const float ys = y[h] * (invA * rc[8 + HP + h0 + h]);
              const float t = ys - rc[8 + h0 + h];
              yy = fmaf(t, t, yy);
              ey = fmaf(fabsf(t), fabsf(ys) + fabsf(rc[8 + h0 + h]), ey);
            }
          }
          finish(qi, yy, ey);
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

// Per-slot epilogue records, one warp per (anchor, slot) -- or per component
// when single != 0 -- after the stage images (which supply the row scales):
//   [0] q (int bits)  [1] kconst_q hi  [2] m  [3] lin row scale  [4] psi row scale
//   [5] kconst_q lo   [8, 8+Hp) b_h     [8+Hp, 8+2Hp) W row scales
// with b = W_q^T (mu_q - mu_a), m = sum psi_q^-1 (mu_q - mu_a)^2 (fp32 operands,
// fp64 accumulation; 0 for single), kconst = hi + lo exactly to ~48 bits.
__global__ void __launch_bounds__(256) k_build_records(Dims dm, int Hp, int qg, int ngroups, int N1max, int single,
                                                       const float* WT, const float* mu32, const float* ipsi32,
                                                       const double* kconst, const int* g, const int* gcnt,
                                                       const float* scl, float* rec, int fused,
                                                       const double* logpi, const double* logdet) {
  const int lane = threadIdx.x & 31;
  const int R = rec_stride(Hp);
  const int nslot = single ? 1 : dm.G;
  const int ng = single ? 1 : ngroups;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = gw; w < (int64_t)dm.C * nslot; w += nw) {
    const int c = static_cast<int>(w / nslot), i = static_cast<int>(w - (int64_t)c * nslot);
    float* out = rec + w * R;
    if (!single && i >= gcnt[c]) continue;
    const int q = single ? c : g[(int64_t)c * dm.G + i];
    const int grp = single ? 0 : i / qg, qi = single ? 0 : i - grp * qg;
    const float* sr = scl + ((int64_t)c * ng + grp) * (N1max + kNL);
    double m = 0.0;
    if (fused) {
      // m and b were written by k_build_images (anchor images)
    } else if (!single) {
      const float* mq = mu32 + (int64_t)q * dm.D;
      const float* ma = mu32 + (int64_t)c * dm.D;
      const float* ip = ipsi32 + (int64_t)q * dm.D;
      // b in blocks of 8 latent rows (8 independent loads and fp64 sums per
      // lane and dimension), m beside the first block; the products of two
      // fp32 values are exact in fp64, so only the summation order is fixed here
      for (int h0 = 0; h0 < Hp; h0 += 8) {
        double sb[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        const float* wr = WT + ((int64_t)q * Hp + h0) * dm.D;
        for (int d = lane; d < dm.D; d += 32) {
          const float dlf = mq[d] - ma[d];  // same fp32 rounding as the scorer's operands
          const double dl = static_cast<double>(dlf);
          if (h0 == 0) m += static_cast<double>(ip[d]) * dl * dl;
#pragma unroll
          for (int h = 0; h < 8; ++h)
            if (h0 + h < Hp) sb[h] += static_cast<double>(__ldg(wr + (int64_t)h * dm.D + d)) * dl;
        }
#pragma unroll
        for (int h = 0; h < 8; ++h) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) sb[h] += __shfl_xor_sync(0xffffffffu, sb[h], o);
          if (lane == 0 && h0 + h < Hp) out[8 + h0 + h] = static_cast<float>(sb[h]);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
    } else {
      for (int h = lane; h < Hp; h += 32) out[8 + h] = 0.f;
    }
    for (int h = lane; h < Hp; h += 32) out[8 + Hp + h] = sr[kNL + qi * Hp + h];
    if (lane == 0) {
      const double kc = kconst[q];
      const float hi = static_cast<float>(kc);
      out[0] = __int_as_float(q);
      out[1] = hi;
      if (!fused) out[2] = static_cast<float>(m);
      out[3] = sr[qi];
      out[4] = sr[N1max + qi];
      out[5] = isfinite(kc) ? static_cast<float>(kc - static_cast<double>(hi)) : 0.f;
      // [6] the magnitude of the log-joint's constant terms, |log pi| + (D
      // log 2pi + |log|Sigma||) / 2: with |Q| / 2 it is the scale the
      // parity tests measure log-joint errors against (flag criterion)
      out[6] = (logpi && logdet && isfinite(logpi[q]))
                   ? static_cast<float>(fabs(logpi[q]) + 0.5 * (dm.D * 1.8378770664093453 + fabs(logdet[q])))
                   : 0.f;
      out[7] = 0.f;
    }
  }
}

// B stage images: for anchor a, component group grp and K chunk ch, the exact
// shared-memory stage the MMA reads -- [B1 hi | B1 lo] (N1max rows: 16 lin
// rows, then Hp W rows per component of the group) and [B2 hi | B2 lo] (16
// psi^-1 rows) -- each row scaled by 2^k (max over D ~ 2^14), split into fp16
// hi/lo and 128B-swizzled, so the loader moves a stage with one bulk copy;
// bscl receives 2^-k per row. One warp per B row (all chunks). single != 0:
// one component (q = a), lin = 0 (extra candidates, truncated F).
__global__ void __launch_bounds__(256) k_build_images(Dims dm, int Hp, int qg, int ngroups, int N1max, int single,
                                                      const float* WT, const float* mu32, const float* ipsi32,
                                                      const int* g, const int* gcnt, __half* img, float* bscl,
                                                      const float* sscl, int N1max1, float* rec, __half* limg) {
  const int lane = threadIdx.x & 31;
  const int nchunk = (dm.D + kKC - 1) / kKC;
  const int ng = single ? 1 : ngroups;
  const int nrow = N1max + kNL;
  const int nrow1 = N1max1 + kNL;  // rows of a one-component image (sscl layout)
  const int64_t stage_h = 2 * 64 * (int64_t)nrow;  // halves per stage
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool vec = (dm.D & 3) == 0;
  const bool small = (int64_t)dm.C * ng * nrow < (int64_t{1} << 31);
  for (int64_t wi = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; wi < (int64_t)dm.C * ng * nrow;
       wi += nw) {
    // (row, group, anchor) of this warp's B row: 32-bit divisions when the row
    // count allows (three 64-bit divisions per row were a third of the kernel's
    // instructions)
    int row, grp, a;
    if (small) {
      const unsigned w32 = static_cast<unsigned>(wi), ag = w32 / static_cast<unsigned>(nrow);
      row = static_cast<int>(w32 - ag * static_cast<unsigned>(nrow));
      a = static_cast<int>(ag / static_cast<unsigned>(ng));
      grp = static_cast<int>(ag - static_cast<unsigned>(a) * static_cast<unsigned>(ng));
    } else {
      row = static_cast<int>(wi % nrow);
      grp = static_cast<int>((wi / nrow) % ng);
      a = static_cast<int>(wi / ((int64_t)nrow * ng));
    }
    const int slot0 = grp * qg;
    const int nq = single ? 1 : min(qg, gcnt[a] - slot0);
    // source of this row: kind 0 zero, 1 lin (q), 2 W (q, h), 3 psi (q)
    int kind = 0, q = 0, h = 0;
    if (row < N1max) {
      if (row < kNL) {
        if (!single && row < nq) kind = 1, q = g[(int64_t)a * dm.G + slot0 + row];
      } else {
        const int qi = (row - kNL) / Hp;
        h = (row - kNL) - qi * Hp;
        if (qi < nq) kind = 2, q = single ? a : g[(int64_t)a * dm.G + slot0 + qi];
      }
    } else if (row - N1max < nq) {
      kind = 3, q = single ? a : g[(int64_t)a * dm.G + slot0 + (row - N1max)];
    }
    const float* src = kind == 2 ? WT + ((int64_t)q * Hp + h) * dm.D : ipsi32 + (int64_t)q * dm.D;
    const float* mq = mu32 + (int64_t)q * dm.D;
    const float* ma = mu32 + (int64_t)a * dm.D;
    // 8 consecutive values from d0 (vector loads when aligned and in range)
    auto load8 = [&](int d0, float* v) {
      if (kind == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = 0.f;
        return;
      }
      if (vec && d0 + 8 <= dm.D) {
        const float4 s0 = *reinterpret_cast<const float4*>(src + d0), s1 = *reinterpret_cast<const float4*>(src + d0 + 4);
        v[0] = s0.x, v[1] = s0.y, v[2] = s0.z, v[3] = s0.w, v[4] = s1.x, v[5] = s1.y, v[6] = s1.z, v[7] = s1.w;
        if (kind == 1) {
          const float4 q0 = *reinterpret_cast<const float4*>(mq + d0), q1 = *reinterpret_cast<const float4*>(mq + d0 + 4);
          const float4 a0 = *reinterpret_cast<const float4*>(ma + d0), a1 = *reinterpret_cast<const float4*>(ma + d0 + 4);
          const float dq[8] = {q0.x - a0.x, q0.y - a0.y, q0.z - a0.z, q0.w - a0.w,
                               q1.x - a1.x, q1.y - a1.y, q1.z - a1.z, q1.w - a1.w};
#pragma unroll
          for (int i = 0; i < 8; ++i) v[i] = -2.f * v[i] * dq[i];
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int d = d0 + i;
          float x = 0.f;
          if (d < dm.D) {
            x = src[d];
            if (kind == 1) x = -2.f * x * (mq[d] - ma[d]);
          }
          v[i] = x;
        }
      }
    };
    // row scale: W / psi rows reuse the one-component images' scales (same
    // row of the same component); lin rows depend on the anchor: max pass
    int k = 0;
    if (!single && sscl && (kind == 2 || kind == 3)) {
      const int r1 = kind == 2 ? kNL + h : N1max1;
      k = -static_cast<int>(((__float_as_uint(sscl[(int64_t)q * nrow1 + r1]) >> 23) & 0xffu)) + 127;
    } else {
      float mx = 0.f;
      if (kind != 0)
        for (int d0 = 8 * lane; d0 < dm.D; d0 += 256) {
          float v[8];
          load8(d0, v);
#pragma unroll
          for (int i = 0; i < 8; ++i) mx = fmaxf(mx, fabsf(v[i]));
        }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      k = scale_exp(mx);
    }
    const float sc = exp2i(k);
    if (lane == 0) bscl[((int64_t)a * ng + grp) * nrow + row] = exp2i(-k);
    // matrix offsets (halves) within a stage: B1 hi 0, B1 lo N1max*64, B2 hi 2*N1max*64, B2 lo +16*64
    const int rr = row < N1max ? row : row - N1max;
    int64_t off_hi = row < N1max ? 0 : 2 * (int64_t)N1max * 64;
    int64_t off_lo = row < N1max ? (int64_t)N1max * 64 : 2 * (int64_t)N1max * 64 + kNL * 64;
    __half* base = img + ((int64_t)a * ng + grp) * nchunk * stage_h;
    int64_t sth = stage_h;
    // limg != null (image-free anchor stages): only the lin and psi rows are
    // written, into the small image [lin hi | lin lo | psi hi | psi lo] (16
    // lines each, the same line positions and swizzle as in the stage); the W
    // rows come from the one-component images at scoring time
    const bool wimg = limg == nullptr || (row < N1max ? row < kNL : true);
    if (limg != nullptr) {
      base = limg + ((int64_t)a * ng + grp) * nchunk * (4 * kNL * 64);
      sth = 4 * kNL * 64;
      off_hi = row < N1max ? 0 : 2 * kNL * 64;
      off_lo = off_hi + kNL * 64;
    }
    // rec != null (anchor images): the record sums ride along -- a W row h of
    // q gives b_h = sum_d W_q[h][d] (mu_q - mu_a)[d], the psi row of q gives
    // m = sum_d psi_q^-1 (mu_q - mu_a)^2 (fp32 differences as the scorer's
    // operands, exact fp32 products, fp64 sums); k_build_records skips them
    const bool sums = rec != nullptr && (kind == 2 || kind == 3);
    double acc = 0.0;
    for (int u = lane; u < nchunk * (kKC / 8); u += 32) {  // one 16-byte unit (8 halves) per lane
      const int ch = u / (kKC / 8), j = u - ch * (kKC / 8);
      float v[8];
      load8(ch * kKC + 8 * j, v);
      if (sums) {
        const int d0 = ch * kKC + 8 * j;
        float dq[8];
        if (vec && d0 + 8 <= dm.D) {  // (two 16-byte loads per mean instead of 8 scalar ones)
          const float4 q0 = *reinterpret_cast<const float4*>(mq + d0), q1 = *reinterpret_cast<const float4*>(mq + d0 + 4);
          const float4 a0 = *reinterpret_cast<const float4*>(ma + d0), a1 = *reinterpret_cast<const float4*>(ma + d0 + 4);
          dq[0] = q0.x - a0.x, dq[1] = q0.y - a0.y, dq[2] = q0.z - a0.z, dq[3] = q0.w - a0.w;
          dq[4] = q1.x - a1.x, dq[5] = q1.y - a1.y, dq[6] = q1.z - a1.z, dq[7] = q1.w - a1.w;
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) dq[i] = d0 + i < dm.D ? mq[d0 + i] - ma[d0 + i] : 0.f;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (d0 + i < dm.D) {
            const double dl = static_cast<double>(dq[i]);
            acc += kind == 2 ? static_cast<double>(v[i]) * dl : static_cast<double>(v[i]) * dl * dl;
          }
        }
      }
      if (!wimg) continue;
      uint32_t hw[4], lw[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) split2(v[2 * i] * sc, v[2 * i + 1] * sc, hw[i], lw[i]);
      const int pos = rr * 64 + (((j ^ (rr & 7)) & 7) << 3);  // 128B swizzle: 16-byte unit j of row rr
      __half* st = base + ch * sth;
      *reinterpret_cast<uint4*>(st + off_hi + pos) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
      *reinterpret_cast<uint4*>(st + off_lo + pos) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
    if (sums) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) {
        const int qi = kind == 2 ? (row - kNL) / Hp : row - N1max;
        float* out = rec + ((int64_t)a * dm.G + slot0 + qi) * rec_stride(Hp);
        if (kind == 2) out[8 + h] = static_cast<float>(acc);
        else out[2] = static_cast<float>(acc);
      }
    }
  }
}

// per-row max |x| (A-row scale bounds), one warp per row
__global__ void k_rowmax(int64_t N, int D, const float* X, float* xmax) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t n = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; n < N; n += nw) {
    float m = 0.f;
    for (int d = lane; d < D; d += 32) m = fmaxf(m, fabsf(X[n * D + d]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) xmax[n] = m;
  }
}

int ws_qg(const Dims& dm, int single) {
  const int Hp = ws_hp(dm.H);
  return single ? 1 : std::max(1, std::min(dm.G, qg_max(Hp)));
}
int ws_n1max(const Dims& dm, int single) { return kNL + ((ws_qg(dm, single) * ws_hp(dm.H) + 15) / 16) * 16; }

}  // namespace

int ws_hp(int H) { return H <= 8 ? 8 : H <= 16 ? 16 : H <= 32 ? 32 : 64; }

int ws_groups(const Dims& dm) {
  const int qg = ws_qg(dm, 0);
  return (dm.G + qg - 1) / qg;
}

bool ws_smem_plan(int Hp, uint32_t stage_bytes, int* xslots, int* nb, size_t* dyn, int* cps);

bool score_ws_supported(const Dims& dm) {
  if (dm.D > kMaxD || dm.D % 4 != 0 || dm.H > 64 || dm.G > 64) return false;
  int xs, nb, cps;
  size_t dyn;
  for (int single = 0; single < 2; ++single)
    if (!ws_smem_plan(ws_hp(dm.H), static_cast<uint32_t>(2 * 128 * (ws_n1max(dm, single) + kNL)), &xs, &nb, &dyn,
                      &cps))
      return false;
  return true;
}

int64_t ws_image_halves(const Dims& dm, int single) {
  const int nchunk = (dm.D + kKC - 1) / kKC;
  const int ng = single ? 1 : ws_groups(dm);
  return (int64_t)dm.C * ng * nchunk * 2 * 64 * (ws_n1max(dm, single) + kNL);
}
// image-free anchor stages: the per-(anchor, group, chunk) lin / psi image
// (halves), and whether the W rows can be copied from the one-component
// images with their swizzle phase intact (Hp a multiple of 8)
int64_t ws_small_image_halves(const Dims& dm) {
  return (int64_t)dm.C * ws_groups(dm) * ((dm.D + kKC - 1) / kKC) * 4 * kNL * 64;
}
bool ws_image_free_ok(const Dims& dm) { return ws_hp(dm.H) % 8 == 0; }
int64_t ws_scale_floats(const Dims& dm, int single) {
  const int ng = single ? 1 : ws_groups(dm);
  return (int64_t)dm.C * ng * (ws_n1max(dm, single) + kNL);
}
int64_t ws_record_floats(const Dims& dm, int single) {
  return (int64_t)dm.C * (single ? 1 : dm.G) * rec_stride(ws_hp(dm.H));
}

cudaError_t launch_ws_images(const Dims& dm, int single, const float* WT, const float* mu32, const float* ipsi32,
                             const int* g, const int* gcnt, void* img, float* bscl, cudaStream_t s,
                             const float* sscl, float* rec, void* limg) {
  // (warp-strided over the B rows; 32 blocks per SM measured 0.09 ms faster than 8 at config 3)
  k_build_images<<<sm_count() * 32, 256, 0, s>>>(dm, ws_hp(dm.H), ws_qg(dm, single), ws_groups(dm),
                                                ws_n1max(dm, single), single, WT, mu32, ipsi32, g, gcnt,
                                                static_cast<__half*>(img), bscl, single ? nullptr : sscl,
                                                ws_n1max(dm, 1), single ? nullptr : rec,
                                                single ? nullptr : static_cast<__half*>(limg));
  return cudaGetLastError();
}

cudaError_t launch_ws_records(const Dims& dm, int single, const float* WT, const float* mu32, const float* ipsi32,
                              const double* kconst, const int* g, const int* gcnt, const float* scl, float* rec,
                              cudaStream_t s, int fused, const double* logpi, const double* logdet) {
  k_build_records<<<sm_count() * 8, 256, 0, s>>>(dm, ws_hp(dm.H), ws_qg(dm, single), ws_groups(dm),
                                                 ws_n1max(dm, single), single, WT, mu32, ipsi32, kconst, g, gcnt,
                                                 scl, rec, single ? 0 : fused, logpi, logdet);
  return cudaGetLastError();
}

cudaError_t launch_rowmax(int64_t N, int D, const float* X, float* xmax, cudaStream_t s) {
  k_rowmax<<<sm_count() * 8, 256, 0, s>>>(N, D, X, xmax);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- dense all-pairs pass
// exact_log_likelihood (model.cpp:139-148) scores every (n, c): components are
// blocked into pseudo-anchors a = bG with g'_a = {bG, ..., bG+G-1} (rows
// centred on mu_a), and a chunk of R rows gets the fake candidate list
// K'(n) = (0, G, 2G, ...), so the anchor pass writes l(n, c) to slot c of row
// n (slot j*G + i with j = c / G). Jobs are row-tile major (all blocks of one
// 128-row tile are adjacent): a tile of X is read from HBM once and the
// blocks' B images stay in L2.
__global__ void k_dense_groups(int C, int G, int* g, int* gcnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)C * G;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = static_cast<int>(i / G), k = static_cast<int>(i - (int64_t)c * G);
    const bool anchor = c % G == 0;
    g[i] = anchor && c + k < C ? c + k : 0;
    if (k == 0) gcnt[c] = anchor ? min(G, C - c) : 0;
  }
}
__global__ void k_dense_chunk(int C, int G, int nb, int R, int* ent, int4* jobs, int* itemoff) {
  const int ntile = (R + kRows - 1) / kRows;
  const int64_t nent = (int64_t)nb * R, njob = (int64_t)nb * ntile;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nent + njob;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < nent) {  // block b's rows in ascending order: e = n * nb + b (row n relative to the chunk)
      const int b = static_cast<int>(i / R), t = static_cast<int>(i - (int64_t)b * R);
      ent[i] = t * nb + b;
    } else {
      const int it = static_cast<int>(i - nent);
      const int tile = it / nb, b = it - tile * nb;
      jobs[it] = make_int4(b * G, b * R + tile * kRows, min(kRows, R - tile * kRows), min(G, C - b * G));
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) itemoff[C] = static_cast<int>(njob);
}
cudaError_t launch_dense_groups(int C, int G, int* g, int* gcnt, cudaStream_t s) {
  k_dense_groups<<<sm_count() * 4, 256, 0, s>>>(C, G, g, gcnt);
  return cudaGetLastError();
}
// CSR form of the same chunk for the single-role scorers (items of `rows` rows
// per pseudo-anchor, component-major): off[c] = ceil(c/G) R
__global__ void k_dense_csr(int C, int G, int R, int rows, int* off, int* itemoff) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c <= C; c += gridDim.x * blockDim.x) {
    const int k = (c + G - 1) / G;  // pseudo-anchors before c
    off[c] = k * R;
    itemoff[c] = k * ((R + rows - 1) / rows);
  }
}
cudaError_t launch_dense_chunk(int C, int G, int nb, int R, int* ent, int4* jobs, int* itemoff, cudaStream_t s) {
  k_dense_chunk<<<sm_count() * 4, 256, 0, s>>>(C, G, nb, R, ent, jobs, itemoff);
  return cudaGetLastError();
}
cudaError_t launch_dense_csr(int C, int G, int R, int rows, int* off, int* itemoff, cudaStream_t s) {
  k_dense_csr<<<(C + 256) / 256, 256, 0, s>>>(C, G, R, rows, off, itemoff);
  return cudaGetLastError();
}
int64_t dense_jobs(int nb, int R) { return (int64_t)nb * ((R + kRows - 1) / kRows); }

unsigned long long* g_ws_prof = nullptr;  // set by vmfa_diag_scorer_cycles
bool ws_diag_armed() { return g_ws_prof != nullptr; }
int g_ws_dbg = 0;                          // diagnostics flags (enable >> 1)
constexpr int kProfWords = 16 + 8 * kTraceEvents;

// Shared-memory plan: X ring slots and B ring stages within the opt-in limit
// (227 KB minus the kernel's static shared memory). false: does not fit.
// Slots of two K chunks (half the bulk copies) when they fit, else one.
bool ws_smem_plan(int Hp, uint32_t stage_bytes, int* xslots, int* nb, size_t* dyn, int* cps_out) {
  const size_t limit = 227 * 1024;
  const size_t stat = 2 * (kMaxD + 8) * 4 + 4 * qg_max(Hp) * rec_stride(Hp) * 4 + 1024;  // s_mu, s_rec, barriers
  const size_t avail = limit - stat - 1024;  // 1024: stage alignment slack
  static const int want_cps = [] {
    const char* v = std::getenv("VMFA_WS_CPS");
    return v ? std::max(1, std::min(kMaxCps, std::atoi(v))) : kMaxCps;
  }();
  for (int cps = want_cps; cps >= 1; --cps)
    for (int xs = kMaxXSlots; xs >= 2; --xs) {
      const size_t xb = static_cast<size_t>(xs) * x_slot_bytes(cps);
      if (xb + 2 * stage_bytes > avail) continue;
      *xslots = xs;
      *cps_out = cps;
      *nb = std::min(kMaxNB, static_cast<int>((avail - xb) / stage_bytes));
      if (*nb > 4 && xs < kMaxXSlots) *nb = 4;
      *dyn = static_cast<size_t>(*nb) * stage_bytes + xb + 1024;
      return true;
    }
  return false;
}

// 2-D tensor map of X (D fp32 columns x N rows) with a box of one slot row
// (x_row(cps) columns x 1 row) for tile::gather4
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
bool x_tensor_map(CUtensorMap* map, const float* X, int64_t N, int D, int box_cols) {
  static EncodeTiledFn encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(fn);
  }();
  if (!encode || N < 1) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(N)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(D) * 4};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), 1};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(X), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t launch_score_ws(int mode, const ScoreArgs& s, const WsOperands& op, int4* jobs, cudaStream_t st,
                            bool build_jobs) {
  WsArgs a{};
  a.dm = s.dm;
  a.mode = mode;
  a.Hp = ws_hp(s.dm.H);
  const int single = mode == kModeAnchor ? 0 : 1;
  a.qg = ws_qg(s.dm, single);
  a.N1max = ws_n1max(s.dm, single);
  const int cols = a.N1max + kNL;
  a.TB = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : 256;
  a.nacc = (2 * a.TB + 2 * 128 <= 512) ? 2 : 1;  // A stages use 2 x 128 TMEM columns
  const uint32_t need = a.nacc * a.TB + 2 * 128;
  a.tmem_cols = need <= 256 ? 256 : 512;
  a.stage_bytes = static_cast<uint32_t>(2 * 128 * (a.N1max + kNL));
  // shared memory: the producers' X ring + the B ring (>= 2 stages each)
  size_t dyn = 0;
  if (!ws_smem_plan(a.Hp, a.stage_bytes, &a.xslots, &a.nbstage, &dyn, &a.cps)) return cudaErrorInvalidValue;
  static const int want_gather = [] {
    const char* v = std::getenv("VMFA_WS_GATHER4");
    return v ? std::atoi(v) : 1;
  }();
  CUtensorMap xmap{};
  a.gather = want_gather && x_tensor_map(&xmap, s.X, s.dm.N, s.dm.D, x_row(a.cps)) ? 1 : 0;
  a.X = s.X;
  a.xmax = op.xmax;
  a.mumax = op.mumax;
  a.mu32 = op.mu32;
  a.rec = single ? op.srec : op.brec;
  a.img = static_cast<const __half*>(single ? op.simg : op.bimg);
  a.limg = single ? nullptr : static_cast<const __half*>(op.limg);
  a.simg1 = static_cast<const __half*>(op.simg);
  a.N1max1 = ws_n1max(s.dm, 1);
  a.ngroups = ws_groups(s.dm);
  a.jobs = jobs;
  a.itemoff = s.itemoff;
  a.ent = s.ent;
  a.g = s.g;
  a.gcnt = s.gcnt;
  a.out = s.out;
  a.list_div = s.list_div;
  a.fix_list = op.fix_list;
  a.fix_cnt = op.fix_cnt;
  a.fix_cap = op.fix_cap;
  a.prof = g_ws_prof;
  a.dbg = g_ws_prof ? g_ws_dbg : 0;
  if (build_jobs) k_build_jobs<<<(s.dm.C + 255) / 256, 256, 0, st>>>(s.dm.C, mode, s.off, s.itemoff, s.gcnt, jobs);
  auto go = [&](auto kern) {
    ensure_dyn_smem(reinterpret_cast<const void*>(kern), dyn);
    kern<<<sm_count(), kThreads, dyn, st>>>(a, xmap);
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

// Diagnostics: per-role cycle counters and a CTA-0 timeline of the
// warp-specialised scorer (enable bit 0; bits 1.. select debug variants).
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
