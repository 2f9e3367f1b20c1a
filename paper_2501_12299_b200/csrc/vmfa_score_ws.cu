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
constexpr int kProd = kProdWarps * 32;
constexpr int kMmaWarp = 8;
constexpr int kEpiWarp0 = 9;
constexpr int kThreads = 13 * 32;
constexpr int kMaxD = 1024;
constexpr int kNL = 16;               // lin rows / psi rows per group (qg <= 16)

struct WsArgs {
  Dims dm;
  int mode;
  int Hp;            // W rows per component (>= 8)
  int qg;            // components per job (group)
  int N1max;         // 16 + round16(qg * Hp)
  int nstage;
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
  const float* lblk; // anchor mode: [C][ngroups][nchunk][4][16][32] lin hi|lo, psi hi|lo tiles
  const float* cblk; // single mode: [C][nchunk][4][16][32] (lin = 0, psi row 0)
  int ngroups;
  const int* off;
  const int* ent;
  const int* itemoff;
  const int* g;
  const int* gcnt;
  float* out;
  unsigned long long* prof;  // optional per-role cycle counters (nullptr: off)
};

// per-role cycle accounting (debug builds of the pipeline; prof == nullptr in production)
enum ProfSite { kPWaitTE, kPSync, kPWaitEmpty, kPBuild, kMWaitTE, kMWaitFull, kMIssue, kEWait, kEWork, kNumSites };
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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
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
__device__ __forceinline__ void prod_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kProd) : "memory"); }

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

struct Job {
  int c, row0, nrows, ncomp;
};
__device__ __forceinline__ Job decode(const WsArgs& a, int item) {
  int lo = 0, hi = a.dm.C;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(a.itemoff + mid) <= item) lo = mid;
    else hi = mid;
  }
  Job j;
  j.c = lo;
  j.row0 = __ldg(a.off + lo) + (item - __ldg(a.itemoff + lo)) * kRows;
  j.nrows = min(kRows, __ldg(a.off + lo + 1) - j.row0);
  j.ncomp = a.mode == kModeAnchor ? __ldg(a.gcnt + lo) : 1;
  return j;
}

struct Meta {
  int e[kRows];
  int comp[kNL];
  int c, g0, nq, nrows;
};

template <int HP>
__global__ void __launch_bounds__(kThreads, 1) k_score_ws(WsArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  __shared__ uint64_t s_full[2], s_empty[2], s_tfull[2], s_tempty[2], s_mready[2];
  __shared__ uint32_t s_tmem;
  __shared__ Meta s_meta[2];
  __shared__ __align__(16) float s_mu[kMaxD];
  const Dims dm = a.dm;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = (smem_u32(smem_dyn) + 1023u) & ~1023u;
  const int nchunk = (dm.D + kKC - 1) / kKC;
  const int total = __ldg(a.itemoff + dm.C);

  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], kProdWarps);
      mbar_init(&s_empty[i], 1);
      mbar_init(&s_tfull[i], 1);
      mbar_init(&s_tempty[i], 4);
      mbar_init(&s_mready[i], kProdWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(a.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (uint32_t i = tid * 16; i < a.stage_bytes * a.nstage; i += kThreads * 16) st4(sbase + i, 0, 0, 0, 0);
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = s_tmem;
  // smem stage map (offsets from a 1024-aligned stage base): B operands only
  const uint32_t offB1 = 0;                                 // B1 hi, then B1 lo (N1max rows each)
  const uint32_t offB2 = offB1 + 2 * a.N1max * 128;         // B2 hi, then B2 lo (16 rows each)
  // TMEM map: accumulators [0, nacc*TB), A stages of 4 x 32 columns after them
  const uint32_t colA = a.nacc * a.TB;

  if (warp < kProdWarps) {
    // ================================================================ producers
    // A ownership: TMEM lane quadrant of this warp, one row per lane, K half ah
    const int ar = 32 * (warp & 3) + lane, ah = warp >> 2;
    uint32_t sc = 0;
    int jb = 0;
    Prof pf{};
    pf.start();
    for (int item = blockIdx.x; item < total; item += gridDim.x) {
      const Job J = decode(a, item);
      for (int g0 = 0; g0 < J.ncomp; g0 += a.qg, ++jb) {
        const int b = a.nacc == 2 ? (jb & 1) : 0;
        const int use_b = a.nacc == 2 ? (jb >> 1) : jb;
        const int nq = min(a.qg, J.ncomp - g0);
        if (use_b >= 1) mbar_wait(&s_tempty[b], (use_b - 1) & 1);
        pf.lap(kPWaitTE);
        prod_sync();  // all producers done with the previous job's s_mu / meta reads
        Meta& M = s_meta[b];
        if (tid < kRows) {
          int e = -1;
          if (tid < J.nrows) e = __ldg(a.ent + J.row0 + tid);
          M.e[tid] = e;
        }
        if (tid < nq) M.comp[tid] = a.mode == kModeAnchor ? __ldg(a.g + (int64_t)J.c * dm.G + g0 + tid) : J.c;
        if (tid == 0) {
          M.c = J.c;
          M.g0 = g0;
          M.nq = nq;
          M.nrows = J.nrows;
        }
        const float* mu_a = a.mu32 + (int64_t)J.c * dm.D;
        for (int d = tid; d < nchunk * kKC; d += kProd) s_mu[d] = d < dm.D ? __ldg(mu_a + d) : 0.f;
        prod_sync();
        if (lane == 0) mbar_arrive(&s_mready[b]);  // meta[b] published to the epilogue
        pf.lap(kPSync);
        const int e = M.e[ar];
        const int n = e < 0 ? -1 : (a.mode == kModeExtra ? e : e / dm.Cp);
        const float* xrow = a.X + (int64_t)(n < 0 ? 0 : n) * dm.D;
        const bool vec = (dm.D & 3) == 0;
        auto load_x = [&](int ch, float4* xv) {
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int d = ch * kKC + 16 * ah + 4 * jj;
            float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
            if (n >= 0 && d < dm.D) {
              if (vec) {
                t = __ldg(reinterpret_cast<const float4*>(xrow + d));
              } else {
                float u[4] = {0.f, 0.f, 0.f, 0.f};
                for (int k = 0; k < 4 && d + k < dm.D; ++k) u[k] = __ldg(xrow + d + k);
                t = make_float4(u[0], u[1], u[2], u[3]);
              }
            }
            xv[jj] = t;
          }
        };
        // register prefetch ring: rows of chunks ch+1 and ch+2 in flight while ch is built
        float4 xcur[4], xn1[4], xn2[4];
        load_x(0, xcur);
        if (nchunk > 1) load_x(1, xn1);
        for (int ch = 0; ch < nchunk; ++ch, ++sc) {
          if (ch + 2 < nchunk) load_x(ch + 2, xn2);
          const int s = a.nstage == 2 ? static_cast<int>(sc & 1u) : 0;
          const uint32_t use = a.nstage == 2 ? (sc >> 1) : sc;
          pf.lap(kPBuild);
          if (use >= 1) mbar_wait(&s_empty[s], (use - 1) & 1u);
          pf.lap(kPWaitEmpty);
          const uint32_t st = sbase + s * a.stage_bytes;
          const int d0 = ch * kKC;
          // B operands: bulk copies of the pre-split, pre-swizzled blocks
          if (tid == 0) {
            const uint32_t blk = HP * 128;
            mbar_expect_tx(&s_full[s], 2 * nq * blk + 4 * kNL * 128);
            for (int qi = 0; qi < nq; ++qi) {
              const float* src = a.WTS + ((int64_t)M.comp[qi] * nchunk + ch) * 2 * HP * 32;
              const uint32_t row = kNL + qi * HP;
              bulk_copy(st + offB1 + row * 128, src, blk, &s_full[s]);
              bulk_copy(st + offB1 + a.N1max * 128 + row * 128, src + HP * 32, blk, &s_full[s]);
            }
            const float* lb = a.mode == kModeAnchor
                                  ? a.lblk + (((int64_t)J.c * a.ngroups + g0 / a.qg) * nchunk + ch) * 4 * kNL * 32
                                  : a.cblk + ((int64_t)J.c * nchunk + ch) * 4 * kNL * 32;
            bulk_copy(st + offB1, lb, kNL * 128, &s_full[s]);                               // lin hi
            bulk_copy(st + offB1 + a.N1max * 128, lb + kNL * 32, kNL * 128, &s_full[s]);    // lin lo
            bulk_copy(st + offB2, lb + 2 * kNL * 32, kNL * 128, &s_full[s]);                // psi hi
            bulk_copy(st + offB2 + kNL * 128, lb + 3 * kNL * 32, kNL * 128, &s_full[s]);    // psi lo
          }
          // A: v = x - mu_a and v^2, split hi/lo, stored into TMEM (lane = row)
          {
            uint32_t vh[16], vl[16], qh[16], ql[16];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const float4 mv = *reinterpret_cast<const float4*>(s_mu + d0 + 16 * ah + 4 * jj);
              const float4 xv = xcur[jj];
              float v[4] = {xv.x - mv.x, xv.y - mv.y, xv.z - mv.z, xv.w - mv.w};
              if (n < 0) v[0] = v[1] = v[2] = v[3] = 0.f;
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                split(v[k], vh[4 * jj + k], vl[4 * jj + k]);
                split(v[k] * v[k], qh[4 * jj + k], ql[4 * jj + k]);
              }
            }
            const uint32_t ta = tmem + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + colA + s * 128 + 16 * ah;
            tmem_st16(ta, vh);
            tmem_st16(ta + 32, vl);
            tmem_st16(ta + 64, qh);
            tmem_st16(ta + 96, ql);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          }
          fence_before();
          fence_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&s_full[s]);
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            xcur[jj] = xn1[jj];
            xn1[jj] = xn2[jj];
          }
        }
      }
    }
    pf.lap(kPBuild);
    if (a.prof && lane == 0)
      for (int i = 0; i < 4; ++i) atomicAdd(a.prof + i, pf.acc[i]);
  } else if (warp == kMmaWarp) {
    // ================================================================ MMA issuer
    uint32_t sc = 0;
    int jb = 0;
    Prof pf{};
    pf.start();
    for (int item = blockIdx.x; item < total; item += gridDim.x) {
      const Job J = decode(a, item);
      for (int g0 = 0; g0 < J.ncomp; g0 += a.qg, ++jb) {
        const int b = a.nacc == 2 ? (jb & 1) : 0;
        const int use_b = a.nacc == 2 ? (jb >> 1) : jb;
        const int nq = min(a.qg, J.ncomp - g0);
        const int N1 = kNL + ((nq * HP + 15) / 16) * 16;
        const uint32_t acc1 = tmem + b * a.TB, acc2 = acc1 + N1;
        if (use_b >= 1) mbar_wait(&s_tempty[b], (use_b - 1) & 1);
        fence_after();
        pf.lap(kMWaitTE);
        for (int ch = 0; ch < nchunk; ++ch, ++sc) {
          const int s = a.nstage == 2 ? static_cast<int>(sc & 1u) : 0;
          const uint32_t use = a.nstage == 2 ? (sc >> 1) : sc;
          mbar_wait(&s_full[s], use & 1u);
          fence_after();
          pf.lap(kMWaitFull);
          if (lane == 0) {
            const uint32_t st = sbase + s * a.stage_bytes;
            const uint32_t id1 = idesc(N1), id2 = idesc(kNL);
            const uint32_t tA = tmem + colA + s * 128;  // v hi | v lo | v^2 hi | v^2 lo
            const uint32_t Av[3] = {tA, tA, tA + 32};
            const uint32_t Aq[3] = {tA + 64, tA + 64, tA + 96};
            const uint32_t B1[3] = {st + offB1, st + offB1 + a.N1max * 128, st + offB1};
            const uint32_t B2[3] = {st + offB2, st + offB2 + kNL * 128, st + offB2};
#pragma unroll
            for (int p = 0; p < 3; ++p) {
#pragma unroll
              for (int k = 0; k < kKC / 8; ++k) {
                const uint32_t acc = (ch > 0 || p > 0 || k > 0) ? 1u : 0u;
                mma_tf32_ts(acc1, Av[p] + k * 8, sdesc(B1[p] + k * 32), id1, acc);
                mma_tf32_ts(acc2, Aq[p] + k * 8, sdesc(B2[p] + k * 32), id2, acc);
              }
            }
            commit(&s_empty[s]);
            if (ch == nchunk - 1) commit(&s_tfull[b]);
          }
          __syncwarp();
          pf.lap(kMIssue);
        }
      }
    }
    if (a.prof && lane == 0)
      for (int i = kMWaitTE; i <= kMIssue; ++i) atomicAdd(a.prof + i, pf.acc[i]);
  } else if (warp >= kEpiWarp0) {
    // ================================================================ epilogue
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    int jb = 0;
    Prof pf{};
    pf.start();
    for (int item = blockIdx.x; item < total; item += gridDim.x) {
      const Job J = decode(a, item);
      for (int g0 = 0; g0 < J.ncomp; g0 += a.qg, ++jb) {
        const int b = a.nacc == 2 ? (jb & 1) : 0;
        const int use_b = a.nacc == 2 ? (jb >> 1) : jb;
        mbar_wait(&s_mready[b], use_b & 1);
        mbar_wait(&s_tfull[b], use_b & 1);
        fence_after();
        pf.lap(kEWait);
        const Meta& M = s_meta[b];
        const int nq = M.nq;
        const int N1 = kNL + ((nq * HP + 15) / 16) * 16;
        const uint32_t trow = tmem + b * a.TB + (static_cast<uint32_t>(quad * 32) << 16);
        float lin[16], d2[16];
        tmem_ld<16>(trow, lin);
        tmem_ld<16>(trow + N1, d2);
        const int e = M.e[r];
        for (int qi = 0; qi < nq; ++qi) {
          float y[HP];
#pragma unroll
          for (int h0 = 0; h0 < HP; h0 += 16) {
            if constexpr (HP >= 16) tmem_ld<16>(trow + kNL + qi * HP + h0, y + h0);
            else tmem_ld<8>(trow + kNL + qi * HP + h0, y + h0);
          }
          const int q = M.comp[qi];
          float m = 0.f;
          float yy = 0.f;
          if (a.mode == kModeAnchor) {
            const float* cst = a.acst + ((int64_t)M.c * dm.G + M.g0 + qi) * (HP + 1);
#pragma unroll
            for (int h = 0; h < HP; ++h) {
              const float t = y[h] - __ldg(cst + h);
              yy = fmaf(t, t, yy);
            }
            m = __ldg(cst + HP);
          } else {
#pragma unroll
            for (int h = 0; h < HP; ++h) yy = fmaf(y[h], y[h], yy);
          }
          float linq = 0.f, d2q = 0.f;
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (i == qi) {
              linq = lin[i];
              d2q = d2[i];
            }
          const double diag = static_cast<double>(d2q) + static_cast<double>(linq) + static_cast<double>(m);
          const float lj = static_cast<float>(__ldg(a.kconst + q) - 0.5 * (diag - static_cast<double>(yy)));
          if (r < M.nrows) {
            if (a.mode == kModeAnchor) {
              const int n = e / dm.Cp, j = e - n * dm.Cp;
              a.out[(int64_t)n * dm.SL + j * dm.G + M.g0 + qi] = lj;
            } else if (a.mode == kModeExtra) {
              a.out[(int64_t)e * dm.SL + dm.Cp * dm.G] = lj;
            } else {
              a.out[e] = lj;
            }
          }
        }
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_tempty[b]);
        pf.lap(kEWork);
      }
    }
    if (a.prof && lane == 0)
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

}  // namespace

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

cudaError_t launch_score_ws(int mode, const ScoreArgs& s, const float* WTS, const float* mu32,
                            const float* ipsi32, const float* acst, const float* lblk, const float* cblk,
                            cudaStream_t st) {
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
  const size_t static_smem = 8 * 1024;
  a.nstage = 2;  // A stages live in TMEM; smem holds the B stages only
  (void)static_smem;
  const size_t dyn = static_cast<size_t>(a.nstage) * a.stage_bytes + 1024;
  a.X = s.X;
  a.WTS = WTS;
  a.mu32 = mu32;
  a.ipsi32 = ipsi32;
  a.kconst = s.kconst;
  a.acst = acst;
  a.lblk = lblk;
  a.cblk = cblk;
  a.ngroups = ws_groups(s.dm);
  a.off = s.off;
  a.ent = s.ent;
  a.itemoff = s.itemoff;
  a.g = s.g;
  a.gcnt = s.gcnt;
  a.out = s.out;
  a.prof = g_ws_prof;
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn));
    kern<<<sm_count(), kThreads, dyn, st>>>(a);
  };
  switch (a.Hp) {
    case 8: go(k_score_ws<8>); break;
    case 16: go(k_score_ws<16>); break;
    case 32: go(k_score_ws<32>); break;
    default: go(k_score_ws<64>); break;
  }
  return cudaGetLastError();
}

}  // namespace vmfa_b200

// Diagnostics: per-role cycle counters of the warp-specialised scorer.
extern "C" int vmfa_diag_scorer_cycles(int enable, unsigned long long* out, int n) {
  using namespace vmfa_b200;
  if (enable && !g_ws_prof) {
    if (cudaMalloc(&g_ws_prof, sizeof(unsigned long long) * 16) != cudaSuccess) return VMFA_ERR_CUDA;
    cudaMemset(g_ws_prof, 0, sizeof(unsigned long long) * 16);
  }
  if (out && g_ws_prof) {
    cudaDeviceSynchronize();
    cudaMemcpy(out, g_ws_prof, sizeof(unsigned long long) * (n < 16 ? n : 16), cudaMemcpyDeviceToHost);
    cudaMemset(g_ws_prof, 0, sizeof(unsigned long long) * 16);
  }
  if (!enable && g_ws_prof) {
    cudaFree(g_ws_prof);
    g_ws_prof = nullptr;
  }
  return VMFA_OK;
}
