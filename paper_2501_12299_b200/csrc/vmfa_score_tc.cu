// vmfa_score_tc.cu — tensor-core (tcgen05, kind::tf32, 3xTF32 split precision)
// scorer of the E-step's candidate log-joints (log_joint, model.cpp:81-95)
// over anchor blocks.
//
// Item = (anchor a, <= 128 rows n with a in K(n)) x (components Q = g_a), or a
// single component (extra candidates, post-M-step truncated F). With the rows
// centred on the anchor, v = x - mu_a, and delta_q = mu_q - mu_a:
//   y_q    = W_q^T v - W_q^T delta_q                     (W = U R^-T, H cols)
//   diag_q = sum_d psi_qd^-1 v_d^2 - 2 sum_d psi_qd^-1 delta_qd v_d
//            + sum_d psi_qd^-1 delta_qd^2
//   l      = log pi_q - 0.5 (D log 2pi + log|Sigma_q| + diag_q - |y_q|^2)
// i.e. three GEMMs over K = D sharing the A rows of the block:
//   GEMM1  [v]   (128 x D) x [W_q columns, q in Q]        -> TMEM cols [0, N1)
//   GEMM3  [v]   (128 x D) x [-2 psi^-1 delta_q]          -> [N1, N1+NL)
//   GEMM2  [v^2] (128 x D) x [psi^-1_q]                   -> [N1+NL, N1+2NL)
// Every operand is split x = hi + lo (tf32) and each product accumulates
// hi*hi + hi*lo + lo*hi in fp32 (3xTF32): fp32-accurate, SURVEY §7 hard part 2.
// The CUDA cores gather the rows (K chunks of 32 dims = one 128-byte swizzle
// row), centre, square, split and store into 128B-swizzled K-major tiles; one
// thread issues the MMAs; chunks are double-buffered on mbarriers signalled by
// tcgen05.commit; the epilogue reads the accumulators with tcgen05.ld.
#include <algorithm>
#include <cstdint>

#include "vmfa_kernels.cuh"

namespace vmfa_b200 {
namespace {

constexpr int kTcRows = 128;     // UMMA_M
constexpr int kTcThreads = 256;  // 8 warps; warp w reads TMEM lane quadrant w % 4
constexpr int kMaxD = 1024;      // centering mean staged in smem
constexpr int kKC = 32;          // K chunk (tf32 elements) = 128 bytes
constexpr int kTileA = kTcRows * 128;  // bytes of one A tile (16 KB)

struct TcArgs {
  Dims dm;
  int mode;
  int Hp;          // padded H (4, 8, 16, 32, 64)
  int qg;          // components per group (TMEM budget)
  int N1, NL;      // GEMM1 / GEMM2,3 widths for a full group
  int nstage;
  uint32_t tmem_cols;
  uint32_t stage_bytes;
  const float* X;
  const float* WT;
  const float* mu32;
  const float* ipsi32;
  const double* kconst;
  const int* off;
  const int* ent;
  const int* itemoff;
  const int* g;
  const int* gcnt;
  float* out;
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
// byte offset of the 16-byte chunk j (0..7) of row r in a 128B-swizzled,
// K-major tile made of 8-row x 128-byte atoms stacked every 1024 bytes
__device__ __forceinline__ uint32_t swz(int r, int j) {
  return static_cast<uint32_t>(((r >> 3) << 10) + ((r & 7) << 7) + (((j ^ (r & 7)) & 7) << 4));
}
// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, SBO = 1024 B
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;           // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;   // SBO: next 8-row atom
  d |= static_cast<uint64_t>(1) << 46;           // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;           // SWIZZLE_128B
  return d;
}
// instruction descriptor: kind::tf32, A/B tf32 K-major, D f32, M=128, N
__device__ __forceinline__ uint32_t idesc(int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(kTcRows >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t id,
                                         uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(id), "r"(accum));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
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
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int W>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float* v);
template <>
__device__ __forceinline__ void tmem_ld<4>(uint32_t taddr, float* v) {
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}
template <>
__device__ __forceinline__ void tmem_ld<8>(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
template <>
__device__ __forceinline__ void tmem_ld<16>(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
template <int W>
__device__ __forceinline__ void tmem_ld_n(uint32_t taddr, float* v) {
  if constexpr (W <= 16) {
    tmem_ld<W>(taddr, v);
  } else {
#pragma unroll
    for (int i = 0; i < W; i += 16) tmem_ld<16>(taddr + i, v + i);
  }
}

// Per-stage smem map (offsets from the 1024-aligned stage base):
//   [0,16K) A v hi | [16K,32K) A v lo | [32K,48K) A v^2 hi | [48K,64K) A v^2 lo
//   B1 hi (N1 rows x 128 B) | B1 lo | B3 hi (NL) | B3 lo | B2 hi (NL) | B2 lo
struct StageMap {
  uint32_t a_vh, a_vl, a_qh, a_ql, b1h, b1l, b3h, b3l, b2h, b2l;
};
__device__ __forceinline__ StageMap stage_map(uint32_t base, int N1, int NL) {
  StageMap m;
  m.a_vh = base;
  m.a_vl = base + kTileA;
  m.a_qh = base + 2 * kTileA;
  m.a_ql = base + 3 * kTileA;
  m.b1h = base + 4 * kTileA;
  m.b1l = m.b1h + N1 * 128;
  m.b3h = m.b1l + N1 * 128;
  m.b3l = m.b3h + NL * 128;
  m.b2h = m.b3l + NL * 128;
  m.b2l = m.b2h + NL * 128;
  return m;
}

constexpr int kMaxUnits = 10;  // B (row, 16-byte chunk) units per thread: (256 + 32) * 8 / 256

template <int HP>
__global__ void __launch_bounds__(kTcThreads, 1) k_score_tc(TcArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  __shared__ uint64_t s_bar[2];
  __shared__ uint32_t s_tmem;
  __shared__ int s_e[kTcRows];
  __shared__ int s_n[kTcRows];
  __shared__ int s_comp[64];
  __shared__ double s_kc[64];
  __shared__ float s_b[256];       // W_q^T delta_q per group component (qg * HP <= 256)
  __shared__ float s_m[16];        // sum psi^-1 delta^2
  __shared__ float s_ld[kTcRows][33];  // lin / diag accumulators per row
  __shared__ __align__(16) float s_mu[kMaxD];  // anchor mean (centering)

  const Dims dm = a.dm;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = (smem_u32(smem_dyn) + 1023u) & ~1023u;

  if (tid == 0) {
    mbar_init(&s_bar[0]);
    mbar_init(&s_bar[1]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(a.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // zero every stage once: B padding rows are never written afterwards
  for (uint32_t i = tid * 16; i < a.stage_bytes * a.nstage; i += kTcThreads * 16) st4(sbase + i, 0, 0, 0, 0);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = s_tmem;
  uint32_t phase[2] = {0u, 0u};
  bool pending[2] = {false, false};

  const int total = __ldg(a.itemoff + dm.C);
  const int nchunk = (dm.D + kKC - 1) / kKC;
  const bool vec_ok = (dm.D & 3) == 0;
  // A ownership: row ar, 16-byte chunks [4*ah, 4*ah+4) of each K chunk
  const int ar = tid & (kTcRows - 1), ah = tid >> 7;

  for (int item = blockIdx.x; item < total; item += gridDim.x) {
    // ---- item prologue
    int lo = 0, hi = dm.C;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(a.itemoff + mid) <= item) lo = mid;
      else hi = mid;
    }
    const int c = lo;  // anchor (or the single component)
    const int row0 = __ldg(a.off + c) + (item - __ldg(a.itemoff + c)) * kTcRows;
    const int nrows = min(kTcRows, __ldg(a.off + c + 1) - row0);
    const int ncomp = a.mode == kModeAnchor ? __ldg(a.gcnt + c) : 1;
    if (tid < kTcRows) {
      int e = -1, n = -1;
      if (tid < nrows) {
        e = __ldg(a.ent + row0 + tid);
        n = a.mode == kModeExtra ? e : e / dm.Cp;
      }
      s_e[tid] = e;
      s_n[tid] = n;
    }
    if (tid < ncomp) {
      const int q = a.mode == kModeAnchor ? __ldg(a.g + (int64_t)c * dm.G + tid) : c;
      s_comp[tid] = q;
      s_kc[tid] = __ldg(a.kconst + q);
    }
    const float* mu_a = a.mu32 + (int64_t)c * dm.D;
    for (int d = tid; d < nchunk * kKC; d += kTcThreads) s_mu[d] = d < dm.D ? __ldg(mu_a + d) : 0.f;
    __syncthreads();
    const int my_n = s_n[ar];
    const float* xrow = a.X + (int64_t)(my_n < 0 ? 0 : my_n) * dm.D;

    auto load_x = [&](int ch, float4* xv) {
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int d = ch * kKC + 4 * (4 * ah + jj);
        float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
        if (my_n >= 0 && d < dm.D) {
          if (vec_ok) {
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

    for (int g0 = 0; g0 < ncomp; g0 += a.qg) {
      const int nq = min(a.qg, ncomp - g0);
      const int N1 = ((nq * HP + 15) / 16) * 16;
      const int NL = 16;
      const int nb1 = nq * HP;       // live GEMM1 rows
      const int nbrows = nb1 + 2 * nq;  // + lin rows + psi^-1 rows
      const int nunits = nbrows * 8;
      double accb[kMaxUnits];
#pragma unroll
      for (int u = 0; u < kMaxUnits; ++u) accb[u] = 0.0;
      float4 xcur[4], xnext[4];
      load_x(0, xcur);
      for (int ch = 0; ch < nchunk; ++ch) {
        if (ch + 1 < nchunk) load_x(ch + 1, xnext);  // prefetch the next chunk's rows
        const int s = a.nstage == 2 ? (ch & 1) : 0;
        if (pending[s]) {
          mbar_wait(&s_bar[s], phase[s]);
          phase[s] ^= 1u;
          pending[s] = false;
        }
        const StageMap m = stage_map(sbase + s * a.stage_bytes, a.N1, a.NL);
        const int d0 = ch * kKC;
        // ---- A: v = x - mu_a, v^2, tf32 hi/lo splits (128B-swizzled, K-major)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j = 4 * ah + jj;
          const float4 mv = *reinterpret_cast<const float4*>(s_mu + d0 + 4 * j);
          const float4 xv = xcur[jj];
          float v[4] = {xv.x - mv.x, xv.y - mv.y, xv.z - mv.z, xv.w - mv.w};
          if (my_n < 0) v[0] = v[1] = v[2] = v[3] = 0.f;
          uint32_t vh[4], vl[4], qh[4], ql[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            split(v[k], vh[k], vl[k]);
            split(v[k] * v[k], qh[k], ql[k]);
          }
          const uint32_t o = swz(ar, j);
          st4(m.a_vh + o, vh[0], vh[1], vh[2], vh[3]);
          st4(m.a_vl + o, vl[0], vl[1], vl[2], vl[3]);
          st4(m.a_qh + o, qh[0], qh[1], qh[2], qh[3]);
          st4(m.a_ql + o, ql[0], ql[1], ql[2], ql[3]);
        }
        // ---- B: units (row, 16-byte chunk j), vectorised loads
#pragma unroll
        for (int uu = 0; uu < kMaxUnits; ++uu) {
          const int u = tid + uu * kTcThreads;
          if (u >= nunits) break;
          const int br = u >> 3, j = u & 7;
          const int d = d0 + 4 * j;
          int kind, qi, h = 0, dr;
          if (br < nb1) {
            kind = 0;
            qi = br / HP;
            h = br - qi * HP;
            dr = br;
          } else if (br < nb1 + nq) {
            kind = 1;
            qi = br - nb1;
            dr = qi;
          } else {
            kind = 2;
            qi = br - nb1 - nq;
            dr = qi;
          }
          const int q = s_comp[g0 + qi];
          float val[4] = {0.f, 0.f, 0.f, 0.f};
          if (d < dm.D) {
            const float4 ma = *reinterpret_cast<const float4*>(s_mu + d);
            float4 mq, w4, ip4;
            const float* muq = a.mu32 + (int64_t)q * dm.D + d;
            const float* ipq = a.ipsi32 + (int64_t)q * dm.D + d;
            const float* wq = a.WT + ((int64_t)q * HP + h) * dm.D + d;
            if (vec_ok) {
              mq = __ldg(reinterpret_cast<const float4*>(muq));
              if (kind == 0) w4 = __ldg(reinterpret_cast<const float4*>(wq));
              else ip4 = __ldg(reinterpret_cast<const float4*>(ipq));
            } else {
              float t0[4] = {0.f, 0.f, 0.f, 0.f}, t1[4] = {0.f, 0.f, 0.f, 0.f};
              for (int k = 0; k < 4 && d + k < dm.D; ++k) {
                t0[k] = __ldg(muq + k);
                t1[k] = kind == 0 ? __ldg(wq + k) : __ldg(ipq + k);
              }
              mq = make_float4(t0[0], t0[1], t0[2], t0[3]);
              w4 = ip4 = make_float4(t1[0], t1[1], t1[2], t1[3]);
            }
            const float dl[4] = {mq.x - ma.x, mq.y - ma.y, mq.z - ma.z, mq.w - ma.w};
            if (kind == 0) {
              const float w[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                val[k] = w[k];
                accb[uu] = fma(static_cast<double>(w[k]), static_cast<double>(dl[k]), accb[uu]);
              }
            } else {
              const float ip[4] = {ip4.x, ip4.y, ip4.z, ip4.w};
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                if (kind == 1) {
                  val[k] = -2.f * ip[k] * dl[k];
                  accb[uu] = fma(static_cast<double>(ip[k]) * dl[k], static_cast<double>(dl[k]), accb[uu]);
                } else {
                  val[k] = ip[k];
                }
              }
            }
          }
          uint32_t bh[4], bl[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) split(val[k], bh[k], bl[k]);
          const uint32_t dh = kind == 0 ? m.b1h : (kind == 1 ? m.b3h : m.b2h);
          const uint32_t dlo = kind == 0 ? m.b1l : (kind == 1 ? m.b3l : m.b2l);
          const uint32_t o = swz(dr, j);
          st4(dh + o, bh[0], bh[1], bh[2], bh[3]);
          st4(dlo + o, bl[0], bl[1], bl[2], bl[3]);
        }
        fence_async_smem();
        fence_before();
        __syncthreads();
        // ---- MMA issue (one thread): 3 split passes x 4 k-steps x 3 GEMMs
        if (tid == 0) {
          fence_after();
          const uint32_t id1 = idesc(N1), idl = idesc(NL);
          const uint32_t A_v[3] = {m.a_vh, m.a_vh, m.a_vl};
          const uint32_t A_q[3] = {m.a_qh, m.a_qh, m.a_ql};
          const uint32_t B1[3] = {m.b1h, m.b1l, m.b1h};
          const uint32_t B3[3] = {m.b3h, m.b3l, m.b3h};
          const uint32_t B2[3] = {m.b2h, m.b2l, m.b2h};
#pragma unroll
          for (int p = 0; p < 3; ++p) {
#pragma unroll
            for (int k = 0; k < kKC / 8; ++k) {
              const uint32_t acc = (ch > 0 || p > 0 || k > 0) ? 1u : 0u;
              const uint32_t ko = k * 32;  // 8 tf32 = 32 bytes along K
              mma_tf32(tmem, sdesc(A_v[p] + ko), sdesc(B1[p] + ko), id1, acc);
              mma_tf32(tmem + N1, sdesc(A_v[p] + ko), sdesc(B3[p] + ko), idl, acc);
              mma_tf32(tmem + N1 + NL, sdesc(A_q[p] + ko), sdesc(B2[p] + ko), idl, acc);
            }
          }
          mma_commit(&s_bar[s]);
        }
        pending[s] = true;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) xcur[jj] = xnext[jj];
      }
      // ---- per-group constants: reduce each B row's 8 chunk partials (8 lanes)
#pragma unroll
      for (int uu = 0; uu < kMaxUnits; ++uu) {
        const int u = tid + uu * kTcThreads;
        if (u - lane >= nunits) break;  // warp-uniform exit: every lane reaches the shuffles
        double v = u < nunits ? accb[uu] : 0.0;
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        const int br = u >> 3;
        if ((u & 7) == 0 && u < nunits) {
          if (br < nb1) s_b[br] = static_cast<float>(v);
          else if (br < nb1 + nq) s_m[br - nb1] = static_cast<float>(v);
        }
      }
      // ---- drain the pipeline, then the epilogue of this group
      for (int s = 0; s < 2; ++s)
        if (pending[s]) {
          mbar_wait(&s_bar[s], phase[s]);
          phase[s] ^= 1u;
          pending[s] = false;
        }
      fence_after();
      const uint32_t trow = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
      if (warp < 4) {
        float t[32];  // lin columns then diag columns (NL == 16, qg <= 16)
        tmem_ld<16>(trow + N1, t);
        tmem_ld<16>(trow + N1 + NL, t + 16);
#pragma unroll
        for (int i = 0; i < 32; ++i) s_ld[tid][i] = t[i];
      }
      __syncthreads();
      const int r = (warp & 3) * 32 + lane;
      const int e = s_e[r];
      for (int qi = warp >> 2; qi < nq; qi += 2) {
        float y[HP];
        tmem_ld_n<HP>(trow + qi * HP, y);
        float yy = 0.f;
#pragma unroll
        for (int h = 0; h < HP; ++h) {
          const float t = y[h] - s_b[qi * HP + h];
          yy = fmaf(t, t, yy);
        }
        const float lin = s_ld[r][qi];
        const float d2 = s_ld[r][16 + qi];
        const double diag = static_cast<double>(d2) + static_cast<double>(lin) + static_cast<double>(s_m[qi]);
        const float lj = static_cast<float>(s_kc[g0 + qi] - 0.5 * (diag - static_cast<double>(yy)));
        if (r < nrows) {
          if (a.mode == kModeAnchor) {
            const int n = e / dm.Cp, j = e - n * dm.Cp;
            a.out[(int64_t)n * dm.SL + j * dm.G + g0 + qi] = lj;
          } else if (a.mode == kModeExtra) {
            a.out[(int64_t)e * dm.SL + dm.Cp * dm.G] = lj;
          } else {
            a.out[e] = lj;
          }
        }
      }
      fence_before();
      __syncthreads();
    }
  }
  fence_after();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols));
}

}  // namespace

bool score_tc_supported(const Dims& dm) {
  return dm.H <= 64 && dm.G <= 64 && dm.D <= kMaxD;
}

cudaError_t launch_score_tc(int mode, const ScoreArgs& s, const float* WT, const float* ipsi32,
                            const float* mu32, cudaStream_t st) {
  TcArgs a{};
  a.dm = s.dm;
  a.mode = mode;
  const int H = s.dm.H;
  a.Hp = ws_hp(H);  // WT rows per component (shared with the warp-specialised scorer)
  const int ncomp_max = mode == kModeAnchor ? s.dm.G : 1;
  // group size: GEMM1 width <= 256 and N1 + 2 NL <= 512 TMEM columns; NL == 16
  int qg = std::min(ncomp_max, std::min(16, 256 / a.Hp));
  a.qg = std::max(qg, 1);
  a.N1 = ((a.qg * a.Hp + 15) / 16) * 16;
  a.NL = 16;
  const int cols = a.N1 + 2 * a.NL;
  a.tmem_cols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
  a.stage_bytes = static_cast<uint32_t>(4 * kTileA + 2 * 128 * (a.N1 + 2 * a.NL));
  const size_t static_smem = 26 * 1024;  // barriers, ids, b/m, lin/diag staging (upper bound)
  a.nstage = (2 * a.stage_bytes + 1024 + static_smem <= 227 * 1024) ? 2 : 1;
  const size_t dyn = static_cast<size_t>(a.nstage) * a.stage_bytes + 1024;
  a.X = s.X;
  a.WT = WT;
  a.mu32 = mu32;
  a.ipsi32 = ipsi32;
  a.kconst = s.kconst;
  a.off = s.off;
  a.ent = s.ent;
  a.itemoff = s.itemoff;
  a.g = s.g;
  a.gcnt = s.gcnt;
  a.out = s.out;
  const int grid = sm_count();
  auto go = [&](auto kern) {
    ensure_dyn_smem(reinterpret_cast<const void*>(kern), dyn);
    kern<<<grid, kTcThreads, dyn, st>>>(a);
  };
  switch (a.Hp) {
    case 8: go(k_score_tc<8>); break;
    case 16: go(k_score_tc<16>); break;
    case 32: go(k_score_tc<32>); break;
    default: go(k_score_tc<64>); break;
  }
  return cudaGetLastError();
}

}  // namespace vmfa_b200
