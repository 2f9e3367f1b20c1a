// vmfa_stats_tc.cu — the sufficient statistics (accumulate_suffstats,
// mstep.cpp:47-101) on the 5th-generation tensor cores.
//
// Per item (component c, <= 256 of its K-pairs (n, q)), centred rows
// v_n = x_n - mu_c (fp32 mu, as the other statistics kernels; k_stats_uncenter
// restores the raw sums):
//   GEMM i   Z   [rows x HP]  = [v] (rows x D) . [V_c^T] (D x HP)     mz = V_c v
//   GEMM ii  Y_v [D x N2]     = [v]^T (D x rows) . [q zhat] (rows x N2)
// with zhat = [mz; 1], plus E = sum q zhat zhat^T in fp64 from the fp32 mz and
// sq_v = sum q v^2 (fp64 shared-memory sums of fp32 partials) on the CUDA
// cores. Both GEMMs are tcgen05.mma.kind::f16 in 3xFP16 (hi*hi + hi*lo +
// lo*hi, 22 significant bits, fp32 accumulation in TMEM), SS form: one smem
// copy of each 64-dimension chunk of split v serves GEMM i as a K-major A
// (rows x dims) and GEMM ii as an MN-major A (dims x rows, two adjacent chunks
// = M 128). Row n of v is scaled by 2^k_n (|v| <= 2^14 from the bound
// max|x_n| + max|mu_c|) for GEMM i; GEMM ii sums over rows (its K), so
// 2^-k_n is folded into its B operand (q zhat), exactly, and every column of
// that operand gets a power-of-two scale from an a-priori bound
// (|V_h|_1 max_n bound_n^2; the fp16 split keeps 22 bits for values down to
// 2^-17 of the bound, far below its looseness).
//
// A tile is 128 rows; per tile GEMM i (Z in one of two TMEM buffers), the
// CUDA-core work (mz, E, GEMM ii's B), then GEMM ii (Y_v accumulates in TMEM
// over the item's tiles); the tiles are pipelined (GEMM i of tile t + 1 runs
// during tile t's CUDA-core work), and each row chunk is produced twice, the
// second time from L2. Roles: warps 0-7
// produce chunks into a 4-slot ring (32 KB each: 128 rows x 64 dims, fp16 hi
// and lo, 128-byte swizzle) and do the CUDA-core work; one thread of warp 8
// issues the MMAs and commits to the ring / phase barriers. Outputs as the
// other statistics kernels: a component's sole item writes Y_v, sq_v, E
// directly, split components write item partials reduced by k_stats_reduce.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "vmfa_kernels.cuh"

namespace vmfa_b200 {
namespace {

constexpr int kTRows = 128;            // rows per tile (M of GEMM i, K of GEMM ii)
constexpr int kTItemRows = 512;        // K-pairs per item (<= 4 tiles; Z of each in TMEM)
constexpr int kTProd = 256;            // producer threads (warps 0-7)
constexpr int kTThreads = kTProd + 32; // + the MMA warp
constexpr int kTSlots = 4;
constexpr uint32_t kTSlotBytes = 32768;  // hi (16 KB) + lo (16 KB)
constexpr int kTMaxChunks = 13;        // D <= 832
constexpr int kTargetE = 14;           // operands scaled to |value| <= 2^14

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ int sexp(float bound) {
  if (!(bound > 0.f)) return 0;
  const uint32_t b = __float_as_uint(bound);
  int e = static_cast<int>((b >> 23) & 0xffu) - 127;
  if ((b & 0x7fffffu) != 0u) e += 1;
  if (((b >> 23) & 0xffu) == 0u) e = -126;
  return max(-100, min(100, kTargetE - e));
}
__device__ __forceinline__ float p2(int k) { return __uint_as_float(static_cast<uint32_t>(k + 127) << 23); }
__device__ __forceinline__ void split(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x0, x1);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
__device__ __forceinline__ void split1(float x, __half& hi, __half& lo) {
  hi = __float2half_rn(x);
  lo = __float2half_rn(x - __half2float(hi));
}
// 128-byte-swizzled byte offset of (line, 16-byte unit) in a 1024-byte-aligned buffer
__device__ __forceinline__ uint32_t swz(int line, int unit) {
  return static_cast<uint32_t>(line * 128 + ((unit ^ (line & 7)) << 4));
}
// smem descriptor, 128-byte swizzle: SBO = 1 KB between 8-line groups;
// LBO = byte offset between 64-element atoms along M/N (MN-major only)
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo_bytes) {
  uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
// kind::f16 instruction descriptor: fp32 D, fp16 A/B, M = 128, A K- or MN-major
__device__ __forceinline__ uint32_t idesc(int N, bool a_mn) {
  return (1u << 4) | (a_mn ? (1u << 15) : 0u) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(kTRows >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void tcommit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void binit(uint64_t* bar, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void barrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
// waits for completion #k (k >= 1) of the barrier (parity (k - 1) & 1);
// traps after ~10 s so a pipeline bug fails the launch instead of hanging
__device__ __forceinline__ void bwait(uint64_t* bar, uint32_t k) {
  const uint32_t parity = (k - 1u) & 1u;
  uint32_t ok = 0;
  long long t0 = 0;
  for (uint32_t spin = 0;; ++spin) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(su32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    if ((spin & 1023u) == 0) {
      const long long now = clock64();
      if (spin == 0) t0 = now;
      else if (now - t0 > 20000000000LL) __trap();
    }
  }
}
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tfence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tfence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tld8(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void producers_sync() { asm volatile("bar.sync 1, %0;" ::"r"(kTProd) : "memory"); }

__device__ __forceinline__ int find_item_t(const int* itemoff, int C, int item) {
  int lo = 0, hi = C;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(itemoff + mid) <= item) lo = mid;
    else hi = mid;
  }
  return lo;
}

struct TcLayout {
  int nch;       // real 64-dimension chunks (ceil(D / 64))
  int npair;     // chunk pairs (M = 128 dimensions of GEMM ii)
  int HP, N2;    // GEMM i / GEMM ii N
  uint32_t off_V, off_B2, off_z, off_sq, off_row, off_q, off_qf, off_k, total;
  uint32_t tmem_cols;  // Z (2 x HP, at 0) + Y_v (npair x N2, at 64)
};
__host__ __device__ inline TcLayout tc_layout(int D, int H) {
  TcLayout L;
  L.nch = (D + 63) / 64;
  L.npair = (L.nch + 1) / 2;
  L.HP = ((H + 15) / 16) * 16;
  L.N2 = ((H + 1 + 15) / 16) * 16;  // (M = 128: N in steps of 16)
  uint32_t o = kTSlots * kTSlotBytes;
  L.off_V = o;
  o += static_cast<uint32_t>(L.nch) * 2 * L.HP * 128;
  L.off_B2 = o;
  o += 2u * 2 * L.N2 * 128;
  L.off_z = o;
  o += static_cast<uint32_t>(kTRows) * (H + 1) * 4;
  o = (o + 7u) & ~7u;
  L.off_sq = o;
  o += static_cast<uint32_t>(L.npair) * 128 * 8;
  L.off_row = o;
  o += kTItemRows * 4;
  L.off_q = (o + 7u) & ~7u;
  o = L.off_q + kTItemRows * 8;
  L.off_qf = o;
  o += kTItemRows * 4;
  L.off_k = o;
  o += kTItemRows * 4;
  L.total = o;
  L.tmem_cols = 512;  // Z (4 tiles x HP <= 64) | Y_v hi*hi (<= 224) | Y_v corrections (<= 224)
  return L;
}

template <int HP, int N2>
__global__ void __launch_bounds__(kTThreads, 1)
    k_stats_tc(StatsArgs a, const float* __restrict__ xmax, const float* __restrict__ mumax,
               const unsigned char* __restrict__ vimg, const int* __restrict__ vexp_g,
               const float* __restrict__ vl1_g, const int* __restrict__ itemoff, int nh1, double* part,
               int64_t part_stride, int dbg) {
  extern __shared__ __align__(1024) unsigned char sm[];
  // (a waiter may lag a barrier by at most one phase: each tile of an item
  // has its own Z barrier, as all 4 can complete before the first is waited on)
  __shared__ uint64_t s_full[kTSlots], s_empty[kTSlots], s_zdone[2], s_b2ready, s_b2free, s_ydone;
  __shared__ uint32_t s_tmem;
  __shared__ int s_item;
  __shared__ double s_sqscale;  // the item's sq_v fixed-point scale 2^e (sums < 2^62)
  __shared__ float s_bmax[8];
  __shared__ int s_colexp[32];
  __shared__ float s_colmax[8][32];
  const Dims dm = a.dm;
  const int D = dm.D, H = dm.H, H1 = H + 1;
  const TcLayout L = tc_layout(D, H);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = su32(sm);
  float* s_z = reinterpret_cast<float*>(sm + L.off_z);           // [128][H1] fp32 zhat rows of one tile
  unsigned long long* s_sq = reinterpret_cast<unsigned long long*>(sm + L.off_sq);  // [npair * 128] sq_v, fixed point
  int* s_row = reinterpret_cast<int*>(sm + L.off_row);           // x row per item row
  double* s_q = reinterpret_cast<double*>(sm + L.off_q);         // q (fp64)
  float* s_qf = reinterpret_cast<float*>(sm + L.off_qf);         // q (fp32)
  int* s_k = reinterpret_cast<int*>(sm + L.off_k);               // row scale exponents
  if (tid == 0) {
    for (int i = 0; i < kTSlots; ++i) {
      binit(&s_full[i], kTProd);
      binit(&s_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) binit(&s_zdone[i], 1);
    binit(&s_b2ready, kTProd);
    binit(&s_b2free, 1);
    binit(&s_ydone, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 8) {  // TMEM: Z (2 tiles x HP columns) at 0, Y_v (npair x N2) at 64
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&s_tmem)),
                 "r"(L.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tfence_before();
  __syncthreads();
  tfence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t tY = tmem + 64, tYc = tmem + 288;  // Y_v: hi*hi products / the two correction products
  const int total = __ldg(itemoff + dm.C);
  // barrier completion counts (identical bookkeeping in every role)
  uint32_t fills[kTSlots] = {0, 0, 0, 0};  // completed fills per slot
  uint32_t nzt[2] = {};                    // completions of each Z buffer's barrier
  uint32_t nb2 = 0, ny = 0;                // b2ready+b2free / ydone completions
  uint32_t gs = 0;                         // global stage counter (slot = gs % 4)
  int c_cur = 0;                           // the item's component (for fill)

  // ---- producers: one ring fill = split v of (tile t, chunk k). The rows
  // of the NEXT fill are loaded into registers before this fill waits for its
  // slot (two register sets, ping-pong), so every thread keeps 8-16 row
  // pieces in flight. Thread: 4 dimensions (dg) x 8 rows (rg).
  struct Piece {
    float4 x[8];
    float4 mu;
  };
  const int dg = tid & 15, rg = tid >> 4;
  auto load = [&](int t, int k, int nr, Piece& P) {
    const int d0 = k * 64 + 4 * dg;
    P.mu = make_float4(0.f, 0.f, 0.f, 0.f);
    if (d0 < D) P.mu = __ldg(reinterpret_cast<const float4*>(a.mu32 + (int64_t)c_cur * D + d0));
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int rr = t * kTRows + rg * 8 + i;
      P.x[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (rr < nr && d0 < D && !(dbg & 2)) P.x[i] = __ldg(reinterpret_cast<const float4*>(a.X + (int64_t)s_row[rr] * D + d0));
    }
  };
  auto store = [&](int t, int k, int nr, const Piece& P, bool do_sq) {
    const int slot = gs % kTSlots;
    if (fills[slot] > 0) bwait(&s_empty[slot], fills[slot]);  // the MMAs of the previous fill are done
    const uint32_t hi = sbase + slot * kTSlotBytes, lo = hi + 16384;
    const int d0 = k * 64 + 4 * dg;
    float sq0 = 0.f, sq1 = 0.f, sq2 = 0.f, sq3 = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = rg * 8 + i, rr = t * kTRows + r;
      const bool live = rr < nr && d0 < D;
      const float v0 = live ? P.x[i].x - P.mu.x : 0.f, v1 = live ? P.x[i].y - P.mu.y : 0.f;
      const float v2 = live ? P.x[i].z - P.mu.z : 0.f, v3 = live ? P.x[i].w - P.mu.w : 0.f;
      if (do_sq && live) {
        const float q = s_qf[rr];
        sq0 = fmaf(q * v0, v0, sq0);
        sq1 = fmaf(q * v1, v1, sq1);
        sq2 = fmaf(q * v2, v2, sq2);
        sq3 = fmaf(q * v3, v3, sq3);
      }
      const float sc = rr < nr ? p2(s_k[rr]) : 1.f;
      uint32_t h01, l01, h23, l23;
      split(v0 * sc, v1 * sc, h01, l01);
      split(v2 * sc, v3 * sc, h23, l23);
      const uint32_t o = swz(r, dg >> 1) + (dg & 1) * 8;
      asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(hi + o), "r"(h01), "r"(h23) : "memory");
      asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(lo + o), "r"(l01), "r"(l23) : "memory");
    }
    if (do_sq) {
      // the warp's two row groups, then exact fixed-point sums (integer
      // atomics: the order of the warps cannot change the result)
      sq0 += __shfl_xor_sync(0xffffffffu, sq0, 16);
      sq1 += __shfl_xor_sync(0xffffffffu, sq1, 16);
      sq2 += __shfl_xor_sync(0xffffffffu, sq2, 16);
      sq3 += __shfl_xor_sync(0xffffffffu, sq3, 16);
      if (lane < 16 && d0 < D) {
        const double f = s_sqscale;
        atomicAdd(&s_sq[d0], static_cast<unsigned long long>(llrint(static_cast<double>(sq0) * f)));
        atomicAdd(&s_sq[d0 + 1], static_cast<unsigned long long>(llrint(static_cast<double>(sq1) * f)));
        atomicAdd(&s_sq[d0 + 2], static_cast<unsigned long long>(llrint(static_cast<double>(sq2) * f)));
        atomicAdd(&s_sq[d0 + 3], static_cast<unsigned long long>(llrint(static_cast<double>(sq3) * f)));
      }
    }
    fence_async();
    barrive(&s_full[slot]);
    ++fills[slot];
    ++gs;
  };
  // ---- the MMA thread: consume one slot (GEMM i) or a slot pair (GEMM ii)
  auto take = [&]() -> int {
    const int slot = gs % kTSlots;
    ++fills[slot];
    bwait(&s_full[slot], fills[slot]);
    tfence_after();
    ++gs;
    return slot;
  };

  for (;;) {
    __syncthreads();
    if (tid == 0) s_item = a.qctr ? atomicAdd(a.qctr, 1) : -1;
    __syncthreads();
    const int item = s_item;
    if (item < 0 || item >= total) break;
    const int c = find_item_t(itemoff, dm.C, item);
    const int r0 = a.off[c] + (item - itemoff[c]) * kTItemRows;
    const int nr = min(a.off[c + 1], r0 + kTItemRows) - r0;
    const int T = (nr + kTRows - 1) / kTRows;
    const bool direct = itemoff[c + 1] - itemoff[c] == 1;
    c_cur = c;

    if (warp < 8) {
      // ---- item setup: rows, q, row scales, mu, V image (per-h scale), sq
      const float mb = __ldg(mumax + c);
      for (int i = tid; i < kTItemRows; i += kTProd) {
        int n = 0, k = 0;
        double q = 0.0;
        if (i < nr) {
          const int e = a.ent[r0 + i];
          n = e / dm.Cp;
          q = a.resp[e];
          k = sexp(__ldg(xmax + n) + mb);
        }
        s_row[i] = n;
        s_q[i] = q;
        s_qf[i] = static_cast<float>(q);
        s_k[i] = k;
      }
      for (int d = tid; d < L.npair * 128; d += kTProd) s_sq[d] = 0ull;
      {  // sq_v <= nr max_n (max|x_n| + max|mu_c|)^2: the fixed-point scale
        float bm = 0.f;
        for (int i = tid; i < nr; i += kTProd) bm = fmaxf(bm, __ldg(xmax + s_row[i]) + mb);
        for (int o = 16; o > 0; o >>= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, o));
        if (lane == 0) s_bmax[warp] = bm;
        producers_sync();
        if (tid == 0) {
          float m = 0.f;
          for (int w = 0; w < 8; ++w) m = fmaxf(m, s_bmax[w]);
          const double B = static_cast<double>(m) * m * static_cast<double>(nr) + 1e-300;
          s_sqscale = ldexp(1.0, 61 - ilogb(B));
        }
      }
      // V image (GEMM i's B, prebuilt per precompute by k_stats_vimg in this
      // smem layout): a linear copy; its row scales and |V_h|_1 beside it
      {
        const uint32_t nb = static_cast<uint32_t>(L.nch) * 2 * HP * 128;
        const uint4* src = reinterpret_cast<const uint4*>(vimg + (int64_t)c * nb);
        uint4* dst = reinterpret_cast<uint4*>(sm + L.off_V);
        for (uint32_t i = tid; i < nb / 16; i += kTProd) dst[i] = __ldg(src + i);
        if (tid < HP) {
          s_colexp[tid] = __ldg(vexp_g + (int64_t)c * HP + tid);
          s_colmax[0][tid] = __ldg(vl1_g + (int64_t)c * HP + tid);
        }
      }
      fence_async();
      producers_sync();
      int vexp[HP];  // (kept in registers by the Z epilogue)
#pragma unroll
      for (int h = 0; h < HP; ++h) vexp[h] = s_colexp[h];
      producers_sync();
      if (tid < N2) {  // GEMM ii's B column scales (from the bounds)
        float mm = 0.f;
        for (int w = 0; w < 8; ++w) mm = fmaxf(mm, s_bmax[w]);
        const float bnd = tid < H ? 1.01f * s_colmax[0][tid] * mm * mm * p2(-13)
                                  : (tid == H ? 1.01f * mm * p2(-13) : 0.f);
        s_colexp[tid] = sexp(bnd);
      }
      producers_sync();
      // ---- tiles, pipelined: GEMM i fills of tile t + 1 go before tile t's
      // epilogue (the MMA computes Z of t + 1 in the other Z buffer meanwhile)
      // and its GEMM ii fills (re-reading tile t's rows while they are in L2)
      const int NE = H1 * (H1 + 1) / 2;
      double eacc = 0.0;  // entry tid (tid < NE)
      int ei = 0, ej = 0;
      if (tid < NE) {
        int t = tid;
        while (t >= H1 - ei) t -= H1 - ei, ++ei;
        ej = ei + t;
      }
      const int NK = 2 * L.npair;
      // tile t's CUDA-core work, before its first GEMM ii fill
      auto epilogue = [&](int t) {
        // mz of tile t (warps 0-3: TMEM lanes = tile rows) into s_z
        if (warp < 4) {
          bwait(&s_zdone[t & 1], nzt[t & 1] + 1);
          tfence_after();
          const int r = warp * 32 + lane, rr = t * kTRows + r;
          float z[HP];
#pragma unroll
          for (int h0 = 0; h0 < HP; h0 += 8)
            tld8(tmem + (static_cast<uint32_t>(warp * 32) << 16) + (t & 1) * HP + h0, z + h0);
          tld_wait();
          const bool live = rr < nr;
#pragma unroll
          for (int h = 0; h < HP; ++h)
            if (h < H) s_z[r * H1 + h] = live ? z[h] * p2(-(s_k[rr] + vexp[h])) : 0.f;
          s_z[r * H1 + H] = live ? 1.f : 0.f;
        }
        ++nzt[t & 1];
        if (nb2 > 0) bwait(&s_b2free, nb2);  // the previous tile's GEMM ii is done with B
        producers_sync();
        // E (fp64, a thread per upper-triangle entry, summed over the tiles)
        const int nt = min(kTRows, nr - t * kTRows);
        if (tid < NE)
          for (int r = 0; r < nt; ++r)
            eacc = fma(s_q[t * kTRows + r], static_cast<double>(s_z[r * H1 + ei]) * static_cast<double>(s_z[r * H1 + ej]),
                       eacc);
        // GEMM ii's B for tile t: q zhat_h 2^(e_h - k_r), K-major (h rows, 64
        // tile rows per 128-byte line, two line blocks)
        const uint32_t b2 = sbase + L.off_B2;
        for (int i = tid; i < kTRows * N2; i += kTProd) {
          const int r = i % kTRows, h = i / kTRows, rr = t * kTRows + r;
          float b = 0.f;
          if (rr < nr && h < H1) b = s_qf[rr] * s_z[r * H1 + h] * p2(s_colexp[h] - s_k[rr]);
          __half bh, bl;
          split1(b, bh, bl);
          const int kc = r >> 6, rl = r & 63;
          const uint32_t o = swz(h, rl >> 3) + (rl & 7) * 2;
          const uint32_t base_h = b2 + (0 * 2 + kc) * N2 * 128, base_l = b2 + (1 * 2 + kc) * N2 * 128;
          asm volatile("st.shared.b16 [%0], %1;" ::"r"(base_h + o), "h"(*reinterpret_cast<uint16_t*>(&bh)) : "memory");
          asm volatile("st.shared.b16 [%0], %1;" ::"r"(base_l + o), "h"(*reinterpret_cast<uint16_t*>(&bl)) : "memory");
        }
        fence_async();
        barrive(&s_b2ready);
        ++nb2;
        producers_sync();  // (s_z is rewritten by the next tile)
      };
      // the item's fills in MMA order: A(0), then per t: A(t + 1), B(t)
      // (A = GEMM i, B = GEMM ii); rows loaded two fills ahead (3 register
      // sets), the GEMM ii fills' loads also ahead of the epilogue
      const int nF = 2 * T * NK;
      auto fdesc = [&](int f, int& t, int& k, bool& b) {
        if (f < NK) {
          t = 0, k = f, b = false;
          return;
        }
        const int j = (f - NK) / NK;
        k = (f - NK) - j * NK;
        if (j < 2 * (T - 1)) {
          b = (j & 1) != 0;
          t = b ? (j - 1) / 2 : j / 2 + 1;
        } else {
          t = T - 1, b = true;
        }
      };
      auto ld = [&](int f, Piece& P) {
        int t, k;
        bool b;
        fdesc(f, t, k, b);
        load(t, k, nr, P);
      };
      auto st = [&](int f, const Piece& P) {
        int t, k;
        bool b;
        fdesc(f, t, k, b);
        if (b && k == 0) epilogue(t);
        store(t, k, nr, P, b);
      };
      {
        Piece P0, P1, P2;
        ld(0, P0);
        if (1 < nF) ld(1, P1);
        for (int f = 0; f < nF; f += 3) {
          if (f + 2 < nF) ld(f + 2, P2);
          st(f, P0);
          if (f + 1 >= nF) break;
          if (f + 3 < nF) ld(f + 3, P0);
          st(f + 1, P1);
          if (f + 2 >= nF) break;
          if (f + 4 < nF) ld(f + 4, P1);
          st(f + 2, P2);
        }
      }
      if (tid < NE) {
        double* pe = direct ? a.E + (int64_t)c * H1 * H1 : part + (int64_t)item * part_stride + (int64_t)nh1 * D + D;
        pe[ej * H1 + ei] = eacc;
        pe[ei * H1 + ej] = eacc;
      }
      // ---- Y_v epilogue (warps 0-3: TMEM lanes = the pair's 128 dimensions)
      producers_sync();
      if (warp < 4) {
        bwait(&s_ydone, ++ny);
        tfence_after();
        double* pp = direct ? nullptr : part + (int64_t)item * part_stride;
        for (int j = 0; j < L.npair; ++j) {
          float y[N2], yc[N2];
#pragma unroll
          for (int h0 = 0; h0 < N2; h0 += 8) {
            tld8(tY + (static_cast<uint32_t>(warp * 32) << 16) + j * N2 + h0, y + h0);
            tld8(tYc + (static_cast<uint32_t>(warp * 32) << 16) + j * N2 + h0, yc + h0);
          }
          tld_wait();
#pragma unroll
          for (int h = 0; h < N2; ++h) y[h] += yc[h];
          const int d = j * 128 + warp * 32 + lane;
          if (d < D) {
#pragma unroll
            for (int h = 0; h < N2; ++h) {
              if (h >= H1) break;
              const double v = static_cast<double>(y[h]) * static_cast<double>(p2(-s_colexp[h]));
              if (direct) a.Y[((int64_t)c * H1 + h) * D + d] = v;
              else pp[(int64_t)h * D + d] = v;
            }
          }
        }
      } else {
        ++ny;
      }
      for (int d = tid; d < D; d += kTProd) {
        const double v = static_cast<double>(s_sq[d]) / s_sqscale;
        if (direct) a.sq[(int64_t)c * D + d] = v;
        else part[(int64_t)item * part_stride + (int64_t)nh1 * D + d] = v;
      }
      tfence_before();
    } else {
      // ---- the MMA warp: every lane walks the schedule (the barrier waits,
      // the counters), lane 0 issues the MMAs and commits
      const bool leader = lane == 0;
      const uint32_t id1 = idesc(HP, false), id2 = idesc(N2, true);
      auto gemm_i = [&](int t) {  // Z of tile t into buffer t & 1
        for (int k = 0; k < 2 * L.npair; ++k) {
          const int slot = take();
          if (k < L.nch && leader && !(dbg & 1)) {
            const uint32_t ah = sbase + slot * kTSlotBytes, al = ah + 16384;
            const uint32_t bh = sbase + L.off_V + (k * 2) * HP * 128, bl = bh + HP * 128;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t o = kk * 32;
              const uint32_t acc = (k > 0 || kk > 0) ? 1u : 0u;
              const uint32_t dz = tmem + (t & 1) * HP;
              mma_ss(dz, desc(al + o, 16), desc(bh + o, 16), id1, acc);
              mma_ss(dz, desc(ah + o, 16), desc(bl + o, 16), id1, 1u);
              mma_ss(dz, desc(ah + o, 16), desc(bh + o, 16), id1, 1u);
            }
          }
          if (leader) {
            tcommit(&s_empty[slot]);
            if (k == 2 * L.npair - 1) tcommit(&s_zdone[t & 1]);
          }
          __syncwarp();
        }
      };
      gemm_i(0);
      for (int t = 0; t < T; ++t) {
        if (t + 1 < T) gemm_i(t + 1);
        bwait(&s_b2ready, ++nb2);
        tfence_after();
        const uint32_t b2 = sbase + L.off_B2;
        for (int j = 0; j < L.npair; ++j) {
          const int s0 = take();
          take();  // the adjacent slot (s0 even): the MN-major atoms 32 KB apart
          if (leader && !(dbg & 1)) {
            const uint32_t ah = sbase + s0 * kTSlotBytes, al = ah + 16384;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const uint32_t oa = kk * 2048;  // 16 tile rows = two 8-row groups
              const uint32_t bh = b2 + (0 * 2 + (kk >> 2)) * N2 * 128 + (kk & 3) * 32;
              const uint32_t bl = b2 + (1 * 2 + (kk >> 2)) * N2 * 128 + (kk & 3) * 32;
              const uint32_t acc = (t > 0 || kk > 0) ? 1u : 0u;
              // the small correction products in their own accumulator (the
              // tensor core's accumulation truncates: the hi*hi sum then sees
              // a third of the additions)
              mma_ss(tYc + j * N2, desc(al + oa, kTSlotBytes), desc(bh, 16), id2, acc);
              mma_ss(tYc + j * N2, desc(ah + oa, kTSlotBytes), desc(bl, 16), id2, 1u);
              mma_ss(tY + j * N2, desc(ah + oa, kTSlotBytes), desc(bh, 16), id2, acc);
            }
          }
          if (leader) {
            tcommit(&s_empty[s0]);
            tcommit(&s_empty[s0 + 1]);
          }
          __syncwarp();
        }
        if (leader) tcommit(&s_b2free);
        __syncwarp();
      }
      if (leader) tcommit(&s_ydone);
      __syncwarp();
      ++ny;
    }
  }
  tfence_before();
  __syncthreads();
  tfence_after();
  if (warp == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(L.tmem_cols));
}

// GEMM i's B for component c, built once per precompute: V_c^T rows h
// (K-major, 64 dimensions per 128-byte swizzled line; hi then lo per chunk),
// row h scaled by 2^e_h (e_h from max_d |V[h][d]|), and |V_h|_1. A block per
// component, a warp per row h.
template <int HP>
__global__ void k_stats_vimg(Dims dm, const float* __restrict__ V32, unsigned char* img, int* vexp, float* vl1) {
  const int D = dm.D, H = dm.H, nch = (D + 63) / 64;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nb = static_cast<int64_t>(nch) * 2 * HP * 128;
  for (int c = blockIdx.x; c < dm.C; c += gridDim.x) {
    const float* Vc = V32 + (int64_t)c * D * H;  // [d][h]
    unsigned char* out = img + c * nb;
    for (int h = warp; h < HP; h += blockDim.x >> 5) {
      float m = 0.f, l1 = 0.f;
      if (h < H)
        for (int d = lane; d < D; d += 32) {
          const float v = fabsf(__ldg(Vc + (int64_t)d * H + h));
          m = fmaxf(m, v);
          l1 += v;
        }
      for (int o = 16; o > 0; o >>= 1) {
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
      }
      const int e = sexp(m);
      if (lane == 0) {
        vexp[(int64_t)c * HP + h] = e;
        vl1[(int64_t)c * HP + h] = l1;
      }
      const float sc = p2(e);
      for (int k = 0; k < nch; ++k) {
        const int d = k * 64 + 2 * lane;  // lane: dims (d, d + 1) of chunk k
        const float v0 = (h < H && d < D) ? __ldg(Vc + (int64_t)d * H + h) * sc : 0.f;
        const float v1 = (h < H && d + 1 < D) ? __ldg(Vc + (int64_t)(d + 1) * H + h) * sc : 0.f;
        uint32_t hv, lv;
        split(v0, v1, hv, lv);
        const uint32_t o = swz(h, lane >> 2) + (lane & 3) * 4;
        *reinterpret_cast<uint32_t*>(out + (k * 2 + 0) * HP * 128 + o) = hv;
        *reinterpret_cast<uint32_t*>(out + (k * 2 + 1) * HP * 128 + o) = lv;
      }
    }
  }
}

}  // namespace

int64_t stats_tc_image_bytes(const Dims& dm) {
  const TcLayout L = tc_layout(dm.D, dm.H);
  return static_cast<int64_t>(dm.C) * L.nch * 2 * L.HP * 128;
}
cudaError_t launch_stats_vimg(const Dims& dm, const float* V32, void* img, int* vexp, float* vl1, cudaStream_t s) {
  k_stats_vimg<16><<<sm_count() * 4, 512, 0, s>>>(dm, V32, static_cast<unsigned char*>(img), vexp, vl1);
  return cudaGetLastError();
}

bool stats_tc_ok(const Dims& dm) {
  return dm.D % 4 == 0 && dm.D <= kTMaxChunks * 64 && dm.H >= 1 && dm.H <= 16 &&
         tc_layout(dm.D, dm.H).total <= 227 * 1024;
}
int stats_tc_rows() { return kTItemRows; }

cudaError_t launch_stats_tc(const StatsArgs& a, const float* xmax, const float* mumax, const int* itemoff, int nh1,
                            double* part, int64_t part_stride, cudaStream_t s) {
  if (!a.vimg || !a.vexp || !a.vl1) return cudaErrorInvalidValue;
  const TcLayout L = tc_layout(a.dm.D, a.dm.H);
  const size_t smem = L.total;
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    static const int dbg = [] {
      const char* v = std::getenv("VMFA_STATS_TC_DBG");  // diagnostics: 1 skip MMAs, 2 skip row loads
      return v ? std::atoi(v) : 0;
    }();
    kern<<<sm_count(), kTThreads, smem, s>>>(a, xmax, mumax, static_cast<const unsigned char*>(a.vimg), a.vexp,
                                             a.vl1, itemoff, nh1, part, part_stride, dbg);
  };
  if (L.HP == 16 && L.N2 == 16) go(k_stats_tc<16, 16>);
  else if (L.HP == 16 && L.N2 == 32) go(k_stats_tc<16, 32>);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace vmfa_b200
