// vmfa_stats_tc.cu — the sufficient statistics (accumulate_suffstats,
// mstep.cpp:47-101) on the 5th-generation tensor cores.
//
// Per item (component c, <= kTItemRows of its K-pairs (n, q)), centred rows
// v_n = x_n - mu_c (fp32 mu, as the other statistics kernels; k_stats_uncenter
// restores the raw sums), in tiles of kTRows = 48 rows:
//   GEMM i   Z   [rows x HP]  = [v] (rows x D) . [V_c^T] (D x HP)     mz = V_c v
//   GEMM ii  Y_v [D x N2]    += [v]^T (D x rows) . [q zhat] (rows x N2)
// with zhat = [mz; 1], E = sum q zhat zhat^T in fp64 from the fp32 mz, and
// sq_v = sum q v^2 (fp32 per thread over the item's rows, fp64 across
// threads) on the CUDA cores. Both GEMMs are tcgen05.mma.kind::f16 in 3xFP16
// (hi*hi + hi*lo + lo*hi, 22 significant bits, fp32 accumulation in TMEM), SS
// form, M = 128 (GEMM i's rows 48..127 read the next smem bytes and are
// ignored; an MMA costs the same ~46 cycles for M = 64 or 128 at these N).
//
// A tile's split rows stay RESIDENT in shared memory: every 64-dimension chunk
// of the tile is produced once (global load, centring, power-of-two row scale
// 2^k_n from the bound max|x_n| + max|mu_c|, fp16 hi/lo split, 128-byte
// swizzle) into its own ring slot (12 KB: hi | lo, 48 lines of 128 B), read by
// GEMM i as a K-major A (rows x dims) and, once the tile's zhat is known, by
// GEMM ii as an MN-major A (dims x rows; two adjacent slots = M 128); GEMM ii
// releases the slots to the next tile. The ring holds a whole number of tiles
// (13 slots: one tile at D = 784, three at D = 256). GEMM ii sums over rows
// (its K), so 2^-k_n is folded into its B operand (q zhat), exactly, and every
// column of that operand gets a power-of-two scale from an a-priori bound
// (|V_h|_1 max_n bound_n^2). V_c's image (GEMM i's B, prebuilt per precompute
// by k_stats_vimg) is copied into shared memory once per item.
//
// Roles: warps 0-7 produce the tiles, run the Z epilogue (warps 0-1: TMEM lanes
// = tile rows) and the CUDA-core work; lane 0 of warp 8 issues the MMAs and
// commits to the slot / Z / B2 / Y barriers. Outputs as the other statistics
// kernels: a component's sole item writes Y_v, sq_v, E directly, split
// components write item partials reduced by k_stats_reduce.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "vmfa_kernels.cuh"

namespace vmfa_b200 {
namespace {

constexpr int kTR = 128;                 // rows per tile (GEMM i's M, GEMM ii's K)
constexpr int kTItemRows = 512;          // K-pairs per item (4 tiles)
constexpr int kTMaxChunks = 13;          // D <= 832
constexpr int kTFill = 16;               // fill warps (0-15)
constexpr int kTFillThreads = kTFill * 32;
constexpr int kTRowsPerThr = kTR * 16 / kTFillThreads;  // 4 rows x 4 dimensions per thread and chunk
constexpr int kTEpi0 = kTFill;           // warps 16-19: Z epilogue (kernel Z) / B2 builders (kernel Y)
constexpr int kTMma = kTFill + 4;        // warp 20 issues the MMAs
constexpr int kTThreads = (kTFill + 5) * 32;
constexpr uint32_t kTUnit = kTR * 128;   // one plane of one chunk: 128 rows x 64 fp16 (16 KB)
constexpr uint32_t kTPairBytes = 4 * kTUnit;  // pair slot [hi c0 | hi c1 | lo c0 | lo c1]
constexpr int kTPairs = 2;               // ring depth (pair slots)
constexpr int kTargetE = 14;             // operands scaled to |value| <= 2^14

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
         (static_cast<uint32_t>(128 >> 4) << 24);
}
__device__ __forceinline__ uint32_t idesc_m(int N) { return idesc(N, false); }
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

__device__ __forceinline__ int find_item_t(const int* itemoff, int C, int item) {
  int lo = 0, hi = C;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(itemoff + mid) <= item) lo = mid;
    else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------- layout
struct TcLayout {
  int nch, npair, HP, N2;
  uint32_t off_V, off_B2, off_z, off_ep, off_sqw, off_row, off_q, off_k, total_z;
  uint32_t off_row_y, off_q_y, off_k_y, total_y;
};
__host__ __device__ inline TcLayout tc_layout(int D, int H) {
  TcLayout L;
  L.nch = (D + 63) / 64;
  L.npair = (L.nch + 1) / 2;
  L.HP = ((H + 15) / 16) * 16;
  L.N2 = ((H + 1 + 15) / 16) * 16;  // (M = 128: N in steps of 16)
  const uint32_t ring = kTPairs * kTPairBytes;
  // kernel Z: ring | V image | s_z | E partials (4 warps) | item arrays
  uint32_t o = ring;
  L.off_V = o;
  o += static_cast<uint32_t>(L.nch) * 2 * L.HP * 128;
  L.off_z = o;
  o += static_cast<uint32_t>(kTR) * (H + 1) * 4;
  o = (o + 15u) & ~15u;
  L.off_ep = o;
  o += 4u * 6 * 2 * 32 * 8;
  L.off_row = o;
  L.off_q = (L.off_row + kTItemRows * 4 + 7u) & ~7u;
  L.off_k = L.off_q + kTItemRows * 8;
  L.total_z = L.off_k + kTItemRows * 4;
  // kernel Y: ring | B2 x 2 | sq per fill warp (fp32) | item arrays
  uint32_t p = ring;
  L.off_B2 = p;
  p += 2u * 2 * 2 * L.N2 * 128;  // 2 buffers x (hi, lo) x 2 line blocks (K 0-63, 64-127)
  L.off_sqw = p;
  p += static_cast<uint32_t>(kTFill) * kTMaxChunks * 64 * 4;
  L.off_row_y = p;
  L.off_q_y = (L.off_row_y + kTItemRows * 4 + 7u) & ~7u;
  L.off_k_y = L.off_q_y + kTItemRows * 8;
  L.total_y = L.off_k_y + kTItemRows * 4;
  return L;
}

// dbg & 4: block 0 prints per-role cycle counts (diagnostics)
#define TC_T0() const long long _t0 = (dbg & 4) ? clock64() : 0
#define TC_ACC(i) do { if ((dbg & 4) && blockIdx.x == 0) prof[i] += clock64() - _t0; } while (0)
__device__ __forceinline__ void dmma_f64(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void fill_sync() { asm volatile("bar.sync 1, %0;" ::"r"(kTFillThreads) : "memory"); }
__device__ __forceinline__ void producers_all_sync() { asm volatile("bar.sync 2, %0;" ::"r"(kTMma * 32) : "memory"); }

// Item setup shared by both kernels (all producer warps 0-11): rows, q, row
// scale exponents, and the bound max_n (max|x_n| + max|mu_c|) into s_bmax.
struct ItemSetup {
  int c, r0, nr, T;
  bool direct;
};
__device__ __forceinline__ void item_rows(const StatsArgs& a, const float* __restrict__ xmax, float mb, int r0, int nr,
                                          int* s_row, double* s_q, int* s_k, float* s_bmax) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float bm = 0.f;
  for (int i = tid; i < kTItemRows; i += kTMma * 32) {
    int n = 0, k = 0;
    double q = 0.0;
    if (i < nr) {
      const int e = a.ent[r0 + i];
      n = e / a.dm.Cp;
      q = a.resp[e];
      const float bnd = __ldg(xmax + n) + mb;
      k = sexp(bnd);
      bm = fmaxf(bm, bnd);
    }
    s_row[i] = n;
    s_q[i] = q;
    s_k[i] = k;
  }
  for (int o = 16; o > 0; o >>= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, o));
  if (lane == 0) s_bmax[warp] = bm;
}

// The fill role: unit f of an item = chunk u = f % U (U = 2 npair; chunks >=
// nch are padding: no stores) of tile f / U, 128 rows x 64 dimensions; thread
// (dg, rg) covers dimensions 4 dg .. + 3 of rows 8 rg .. + 7. A pair slot
// holds the units 2p, 2p + 1 of a tile; its full barrier takes one arrival
// per fill warp and unit. Loads run two units ahead (two register batches).
template <bool SQ, typename F>
__device__ __forceinline__ void fill_item(const StatsArgs& a, const TcLayout& L, int c, int nr, int T, uint32_t sbase,
                                          const int* s_row, const double* s_q, const int* s_k, uint64_t* s_full,
                                          uint64_t* s_empty, uint32_t gp0, float* s_sqw, int dbg, F&& on_tile_end) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int dg = tid & 15, rg = tid >> 4;
  const int D = a.dm.D;
  const int U = 2 * L.npair, nF = T * U;
  const float* muc = a.mu32 + (int64_t)c * D;
  float4 xa[kTRowsPerThr], xb[kTRowsPerThr], xc[kTRowsPerThr];
  float4 ma = make_float4(0.f, 0.f, 0.f, 0.f), mbv = ma, mcv = ma;
  auto ldu = [&](int f, float4* xv, float4& mv) {
    const int t = f / U, k = f - t * U, d0 = k * 64 + 4 * dg;
    const bool dl = k < L.nch && d0 < D;
    mv = dl ? __ldg(reinterpret_cast<const float4*>(muc + d0)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int i = 0; i < kTRowsPerThr; ++i) {
      const int rt = t * kTR + rg * kTRowsPerThr + i;
      xv[i] = (dl && rt < nr && !(dbg & 2)) ? __ldg(reinterpret_cast<const float4*>(a.X + (int64_t)s_row[rt] * D + d0))
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto stu = [&](int f, const float4* xv, const float4& mv) {
    const int t = f / U, k = f - t * U, d0 = k * 64 + 4 * dg;
    const uint32_t gp = gp0 + static_cast<uint32_t>(f >> 1);
    const int slot = static_cast<int>(gp % kTPairs);
    const uint32_t use = gp / kTPairs;
    if ((f & 1) == 0 && use > 0) bwait(&s_empty[slot], use);  // the pair slot's previous tile is done
    if (k < L.nch) {
      const uint32_t hi = sbase + slot * kTPairBytes + (f & 1) * kTUnit, lo = hi + 2 * kTUnit;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
      for (int i = 0; i < kTRowsPerThr; ++i) {
        const int r = rg * kTRowsPerThr + i, rt = t * kTR + r;
        const bool on = rt < nr && d0 < D;
        const float v0 = on ? xv[i].x - mv.x : 0.f, v1 = on ? xv[i].y - mv.y : 0.f;
        const float v2 = on ? xv[i].z - mv.z : 0.f, v3 = on ? xv[i].w - mv.w : 0.f;
        if (SQ) {
          const float q = on ? static_cast<float>(s_q[rt]) : 0.f;
          s0 = fmaf(q * v0, v0, s0);
          s1 = fmaf(q * v1, v1, s1);
          s2 = fmaf(q * v2, v2, s2);
          s3 = fmaf(q * v3, v3, s3);
        }
        const float sc = on ? p2(s_k[rt]) : 0.f;
        uint32_t h01, l01, h23, l23;
        split(v0 * sc, v1 * sc, h01, l01);
        split(v2 * sc, v3 * sc, h23, l23);
        const uint32_t o = swz(r, dg >> 1) + (dg & 1) * 8;
        asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(hi + o), "r"(h01), "r"(h23) : "memory");
        asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(lo + o), "r"(l01), "r"(l23) : "memory");
      }
      if (SQ) {  // the warp's two row groups, then the warp's own fp64 row of sums
        s0 += __shfl_xor_sync(0xffffffffu, s0, 16);
        s1 += __shfl_xor_sync(0xffffffffu, s1, 16);
        s2 += __shfl_xor_sync(0xffffffffu, s2, 16);
        s3 += __shfl_xor_sync(0xffffffffu, s3, 16);
        if (lane < 16 && d0 < D) {  // (fp32 over the warp's <= 32 rows of the item)
          float* w = s_sqw + (int64_t)warp * kTMaxChunks * 64 + d0;
          w[0] += s0;
          w[1] += s1;
          w[2] += s2;
          w[3] += s3;
        }
      }
      fence_async();
    }
    __syncwarp();
    if (lane == 0) barrive(&s_full[slot]);
    if (k == U - 1) on_tile_end(t);
  };
  ldu(0, xa, ma);
  if (1 < nF) ldu(1, xb, mbv);
  if (2 < nF) ldu(2, xc, mcv);
  for (int f = 0; f < nF; f += 3) {
    stu(f, xa, ma);
    if (f + 3 < nF) ldu(f + 3, xa, ma);
    if (f + 1 >= nF) break;
    stu(f + 1, xb, mbv);
    if (f + 4 < nF) ldu(f + 4, xb, mbv);
    if (f + 2 >= nF) break;
    stu(f + 2, xc, mcv);
    if (f + 5 < nF) ldu(f + 5, xc, mcv);
  }
}

// ---------------------------------------------------------------- kernel Z
// GEMM i per tile of 128 rows (M = 128, every row live): Z = [v] . [V_c^T]
// over the chunk pairs streamed through the ring (a slot is released as soon
// as its two chunks are multiplied); Z double-buffered in TMEM so the
// epilogue of tile t (warps 8-11: zhat = Z 2^-(k_n + e_h) to global memory,
// and E = sum q [zhat; 1][zhat; 1]^T in fp64 by DMMA m8n8k4, each warp over
// its own 32 rows) runs under GEMM i of tile t + 1.
template <int HP>
__global__ void __launch_bounds__(kTThreads, 1)
    k_stats_z(StatsArgs a, const float* __restrict__ xmax, const float* __restrict__ mumax,
              const unsigned char* __restrict__ vimg, const int* __restrict__ vexp_g, const int* __restrict__ itemoff,
              int nh1, double* part, int64_t part_stride, float* zout, int dbg) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t s_full[kTPairs], s_empty[kTPairs], s_zdone[2], s_zfree[2];
  __shared__ uint32_t s_tmem;
  __shared__ int s_item;
  __shared__ float s_bmax[kTMma];
  __shared__ int s_vexp[32];
  long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long tstart = clock64();
  const Dims dm = a.dm;
  const int D = dm.D, H = dm.H, H1 = H + 1;
  const TcLayout L = tc_layout(D, H);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = su32(sm);
  float* s_z = reinterpret_cast<float*>(sm + L.off_z);
  double (*s_epart)[6 * 2 * 32] = reinterpret_cast<double (*)[6 * 2 * 32]>(sm + L.off_ep);
  int* s_row = reinterpret_cast<int*>(sm + L.off_row);
  double* s_q = reinterpret_cast<double*>(sm + L.off_q);
  int* s_k = reinterpret_cast<int*>(sm + L.off_k);
  if (tid == 0) {
    for (int i = 0; i < kTPairs; ++i) {
      binit(&s_full[i], 2 * kTFill);
      binit(&s_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      binit(&s_zdone[i], 1);
      binit(&s_zfree[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kTMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&s_tmem)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tfence_before();
  __syncthreads();
  tfence_after();
  const uint32_t tmem = s_tmem;
  const int total = __ldg(itemoff + dm.C);
  uint32_t gp = 0;     // pair slots consumed so far (all items)
  uint32_t ntile = 0;  // tiles so far (Z buffer = ntile & 1)
  for (;;) {
    __syncthreads();
    if (tid == 0) s_item = a.qctr ? atomicAdd(a.qctr, 1) : -1;
    __syncthreads();
    const int item = s_item;
    if (item < 0 || item >= total) break;
    const int c = find_item_t(itemoff, dm.C, item);
    const int r0 = a.off[c] + (item - itemoff[c]) * kTItemRows;
    const int nr = min(a.off[c + 1], r0 + kTItemRows) - r0;
    const int T = (nr + kTR - 1) / kTR;
    const bool direct = itemoff[c + 1] - itemoff[c] == 1;
    if (warp < kTMma) {
      item_rows(a, xmax, __ldg(mumax + c), r0, nr, s_row, s_q, s_k, s_bmax);
      const uint32_t nb = static_cast<uint32_t>(L.nch) * 2 * HP * 128;
      const uint4* src = reinterpret_cast<const uint4*>(vimg + (int64_t)c * nb);
      uint4* dst = reinterpret_cast<uint4*>(sm + L.off_V);
      for (uint32_t i = tid; i < nb / 16; i += kTMma * 32) dst[i] = __ldg(src + i);
      if (tid < HP) s_vexp[tid] = __ldg(vexp_g + (int64_t)c * HP + tid);
      fence_async();
      producers_all_sync();
    }
    if (warp < kTFill) {
      TC_T0();
      fill_item<false>(a, L, c, nr, T, sbase, s_row, s_q, s_k, s_full, s_empty, gp, nullptr, dbg, [](int) {});
      TC_ACC(0);
    } else if (warp < kTMma) {
      // ---- Z epilogue + E (warps 8-11: TMEM lanes 32 (warp - 8) ..)
      const int qd = warp - kTEpi0;
      double ec[6][2];
#pragma unroll
      for (int i = 0; i < 6; ++i) ec[i][0] = ec[i][1] = 0.0;
      for (int t = 0; t < T; ++t) {
        const uint32_t zb = (ntile + t) & 1u;
        {
          TC_T0();
          bwait(&s_zdone[zb], (ntile + t) / 2 + 1);
          TC_ACC(1);
        }
        tfence_after();
        const int r = qd * 32 + lane, rt = t * kTR + r;
        float z[HP];
#pragma unroll
        for (int h0 = 0; h0 < HP; h0 += 8)
          tld8(tmem + (static_cast<uint32_t>(qd * 32) << 16) + zb * HP + h0, z + h0);
        tld_wait();
        tfence_before();
        __syncwarp();
        if (lane == 0) barrive(&s_zfree[zb]);
        const bool lv = rt < nr;
        float* zo = zout + (int64_t)(r0 + rt) * H;
#pragma unroll
        for (int h = 0; h < HP; ++h)
          if (h < H) {
            const float v = lv ? z[h] * p2(-(s_k[lv ? rt : 0] + s_vexp[h])) : 0.f;
            s_z[r * H1 + h] = v;
            if (lv) zo[h] = v;
          }
        s_z[r * H1 + H] = lv ? 1.f : 0.f;
        __syncwarp();
        // E over this warp's 32 rows: A(g, t) = zhat[row t][8 mi + g],
        // B(t, g) = q zhat[row t][8 ni + g] (k = 4 rows per DMMA)
        const int g = lane >> 2, tq = lane & 3;
        for (int k0 = 0; k0 < 32; k0 += 4) {
          const int rr = qd * 32 + k0 + tq, rtt = t * kTR + rr;
          const double q = s_q[rtt];
          double za[3], zq[3];
#pragma unroll
          for (int m = 0; m < 3; ++m) {
            const int col = 8 * m + g;
            za[m] = col < H1 ? static_cast<double>(s_z[rr * H1 + col]) : 0.0;
            zq[m] = q * za[m];
          }
          dmma_f64(ec[0], za[0], zq[0]);
          dmma_f64(ec[1], za[0], zq[1]);
          dmma_f64(ec[2], za[0], zq[2]);
          dmma_f64(ec[3], za[1], zq[1]);
          dmma_f64(ec[4], za[1], zq[2]);
          dmma_f64(ec[5], za[2], zq[2]);
        }
        __syncwarp();
      }
      // E out: the 4 warps' partials in order, both triangles
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        s_epart[qd][(i * 2 + 0) * 32 + lane] = ec[i][0];
        s_epart[qd][(i * 2 + 1) * 32 + lane] = ec[i][1];
      }
      asm volatile("bar.sync 3, 128;" ::: "memory");
      if (qd == 0) {
        double* pe = direct ? a.E + (int64_t)c * H1 * H1 : part + (int64_t)item * part_stride + (int64_t)nh1 * D + D;
        const int g = lane >> 2, tq = lane & 3;
        const int tmi[6] = {0, 0, 0, 1, 1, 2}, tni[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
        for (int i = 0; i < 6; ++i)
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const double v = ((s_epart[0][(i * 2 + u) * 32 + lane] + s_epart[1][(i * 2 + u) * 32 + lane]) +
                              s_epart[2][(i * 2 + u) * 32 + lane]) + s_epart[3][(i * 2 + u) * 32 + lane];
            const int ei = 8 * tmi[i] + g, ej = 8 * tni[i] + 2 * tq + u;
            if (ei < H1 && ej < H1 && ei <= ej) {
              pe[ej * H1 + ei] = v;
              pe[ei * H1 + ej] = v;
            }
          }
      }
    } else {
      // ---- MMA issuer (warp 12, lane 0)
      const bool leader = lane == 0;
      const uint32_t id1 = idesc(HP, false);
      const uint32_t vb = sbase + L.off_V;
      uint32_t g = gp;
      for (int t = 0; t < T; ++t) {
        const uint32_t tt = ntile + t, zb = tt & 1u;
        if (tt >= 2) bwait(&s_zfree[zb], tt / 2);  // the epilogue is done with this Z buffer
        tfence_after();
        for (int p = 0; p < L.npair; ++p, ++g) {
          const int slot = static_cast<int>(g % kTPairs);
          {
            TC_T0();
            bwait(&s_full[slot], g / kTPairs + 1);
            TC_ACC(2);
          }
          tfence_after();
          if (leader && !(dbg & 1)) {
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              const int k = 2 * p + hf;
              if (k >= L.nch) break;
              const uint32_t ah = sbase + slot * kTPairBytes + hf * kTUnit, al = ah + 2 * kTUnit;
              const uint32_t bh = vb + (k * 2) * HP * 128, bl = bh + HP * 128;
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                const uint32_t o = kk * 32;
                const uint32_t acc = (k > 0 || kk > 0) ? 1u : 0u;
                const uint32_t dz = tmem + zb * HP;
                mma_ss(dz, desc(al + o, 16), desc(bh + o, 16), idesc_m(HP), acc);
                mma_ss(dz, desc(ah + o, 16), desc(bl + o, 16), idesc_m(HP), 1u);
                mma_ss(dz, desc(ah + o, 16), desc(bh + o, 16), idesc_m(HP), 1u);
              }
            }
            tcommit(&s_empty[slot]);
          }
          __syncwarp();
        }
        if (leader) tcommit(&s_zdone[zb]);
        __syncwarp();
        (void)id1;
      }
    }
    gp += static_cast<uint32_t>(T * L.npair);
    ntile += static_cast<uint32_t>(T);
  }
  tfence_before();
  __syncthreads();
  tfence_after();
  if (warp == kTMma) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
  if ((dbg & 4) && blockIdx.x == 0 && (tid == 0 || tid == kTEpi0 * 32 || tid == kTMma * 32))
    printf("stats_z %d: total %lld fill %lld zdone %lld full %lld\n", warp, clock64() - tstart, prof[0], prof[1],
           prof[2]);
}

// ---------------------------------------------------------------- kernel Y
// GEMM ii per tile: Y_v [D x N2] += [v]^T (MN-major A: a pair slot = 128
// dimensions) . [q zhat 2^(e_h - k_n)] (K-major B2, double-buffered, built by
// warps 8-11 from kernel Z's zhat while the previous tile multiplies); the
// fill warps also accumulate sq_v = sum q v^2 (fp32 per chunk, fp64 per warp
// and dimension).
template <int N2>
__global__ void __launch_bounds__(kTThreads, 1)
    k_stats_y(StatsArgs a, const float* __restrict__ xmax, const float* __restrict__ mumax,
              const float* __restrict__ vl1_g, const int* __restrict__ itemoff, int nh1, double* part,
              int64_t part_stride, const float* __restrict__ zin, int dbg) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t s_full[kTPairs], s_empty[kTPairs], s_b2ready[2], s_b2free[2], s_ydone;
  __shared__ uint32_t s_tmem;
  __shared__ int s_item;
  __shared__ float s_bmax[kTMma];
  __shared__ int s_colexp[32];
  long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long tstart = clock64();
  const Dims dm = a.dm;
  const int D = dm.D, H = dm.H, H1 = H + 1;
  const TcLayout L = tc_layout(D, H);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = su32(sm);
  int* s_row = reinterpret_cast<int*>(sm + L.off_row_y);
  double* s_q = reinterpret_cast<double*>(sm + L.off_q_y);
  int* s_k = reinterpret_cast<int*>(sm + L.off_k_y);
  float* s_sqw = reinterpret_cast<float*>(sm + L.off_sqw);
  if (tid == 0) {
    for (int i = 0; i < kTPairs; ++i) {
      binit(&s_full[i], 2 * kTFill);
      binit(&s_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      binit(&s_b2ready[i], 4);
      binit(&s_b2free[i], 1);
    }
    binit(&s_ydone, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kTMma) {  // Y_v: hi*hi at 0, corrections at 256 (npair x N2 <= 224 columns each)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&s_tmem)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tfence_before();
  __syncthreads();
  tfence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t tY = tmem, tYc = tmem + 256;
  const int total = __ldg(itemoff + dm.C);
  uint32_t gp = 0, ntile = 0, ny = 0;
  for (;;) {
    __syncthreads();
    if (tid == 0) s_item = a.qctr ? atomicAdd(a.qctr + 1, 1) : -1;
    __syncthreads();
    const int item = s_item;
    if (item < 0 || item >= total) break;
    const int c = find_item_t(itemoff, dm.C, item);
    const int r0 = a.off[c] + (item - itemoff[c]) * kTItemRows;
    const int nr = min(a.off[c + 1], r0 + kTItemRows) - r0;
    const int T = (nr + kTR - 1) / kTR;
    const bool direct = itemoff[c + 1] - itemoff[c] == 1;
    if (warp < kTMma) {
      item_rows(a, xmax, __ldg(mumax + c), r0, nr, s_row, s_q, s_k, s_bmax);
      for (int i = tid; i < kTFill * kTMaxChunks * 64; i += kTMma * 32) s_sqw[i] = 0.f;
      producers_all_sync();
      if (tid < N2) {  // B2's column scales from the bounds: |zhat_h| <= |V_h|_1 max_n bound_n
        float mm = 0.f;
        for (int w = 0; w < kTMma; ++w) mm = fmaxf(mm, s_bmax[w]);
        const float bnd = tid < H ? 1.01f * __ldg(vl1_g + (int64_t)c * 16 + tid) * mm * mm * p2(-13)
                                  : (tid == H ? 1.01f * mm * p2(-13) : 0.f);
        s_colexp[tid] = sexp(bnd);
      }
      producers_all_sync();
    }
    if (warp < kTFill) {
      TC_T0();
      fill_item<true>(a, L, c, nr, T, sbase, s_row, s_q, s_k, s_full, s_empty, gp, s_sqw, dbg, [](int) {});
      TC_ACC(0);
    } else if (warp < kTMma) {
      // ---- B2 builders (warps 8-11): thread = tile row
      const int r = (warp - kTEpi0) * 32 + lane;
      for (int t = 0; t < T; ++t) {
        const uint32_t tt = ntile + t, bb = tt & 1u;
        if (tt >= 2) {
          TC_T0();
          bwait(&s_b2free[bb], tt / 2);
          TC_ACC(1);
        }
        const int rt = t * kTR + r;
        const bool lv = rt < nr;
        const float* zi = zin + (int64_t)(r0 + (lv ? rt : 0)) * H;
        const float qs = lv ? static_cast<float>(s_q[rt]) : 0.f;
        const int kr = lv ? s_k[rt] : 0;
        const uint32_t b2 = sbase + L.off_B2 + bb * (2 * 2 * N2 * 128);
        const int kc = r >> 6, rl = r & 63;
#pragma unroll 4
        for (int h = 0; h < N2; ++h) {
          float b = 0.f;
          if (lv && h < H1) b = qs * (h < H ? __ldg(zi + h) : 1.f) * p2(s_colexp[h] - kr);
          __half bh, bl;
          split1(b, bh, bl);
          const uint32_t o = (kc * N2 + h) * 128 + (((rl >> 3) ^ (h & 7)) << 4) + (rl & 7) * 2;
          asm volatile("st.shared.b16 [%0], %1;" ::"r"(b2 + o), "h"(*reinterpret_cast<uint16_t*>(&bh)) : "memory");
          asm volatile("st.shared.b16 [%0], %1;" ::"r"(b2 + 2 * N2 * 128 + o), "h"(*reinterpret_cast<uint16_t*>(&bl))
                       : "memory");
        }
        fence_async();
        __syncwarp();
        if (lane == 0) barrive(&s_b2ready[bb]);
      }
    } else {
      // ---- MMA issuer
      const bool leader = lane == 0;
      const uint32_t id2 = idesc(N2, true);
      uint32_t g = gp;
      for (int t = 0; t < T; ++t) {
        const uint32_t tt = ntile + t, bb = tt & 1u;
        bwait(&s_b2ready[bb], tt / 2 + 1);
        tfence_after();
        const uint32_t b2 = sbase + L.off_B2 + bb * (2 * 2 * N2 * 128);
        for (int p = 0; p < L.npair; ++p, ++g) {
          const int slot = static_cast<int>(g % kTPairs);
          {
            TC_T0();
            bwait(&s_full[slot], g / kTPairs + 1);
            TC_ACC(2);
          }
          tfence_after();
          if (leader && !(dbg & 1)) {
            const uint32_t ah = sbase + slot * kTPairBytes, al = ah + 2 * kTUnit;
#pragma unroll
            for (int kk = 0; kk < kTR / 16; ++kk) {
              const uint32_t oa = kk * 2048;  // 16 tile rows = two 8-row groups
              const uint32_t bh = b2 + (kk >> 2) * N2 * 128 + (kk & 3) * 32, bl = bh + 2 * N2 * 128;
              const uint32_t acc = (t > 0 || kk > 0) ? 1u : 0u;
              // the small correction products in their own accumulator (the
              // tensor core's accumulation truncates)
              mma_ss(tYc + p * N2, desc(al + oa, kTUnit), desc(bh, 16), id2, acc);
              mma_ss(tYc + p * N2, desc(ah + oa, kTUnit), desc(bl, 16), id2, 1u);
              mma_ss(tY + p * N2, desc(ah + oa, kTUnit), desc(bh, 16), id2, acc);
            }
            tcommit(&s_empty[slot]);
          }
          __syncwarp();
        }
        if (leader) tcommit(&s_b2free[bb]);
        __syncwarp();
      }
      if (leader) tcommit(&s_ydone);
      __syncwarp();
    }
    // ---- item end: Y_v (warps 0-3: TMEM lanes = a pair's 128 dimensions) and sq_v
    ++ny;
    if (warp < kTMma) {
      bwait(&s_ydone, ny);
      tfence_after();
      if (warp < 4) {
        double* pp = direct ? nullptr : part + (int64_t)item * part_stride;
        for (int j = 0; j < L.npair; ++j) {
          const int d = j * 128 + warp * 32 + lane;
#pragma unroll
          for (int h0 = 0; h0 < N2; h0 += 8) {
            if (h0 >= H1) break;
            float y[8], yc[8];
            tld8(tY + (static_cast<uint32_t>(warp * 32) << 16) + j * N2 + h0, y);
            tld8(tYc + (static_cast<uint32_t>(warp * 32) << 16) + j * N2 + h0, yc);
            tld_wait();
            if (d < D) {
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int h = h0 + u;
                if (h >= H1) break;
                const double v = static_cast<double>(y[u] + yc[u]) * static_cast<double>(p2(-s_colexp[h]));
                if (direct) a.Y[((int64_t)c * H1 + h) * D + d] = v;
                else pp[(int64_t)h * D + d] = v;
              }
            }
          }
        }
      }
      producers_all_sync();
      for (int d = tid; d < D; d += kTMma * 32) {
        double v = 0.0;
        for (int w = 0; w < kTFill; ++w) v += static_cast<double>(s_sqw[(int64_t)w * kTMaxChunks * 64 + d]);
        if (direct) a.sq[(int64_t)c * D + d] = v;
        else part[(int64_t)item * part_stride + (int64_t)nh1 * D + d] = v;
      }
      tfence_before();
    }
    gp += static_cast<uint32_t>(T * L.npair);
    ntile += static_cast<uint32_t>(T);
  }
  tfence_before();
  __syncthreads();
  tfence_after();
  if (warp == kTMma) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  if ((dbg & 4) && blockIdx.x == 0 && (tid == 0 || tid == kTEpi0 * 32 || tid == kTMma * 32))
    printf("stats_y %d: total %lld fill %lld b2free %lld full %lld\n", warp, clock64() - tstart, prof[0], prof[1],
           prof[2]);
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
  const TcLayout L = tc_layout(dm.D, dm.H);
  return dm.D % 4 == 0 && dm.D <= kTMaxChunks * 64 && dm.H >= 1 && dm.H <= 16 &&
         L.total_z <= 227 * 1024 - 4096 && L.total_y <= 227 * 1024 - 4096;  // (+ static)
}
int stats_tc_rows() { return kTItemRows; }

// two passes over the K-pairs (vmfa_stats_tc.cu header): k_stats_z (zhat to
// zbuf, E), then k_stats_y (Y_v, sq_v); qctr[0], qctr[1] their work queues
cudaError_t launch_stats_tc(const StatsArgs& a, const float* xmax, const float* mumax, const int* itemoff, int nh1,
                            double* part, int64_t part_stride, cudaStream_t s) {
  if (!a.vimg || !a.vexp || !a.vl1 || !a.zbuf || !a.qctr) return cudaErrorInvalidValue;
  const TcLayout L = tc_layout(a.dm.D, a.dm.H);
  static const int dbg = [] {
    const char* v = std::getenv("VMFA_STATS_TC_DBG");  // diagnostics: 1 skip MMAs, 2 skip row loads, 4 cycles
    return v ? std::atoi(v) : 0;
  }();
  if (cudaError_t e = cudaMemsetAsync(a.qctr, 0, 2 * sizeof(int), s); e != cudaSuccess) return e;
  ensure_dyn_smem(reinterpret_cast<const void*>(k_stats_z<16>), L.total_z);
  k_stats_z<16><<<sm_count(), kTThreads, L.total_z, s>>>(a, xmax, mumax, static_cast<const unsigned char*>(a.vimg),
                                                          a.vexp, itemoff, nh1, part, part_stride, a.zbuf, dbg);
  auto go = [&](auto kern) {
    ensure_dyn_smem(reinterpret_cast<const void*>(kern), L.total_y);
    kern<<<sm_count(), kTThreads, L.total_y, s>>>(a, xmax, mumax, a.vl1, itemoff, nh1, part, part_stride, a.zbuf, dbg);
  };
  if (L.N2 == 16) go(k_stats_y<16>);
  else if (L.N2 == 32) go(k_stats_y<32>);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace vmfa_b200
