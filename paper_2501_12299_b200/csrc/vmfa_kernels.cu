// vmfa_kernels.cu — sm_100a kernels of one v-MFA EM iteration.
//
// Design: the E-step scoring is organised around ANCHOR BLOCKS.
// For every component a, the points n with a in K(n) (the inverted K map, a
// stable counting sort) need every component of g_a, because
// S(n) = U_{a in K(n)} g_a U {r_n} (estep.cpp:83-101). A block (64 gathered
// rows of a) x (g_a) is therefore dense: the rows are staged once in shared
// memory and every component of g_a is scored against them, so each gathered
// row is read from HBM/L2 C' times per iteration instead of |S(n)| times.
// Duplicates across anchors are scored but dropped by k_select, which also
// reproduces the reference's insertion order, tie rules and counters exactly.
#include <algorithm>
#include <mutex>
#include <utility>
#include <vector>
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "vmfa_kernels.cuh"
#include "vmfa_rng.hpp"

namespace vmfa_b200 {

namespace {

constexpr double kLog2Pi = 1.8378770664093453;  // numerics.hpp:10
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ int find_item(const int* itemoff, int C, int item) {
  // largest c with itemoff[c] <= item (itemoff is non-decreasing, size C+1)
  int lo = 0, hi = C;  // invariant itemoff[lo] <= item < itemoff[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(itemoff + mid) <= item) lo = mid;
    else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------- small utilities
__global__ void k_iota(int* v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = static_cast<int>(i);
}
__global__ void k_fill_i32(int* v, int64_t n, int value) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = value;
}
__global__ void k_keys_from_i32(const int* src, unsigned* keys, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = static_cast<unsigned>(src[i]);
}
// off[c] = first index i with sorted[i] >= c (lower bound); off[C] = #keys < C.
__global__ void k_offsets_sorted(const unsigned* sorted, int64_t n, int C, int* off) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c <= C; c += gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (sorted[mid] < static_cast<unsigned>(c)) lo = mid + 1;
      else hi = mid;
    }
    off[c] = static_cast<int>(lo);
  }
}
__global__ void k_hist(const unsigned* keys, int64_t n, int C, int* cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned k = keys[i];
    if (k < static_cast<unsigned>(C)) atomicAdd(cnt + k, 1);
  }
}
// CSR offsets from sorted keys in [0, C] by one pass over the keys:
// off[c] = #keys < c; row i writes the c in (key[i-1], key[i]] (the
// intervals partition [0, C], each offset is written once)
__global__ void k_offsets_scan(const unsigned* sorted, int64_t n, int C, int* off) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
    const int prev = i > 0 ? static_cast<int>(sorted[i - 1]) : -1;
    const int cur = i < n ? static_cast<int>(sorted[i]) : C;
    for (int c = prev + 1; c <= cur; ++c) off[c] = static_cast<int>(i);
  }
}
// items = exclusive scan of max(min1, ceil((off[c+1] - off[c]) / rows)) over
// c < C (items[C] = total), one 1024-thread block (C is at most ~10^5)
__global__ void __launch_bounds__(1024) k_items_scan(const int* off, int C, int rows, int min1, int* items) {
  __shared__ int s_warp[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = (C + 1 + 1023) / 1024;
  const int c0 = tid * per, c1 = min(C + 1, c0 + per);
  int sum = 0;
  for (int c = c0; c < c1; ++c) sum += c < C ? max(min1, (off[c + 1] - off[c] + rows - 1) / rows) : 0;
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = s_warp[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(kFull, w, o);
      if (lane >= o) w += t;
    }
    s_warp[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  int run = incl - sum + (warp > 0 ? s_warp[warp - 1] : 0);
  for (int c = c0; c < c1; ++c) {
    items[c] = run;
    run += c < C ? max(min1, (off[c + 1] - off[c] + rows - 1) / rows) : 0;
  }
}
__global__ void k_chunks_from_off(const int* off, int C, int rows, int min1, int* chunks) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c <= C; c += gridDim.x * blockDim.x) {
    if (c == C) {
      chunks[c] = 0;
      continue;
    }
    const int n = off[c + 1] - off[c];
    chunks[c] = max(min1, (n + rows - 1) / rows);
  }
}
__global__ void k_chunks(const int* cnt, int C, int rows, int* chunks) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c <= C; c += gridDim.x * blockDim.x)
    chunks[c] = c < C ? (cnt[c] + rows - 1) / rows : 0;
}

// ---------------------------------------------------------------- K0: extra candidate
// r_n = uniform_component(seed, iteration, n_global, C) (rng.hpp:91-98,
// estep.cpp:259-260). rkey = r_n if it is not already in U_{a in K(n)} g_a,
// else the sentinel C (the reference pushes it and the epoch-stamp drops it).
__global__ void k_extra(Dims dm, const int* __restrict__ K, const int* __restrict__ g,
                        const int* __restrict__ gcnt, const unsigned long long* __restrict__ sit, int* rx,
                        unsigned* rkey) {
  // (seed, E-step index) from device memory: one captured CUDA graph serves every iteration
  const uint64_t seed = sit[0], it = sit[1];
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < dm.N; n += (int64_t)gridDim.x * blockDim.x) {
    const int r = extra_candidate(seed, it, static_cast<uint64_t>(dm.n0 + n), dm.C);
    bool dup = false;
    for (int j = 0; j < dm.Cp && !dup; ++j) {
      const int a = K[n * dm.Cp + j];
      const int m = gcnt[a];
      for (int i = 0; i < m; ++i)
        if (g[(int64_t)a * dm.G + i] == r) {
          dup = true;
          break;
        }
    }
    rx[n] = r;
    rkey[n] = dup ? static_cast<unsigned>(dm.C) : static_cast<unsigned>(r);
  }
}

// ---------------------------------------------------------------- K2: scoring (FFMA)
// One warp scores one component against the 64 staged rows of the item: lane l
// owns rows 2l and 2l+1; per dimension it reads the row pair from the
// transposed smem tile and the component's packed parameter row (broadcast
// ld.global.nc), computing v = x - mu, diag += v^2/psi and y = W^T v in fp32.
// l(n,c) = kconst_c - 0.5 (diag - |y|^2), combined in fp64 (model.cpp:87-94).
template <int HC>
__device__ __forceinline__ void score_pair_rows(const float* __restrict__ xs, int D, int H,
                                                int Hc, int HP, const float* __restrict__ Pc,
                                                int lane, float& diag0, float& diag1,
                                                float& yy0, float& yy1) {
  diag0 = diag1 = yy0 = yy1 = 0.f;
  for (int h0 = 0; h0 < Hc; h0 += HC) {
    float a0[HC], a1[HC];
#pragma unroll
    for (int h = 0; h < HC; ++h) a0[h] = a1[h] = 0.f;
    const bool first = (h0 == 0);
#pragma unroll 2
    for (int d = 0; d < D; ++d) {
      const float2 xv = *reinterpret_cast<const float2*>(xs + d * kXsStride + 2 * lane);
      const float* pd = Pc + (int64_t)d * HP;
      const float2 mp = __ldg(reinterpret_cast<const float2*>(pd + Hc));
      const float v0 = xv.x - mp.x, v1 = xv.y - mp.x;
      if (first) {
        diag0 = fmaf(v0 * mp.y, v0, diag0);
        diag1 = fmaf(v1 * mp.y, v1, diag1);
      }
#pragma unroll
      for (int h = 0; h < HC; h += 4) {
        const float4 w = __ldg(reinterpret_cast<const float4*>(pd + h0 + h));
        a0[h + 0] = fmaf(w.x, v0, a0[h + 0]);
        a1[h + 0] = fmaf(w.x, v1, a1[h + 0]);
        a0[h + 1] = fmaf(w.y, v0, a0[h + 1]);
        a1[h + 1] = fmaf(w.y, v1, a1[h + 1]);
        a0[h + 2] = fmaf(w.z, v0, a0[h + 2]);
        a1[h + 2] = fmaf(w.z, v1, a1[h + 2]);
        a0[h + 3] = fmaf(w.w, v0, a0[h + 3]);
        a1[h + 3] = fmaf(w.w, v1, a1[h + 3]);
      }
    }
#pragma unroll
    for (int h = 0; h < HC; ++h) {
      yy0 = fmaf(a0[h], a0[h], yy0);
      yy1 = fmaf(a1[h], a1[h], yy1);
    }
  }
  (void)H;
}

template <int MODE, int HC>
__global__ void __launch_bounds__(kScoreThreads)
k_score(ScoreArgs a) {
  extern __shared__ __align__(16) float xs[];  // [D][kXsStride]
  __shared__ int s_n[kScoreRows];
  __shared__ int s_e[kScoreRows];
  const Dims dm = a.dm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int total = __ldg(a.itemoff + dm.C);
  for (int item = blockIdx.x; item < total; item += gridDim.x) {
    const int c = find_item(a.itemoff, dm.C, item);
    const int row0 = __ldg(a.off + c) + (item - __ldg(a.itemoff + c)) * kScoreRows;
    const int nrows = min(kScoreRows, __ldg(a.off + c + 1) - row0);
    if (tid < kScoreRows) {
      int e = -1, n = -1;
      if (tid < nrows) {
        e = __ldg(a.ent + row0 + tid);
        n = MODE == kModeExtra ? e : e / dm.Cp;
      }
      s_e[tid] = e;
      s_n[tid] = n;
    }
    __syncthreads();
    // gather rows, transposed into xs[d][r] (coalesced global reads along d)
    for (int r = warp; r < kScoreRows; r += kScoreThreads / 32) {
      const int n = s_n[r];
      const float* xr = a.X + (int64_t)(n < 0 ? 0 : n) * dm.D;
      for (int d = lane; d < dm.D; d += 32) xs[d * kXsStride + r] = n < 0 ? 0.f : __ldg(xr + d);
    }
    __syncthreads();
    const int ncomp = MODE == kModeAnchor ? __ldg(a.gcnt + c) : 1;
    for (int ci = warp; ci < ncomp; ci += kScoreThreads / 32) {
      const int comp = MODE == kModeAnchor ? __ldg(a.g + (int64_t)c * dm.G + ci) : c;
      const float* Pc = a.P + (int64_t)comp * dm.D * a.L.HP;
      float d0, d1, y0, y1;
      score_pair_rows<HC>(xs, dm.D, dm.H, a.L.Hc, a.L.HP, Pc, lane, d0, d1, y0, y1);
      const double kc = __ldg(a.kconst + comp);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int r = 2 * lane + k;
        if (r >= nrows) continue;
        const double diag = k == 0 ? d0 : d1, yy = k == 0 ? y0 : y1;
        const float lj = static_cast<float>(kc - 0.5 * (diag - yy));
        const int e = s_e[r];
        if (MODE == kModeAnchor) {
          const int n = e / dm.Cp, j = e - n * dm.Cp;
          a.out[(int64_t)n * dm.SL + j * dm.G + ci] = lj;
        } else if (MODE == kModeExtra) {
          a.out[(int64_t)e * dm.SL + dm.Cp * dm.G] = lj;
        } else {
          a.out[e] = lj;
        }
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- K3: selection (warp per row)
// Reconstructs S(n) in the reference's insertion order (slot s = j*G + i for
// g_{K(n)[j]}[i], then the extra), keeps the first occurrence of each component
// (epoch-stamp dedup, estep.cpp:83-101), selects the top-C' by (l desc, index
// asc) (estep.cpp:103-122), labels the row by the first strict maximum over the
// ascending K row (estep.cpp:157-166) and computes the fp64 responsibilities
// and LSE of block 4 (estep.cpp:316-335).
// A component scored by several anchors keeps the value of its most accurate
// slot: the anchor-centred expansion of (x - mu_q) around mu_a loses
// sum (x - mu_a)^2 / psi_q relative precision, so a self slot (q == a: the
// expansion is exact, delta = 0) or the uncovered extra (one-component pass)
// wins, else the anchor closest to x (largest own log-joint l(n, a)).
struct Cand {
  float l;
  int c;
  int slot;
  int valid;
};
__device__ __forceinline__ bool better(const Cand& x, const Cand& y) {
  if (x.valid != y.valid) return x.valid > y.valid;
  if (x.l != y.l) return x.l > y.l;
  return x.c < y.c;
}

// Order-preserving 64-bit key: larger key = larger l, ties -> smaller index.
__device__ __forceinline__ unsigned long long sel_key(float l, int c) {
  unsigned u = __float_as_uint(l);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);  // monotone float -> uint
  return (static_cast<unsigned long long>(u) << 32) | static_cast<unsigned>(0x7fffffff - c);
}

template <int NS>
__global__ void __launch_bounds__(256) k_select(SelectArgs a) {
  // per-warp bitmap of the components already seen in earlier slot rounds
  // (first-occurrence dedup across rounds; bits are cleared after each row)
  extern __shared__ unsigned s_seen[];
  const Dims dm = a.dm;
  const int lane = threadIdx.x & 31;
  const int W = (dm.C + 31) >> 5;
  for (int i = threadIdx.x; i < W * (blockDim.x >> 5); i += blockDim.x) s_seen[i] = 0u;
  __syncthreads();
  unsigned* seen = s_seen + (threadIdx.x >> 5) * W;
  // per warp: own log-joint of each anchor j (its self slot) and its rank, <= 8 anchors
  float* qual = reinterpret_cast<float*>(s_seen + W * (blockDim.x >> 5)) + (threadIdx.x >> 5) * 8;
  int* qrank = reinterpret_cast<int*>(s_seen + W * (blockDim.x >> 5)) + 64 + (threadIdx.x >> 5) * 8;
  // per warp: hash of the row's scored components -> best (rank, slot)
  constexpr int kHB = NS <= 1 ? 6 : NS <= 2 ? 7 : NS <= 4 ? 8 : 9;
  constexpr unsigned kHS = 1u << kHB;
  int* hkey = reinterpret_cast<int*>(s_seen + W * (blockDim.x >> 5)) + 128 + (threadIdx.x >> 5) * (2 * kHS);
  unsigned* hval = reinterpret_cast<unsigned*>(hkey) + kHS;
  if constexpr (NS > 2) {  // (the table exists only where it is used)
    for (int i = lane; i < static_cast<int>(kHS); i += 32) hkey[i] = -1, hval[i] = 0u;
    __syncwarp();
  }
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int CpG = dm.Cp * dm.G;
  const float invG = 1.0f / static_cast<float>(dm.G);
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int64_t n = warp0; n < dm.N; n += nwarps) {
    int comp[NS];
    bool uniq[NS];
    float lj[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const int s = k * 32 + lane;
      int cmp = -1;
      if (s < CpG) {
        // s / G exactly: (s + 0.5) / G stays >= 0.5 / G away from an integer
        const int j = __float2int_rz((static_cast<float>(s) + 0.5f) * invG), i = s - j * dm.G;
        const int an = a.K[n * dm.Cp + j];
        if (i < a.gcnt[an]) cmp = a.g[(int64_t)an * dm.G + i];
      } else if (s == CpG) {
        cmp = a.rx[n];
      }
      comp[k] = cmp;
    }
    // first-occurrence dedup in slot order (s = k*32 + lane): within a round by
    // __match_any_sync (keep the lowest lane), across rounds by the bitmap
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const unsigned m = __match_any_sync(kFull, comp[k]);
      bool u = comp[k] >= 0 && (m & lt_mask) == 0u;
      if (k > 0 && u) u = ((seen[comp[k] >> 5] >> (comp[k] & 31)) & 1u) == 0u;
      uniq[k] = u;
      if (k + 1 < NS) {
        __syncwarp();
        if (u) atomicOr(&seen[comp[k] >> 5], 1u << (comp[k] & 31));
        __syncwarp();
      }
    }
    __syncwarp();  // the last round's bitmap reads precede the clearing
#pragma unroll
    for (int k = 0; k + 1 < NS; ++k)
      if (uniq[k]) atomicAnd(&seen[comp[k] >> 5], ~(1u << (comp[k] & 31)));
    // slot values; the extra slot holds a value only when it is not a
    // duplicate (k_extra leaves covered extras unscored)
    float pri[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const int s = k * 32 + lane;
      float v = -INFINITY;
      const bool scored = comp[k] >= 0 && (s < CpG || uniq[k]);
      if (scored) {
        v = a.LJ[n * dm.SL + s];
        if (v != v) v = -INFINITY;  // NaN ranks last (reference comparator undefined)
      }
      lj[k] = v;
      pri[k] = -INFINITY;
      if (s < CpG && comp[k] >= 0) {
        const int j = __float2int_rz((static_cast<float>(s) + 0.5f) * invG);
        if (comp[k] == a.K[n * dm.Cp + j]) {
          qual[j] = v;
          pri[k] = INFINITY;
        }
      } else if (s == CpG && scored) {
        pri[k] = INFINITY;
      }
    }
    __syncwarp();
    bool dups = false;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const int s = k * 32 + lane;
      if (s < CpG && comp[k] >= 0 && pri[k] != INFINITY)
        pri[k] = qual[__float2int_rz((static_cast<float>(s) + 0.5f) * invG)];
      dups |= comp[k] >= 0 && !uniq[k];
    }
    // the first occurrence takes the value of the best slot of its component:
    // the largest priority, the smallest slot on a tie. Only duplicate slots
    // can beat a first occurrence, so they alone are visited (warp-uniform
    // loop over their ballot); priorities travel as ranks packed with the
    // component (anchor j: #{j' : qual[j'] < qual[j]}, equal values equal
    // ranks, -inf 0 like an unscored slot, +inf 15), the value is fetched once
    if (__any_sync(kFull, dups)) {
      if (lane < dm.Cp) {
        const float qj = qual[lane];
        int r = 0;
        for (int j2 = 0; j2 < dm.Cp; ++j2) r += qual[j2] < qj;
        qrank[lane] = r;
      }
      __syncwarp();
      int bs[NS];
      if constexpr (NS <= 2) {
        // NS <= 2 (at most 64 slots): only duplicate slots can beat a first
        // occurrence, so they alone are visited (warp-uniform loop over their
        // ballot), ranks packed with the component in one 32-bit shuffle
        unsigned pk[NS];
        int br[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) {
          const int s = k * 32 + lane;
          int rk = pri[k] == INFINITY ? 15 : 0;
          if (s < CpG && comp[k] >= 0 && pri[k] != INFINITY)
            rk = qrank[__float2int_rz((static_cast<float>(s) + 0.5f) * invG)];
          pk[k] = comp[k] >= 0 ? (static_cast<unsigned>(comp[k]) << 4) | static_cast<unsigned>(rk) : 0xffffffffu;
          br[k] = rk;
          bs[k] = s;
        }
#pragma unroll
        for (int k2 = 0; k2 < NS; ++k2) {
          unsigned dm2 = __ballot_sync(kFull, comp[k2] >= 0 && !uniq[k2]);
          while (dm2) {
            const int t = __ffs(dm2) - 1;
            dm2 &= dm2 - 1;
            const unsigned o = __shfl_sync(kFull, pk[k2], t);
            const int orank = static_cast<int>(o & 15u);
#pragma unroll
            for (int k = 0; k < NS; ++k)
              if (uniq[k] && static_cast<int>(o >> 4) == comp[k] && orank > br[k]) {
                br[k] = orank;
                bs[k] = k2 * 32 + t;
              }
          }
        }
      } else {
        // every scored slot posts (rank, slot) under its component in a small
        // per-warp hash (linear probing, <= 50 % load): the maximum of
        // rank << 8 | (255 - slot) is the best slot, the smallest one on a tie
        int pos[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) {
          const int s = k * 32 + lane;
          bs[k] = s;
          pos[k] = -1;
          // (a duplicate extra slot is unscored and never wins)
          if (comp[k] < 0 || (s >= CpG && !uniq[k])) continue;
          int rk = pri[k] == INFINITY ? 15 : 0;
          if (s < CpG && pri[k] != INFINITY) rk = qrank[__float2int_rz((static_cast<float>(s) + 0.5f) * invG)];
          unsigned h = (static_cast<unsigned>(comp[k]) * 2654435761u) >> (32 - kHB);
          for (;;) {
            const int old = atomicCAS(&hkey[h], -1, comp[k]);
            if (old == -1 || old == comp[k]) break;
            h = (h + 1u) & (kHS - 1);
          }
          pos[k] = static_cast<int>(h);
          atomicMax(&hval[h], (static_cast<unsigned>(rk) << 8) | static_cast<unsigned>(255 - s));
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < NS; ++k)
          if (uniq[k]) bs[k] = 255 - static_cast<int>(hval[pos[k]] & 255u);
        __syncwarp();
#pragma unroll
        for (int k = 0; k < NS; ++k)
          if (pos[k] >= 0) hkey[pos[k]] = -1, hval[pos[k]] = 0u;
      }
      float ljw[NS];
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        float w = lj[k];
#pragma unroll
        for (int k2 = 0; k2 < NS; ++k2) {
          const float ov = __shfl_sync(kFull, lj[k2], bs[k] & 31);
          if (k2 == (bs[k] >> 5)) w = ov;
        }
        ljw[k] = w;
      }
#pragma unroll
      for (int k = 0; k < NS; ++k) lj[k] = ljw[k];
    }
#pragma unroll
    for (int k = 0; k < NS; ++k)
      if (!uniq[k]) lj[k] = 0.f;
    __syncwarp();
    // compaction of the retained joints (reference layout, insertion order)
    int base = 0;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const unsigned b = __ballot_sync(kFull, uniq[k]);
      if (uniq[k]) {
        const int pos = base + __popc(b & lt_mask);
        a.ret_idx[n * dm.stride + pos] = comp[k];
        a.ret_lj[n * dm.stride + pos] = lj[k];
      }
      base += __popc(b);
    }
    const int m = base;
    // top-C' by (l desc, index asc) on packed keys (0 = no candidate); round
    // r's winner is held by lane r
    unsigned long long key[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) key[k] = uniq[k] ? sel_key(lj[k], comp[k]) : 0ull;
    int myc = 0;
    float myl = -INFINITY;
    int best_c = 0;
    float best_l = -INFINITY;
    for (int r = 0; r < dm.Cp; ++r) {
      unsigned long long best = 0ull;
#pragma unroll
      for (int k = 0; k < NS; ++k) best = key[k] > best ? key[k] : best;
      // warp max of the 64-bit keys: high words by a redux, low words among the ties
      const unsigned hi = __reduce_max_sync(kFull, static_cast<unsigned>(best >> 32));
      const unsigned lo = __reduce_max_sync(
          kFull, static_cast<unsigned>(best >> 32) == hi ? static_cast<unsigned>(best) : 0u);
      best = (static_cast<unsigned long long>(hi) << 32) | lo;
      if (best == 0ull) {
        if (lane == 0) atomicOr(a.status, 1);  // InsufficientCandidates
        continue;
      }
      const int c = 0x7fffffff - static_cast<int>(best & 0xffffffffu);
      unsigned u = static_cast<unsigned>(best >> 32);
      u = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
      const float l = __uint_as_float(u);
      if (lane == r) myc = c, myl = l;
      // label (estep.cpp:157-166): the first member of the sorted K replaced
      // only by a strictly larger l = the largest l, ties to the smaller index
      if (r == 0) best_c = c, best_l = l;
#pragma unroll
      for (int k = 0; k < NS; ++k)
        if (key[k] == best) key[k] = 0ull;  // unique keys: only the owner matches
    }
    // K sorted ascending by component (estep.cpp:121): rank of member `lane`
    int rank = 0;
    for (int j = 0; j < dm.Cp; ++j) rank += __shfl_sync(kFull, myc, j) < myc;
    // block 4: fp64 log-sum-exp and responsibilities (numerics.hpp:15-22); lane j
    // evaluates member j's exponential, the terms are summed in K order
    const double mx = static_cast<double>(best_l);
    const double term = (lane < dm.Cp && isfinite(mx)) ? exp(static_cast<double>(myl) - mx) : 0.0;
    double l = mx;
    if (isfinite(mx)) {
      double s2 = 0.0;
      for (int k = 0; k < dm.Cp; ++k) {
        const int src = __ffs(__ballot_sync(kFull, lane < dm.Cp && rank == k)) - 1;
        s2 += __shfl_sync(kFull, term, src < 0 ? 0 : src);
      }
      l = mx + log(s2);
    }
    if (lane < dm.Cp) {
      a.K[n * dm.Cp + rank] = myc;
      a.resp[n * dm.Cp + rank] = exp(static_cast<double>(myl) - l);
    }
    if (lane == 0) {
      a.labels[n] = best_c;
      a.lablj[n] = best_l;
      a.lse[n] = l;
      a.ret_cnt[n] = m;
    }
  }
}

// ---------------------------------------------------------------- K4: g update (CTA per component)
// Block 3 (estep.cpp:286-312): for n in I_c and each retained ct != c with
// pi_ct > 0, accumulate value = (l(n,c) - log pi_c) - (l(n,ct) - log pi_ct)
// [kl] or -l(n,ct) [euclid] into (sum, count) per ct; then update_g
// (estep.cpp:204-220): g_c = {c} U the G-1 smallest (sum/count, ct), sorted.
// Sums are exact fixed-point integers (split hi/lo int64), so the
// accumulation order -- and the number of ranks -- cannot change them.
// value = hi 2^-10 + lo 2^-30, lo in [0, 2^20): |value| saturates at 2^40
// (1.1e12; a term's hi stays below 2^50, so a key's sum overflows only past
// 2^53 in total, i.e. ~8e6 terms of 1e9 each), and lo sums overflow only past
// 2^43 terms. The resolution 2^-30 is far below the fp32 log-joints the
// values are formed from (tests/test_multirank_gloo.py restates the encoding,
// tests/test_gpu_parity.py drives values past the saturation bound).
__device__ __forceinline__ void to_fixed(double v, long long& hi, long long& lo) {
  const double kMax = 1099511627776.0;  // 2^40
  if (!(v == v)) v = kMax;
  v = fmin(fmax(v, -kMax), kMax);
  const double y = v * 1024.0;  // 2^10
  const double f = floor(y);
  hi = static_cast<long long>(f);
  lo = static_cast<long long>((y - f) * 1048576.0);  // 2^20
}
__device__ __forceinline__ double from_fixed(long long hi, long long lo) {
  return static_cast<double>(hi) * (1.0 / 1024.0) + static_cast<double>(lo) * (1.0 / 1073741824.0);
}
constexpr int kGupdBatch = 4;  // points in flight per warp in k_gupdate
constexpr int kGupdProbes = 32;  // probe limit of a dense-rows item's hash
__device__ __forceinline__ unsigned hash_key(int k) { return static_cast<unsigned>(k) * 2654435761u; }
// Exact 64-bit integer add into shared memory from two native 32-bit atomics
// (a 64-bit shared atomicAdd compiles to a CAS spin loop on sm_100): the low
// word's add returns its old value, so its wrap-around is detected exactly
// and carried into the high word. The pair is read only after a barrier.
__device__ __forceinline__ void smem_add_u64(unsigned long long* addr, unsigned long long v) {
  unsigned* w = reinterpret_cast<unsigned*>(addr);
  const unsigned lo = static_cast<unsigned>(v), hi = static_cast<unsigned>(v >> 32);
  const unsigned old = atomicAdd(w, lo);
  const unsigned up = hi + (old + lo < old ? 1u : 0u);
  if (up) atomicAdd(w + 1, up);
}

struct KeyMin {
  double v;
  int c;
};
__device__ __forceinline__ bool kless(const KeyMin& x, const KeyMin& y) {
  if (x.v != y.v) return x.v < y.v;
  return x.c < y.c;
}

__device__ __forceinline__ void sort_small(int* v, int m) {
  for (int i = 1; i < m; ++i) {
    const int x = v[i];
    int j = i - 1;
    while (j >= 0 && v[j] > x) {
      v[j + 1] = v[j];
      --j;
    }
    v[j + 1] = x;
  }
}

// Items are (component c, chunk of <= a.pts_per_item points of I_c). A
// component with one item accumulates and selects in shared memory; chunks of
// larger components (and every component in exchange mode) add their exact
// integer partial sums into row c of the dense table xc (order-independent),
// and k_gselect_dense selects from the rows.
__global__ void __launch_bounds__(kGupdThreads) k_gupdate(GupdArgs a, int capmax) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  long long* t_hi = reinterpret_cast<long long*>(smem_raw);
  long long* t_lo = t_hi + capmax;
  int* t_key = reinterpret_cast<int*>(t_lo + capmax);
  int* t_cnt = t_key + capmax;
  __shared__ KeyMin red[kGupdThreads / 32];
  __shared__ int red_i[kGupdThreads / 32];
  __shared__ int s_sel[64];
  __shared__ int s_nsel, s_win;
  const Dims dm = a.dm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = kGupdThreads / 32;
  const int64_t CC = (int64_t)dm.C * dm.C;
  // capmax < 0: the dense table (one (cnt, hi, lo) entry per component,
  // indexed by c~, no probing) lives in shared memory (C <= kGupdDenseMax);
  // otherwise the per-CTA global tables back the hash
  // (shared layout: hi [C] u64 | lo [C] u64 | cnt [C] u32 -- 20 bytes per component)
  const bool sdense = capmax < 0;
  long long* g_cnt = a.gt_cnt + (int64_t)blockIdx.x * dm.C;
  long long* g_hi = sdense ? reinterpret_cast<long long*>(smem_raw) : a.gt_hi + (int64_t)blockIdx.x * dm.C;
  long long* g_lo = sdense ? g_hi + dm.C : a.gt_lo + (int64_t)blockIdx.x * dm.C;
  unsigned* d_cnt = reinterpret_cast<unsigned*>(smem_raw + 16 * static_cast<size_t>(dm.C));
  const int total = a.itemoff[dm.C];
  for (int item = blockIdx.x; item < total; item += gridDim.x) {
    const int c = find_item(a.itemoff, dm.C, item);
    const int nitems = a.itemoff[c + 1] - a.itemoff[c];
    const int p0 = a.part_off[c] + (item - a.itemoff[c]) * a.pts_per_item;
    const int p1 = min(a.part_off[c + 1], p0 + a.pts_per_item);
    const int npts = max(0, p1 - p0);
    const bool to_rows = a.exchange || nitems > 1 || a.force_rows || a.list;
    const long long bound = llmin((long long)dm.C - 1, (long long)npts * (dm.stride - 1));
    int cap = 32;
    bool use_smem;
    if (sdense) {
      use_smem = false;
    } else if (to_rows && (a.xc || a.list)) {  // small table sized for the typical key count; overflow adds into row c of xc (or the list)
      while (cap < 2 * bound && cap < min(capmax, kGupdRowsCap)) cap <<= 1;
      use_smem = true;
    } else {
      while (cap < 2 * bound && cap < 2 * capmax) cap <<= 1;
      use_smem = cap <= capmax;
    }
    if (npts > 0) {
      if (use_smem) {
        for (int i = tid; i < cap; i += kGupdThreads) {
          t_key[i] = -1;
          t_cnt[i] = 0;
          t_hi[i] = 0;
          t_lo[i] = 0;
        }
      } else {
        for (int i = tid; i < dm.C; i += kGupdThreads) {
          if (sdense) d_cnt[i] = 0u;
          else g_cnt[i] = 0;
          g_hi[i] = 0;
          g_lo[i] = 0;
        }
      }
      __syncthreads();
      const double logpi_c = a.logpi[c];
      // kGupdBatch points per warp step: every load of the batch is issued
      // before any is consumed (the per-point chains are latency-bound)
      for (int pb = p0 + warp; pb < p1; pb += nw * kGupdBatch) {
        int nn[kGupdBatch], mm[kGupdBatch];
        float lb[kGupdBatch];
#pragma unroll
        for (int u = 0; u < kGupdBatch; ++u) {
          const int p = pb + u * nw;
          nn[u] = p < p1 ? a.part_ent[p] : -1;
        }
#pragma unroll
        for (int u = 0; u < kGupdBatch; ++u) {
          mm[u] = nn[u] >= 0 ? a.ret_cnt[nn[u]] : 0;
          lb[u] = nn[u] >= 0 ? a.lablj[nn[u]] : 0.f;
        }
        int mmax = 0;
#pragma unroll
        for (int u = 0; u < kGupdBatch; ++u) mmax = max(mmax, mm[u]);
        for (int jb = 0; jb < mmax; jb += 32) {
          const int j = jb + lane;
          int cts[kGupdBatch];
          float lts[kGupdBatch];
#pragma unroll
          for (int u = 0; u < kGupdBatch; ++u) {
            cts[u] = j < mm[u] ? a.ret_idx[(int64_t)nn[u] * dm.stride + j] : -1;
            lts[u] = j < mm[u] ? a.ret_lj[(int64_t)nn[u] * dm.stride + j] : 0.f;
          }
          double lps[kGupdBatch];
#pragma unroll
          for (int u = 0; u < kGupdBatch; ++u) lps[u] = (cts[u] >= 0 && cts[u] != c) ? a.logpi[cts[u]] : -INFINITY;
#pragma unroll
          for (int u = 0; u < kGupdBatch; ++u) {
          const int ct = cts[u];
          const double lpt = lps[u];
          if (ct < 0 || ct == c || lpt == -INFINITY) continue;  // pi_ct <= 0 (estep.cpp:301)
          const double cond_c = static_cast<double>(lb[u]) - logpi_c;
          const double lt = static_cast<double>(lts[u]);
          const double v = a.mode == 0 ? cond_c - (lt - lpt) : -lt;
          long long hi, lo;
          to_fixed(v, hi, lo);
          if (use_smem) {
            // linear probing; an item adding into the dense rows stops after
            // kGupdProbes slots and adds straight into row c (exact integer
            // sums, so where a key's parts land does not matter): a table
            // filled by a large component (config 3: ~4000 keys in 2048 slots)
            // would otherwise scan every slot per insertion
            unsigned h = hash_key(ct) & (cap - 1);
            const int plim = to_rows ? min(cap, kGupdProbes) : cap;
            int probes = 0;
            bool full = false;
            while (true) {
              const int prev = atomicCAS(t_key + h, -1, ct);
              if (prev == -1 || prev == ct) break;
              h = (h + 1) & (cap - 1);
              if (++probes >= plim) {
                full = true;
                break;
              }
            }
            if (full && a.list) {  // (to_rows items only: one list entry for this occurrence)
              const unsigned long long w = atomicAdd(a.cl_n, 1ULL);
              if ((long long)w < a.cl_cap) {
                a.cl_key[w] = (static_cast<unsigned>(c) << a.cl_kb) | static_cast<unsigned>(ct);
                a.cl_cnt[w] = 1;
                a.cl_hi[w] = hi;
                a.cl_lo[w] = lo;
              } else {
                atomicExch(a.cl_ovf, 1);
              }
            } else if (full) {  // (to_rows items only: exact integer adds straight into row c)
              const int64_t at = (int64_t)c * dm.C + ct;
              atomicAdd(reinterpret_cast<unsigned long long*>(a.xc + at), 1ULL);
              atomicAdd(reinterpret_cast<unsigned long long*>(a.xc + CC + at), static_cast<unsigned long long>(hi));
              atomicAdd(reinterpret_cast<unsigned long long*>(a.xc + 2 * CC + at), static_cast<unsigned long long>(lo));
            } else {
              atomicAdd(t_cnt + h, 1);
              smem_add_u64(reinterpret_cast<unsigned long long*>(t_hi + h), static_cast<unsigned long long>(hi));
              smem_add_u64(reinterpret_cast<unsigned long long*>(t_lo + h), static_cast<unsigned long long>(lo));
            }
          } else if (sdense) {  // (shared-memory atomics: the pointers below are known to be shared)
            unsigned long long* d = reinterpret_cast<unsigned long long*>(smem_raw);
            atomicAdd(reinterpret_cast<unsigned*>(smem_raw + 16 * static_cast<size_t>(dm.C)) + ct, 1u);
            smem_add_u64(d + ct, static_cast<unsigned long long>(hi));
            smem_add_u64(d + dm.C + ct, static_cast<unsigned long long>(lo));
          } else {  // (the per-CTA global tables)
            const int64_t gb = (int64_t)blockIdx.x * dm.C + ct;
            atomicAdd(reinterpret_cast<unsigned long long*>(a.gt_cnt + gb), 1ULL);
            atomicAdd(reinterpret_cast<unsigned long long*>(a.gt_hi + gb), static_cast<unsigned long long>(hi));
            atomicAdd(reinterpret_cast<unsigned long long*>(a.gt_lo + gb), static_cast<unsigned long long>(lo));
          }
          }
        }
      }
      __syncthreads();
    }
    const int tab_n = npts == 0 ? 0 : (use_smem ? cap : dm.C);
    auto entry = [&](int i, int& ct, long long& cnt, long long& hi, long long& lo) {
      if (use_smem) {
        ct = t_key[i];
        cnt = t_cnt[i];
        hi = t_hi[i];
        lo = t_lo[i];
      } else {
        ct = i;
        cnt = sdense ? static_cast<long long>(d_cnt[i]) : g_cnt[i];
        hi = g_hi[i];
        lo = g_lo[i];
      }
    };
    if (a.dump) {
      for (int i = tid; i < tab_n; i += kGupdThreads) {
        int ct;
        long long cnt, hi, lo;
        entry(i, ct, cnt, hi, lo);
        if (ct < 0 || cnt <= 0) continue;
        const unsigned long long w = atomicAdd(a.dump_n, 1ULL);
        if ((long long)w < a.dump_cap) {
          a.dump_c[w] = c;
          a.dump_ct[w] = ct;
          a.dump_cnt[w] = cnt;
          a.dump_hi[w] = hi;
          a.dump_lo[w] = lo;
        }
      }
    }
    if (to_rows && a.list) {
      // the item's table appended to the list, one slot reservation per warp
      for (int i0 = 0; i0 < tab_n; i0 += kGupdThreads) {
        const int i = i0 + tid;
        int ct = -1;
        long long cnt = 0, hi = 0, lo = 0;
        if (i < tab_n) entry(i, ct, cnt, hi, lo);
        const bool valid = ct >= 0 && cnt > 0;
        const unsigned m = __ballot_sync(kFull, valid);
        if (!m) continue;
        const int leader = __ffs(m) - 1;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(a.cl_n, static_cast<unsigned long long>(__popc(m)));
        base = __shfl_sync(kFull, base, leader);
        if (valid) {
          const unsigned long long w = base + __popc(m & ((1u << lane) - 1u));
          if ((long long)w < a.cl_cap) {
            a.cl_key[w] = (static_cast<unsigned>(c) << a.cl_kb) | static_cast<unsigned>(ct);
            a.cl_cnt[w] = cnt;
            a.cl_hi[w] = hi;
            a.cl_lo[w] = lo;
          } else {
            atomicExch(a.cl_ovf, 1);
          }
        }
      }
      __syncthreads();
      continue;
    }
    if (to_rows) {
      for (int i = tid; i < tab_n; i += kGupdThreads) {
        int ct;
        long long cnt, hi, lo;
        entry(i, ct, cnt, hi, lo);
        if (ct < 0 || cnt <= 0) continue;
        const int64_t at = (int64_t)c * dm.C + ct;
        atomicAdd(reinterpret_cast<unsigned long long*>(a.xc + at), static_cast<unsigned long long>(cnt));
        atomicAdd(reinterpret_cast<unsigned long long*>(a.xc + CC + at), static_cast<unsigned long long>(hi));
        atomicAdd(reinterpret_cast<unsigned long long*>(a.xc + 2 * CC + at), static_cast<unsigned long long>(lo));
      }
      __syncthreads();
      continue;
    }
    // update_g: the keys (avg, ct) are computed once, in place of the sums
    // (+inf: no key; averages are finite, the values saturate at 2^40), then
    // G-1 rounds of a block-wide argmin, the winner's key set to +inf
    double* kv = reinterpret_cast<double*>(use_smem ? t_hi : g_hi);
    for (int i = tid; i < tab_n; i += kGupdThreads) {
      int ct;
      long long cnt, hi, lo;
      entry(i, ct, cnt, hi, lo);
      kv[i] = (ct < 0 || cnt <= 0) ? INFINITY : from_fixed(hi, lo) / static_cast<double>(cnt);
    }
    if (tid == 0) s_nsel = 0;
    __syncthreads();
    // G-1 rounds of a block-wide argmin over the threads' own minima (slot i
    // belongs to thread i mod kGupdThreads); only the winner's owner rescans
    // its slots after the winning key is retired
    KeyMin mine{INFINITY, 0x7fffffff};
    int mi = -1;
    auto own_min = [&]() {
      mine = KeyMin{INFINITY, 0x7fffffff};
      mi = -1;
      for (int i = tid; i < tab_n; i += kGupdThreads) {
        const double v = kv[i];
        if (v == INFINITY) continue;
        const KeyMin k{v, use_smem ? t_key[i] : i};
        if (kless(k, mine)) mine = k, mi = i;
      }
    };
    if (npts > 0) own_min();
    for (int r = 0; r < dm.G - 1 && npts > 0; ++r) {
      KeyMin best = mine;
      int bi = mi;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        KeyMin oth{__shfl_xor_sync(kFull, best.v, o), __shfl_xor_sync(kFull, best.c, o)};
        const int obi = __shfl_xor_sync(kFull, bi, o);
        if (kless(oth, best)) best = oth, bi = obi;
      }
      if (lane == 0) red[warp] = best, red_i[warp] = bi;
      __syncthreads();
      if (tid == 0) {
        KeyMin b = red[0];
        int ib = red_i[0];
        for (int w = 1; w < nw; ++w)
          if (kless(red[w], b)) b = red[w], ib = red_i[w];
        s_win = b.c != 0x7fffffff ? ib : -1;
        if (b.c != 0x7fffffff) s_sel[s_nsel++] = b.c;
      }
      __syncthreads();
      const int win = s_win;
      if (win < 0) break;  // no more keys
      if (tid == win % kGupdThreads) {
        kv[win] = INFINITY;
        own_min();
      }
    }
    if (tid == 0) {
      int out[64];
      int m = 0;
      out[m++] = c;
      for (int q = 0; q < s_nsel; ++q) out[m++] = s_sel[q];
      sort_small(out, m);
      for (int i = 0; i < dm.G; ++i) a.g_new[(int64_t)c * dm.G + i] = i < m ? out[i] : -1;
      a.gcnt_new[c] = m;
    }
    __syncthreads();
  }
}

// g selection from dense rows of xc: every component in exchange (multi-rank)
// mode, else the components split over several items. Rows are zeroed after
// reading so the table is clean for the next E-step.
__global__ void __launch_bounds__(kGupdThreads) k_gselect_dense(Dims dm, long long* xc,
                                                                const int* itemoff, int all,
                                                                int* g_new, int* gcnt_new) {
  __shared__ KeyMin red[kGupdThreads / 32];
  __shared__ int s_sel[64];
  __shared__ int s_nsel;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = kGupdThreads / 32;
  const int64_t CC = (int64_t)dm.C * dm.C;
  for (int c = blockIdx.x; c < dm.C; c += gridDim.x) {
    if (!all && itemoff[c + 1] - itemoff[c] <= 1) continue;
    if (tid == 0) s_nsel = 0;
    __syncthreads();
    long long* rc = xc + (int64_t)c * dm.C;
    // G-1 rounds of a block argmin over the threads' own minima (entry ct
    // belongs to thread ct mod kGupdThreads); a winner's count is zeroed in the
    // row (the row is cleared below anyway) and only its owner rescans
    KeyMin mine{INFINITY, 0x7fffffff};
    auto own_min = [&]() {
      mine = KeyMin{INFINITY, 0x7fffffff};
      for (int ct = tid; ct < dm.C; ct += kGupdThreads) {
        const long long cnt = rc[ct];
        if (cnt <= 0) continue;
        const KeyMin k{from_fixed(rc[CC + ct], rc[2 * CC + ct]) / static_cast<double>(cnt), ct};
        if (kless(k, mine)) mine = k;
      }
    };
    own_min();
    for (int r = 0; r < dm.G - 1; ++r) {
      KeyMin best = mine;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        KeyMin oth{__shfl_xor_sync(kFull, best.v, o), __shfl_xor_sync(kFull, best.c, o)};
        if (kless(oth, best)) best = oth;
      }
      if (lane == 0) red[warp] = best;
      __syncthreads();
      if (tid == 0) {
        KeyMin b = red[0];
        for (int w = 1; w < nw; ++w)
          if (kless(red[w], b)) b = red[w];
        if (b.c != 0x7fffffff) s_sel[s_nsel++] = b.c;
      }
      __syncthreads();
      if (s_nsel <= r) break;
      const int win = s_sel[r];
      if (tid == win % kGupdThreads) {
        rc[win] = 0;
        own_min();
      }
    }
    if (tid == 0) {
      int out[64];
      int m = 0;
      out[m++] = c;
      for (int q = 0; q < s_nsel; ++q) out[m++] = s_sel[q];
      sort_small(out, m);
      for (int i = 0; i < dm.G; ++i) g_new[(int64_t)c * dm.G + i] = i < m ? out[i] : -1;
      gcnt_new[c] = m;
    }
    for (int ct = tid; ct < dm.C; ct += kGupdThreads) {
      rc[ct] = 0;
      rc[CC + ct] = 0;
      rc[2 * CC + ct] = 0;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- sparse co-occurrence (large C)
// The list of exact (c, c~) partial sums appended by k_gupdate (list mode)
// is sorted by key = c << kb | c~ (the radix sort of vmfa_sort.cu over 2 kb bits), reduced
// by key (exact int64 sums: the order of the parts does not matter, so g is
// bit-identical to the dense rows' for any item split or rank count), and g_c
// is selected per component from its unique entries exactly as
// k_gselect_dense does from a dense row (update_g, estep.cpp:204-220).
__global__ void k_cooc_heads(CoocArgs a) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += gridDim.x * blockDim.x)
    a.head[i] = (i == 0 || a.key[i] != a.key[i - 1]) ? 1 : 0;
}
// after the inclusive scan of the heads: head[i] = 1 + unique index of entry i
__global__ void k_cooc_sums(CoocArgs a) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += gridDim.x * blockDim.x) {
    const int u = a.head[i] - 1;
    const int src = a.perm[i];
    if (i == 0 || a.key[i] != a.key[i - 1]) a.u_key[u] = a.key[i];
    atomicAdd(reinterpret_cast<unsigned long long*>(a.u_cnt + u), static_cast<unsigned long long>(a.cnt[src]));
    atomicAdd(reinterpret_cast<unsigned long long*>(a.u_hi + u), static_cast<unsigned long long>(a.hi[src]));
    atomicAdd(reinterpret_cast<unsigned long long*>(a.u_lo + u), static_cast<unsigned long long>(a.lo[src]));
  }
}
// u_off[c] = first unique entry of component >= c (binary search; nu from the scan)
__global__ void k_cooc_offsets(CoocArgs a) {
  const int nu = a.n > 0 ? a.head[a.n - 1] : 0;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c <= a.dm.C; c += gridDim.x * blockDim.x) {
    int lo = 0, hi = nu;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (static_cast<int>(a.u_key[mid] >> a.kb) < c) lo = mid + 1;
      else hi = mid;
    }
    a.u_off[c] = lo;
  }
}
// warp per component: G - 1 rounds of a warp argmin over (avg, c~)
__global__ void k_cooc_select(CoocArgs a, int c0, int c1, int zero_others, int* g_new, int* gcnt_new) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const unsigned cmask = (1u << a.kb) - 1u;
  for (int c = blockIdx.x * wpb + (threadIdx.x >> 5); c < a.dm.C; c += gridDim.x * wpb) {
    if (c < c0 || c >= c1) {
      if (zero_others) {
        for (int i = lane; i < a.dm.G; i += 32) g_new[(int64_t)c * a.dm.G + i] = 0;
        if (lane == 0) gcnt_new[c] = 0;
      }
      continue;
    }
    const int e0 = a.u_off[c], e1 = a.u_off[c + 1];
    int sel[64];
    int ns = 0;
    for (int r = 0; r < a.dm.G - 1; ++r) {
      KeyMin best{INFINITY, 0x7fffffff};
      for (int e = e0 + lane; e < e1; e += 32) {
        const long long cnt = a.u_cnt[e];
        if (cnt <= 0) continue;
        const int ct = static_cast<int>(a.u_key[e] & cmask);
        bool taken = false;
        for (int q = 0; q < ns; ++q) taken |= (sel[q] == ct);
        if (taken) continue;
        const KeyMin k{from_fixed(a.u_hi[e], a.u_lo[e]) / static_cast<double>(cnt), ct};
        if (kless(k, best)) best = k;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        KeyMin oth{__shfl_xor_sync(kFull, best.v, o), __shfl_xor_sync(kFull, best.c, o)};
        if (kless(oth, best)) best = oth;
      }
      if (best.c == 0x7fffffff) break;
      sel[ns++] = best.c;
    }
    if (lane == 0) {
      int out[64];
      int m = 0;
      out[m++] = c;
      for (int q = 0; q < ns; ++q) out[m++] = sel[q];
      sort_small(out, m);
      for (int i = 0; i < a.dm.G; ++i) g_new[(int64_t)c * a.dm.G + i] = i < m ? out[i] : -1;
      gcnt_new[c] = m;
    }
  }
}

// ---------------------------------------------------------------- mbarrier / bulk-copy helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void xbar_init(uint64_t* bar, int count = 1) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void xbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void xbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_row(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

// phase timing of k_stats (diagnostics, built with -DVMFA_STATS_PROF): CTA 0,
// thread 0, cycles between marks
__device__ unsigned long long g_stats_prof[16];
__device__ int g_stats_prof_on;
#ifdef VMFA_STATS_PROF
#define SPROF(k)                                                                         \
  do {                                                                                   \
    if (sprof_on) {                                                                      \
      const unsigned long long now_ = clock64();                                         \
      if ((k) > 0) g_stats_prof[(k)] += now_ - sprof_t;                                  \
      sprof_t = now_;                                                                    \
    }                                                                                    \
  } while (0)
#else
#define SPROF(k) \
  do {           \
  } while (0)
#endif

// ---------------------------------------------------------------- K5: sufficient statistics
// CTA per component a over its K-pairs (n, q) in ascending (n, j) order
// (accumulate_point, mstep.cpp:47-67): mz = V_a (x - mu_a) (fp32 dot products),
// then fp64: N += q; E += q [mz;1][mz;1]^T (+ N Sigma_z at the end);
// Y[:, h] += q x zhat_h; sq += q x^2. Fixed order per component =>
// deterministic; no atomics.
constexpr int kStatsBatch = 32;
constexpr int kStatsMaxRows = 1024;  // K-pairs per statistics item (upper bound)
constexpr int kStatsMaxRowsBig = 1536;  // ... of k_stats_mma's BIG variant (one CTA per SM: room for longer items)
constexpr int kStatsMaxBuf = 6;      // row-batch ring depth (bulk-copy path)
constexpr int kStatsMaxH1 = 17;   // columns of Y per pass

// Items are (component, chunk of <= rows_per_item K-pairs): large components
// are split so no CTA owns a disproportionate share (SURVEY §7 hard part 3).
// Per batch of 32 rows (cp.async double-buffered into smem):
//   (i)  mz = V (x - mu) (mstep.cpp:52-53): lane = row, warp = 1/8 of the
//        dimensions, V rows broadcast from smem; warp partials summed in smem.
//   (ii) Y_v += q v zhat^T, sq_v += q v^2 (v = x - mu, fp32 register tiles of
//        4 dims x NH1 columns per thread over a row group, scaled by the
//        item's largest q); E += q [zhat;1][zhat;1]^T in fp64, one thread per
//        upper-triangle entry (N = E(H,H)).
// Sole-item components write their statistics directly; split components
// write fp64 partials summed by k_stats_reduce in item order (deterministic).
// Partial layout per item (pass col0): [Y cols col0.. (NH1 x D) | sq (D) |
// E ((H+1)^2) | N] -- sq/E/N only in the first pass, E only when H+1 <= NH1.
constexpr int kStatsXChunk = 4;  // phase (i): float4s of the row loaded ahead
constexpr int kXPad = 4;  // s_x row stride D + 4: conflict-free LDS.128 across rows

template <int NH1, int ND>
__global__ void __launch_bounds__(kStatsThreads, NH1 > 9 ? 1 : 2) k_stats(StatsArgs a, const int* __restrict__ itemoff,
                                                        int rows_per_item, int col0, double* part,
                                                        int64_t part_stride, int nbuf) {
  // smem: s_x [nbuf][B][XS] | s_V [D][VS] | s_mu [D+pad] | s_pz [8][B][NZ] | s_zf [B][ZS] (float)
  extern __shared__ __align__(16) float s_x[];
  // phase (i) computes the NZ latent columns of this pass; the constant column
  // of [zhat; 1] is implicit (NH1 = 5, 9 passes hold all of H + 1 <= NH1)
  constexpr int NZ = NH1 == kStatsMaxH1 ? NH1 : NH1 - 1;
  constexpr int VS = (NZ + 3) / 4 * 4;   // V row stride (16-byte rows for LDS.128)
  constexpr int ZS = (NH1 + 3) / 4 * 4;  // [zhat;1] row stride in s_zf
  __shared__ double s_red[kStatsThreads / 32];
  __shared__ double s_accE[kStatsThreads];  // E entry of thread tid (fp64)
  __shared__ uint64_t s_xbar[kStatsMaxBuf];  // row-batch arrival (bulk copies, D % 4 == 0)
  __shared__ int s_eall[kStatsMaxRows];      // the item's rows of X
  __shared__ double s_qall[kStatsMaxRows];   // ... and responsibilities / qmax
  __shared__ float s_qfall[kStatsMaxRows];   // the same in fp32 (phase ii)
  const Dims dm = a.dm;
  const int H = dm.H, H1 = H + 1, D = dm.D;
  const int XS = (D + 3) / 4 * 4 + kXPad;
  float* s_V = s_x + (int64_t)nbuf * kStatsBatch * XS;
  float* s_mu = s_V + (int64_t)D * VS;
  float* s_pz = s_mu + (D + 3) / 4 * 4 + 4;  // [8][B][NZ]
  float* s_zf = s_pz + 8 * kStatsBatch * NZ;  // [B][ZS]
  double* s_zd = reinterpret_cast<double*>(s_zf + kStatsBatch * ZS);  // [B][ZS] (E)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool first = col0 == 0;
  const bool full_e = first && (H1 <= NH1);
  const bool vec = (D & 3) == 0;
  // register tiles over the "dimensions" [0, D) of the centred row; E = sum q
  // [zhat;1][zhat;1]^T is accumulated separately in fp64 (one thread per
  // upper-triangle entry): its conditioning follows N_c Sigma_z, which fp32
  // sums cannot resolve for collapsed components
  const int Dp = (D + 3) / 4 * 4;
  const int GD = Dp / 4;
  // E: thread = (upper-triangle entry, row group); row groups summed in order at the item end
  const int NE = H1 * (H1 + 1) / 2;
  const int EG = max(1, kStatsThreads / NE);
  const int eg = tid / NE;
  int ei = -1, ej = -1;  // this thread's E entry (i <= j)
  if (full_e && eg < EG) {
    int t = tid - eg * NE;
    for (int i = 0; i < H1 && ei < 0; ++i) {
      if (t < H1 - i) ei = i, ej = i + t;
      else t -= H1 - i;
    }
  }
  const int RG = max(1, kStatsThreads / GD);
  const int my_dg = tid % GD, my_rg = tid / GD;
  const bool tile_on = my_rg < RG && tid < RG * GD;
  const int dsl = ((D + 7) / 8 + 3) / 4 * 4;  // phase (i) dims per warp, multiple of 4
  const int dw0 = warp * dsl, dw1 = min(D, dw0 + dsl);
  const int total = __ldg(itemoff + dm.C);
  // row gather: one bulk copy per row (D % 4 == 0; lane-parallel 16-byte
  // cp.async measured slower), else 4-byte cp.async with completion tracked by
  // the buffer's mbarrier (every thread's cp.async.mbarrier.arrive.noinc)
  const bool bulk = vec;
  if (tid == 0)
    for (int i = 0; i < kStatsMaxBuf; ++i) xbar_init(&s_xbar[i], bulk ? 1 : kStatsThreads);
  __syncthreads();
  uint32_t xpar = 0u;  // bit b: phase parity of row buffer b's barrier (same in every thread)
#ifdef VMFA_STATS_PROF
  unsigned long long sprof_t = 0;
  const bool sprof_on = blockIdx.x == 0 && threadIdx.x == 0 && g_stats_prof_on;
#endif
  __shared__ int s_item;
  // items from a global work queue (dynamic balance; results depend only on the item)
  auto next_item = [&](int cur) -> int {
    if (!a.qctr) return cur < 0 ? static_cast<int>(blockIdx.x) : cur + static_cast<int>(gridDim.x);
    __syncthreads();
    if (tid == 0) s_item = atomicAdd(a.qctr, 1);
    __syncthreads();
    return s_item;
  };
  for (int item = next_item(-1); item < total; item = next_item(item)) {
    const int c = find_item(itemoff, dm.C, item);
    const int r0 = a.off[c] + (item - itemoff[c]) * rows_per_item;
    const int r1 = min(a.off[c + 1], r0 + rows_per_item);
    const int nr = r1 - r0;
    const bool direct = itemoff[c + 1] - itemoff[c] == 1;  // sole item: write the statistics
    // responsibilities are scaled by the item's largest q before the fp32
    // accumulation (no underflow; N_c == 0 exactly iff every q == 0)
    double qmax = 0.0;
    __syncthreads();  // previous item done with the shared buffers
    // the item's entries and responsibilities, staged once (one latency per item)
    for (int i = tid; i < nr; i += kStatsThreads) {
      const int e = a.ent[r0 + i];
      const double q = a.resp[e];
      s_eall[i] = e / dm.Cp;  // the row of X
      s_qall[i] = q;
      qmax = fmax(qmax, q);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) qmax = fmax(qmax, __shfl_xor_sync(kFull, qmax, o));
    if (lane == 0) s_red[warp] = qmax;
    for (int i = tid; i < D * VS; i += kStatsThreads) {
      const int d = i / VS, h = i - d * VS;
      s_V[i] = (h < NZ && col0 + h < H) ? __ldg(a.V32 + (int64_t)c * D * H + (int64_t)d * H + col0 + h) : 0.f;
    }
    for (int d = tid; d < Dp + 4; d += kStatsThreads) s_mu[d] = d < D ? __ldg(a.mu32 + (int64_t)c * D + d) : 0.f;
    __syncthreads();
    qmax = 0.0;
#pragma unroll
    for (int w = 0; w < kStatsThreads / 32; ++w) qmax = fmax(qmax, s_red[w]);
    const double qdiv = qmax > 0.0 ? qmax : 1.0;  // divide (1/qmax overflows for denormal qmax)
    // every thread rescales the entries it staged (read after the first batch's barriers)
    for (int i = tid; i < nr; i += kStatsThreads) {
      const double q = s_qall[i] / qdiv;
      s_qall[i] = q;
      s_qfall[i] = static_cast<float>(q);
    }
    float accY[ND][4][NH1];
    float accS[ND][4];
    float mreg[ND][4];  // this thread's mean entries (phase ii)
    if (ei >= 0) s_accE[tid] = 0.0;
#pragma unroll
    for (int k = 0; k < ND; ++k)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        accS[k][i] = 0.f;
        mreg[k][i] = s_mu[min(4 * (my_dg + k * GD) + i, Dp + 3)];
#pragma unroll
        for (int h = 0; h < NH1; ++h) accY[k][i][h] = 0.f;
      }
    const int nbat = (nr + kStatsBatch - 1) / kStatsBatch;
    auto issue_rows = [&](int b, int buf) {
      float* dst = s_x + (int64_t)buf * kStatsBatch * XS;
      const int nb = min(kStatsBatch, nr - b * kStatsBatch);
      const int* eb = s_eall + b * kStatsBatch;
      if (bulk) {
        // one bulk copy per row, issued by four lanes of every warp (the
        // copies of a warp are issued one after another, so the batch is
        // spread over the warps); thread 0 arms the barrier with the total
        // (a copy may complete before the arm: the transaction count is signed)
        if (tid == 0) xbar_expect(&s_xbar[buf], static_cast<uint32_t>(nb) * D * 4u);
        if (lane < kStatsBatch / (kStatsThreads / 32)) {
          const int r = warp * (kStatsBatch / (kStatsThreads / 32)) + lane;
          if (r < nb) bulk_row(smem_addr(dst + (int64_t)r * XS), a.X + (int64_t)eb[r] * D, D * 4u, &s_xbar[buf]);
        }
      } else {
        for (int i = tid; i < nb * D; i += kStatsThreads) {
          const int r = i / D, f = i - r * D;
          const float* src = a.X + (int64_t)eb[r] * D + f;
          const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(dst + (int64_t)r * XS + f));
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(src) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(&s_xbar[buf])) : "memory");
      }
    };
    // ring of nbuf row buffers: batch bi + nbuf - 1 is issued once every
    // thread has passed batch bi's first barrier (its buffer's last readers,
    // batch bi - 1, are done); two barriers per batch
    for (int b = 0; b < min(nbuf - 1, nbat); ++b) issue_rows(b, b);
    for (int bi = 0; bi < nbat; ++bi) {
      const int buf = bi % nbuf;
      const int nb = min(kStatsBatch, nr - bi * kStatsBatch);
      SPROF(0);
      if (nbuf == 1) issue_rows(bi, 0);
      xbar_wait(&s_xbar[buf], (xpar >> buf) & 1u);
      xpar ^= 1u << buf;
      SPROF(2);
      const float* xb = s_x + (int64_t)buf * kStatsBatch * XS;
      // (i) partial mz over this warp's dimension slice, lane = row
      {
        float acc[NZ];
#pragma unroll
        for (int h = 0; h < NZ; ++h) acc[h] = 0.f;
        const float* xr = xb + (int64_t)lane * XS;
        if (lane < nb && vec) {
          // chunks of 4 * kStatsXChunk dimensions: the row's chunk is loaded first (ILP), then
          // the broadcast V rows stream through the FMAs
          for (int d0 = dw0; d0 < dw1; d0 += 4 * kStatsXChunk) {
            float4 xv[kStatsXChunk];
#pragma unroll
            for (int j = 0; j < kStatsXChunk; ++j)
              if (d0 + 4 * j < dw1) xv[j] = *reinterpret_cast<const float4*>(xr + d0 + 4 * j);
#pragma unroll
            for (int j = 0; j < kStatsXChunk; ++j) {
              const int d = d0 + 4 * j;
              if (d >= dw1) break;
              const float4 mv = *reinterpret_cast<const float4*>(s_mu + d);
              const float v4[4] = {xv[j].x - mv.x, xv[j].y - mv.y, xv[j].z - mv.z, xv[j].w - mv.w};
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float* vr = s_V + (d + k) * VS;
#pragma unroll
                for (int h4 = 0; h4 < VS; h4 += 4) {
                  const float4 w = *reinterpret_cast<const float4*>(vr + h4);
                  if (h4 + 0 < NZ) acc[h4 + 0] = fmaf(w.x, v4[k], acc[h4 + 0]);
                  if (h4 + 1 < NZ) acc[h4 + 1] = fmaf(w.y, v4[k], acc[h4 + 1]);
                  if (h4 + 2 < NZ) acc[h4 + 2] = fmaf(w.z, v4[k], acc[h4 + 2]);
                  if (h4 + 3 < NZ) acc[h4 + 3] = fmaf(w.w, v4[k], acc[h4 + 3]);
                }
              }
            }
          }
        } else if (lane < nb) {
          for (int d = dw0; d < dw1; d += 4) {
            const float4 xv = *reinterpret_cast<const float4*>(xr + d);
            const float4 mv = *reinterpret_cast<const float4*>(s_mu + d);
            const float v4[4] = {xv.x - mv.x, xv.y - mv.y, xv.z - mv.z, xv.w - mv.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if (d + k >= dw1) break;
              const float* vr = s_V + (d + k) * VS;
#pragma unroll
              for (int h4 = 0; h4 < VS; h4 += 4) {
                const float4 w = *reinterpret_cast<const float4*>(vr + h4);
                if (h4 + 0 < NZ) acc[h4 + 0] = fmaf(w.x, v4[k], acc[h4 + 0]);
                if (h4 + 1 < NZ) acc[h4 + 1] = fmaf(w.y, v4[k], acc[h4 + 1]);
                if (h4 + 2 < NZ) acc[h4 + 2] = fmaf(w.z, v4[k], acc[h4 + 2]);
                if (h4 + 3 < NZ) acc[h4 + 3] = fmaf(w.w, v4[k], acc[h4 + 3]);
              }
            }
          }
        }
        float* pz = s_pz + ((int64_t)warp * kStatsBatch + lane) * NZ;
#pragma unroll
        for (int h = 0; h < NZ; ++h) pz[h] = acc[h];
      }
      SPROF(4);
      __syncthreads();
      SPROF(5);
      if (nbuf >= 2 && bi + nbuf - 1 < nbat) issue_rows(bi + nbuf - 1, (bi + nbuf - 1) % nbuf);
      SPROF(9);
      for (int i = tid; i < kStatsBatch * ZS; i += kStatsThreads) {
        const int r = i / ZS, h = i - r * ZS;
        const int hh = col0 + h;
        float z = 0.f;
        if (h < NZ && hh < H) {
#pragma unroll
          for (int w = 0; w < 8; ++w) z += s_pz[((int64_t)w * kStatsBatch + r) * NZ + h];
        } else if (h < NH1 && hh == H) {
          z = 1.f;
        }
        s_zf[i] = z;
        s_zd[i] = z;
      }
      SPROF(6);
      __syncthreads();
      SPROF(7);
      const double* s_q = s_qall + bi * kStatsBatch;
      const float* s_qf = s_qfall + bi * kStatsBatch;
      if (ei >= 0) {  // E(ei, ej) += q z_i z_j (z kept in fp64 too: fp32 z products are exact in fp64)
        double acc = s_accE[tid];
        for (int r = eg; r < nb; r += EG) acc = fma(s_q[r], s_zd[r * ZS + ei] * s_zd[r * ZS + ej], acc);
        s_accE[tid] = acc;
      }
      // (ii) register tiles: 4 "dimensions" x NH1 columns, rows my_rg::RG;
      // rows in pairs: both rows' operands are loaded before the FMAs
      if (tile_on) {
        auto load_row = [&](int r, float4 (&xo)[ND], float (&zo)[NH1], float& qo) {
          qo = s_qf[r];
          const float* zr = s_zf + r * ZS;
#pragma unroll
          for (int h4 = 0; h4 < NH1; h4 += 4) {
            if (h4 + 4 <= NH1) {
              const float4 z4 = *reinterpret_cast<const float4*>(zr + h4);
              zo[h4] = z4.x, zo[h4 + 1] = z4.y, zo[h4 + 2] = z4.z, zo[h4 + 3] = z4.w;
            } else {
#pragma unroll
              for (int h = h4; h < NH1; ++h) zo[h] = zr[h];
            }
          }
          const float* xr = xb + (int64_t)r * XS;
#pragma unroll
          for (int k = 0; k < ND; ++k) {
            const int d = 4 * (my_dg + k * GD);
            if (vec || d + 3 < D) {
              xo[k] = *reinterpret_cast<const float4*>(xr + d);
            } else {  // tail dimensions contribute v = 0
              xo[k].x = d + 0 < D ? xr[d + 0] : mreg[k][0];
              xo[k].y = d + 1 < D ? xr[d + 1] : mreg[k][1];
              xo[k].z = d + 2 < D ? xr[d + 2] : mreg[k][2];
              xo[k].w = d + 3 < D ? xr[d + 3] : mreg[k][3];
            }
          }
        };
        auto fma_row = [&](const float4 (&xv)[ND], const float (&zv)[NH1], float qf) {
#pragma unroll
          for (int k = 0; k < ND; ++k) {
            if (k > 0 && my_dg + k * GD >= GD) break;
            const float vs[4] = {xv[k].x - mreg[k][0], xv[k].y - mreg[k][1], xv[k].z - mreg[k][2],
                                 xv[k].w - mreg[k][3]};
            float qv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              qv[i] = qf * vs[i];
              if (first) accS[k][i] = fmaf(qv[i], vs[i], accS[k][i]);
            }
#pragma unroll
            for (int h = 0; h < NH1; ++h) {
#pragma unroll
              for (int i = 0; i < 4; ++i) accY[k][i][h] = fmaf(qv[i], zv[h], accY[k][i][h]);
            }
          }
        };
        int r = my_rg;
        for (; r + RG < nb; r += 2 * RG) {  // two rows' operands in flight
          float4 xa[ND], xb2[ND];
          float za[NH1], zb[NH1];
          float qa, qb;
          load_row(r, xa, za, qa);
          load_row(r + RG, xb2, zb, qb);
          fma_row(xa, za, qa);
          fma_row(xb2, zb, qb);
        }
        if (r < nb) {
          float4 xa[ND];
          float za[NH1];
          float qa;
          load_row(r, xa, za, qa);
          fma_row(xa, za, qa);
        }
      }
      SPROF(8);
      if (nbuf == 1) __syncthreads();  // the next issue reuses this batch's buffer
    }
    // combine the row groups of each dimension group through smem (fp64),
    // reusing the row buffers, then write (direct or partial) scaled by qmax
    double* red = reinterpret_cast<double*>(s_x);  // >= RG * GD * 4 * (NH1 + 1) doubles
    double* pp = direct ? nullptr : part + (int64_t)item * part_stride;
    double* pe = direct ? a.E + (int64_t)c * H1 * H1 : pp + (int64_t)NH1 * D + D;
    __syncthreads();  // every row group's E entry (and phase ii) done
    if (ei >= 0 && eg == 0) {
      double e = 0.0;
      for (int g = 0; g < EG; ++g) e += s_accE[tid + g * NE];
      pe[ej * H1 + ei] = e * qmax;
      pe[ei * H1 + ej] = e * qmax;
    }
#pragma unroll
    for (int k = 0; k < ND; ++k) {
      __syncthreads();
      if (tile_on && my_rg > 0) {
        double* dst = red + ((int64_t)(my_rg - 1) * GD + my_dg) * 4 * (NH1 + 1);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
#pragma unroll
          for (int h = 0; h < NH1; ++h) dst[i * (NH1 + 1) + h] = accY[k][i][h];
          dst[i * (NH1 + 1) + NH1] = accS[k][i];
        }
      }
      __syncthreads();
      if (tile_on && my_rg == 0) {
        double ty[4][NH1], ts[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          ts[i] = accS[k][i];
#pragma unroll
          for (int h = 0; h < NH1; ++h) ty[i][h] = accY[k][i][h];
        }
        for (int gg = 1; gg < RG; ++gg) {
          const double* src = red + ((int64_t)(gg - 1) * GD + my_dg) * 4 * (NH1 + 1);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
#pragma unroll
            for (int h = 0; h < NH1; ++h) ty[i][h] += src[i * (NH1 + 1) + h];
            ts[i] += src[i * (NH1 + 1) + NH1];
          }
        }
        const int g = my_dg + k * GD;
        if (k == 0 || g < GD) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int d = 4 * g + i;
            if (d >= D) continue;
            if (direct) {
#pragma unroll
              for (int h = 0; h < NH1; ++h)
                if (col0 + h < H1) a.Y[((int64_t)c * H1 + col0 + h) * D + d] = ty[i][h] * qmax;
              if (first) a.sq[(int64_t)c * D + d] = ts[i] * qmax;
            } else {
#pragma unroll
              for (int h = 0; h < NH1; ++h) pp[(int64_t)h * D + d] = ty[i][h] * qmax;
              if (first) pp[(int64_t)NH1 * D + d] = ts[i] * qmax;
            }
          }
        }
      }
    }
  }
}

// E for H+1 > kStatsMaxH1: item-based, full zhat per row; partial [E | -].
// zhat = [V (x - mu); 1] by a warp per row with lanes over the latent columns
// (coalesced V rows, x and mu broadcast); E += q zhat zhat^T in fp64 by 4x4
// register tiles of the upper triangle (16 DFMA per 8 shared loads), the
// lower triangle mirrored at the end.
constexpr int kEZS = 68;  // padded zhat row (H1 <= 65 -> 17 tiles of 4)
__global__ void __launch_bounds__(kStatsThreads) k_stats_E(StatsArgs a, const int* __restrict__ itemoff,
                                                          int rows_per_item, double* part,
                                                          int64_t part_stride) {
  extern __shared__ __align__(16) double s_zz[];  // [2][kStatsBatch][kEZS]: q zhat, zhat
  double* s_qz = s_zz;
  double* s_z = s_zz + kStatsBatch * kEZS;
  const Dims dm = a.dm;
  const int H = dm.H, H1 = H + 1, D = dm.D;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = kStatsThreads / 32;
  const int NT = (H1 + 3) / 4;  // 4-blocks per side
  // this thread's upper-triangle tile (bi <= bj), or none
  int bi = -1, bj = -1;
  {
    int t = tid;
    for (int i = 0; i < NT && bi < 0; ++i) {
      if (t < NT - i) bi = i, bj = i + t;
      else t -= NT - i;
    }
  }
  const int total = __ldg(itemoff + dm.C);
  for (int item = blockIdx.x; item < total; item += gridDim.x) {
    const int c = find_item(itemoff, dm.C, item);
    const int r0 = a.off[c] + (item - itemoff[c]) * rows_per_item;
    const int r1 = min(a.off[c + 1], r0 + rows_per_item);
    const float* Vc = a.V32 + (int64_t)c * D * H;
    const float* mc = a.mu32 + (int64_t)c * D;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int b0 = r0; b0 < r1; b0 += kStatsBatch) {
      const int nb = min(kStatsBatch, r1 - b0);
      __syncthreads();  // previous batch's tiles done with s_qz / s_z
      for (int r = warp; r < kStatsBatch; r += nw) {
        double q = 0.0;
        float z0 = 0.f, z1 = 0.f;  // columns lane, lane + 32
        if (r < nb) {
          const int e = a.ent[b0 + r];
          const float* x = a.X + (int64_t)(e / dm.Cp) * D;
          q = a.resp[e];
          const bool h0 = lane < H, h1 = lane + 32 < H;
          for (int d = 0; d < D; ++d) {
            const float v = __ldg(x + d) - __ldg(mc + d);
            const float* vr = Vc + (int64_t)d * H;
            if (h0) z0 = fmaf(__ldg(vr + lane), v, z0);
            if (h1) z1 = fmaf(__ldg(vr + lane + 32), v, z1);
          }
        }
        for (int h = lane; h < kEZS; h += 32) {
          const double z = r >= nb ? 0.0 : (h < H ? static_cast<double>(h < 32 ? z0 : z1)
                                                  : (h == H ? 1.0 : 0.0));
          s_z[r * kEZS + h] = z;
          s_qz[r * kEZS + h] = q * z;
        }
      }
      __syncthreads();
      if (bi >= 0) {
        for (int r = 0; r < nb; ++r) {
          const double* qr = s_qz + r * kEZS + 4 * bi;
          const double* zr = s_z + r * kEZS + 4 * bj;
          const double q0 = qr[0], q1 = qr[1], q2 = qr[2], q3 = qr[3];
          const double z0 = zr[0], z1 = zr[1], z2 = zr[2], z3 = zr[3];
          const double qv[4] = {q0, q1, q2, q3}, zv[4] = {z0, z1, z2, z3};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fma(qv[i], zv[j], acc[i][j]);
        }
      }
    }
    double* pe = part + (int64_t)item * part_stride;
    if (bi >= 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int ii = 4 * bi + i, jj = 4 * bj + j;
          if (ii >= H1 || jj >= H1) continue;
          if (bi == bj && ii > jj) continue;  // the diagonal tile's lower half comes from its upper
          pe[jj * H1 + ii] = acc[i][j];
          pe[ii * H1 + jj] = acc[i][j];
        }
    }
  }
}

// ---------------------------------------------------------------- K5 on the tensor cores (H + 1 <= 16)
// The same statistics as k_stats (accumulate_point, mstep.cpp:47-67, centred
// on the fp32 mean as there), with both contractions as warp-level
// mma.sync.m16n8k8 tf32 in 3xTF32 split precision (x = hi + lo, products
// hi*hi + hi*lo + lo*hi, fp32 accumulation: ~21 significant bits, the fp32
// FFMA form's accuracy at a quarter of its instructions; tools/micro/
// mma_sync_tput.cu measures 0.465 mma/clk/SM = 476 FMA/clk against FFMA's 125):
//   (i)  Z = Vc V^T: M = 16 rows of the batch, N = 8 latent columns, K = D
//        (split in quarters over the warps, partials summed in smem);
//   (ii) Y_v^T += (Q Zhat)^T Vc: M = 16 columns of [zhat; 1] (padded),
//        N = 8 dimensions, K = 8 rows; each warp owns D/64 dimension tiles for
//        the whole item, so its accumulators are the item's Y_v columns (no
//        cross-warp reduction); sq_v = sum q v^2 rides on the phase (ii) loads.
// E stays fp64 on the CUDA cores (one thread per upper-triangle entry and row
// group), as in k_stats. Items, work queue, qmax scaling, the direct/partial
// split and the partial layout (nh1 = 5/9/17) are k_stats's, so
// k_stats_reduce / k_stats_uncenter / k_stats_sz are shared.
constexpr int kSmBatch = 32;  // rows per batch (2 m-tiles of phase i, 4 k-steps of phase ii)
constexpr int kSmZD = 17;     // s_zd row stride (fp64)

// round to the nearest tf32 (ties away) by integer add + mask: two ALU
// instructions (cvt.rna.tf32.f32 lowers to ~6 with its inf/nan guards);
// finite inputs only (the statistics operands are finite)
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}
__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// acc += a * b in 3xTF32 (small terms first). The three products of one
// k-step go into a fresh accumulator and are added to acc with round-to-
// nearest FADDs: the tensor core's internal accumulation truncates, and
// chaining hundreds of k-steps through it biases long sums (measured ~30x the
// FFMA error on the statistics; tools/diag_stats_err.py)
__device__ __forceinline__ void mma3(float (&acc)[4], const float (&ah)[4], const float (&al)[4], float b0h,
                                     float b1h, float b0l, float b1l) {
  const uint32_t h[4] = {__float_as_uint(ah[0]), __float_as_uint(ah[1]), __float_as_uint(ah[2]),
                         __float_as_uint(ah[3])};
  const uint32_t l[4] = {__float_as_uint(al[0]), __float_as_uint(al[1]), __float_as_uint(al[2]),
                         __float_as_uint(al[3])};
  float c[4] = {0.f, 0.f, 0.f, 0.f};
  mma_tf32(c, l, __float_as_uint(b0h), __float_as_uint(b1h));
  mma_tf32(c, h, __float_as_uint(b0l), __float_as_uint(b1l));
  mma_tf32(c, h, __float_as_uint(b0h), __float_as_uint(b1h));
#pragma unroll
  for (int k = 0; k < 4; ++k) acc[k] += c[k];
}
// the same three products chained into acc (callers keep the chain short)
__device__ __forceinline__ void mma3c(float (&acc)[4], const float (&ah)[4], const float (&al)[4], float b0h,
                                      float b1h, float b0l, float b1l) {
  const uint32_t h[4] = {__float_as_uint(ah[0]), __float_as_uint(ah[1]), __float_as_uint(ah[2]),
                         __float_as_uint(ah[3])};
  const uint32_t l[4] = {__float_as_uint(al[0]), __float_as_uint(al[1]), __float_as_uint(al[2]),
                         __float_as_uint(al[3])};
  mma_tf32(acc, l, __float_as_uint(b0h), __float_as_uint(b1h));
  mma_tf32(acc, h, __float_as_uint(b0l), __float_as_uint(b1l));
  mma_tf32(acc, h, __float_as_uint(b0h), __float_as_uint(b1h));
}

// BIG (D > 512 or H + 1 = 17, e.g. config 3: D = 784, H = 16): 16-row
// batches, one CTA per SM (up to 255 registers: 13-16 dimension tiles per
// warp), V fragments split on the fly (the pre-split table would not fit next
// to the row ring), fresh accumulators per k-step, and with H + 1 = 17 the
// constant column of [zhat; 1] (Y_v[:, H] = sum q v) accumulated by FFMA next
// to sq_v while the m16 tile holds the 16 latent columns.
__device__ __forceinline__ void dmma_e(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
template <int NTH, int NTW, bool BIG>
__global__ void __launch_bounds__(kStatsThreads, BIG ? 1 : 2) k_stats_mma(StatsArgs a, const int* __restrict__ itemoff,
                                                               int rows_per_item, int nh1, double* part,
                                                               int64_t part_stride, int nbuf) {
  constexpr int BR = BIG ? 16 : kSmBatch;  // rows per batch
  constexpr int MT = BR / 16;              // phase (i) m-tiles
  constexpr int KP = 8 / MT;               // phase (i) K parts
  // smem (dynamic): s_x [nbuf][BR][XS] | s_Vb [KS][NTH][32] float4 (BIG: float2) | s_mu [D]
  extern __shared__ __align__(16) float s_x[];
  __shared__ __align__(16) float s_pz[KP][BR][16];  // phase (i) K-part partials
  __shared__ __align__(16) float4 s_Af[BR / 8][32][2];  // phase (ii) A fragments (hi, lo) per k-step, lane
  __shared__ double s_zd[BR * kSmZD];  // [zhat; 1] rows in fp64 (E)
  __shared__ double s_red[kStatsThreads / 32];
  __shared__ double s_accE[BIG ? 1 : kStatsThreads];
  __shared__ uint64_t s_xbar[kStatsMaxBuf];
  // K-pairs per item, at most (the longer items where the static arrays fit: D <= 832)
  constexpr int MAXR = BIG && NTW <= 13 ? kStatsMaxRowsBig : kStatsMaxRows;
  __shared__ int s_eall[MAXR];
  __shared__ double s_qall[MAXR];
  __shared__ int s_item;
  __shared__ float s_qb[BR];  // the batch's responsibilities (fp32; 0 past the item end)
  const Dims dm = a.dm;
  const int H = dm.H, H1 = H + 1, D = dm.D;
  const int XS = D + 4;  // row stride: XS % 32 == 4 for D % 32 == 0 (conflict-free phase i)
  const int KS = D / 8;  // k-steps of phase (i) / dimension tiles of phase (ii)
  float4* s_Vb = reinterpret_cast<float4*>(s_x + (int64_t)nbuf * BR * XS);
  float2* s_Vu = reinterpret_cast<float2*>(s_Vb);  // BIG: unsplit (b0, b1)
  float* s_mu = BIG ? reinterpret_cast<float*>(s_Vu + (int64_t)KS * NTH * 32)
                    : reinterpret_cast<float*>(s_Vb + (int64_t)KS * NTH * 32);
  const bool cfma = H1 > 16;  // constant column by FFMA (BIG only)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  __shared__ double s_ecc[12][32];  // E tiles (warp 0's DMMA fragments, kept in shared memory between batches)
  // E: thread = (upper-triangle entry, row group)
  const int NE = H1 * (H1 + 1) / 2;
  const int EG = max(1, kStatsThreads / NE);
  const int eg = tid / NE;
  int ei = -1, ej = -1;
  if (eg < EG) {
    int t = tid - eg * NE;
    for (int i = 0; i < H1 && ei < 0; ++i) {
      if (t < H1 - i) ei = i, ej = i + t;
      else t -= H1 - i;
    }
  }
  // phase (i): warp = (m-tile, K part)
  const int pm = warp % MT, pq = warp / MT;
  const int ks0 = pq * KS / KP, ks1 = (pq + 1) * KS / KP;
  const int total = __ldg(itemoff + dm.C);
  if (tid == 0)
    for (int i = 0; i < kStatsMaxBuf; ++i) xbar_init(&s_xbar[i], 1);
  // rows past an item's end keep a previous batch's (finite) rows and get q = 0;
  // zeroed once so the first batches never see uninitialised (NaN) words
  for (int i = tid; i < nbuf * BR * XS; i += kStatsThreads) s_x[i] = 0.f;
  __syncthreads();
  uint32_t xpar = 0u;
  auto next_item = [&](int cur) -> int {
    if (!a.qctr) return cur < 0 ? static_cast<int>(blockIdx.x) : cur + static_cast<int>(gridDim.x);
    __syncthreads();
    if (tid == 0) s_item = atomicAdd(a.qctr, 1);
    __syncthreads();
    return s_item;
  };
  for (int item = next_item(-1); item < total; item = next_item(item)) {
    const int c = find_item(itemoff, dm.C, item);
    const int r0 = a.off[c] + (item - itemoff[c]) * rows_per_item;
    const int r1 = min(a.off[c + 1], r0 + rows_per_item);
    const int nr = r1 - r0;
    const bool direct = itemoff[c + 1] - itemoff[c] == 1;
    double qmax = 0.0;
    __syncthreads();
    for (int i = tid; i < nr; i += kStatsThreads) {
      const int e = a.ent[r0 + i];
      const double q = a.resp[e];
      s_eall[i] = e / dm.Cp;
      s_qall[i] = q;
      qmax = fmax(qmax, q);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) qmax = fmax(qmax, __shfl_xor_sync(kFull, qmax, o));
    if (lane == 0) s_red[warp] = qmax;
    // V^T fragments of phase (i), split: b0 = V[h][d = 8ks + tig], b1 = V[h][d + 4], h = 8nt + gid
    const float* Vc = a.V32 + (int64_t)c * D * H;
    for (int i = tid; i < KS * NTH * 32; i += kStatsThreads) {
      const int l = i & 31, t = i >> 5;
      const int ks = t / NTH, nt = t - ks * NTH;
      const int h = 8 * nt + (l >> 2), d = 8 * ks + (l & 3);
      const float b0 = h < H ? __ldg(Vc + (int64_t)d * H + h) : 0.f;
      const float b1 = h < H ? __ldg(Vc + (int64_t)(d + 4) * H + h) : 0.f;
      if (BIG) {
        s_Vu[i] = make_float2(b0, b1);
      } else {
        const float b0h = tf32_hi(b0), b1h = tf32_hi(b1);
        s_Vb[i] = make_float4(b0h, b1h, b0 - b0h, b1 - b1h);
      }
    }
    for (int d = tid; d < D; d += kStatsThreads) s_mu[d] = __ldg(a.mu32 + (int64_t)c * D + d);
    __syncthreads();
    qmax = 0.0;
#pragma unroll
    for (int w = 0; w < kStatsThreads / 32; ++w) qmax = fmax(qmax, s_red[w]);
    const double qdiv = qmax > 0.0 ? qmax : 1.0;
    const int nbat = (nr + BR - 1) / BR;
    for (int i = tid; i < nbat * BR; i += kStatsThreads) s_qall[i] = i < nr ? s_qall[i] / qdiv : 0.0;
    if (BIG && warp == 0)
#pragma unroll
      for (int i = 0; i < 12; ++i) s_ecc[i][lane] = 0.0;
    if (!BIG && ei >= 0) s_accE[tid] = 0.0;
    float acc[NTW][4];
    double sqd[NTW];  // sq_v: fp32 over a batch's rows per lane, then fp64
    double yhd[NTW];  // Y_v[:, H] when cfma
    float muj[NTW];
#pragma unroll
    for (int i = 0; i < NTW; ++i) {
      sqd[i] = 0.0;
      yhd[i] = 0.0;
      acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
      muj[i] = s_mu[8 * min(warp + 8 * i, KS - 1) + gid];
    }
    auto issue_rows = [&](int b, int buf) {
      float* dst = s_x + (int64_t)buf * BR * XS;
      const int nb = min(BR, nr - b * BR);
      const int* eb = s_eall + b * BR;
      if (tid == 0) xbar_expect(&s_xbar[buf], static_cast<uint32_t>(nb) * D * 4u);
      if (lane < BR / (kStatsThreads / 32)) {
        const int r = warp * (BR / (kStatsThreads / 32)) + lane;
        if (r < nb) bulk_row(smem_addr(dst + (int64_t)r * XS), a.X + (int64_t)eb[r] * D, D * 4u, &s_xbar[buf]);
      }
    };
    for (int b = 0; b < min(nbuf - 1, nbat); ++b) issue_rows(b, b);
    for (int bi = 0, buf = 0; bi < nbat; ++bi, buf = buf + 1 == nbuf ? 0 : buf + 1) {
      const int nb = min(BR, nr - bi * BR);
      xbar_wait(&s_xbar[buf], (xpar >> buf) & 1u);
      xpar ^= 1u << buf;
      const float* xb = s_x + (int64_t)buf * BR * XS;
      // (i) Z partial over this warp's K quarter: A = v rows 16pm.., B = V^T
      {
        // three independent chains (lo*hi, hi*lo, hi*hi) hide the HMMA latency
        float z3[3][NTH][4];
#pragma unroll
        for (int t = 0; t < 3; ++t)
#pragma unroll
          for (int nt = 0; nt < NTH; ++nt) z3[t][nt][0] = z3[t][nt][1] = z3[t][nt][2] = z3[t][nt][3] = 0.f;
        const float* xr0 = xb + (int64_t)(16 * pm + gid) * XS + tig;
        const float* xr1 = xr0 + 8 * XS;
#pragma unroll 4
        for (int ks = ks0; ks < ks1; ++ks) {
          const int d = 8 * ks;
          const float m0 = s_mu[d + tig], m1 = s_mu[d + tig + 4];
          const float v[4] = {xr0[d] - m0, xr1[d] - m0, xr0[d + 4] - m1, xr1[d + 4] - m1};
          float ah[4], al[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            ah[k] = tf32_hi(v[k]);
            al[k] = v[k] - ah[k];
          }
#pragma unroll
          for (int nt = 0; nt < NTH; ++nt) {
            float4 bv;
            if (BIG) {
              const float2 u = s_Vu[((int64_t)ks * NTH + nt) * 32 + lane];
              const float b0h = tf32_hi(u.x), b1h = tf32_hi(u.y);
              bv = make_float4(b0h, b1h, u.x - b0h, u.y - b1h);
            } else {
              bv = s_Vb[((int64_t)ks * NTH + nt) * 32 + lane];
            }
            const uint32_t h[4] = {__float_as_uint(ah[0]), __float_as_uint(ah[1]), __float_as_uint(ah[2]),
                                   __float_as_uint(ah[3])};
            const uint32_t l[4] = {__float_as_uint(al[0]), __float_as_uint(al[1]), __float_as_uint(al[2]),
                                   __float_as_uint(al[3])};
            mma_tf32(z3[0][nt], l, __float_as_uint(bv.x), __float_as_uint(bv.y));
            mma_tf32(z3[1][nt], h, __float_as_uint(bv.z), __float_as_uint(bv.w));
            mma_tf32(z3[2][nt], h, __float_as_uint(bv.x), __float_as_uint(bv.y));
          }
        }
        float z[NTH][4];
#pragma unroll
        for (int nt = 0; nt < NTH; ++nt)
#pragma unroll
          for (int k = 0; k < 4; ++k) z[nt][k] = (z3[0][nt][k] + z3[1][nt][k]) + z3[2][nt][k];
#pragma unroll
        for (int nt = 0; nt < NTH; ++nt) {
          *reinterpret_cast<float2*>(&s_pz[pq][16 * pm + gid][8 * nt + 2 * tig]) = make_float2(z[nt][0], z[nt][1]);
          *reinterpret_cast<float2*>(&s_pz[pq][16 * pm + gid + 8][8 * nt + 2 * tig]) =
              make_float2(z[nt][2], z[nt][3]);
        }
      }
      __syncthreads();
      if (nbuf >= 2 && bi + nbuf - 1 < nbat) issue_rows(bi + nbuf - 1, buf == 0 ? nbuf - 1 : buf - 1);
      // combine: zhat rows (fp64 for E) and the q-scaled phase (ii) A fragments
      const double* s_q = s_qall + bi * BR;
      if (tid < BR * 8) {
        // thread = (k-step, lane, row half): row r, columns gid and gid + 8
        const int ks = tid >> 6, ln = (tid >> 1) & 31, up = tid & 1;
        const int r = 8 * ks + (ln & 3) + 4 * up, h0 = ln >> 2, h1 = h0 + 8;
        auto zval = [&](int h) -> float {
          if (r >= nb || h > H) return 0.f;
          if (h == H) return 1.f;
          float z = 0.f;
#pragma unroll
          for (int k = 0; k < KP; ++k) z += s_pz[k][r][h];
          return z;
        };
        const float z0 = zval(h0), z1 = zval(h1);
        if (h0 < H1) s_zd[r * kSmZD + h0] = z0;
        if (h1 < H1) s_zd[r * kSmZD + h1] = z1;
        if (cfma && h0 == 0) s_zd[r * kSmZD + H] = r < nb ? 1.0 : 0.0;
        const float qf = static_cast<float>(s_q[r]);
        if (h0 == 0) s_qb[r] = qf;
        const float qz0 = qf * z0, qz1 = qf * z1;
        const float hi0 = tf32_hi(qz0), hi1 = tf32_hi(qz1);
        reinterpret_cast<float2*>(&s_Af[ks][ln][0])[up] = make_float2(hi0, hi1);
        reinterpret_cast<float2*>(&s_Af[ks][ln][1])[up] = make_float2(qz0 - hi0, qz1 - hi1);
      }
      __syncthreads();
      if (!BIG && ei >= 0) {  // (16 columns or fewer: a thread per upper-triangle entry)
        double e = s_accE[tid];
        for (int r = eg; r < nb; r += EG) e = fma(s_q[r], s_zd[r * kSmZD + ei] * s_zd[r * kSmZD + ej], e);
        s_accE[tid] = e;
      }
      if (BIG && warp == 0) {
        double ecc[6][2];
#pragma unroll
        for (int i = 0; i < 6; ++i) ecc[i][0] = s_ecc[2 * i][lane], ecc[i][1] = s_ecc[2 * i + 1][lane];
        // E += [zhat; 1]^T diag(q) [zhat; 1] over the batch rows by fp64 DMMA
        // m8n8k4 (k = 4 rows): A(g, t) = zhat[row t][8 mi + g], B(t, g) =
        // q_row zhat[row t][8 ni + g]; the 6 upper 8x8 tiles of the 24 x 24
        // padding (H1 <= 17), accumulated by warp 0 over the item
#pragma unroll
        for (int k0 = 0; k0 < BR; k0 += 4) {
          const int r = k0 + tig;
          const double q = r < nb ? s_q[r] : 0.0;
          double za[3], zq[3];
#pragma unroll
          for (int m = 0; m < 3; ++m) {
            const int col = 8 * m + gid;
            za[m] = (col < H1 && r < nb) ? s_zd[r * kSmZD + col] : 0.0;
            zq[m] = q * za[m];
          }
          dmma_e(ecc[0], za[0], zq[0]);
          dmma_e(ecc[1], za[0], zq[1]);
          dmma_e(ecc[2], za[0], zq[2]);
          dmma_e(ecc[3], za[1], zq[1]);
          dmma_e(ecc[4], za[1], zq[2]);
          dmma_e(ecc[5], za[2], zq[2]);
        }
#pragma unroll
        for (int i = 0; i < 6; ++i) s_ecc[2 * i][lane] = ecc[i][0], s_ecc[2 * i + 1][lane] = ecc[i][1];
      }
      // (ii) Y_v^T += (Q zhat)^T v over the batch's 4 k-steps (rows past nb:
      // q = 0 and A = 0, stale finite v), chained per batch, then one FADD
      // per accumulator into the item's sums
      float sqa[NTW], yha[NTW];
      float accb[BIG ? 1 : NTW][4], accl[BIG ? 1 : NTW][4];  // hi*hi chain and the correction products' chain
#pragma unroll
      for (int i = 0; i < NTW; ++i) sqa[i] = yha[i] = 0.f;
#pragma unroll
      for (int i = 0; i < (BIG ? 1 : NTW); ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) accb[i][k] = accl[i][k] = 0.f;
#pragma unroll
      for (int ks = 0; ks < BR / 8; ++ks) {
        const float4 Ah = s_Af[ks][lane][0], Al = s_Af[ks][lane][1];
        const float ah[4] = {Ah.x, Ah.y, Ah.z, Ah.w}, al[4] = {Al.x, Al.y, Al.z, Al.w};
        const int ra = 8 * ks + tig, rb = ra + 4;
        const float qa = s_qb[ra], qb = s_qb[rb];
        const float* xa = xb + (int64_t)ra * XS + gid;
        const float* xb2 = xb + (int64_t)rb * XS + gid;
#pragma unroll
        for (int i = 0; i < NTW; ++i) {
          // tiles past D/8 (D < 64 NTW) repeat the last tile; their sums are not written
          const int j = min(warp + 8 * i, KS - 1);
          const float va = xa[8 * j] - muj[i];
          const float vb = xb2[8 * j] - muj[i];
          const float qva = qa * va, qvb = qb * vb;
          sqa[i] = fmaf(qva, va, sqa[i]);
          sqa[i] = fmaf(qvb, vb, sqa[i]);
          if (BIG) yha[i] += qva + qvb;
          const float vah = tf32_hi(va), vbh = tf32_hi(vb);
          if (BIG) {
            mma3(acc[i], ah, al, vah, vbh, va - vah, vb - vbh);
          } else {
            const int ii = BIG ? 0 : i;
            const uint32_t h[4] = {__float_as_uint(ah[0]), __float_as_uint(ah[1]), __float_as_uint(ah[2]),
                                   __float_as_uint(ah[3])};
            const uint32_t l[4] = {__float_as_uint(al[0]), __float_as_uint(al[1]), __float_as_uint(al[2]),
                                   __float_as_uint(al[3])};
            mma_tf32(accl[ii], l, __float_as_uint(vah), __float_as_uint(vbh));
            mma_tf32(accl[ii], h, __float_as_uint(va - vah), __float_as_uint(vb - vbh));
            mma_tf32(accb[ii], h, __float_as_uint(vah), __float_as_uint(vbh));
          }
        }
      }
#pragma unroll
      for (int i = 0; i < NTW; ++i) {
        sqd[i] += sqa[i];
        if (BIG) yhd[i] += yha[i];
        if (!BIG) {
#pragma unroll
          for (int k = 0; k < 4; ++k) acc[i][k] += accl[BIG ? 0 : i][k] + accb[BIG ? 0 : i][k];
        }
      }
      if (nbuf == 1) __syncthreads();
    }
    // write: E (fp64, row groups summed in order), Y_v columns and sq_v, scaled by qmax
    double* pp = direct ? nullptr : part + (int64_t)item * part_stride;
    double* pe = direct ? a.E + (int64_t)c * H1 * H1 : pp + (int64_t)nh1 * D + D;
    __syncthreads();
    if (!BIG && ei >= 0 && eg == 0) {
      double e = 0.0;
      for (int g = 0; g < EG; ++g) e += s_accE[tid + g * NE];
      pe[ej * H1 + ei] = e * qmax;
      pe[ei * H1 + ej] = e * qmax;
    }
    if (BIG && warp == 0) {
      const int tmi[6] = {0, 0, 0, 1, 1, 2}, tni[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
      for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int e0 = 8 * tmi[i] + gid, e1 = 8 * tni[i] + 2 * tig + u;
          if (e0 < H1 && e1 < H1 && e0 <= e1) {
            pe[e1 * H1 + e0] = s_ecc[2 * i + u][lane] * qmax;
            pe[e0 * H1 + e1] = s_ecc[2 * i + u][lane] * qmax;
          }
        }
    }
#pragma unroll
    for (int i = 0; i < NTW; ++i) {
      const int j = warp + 8 * i;
      double s = sqd[i], yh = yhd[i];
      s += __shfl_xor_sync(kFull, s, 1);
      s += __shfl_xor_sync(kFull, s, 2);
      if (BIG) {
        yh += __shfl_xor_sync(kFull, yh, 1);
        yh += __shfl_xor_sync(kFull, yh, 2);
      }
      if (j >= KS) continue;
      const int d = 8 * j + 2 * tig;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int h = gid + 8 * (k >> 1), dd = d + (k & 1);
        if (h >= H1) continue;
        const double y = static_cast<double>(acc[i][k]) * qmax;
        if (direct) a.Y[((int64_t)c * H1 + h) * D + dd] = y;
        else pp[(int64_t)h * D + dd] = y;
      }
      if (tig == 0) {
        const double v = s * qmax;
        if (direct) a.sq[(int64_t)c * D + 8 * j + gid] = v;
        else pp[(int64_t)nh1 * D + 8 * j + gid] = v;
        if (cfma) {  // Y_v[:, H] (the constant column)
          const double y = yh * qmax;
          if (direct) a.Y[((int64_t)c * H1 + H) * D + 8 * j + gid] = y;
          else pp[(int64_t)H * D + 8 * j + gid] = y;
        }
      }
    }
  }
}

// Sum a component's item partials in item order into the statistics buffer.
// kind 0: Y/sq/E/N pass at column block col0 (width nh1); kind 1: E only.
__global__ void __launch_bounds__(256) k_stats_reduce(Dims dm, const int* __restrict__ itemoff,
                                                      const double* part, int64_t part_stride,
                                                      int kind, int col0, int nh1, int full_e,
                                                      double* Nc, double* E, double* Y, double* sq) {
  // one thread per output element of every component (coalesced over the
  // partial rows); items summed in item order (deterministic)
  const int D = dm.D, H1 = dm.H + 1;
  const int ncols = min(nh1, H1 - col0);
  const int64_t ny = kind == 1 ? 0 : (int64_t)ncols * D;
  const int64_t nsq = (kind == 0 && col0 == 0) ? D : 0;
  const int64_t ne = (kind == 1 || (col0 == 0 && full_e)) ? (int64_t)H1 * H1 : 0;
  const int64_t per = ny + nsq + ne;
  (void)Nc;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)dm.C * per;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int c = static_cast<int>(t / per);
    const int64_t k = t - (int64_t)c * per;
    const int i0 = __ldg(itemoff + c), i1 = __ldg(itemoff + c + 1);
    if (kind == 0 && i1 - i0 == 1) continue;  // written directly by k_stats
    int64_t src;
    double* dst;
    if (k < ny) {
      src = k;
      dst = Y + ((int64_t)c * H1 + col0) * D + k;
    } else if (k < ny + nsq) {
      src = (int64_t)nh1 * D + (k - ny);
      dst = sq + (int64_t)c * D + (k - ny);
    } else {
      src = kind == 1 ? (k - ny - nsq) : (int64_t)nh1 * D + D + (k - ny - nsq);
      dst = E + (int64_t)c * H1 * H1 + (k - ny - nsq);
    }
    double s = 0.0;
    for (int it = i0; it < i1; ++it) s += part[(int64_t)it * part_stride + src];
    *dst = s;
  }
}

// Restore the raw statistics from the centred ones (mu = the fp32 mean the
// rows were centred on): Y[:, h] = Y_v[:, h] + mu * E(h, H), sq = sq_v +
// 2 mu Y_v[:, H] + mu^2 N_c, with N_c = E(H, H) = sum q.
__global__ void k_stats_uncenter(Dims dm, const float* mu32, double* Nc, const double* E, double* Y,
                                 double* sq) {
  const int H1 = dm.H + 1, D = dm.D;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)dm.C * D;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = static_cast<int>(i / D), d = static_cast<int>(i - (int64_t)c * D);
    const double* Ec = E + (int64_t)c * H1 * H1;
    const double n = Ec[(int64_t)dm.H * H1 + dm.H];
    const double mu = static_cast<double>(mu32[i]);
    double* Yc = Y + (int64_t)c * H1 * D;
    const double yvH = Yc[(int64_t)dm.H * D + d];
    sq[i] += 2.0 * mu * yvH + mu * mu * n;
    for (int h = 0; h < H1; ++h) Yc[(int64_t)h * D + d] += mu * Ec[(int64_t)dm.H * H1 + h];
    if (d == 0) Nc[c] = n;
  }
}

// E_tl += N_c * Sigma_z (the per-row q Sigma_z terms of mstep.cpp:56, summed)
__global__ void k_stats_sz(Dims dm, const double* Nc, const double* Sz, double* E) {
  const int H = dm.H, H1 = H + 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)dm.C * H * H;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = static_cast<int>(i / (H * H));
    const int rem = static_cast<int>(i - (int64_t)c * H * H);
    const int col = rem / H, row = rem - col * H;
    E[(int64_t)c * H1 * H1 + col * H1 + row] += Nc[c] * Sz[i];
  }
}

// ---------------------------------------------------------------- small fp64 dense helpers (warp 0)
// Cholesky of the n x n SPD matrix A (col-major in smem) into R (row-major
// lower, smem). Returns via *ok (smem). Warp-cooperative over rows.
__device__ void warp_cholesky(const double* A, double* R, int n, int* ok) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < n * n; i += 32) R[i] = 0.0;
  __syncwarp();
  int good = 1;
  for (int j = 0; j < n; ++j) {
    double s = 0.0;
    for (int k = lane; k < j; k += 32) s += R[j * n + k] * R[j * n + k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    const double dj = A[j * n + j] - s;
    if (!(dj > 0.0) || !isfinite(dj)) {
      good = 0;
      break;
    }
    const double rjj = sqrt(dj);
    if (lane == 0) R[j * n + j] = rjj;
    for (int i = j + 1 + lane; i < n; i += 32) {
      double t = A[j * n + i];
      for (int k = 0; k < j; ++k) t -= R[i * n + k] * R[j * n + k];
      R[i * n + j] = t / rjj;
    }
    __syncwarp();
  }
  if (lane == 0) *ok = good;
}
// In-place solve of (R R^T) x = b for one right-hand side held by one thread.
__device__ __forceinline__ void chol_solve_thread(const double* R, double* b, int n) {
  for (int i = 0; i < n; ++i) {
    double s = b[i];
    for (int k = 0; k < i; ++k) s -= R[i * n + k] * b[k];
    b[i] = s / R[i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int k = i + 1; k < n; ++k) s -= R[k * n + i] * b[k];
    b[i] = s / R[i * n + i];
  }
}

// chol_solve_thread with compile-time loop bounds (b stays in registers; n <= HM)
template <int HM>
__device__ __forceinline__ void chol_solve_thread_t(const double* R, double* b, int n) {
#pragma unroll
  for (int i = 0; i < HM; ++i)
    if (i < n) {
      double s = b[i];
#pragma unroll
      for (int k = 0; k < i; ++k) s -= R[i * n + k] * b[k];
      b[i] = s / R[i * n + i];
    }
#pragma unroll
  for (int i = HM - 1; i >= 0; --i)
    if (i < n) {
      double s = b[i];
#pragma unroll
      for (int k = i + 1; k < HM; ++k)
        if (k < n) s -= R[k * n + i] * b[k];
      b[i] = s / R[i * n + i];
    }
}

__device__ __forceinline__ void dmma_f64_pre(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void set_status(unsigned long long* st, int c, int code) {
  atomicMin(st, (static_cast<unsigned long long>(c) << 8) | static_cast<unsigned long long>(code));
}

constexpr int kMaxH1 = 65;

// ---------------------------------------------------------------- K7: update_params
// The reference solves E_c A^T = Y_c^T with Eigen's LDLT (mstep.cpp:129-130):
// a left-looking LDL^T with diagonal pivoting. Restated semantics (Eigen >= 3.3,
// LDLT.h, ldlt_inplace<Lower>::unblocked and LDLT::_solve_impl):
//   * step k pivots on the largest |diagonal| among rows k.. (first index on a
//     tie) -- the trailing diagonal is the permuted ORIGINAL one, the Schur
//     update of entry (k,k) happens only at step k;
//   * d_k = A_kk - sum_j L_kj d_j L_kj; L_ik = (A_ik - sum_j L_ij d_j L_kj)/d_k
//     when d_k != 0, else the column must already be zero;
//   * the factorisation fails (info != Success) when a zero pivot is followed
//     by a non-zero one, or a zero pivot has a non-zero column; a matrix with
//     an all-zero diagonal "succeeds" with D = 0;
//   * solve: x = P^T L^-T D^+ L^-1 P b with D^+_i = 1/d_i if |d_i| > DBL_MIN
//     else 0 (pseudo-inverse of D).
// A: n x n column-major, full symmetric on entry; overwritten by L (strictly
// lower) and D (diagonal). perm: transpositions. Warp-cooperative.
__device__ void warp_ldlt(double* A, double* temp, int* perm, int n, int* ok) {
  const int lane = threadIdx.x & 31;
  auto M = [&](int r, int c) -> double& { return A[c * n + r]; };
  bool ret = true, found_zero = false;
  for (int k = 0; k < n; ++k) {
    // (1) largest |diagonal| among k.. (first index on a tie)
    double best = -1.0;
    int bi = n;
    for (int j = k + lane; j < n; j += 32) {
      const double v = fabs(M(j, j));
      if (v > best) best = v, bi = j;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(kFull, best, o);
      const int oi = __shfl_xor_sync(kFull, bi, o);
      if (ov > best || (ov == best && oi < bi)) best = ov, bi = oi;
    }
    const int p = bi < n ? bi : k;
    if (lane == 0) perm[k] = p;
    if (p != k) {  // symmetric transposition of rows / columns k and p
      for (int c = lane; c < n; c += 32) {
        const double t = M(k, c);
        M(k, c) = M(p, c);
        M(p, c) = t;
      }
      __syncwarp();
      for (int r = lane; r < n; r += 32) {
        const double t = M(r, k);
        M(r, k) = M(r, p);
        M(r, p) = t;
      }
      __syncwarp();
    }
    // (2) left-looking update of column k
    for (int j = lane; j < k; j += 32) temp[j] = M(j, j) * M(k, j);
    __syncwarp();
    double s = 0.0;
    for (int j = lane; j < k; j += 32) s += M(k, j) * temp[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    const double akk = M(k, k) - s;
    const bool valid = fabs(akk) > 0.0;
    if (k == 0 && !valid) {  // all-zero diagonal: D = 0, identity transpositions
      for (int j = lane; j < n; j += 32) perm[j] = j;
      __syncwarp();
      break;
    }
    int col_zero = 1;
    for (int i = k + 1 + lane; i < n; i += 32) {
      double t = M(i, k);
      for (int j = 0; j < k; ++j) t -= M(i, j) * temp[j];
      if (valid) t /= akk;
      else col_zero &= (t == 0.0);
      M(i, k) = t;
    }
    col_zero = __all_sync(kFull, col_zero);
    __syncwarp();
    if (lane == 0) M(k, k) = akk;
    if (!valid && k + 1 < n) ret = ret && col_zero;
    if (found_zero && valid) ret = false;
    else if (!valid) found_zero = true;
    __syncwarp();
  }
  if (lane == 0) *ok = ret ? 1 : 0;
}
// x = P^T L^-T D^+ L^-1 P b for one right-hand side held by one thread.
__device__ __forceinline__ void ldlt_solve_thread(const double* A, const int* perm, double* b, int n) {
  for (int k = 0; k < n; ++k) {
    const int p = perm[k];
    const double t = b[k];
    b[k] = b[p];
    b[p] = t;
  }
  for (int i = 0; i < n; ++i) {
    double s = b[i];
    for (int j = 0; j < i; ++j) s -= A[j * n + i] * b[j];
    b[i] = s;
  }
  for (int i = 0; i < n; ++i) {
    const double d = A[i * n + i];
    b[i] = fabs(d) > DBL_MIN ? b[i] / d : 0.0;
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int j = i + 1; j < n; ++j) s -= A[i * n + j] * b[j];
    b[i] = s;
  }
  for (int k = n - 1; k >= 0; --k) {
    const int p = perm[k];
    const double t = b[k];
    b[k] = b[p];
    b[p] = t;
  }
}

// CTA per component (mstep.cpp:117-153): freeze on N_c == 0 exactly; else
// pi = N_c/N, A^T = E^-1 Y^T by LDLT (one trace-scaled jitter retry on
// failure or a non-finite solution, else SingularEc), Lambda / mu from A,
// sigma^2 = max(floor, (sq - sum_h Y.A)/N_c).
// HM != 0: H + 1 <= HM, the per-dimension solve in registers (the
// transpositions composed once into s_idx: b is gathered permuted, the
// solution scattered back to natural order through shared memory s_x)
template <int HM>
__global__ void __launch_bounds__(128) k_update(UpdateArgs a) {
  extern __shared__ __align__(16) double s_upd[];
  __shared__ int s_ok, s_fin;
  __shared__ int s_perm[kMaxH1], s_idx[kMaxH1];
  __shared__ double s_tmp[kMaxH1], s_dinv[kMaxH1];
  const Dims dm = a.dm;
  const int H = dm.H, H1 = H + 1, D = dm.D;
  double* sE = s_upd;              // E_c (+ jitter)
  double* sF = s_upd + H1 * H1;    // LDLT factors
  double* s_x = sF + H1 * H1;      // [H1][blockDim] natural-order solutions (HM != 0)
  const int tid = threadIdx.x;
  for (int c = blockIdx.x; c < dm.C; c += gridDim.x) {
    const double nc = a.Nc[c];
    if (nc == 0.0) {  // mstep.cpp:119-126
      for (int d = tid; d < D; d += blockDim.x) {
        a.mu[(int64_t)c * D + d] = a.mu_prev[(int64_t)c * D + d];
        a.psi[(int64_t)c * D + d] = a.psi_prev[(int64_t)c * D + d];
      }
      for (int i = tid; i < D * H; i += blockDim.x) a.lam[(int64_t)c * D * H + i] = a.lam_prev[(int64_t)c * D * H + i];
      if (tid == 0) a.pi[c] = 0.0;
      continue;
    }
    for (int i = tid; i < H1 * H1; i += blockDim.x) sE[i] = a.E[(int64_t)c * H1 * H1 + i];
    __syncthreads();
    bool solved = false;
    for (int attempt = 0; attempt < 2 && !solved; ++attempt) {
      if (attempt == 1) {  // mstep.cpp:133-135: E_c += 1e-10 tr(E_c)/(H+1) I
        if (tid == 0) {
          double tr = 0.0;
          for (int i = 0; i < H1; ++i) tr += sE[i * H1 + i];
          const double jit = 1e-10 * tr / H1;
          for (int i = 0; i < H1; ++i) sE[i * H1 + i] += jit;
        }
        __syncthreads();
      }
      for (int i = tid; i < H1 * H1; i += blockDim.x) sF[i] = sE[i];
      __syncthreads();
      if (tid < 32) warp_ldlt(sF, s_tmp, s_perm, H1, &s_ok);
      if (tid == 0) s_fin = 1;
      __syncthreads();
      if (!s_ok) continue;
      // solve per d and write (provisionally) -- all finite required
      if constexpr (HM != 0) {
        if (tid < H1) {
          const double dd = sF[tid * H1 + tid];
          s_dinv[tid] = fabs(dd) > DBL_MIN ? 1.0 / dd : 0.0;
        }
        if (tid == 0) {
          for (int i = 0; i < H1; ++i) s_idx[i] = i;
          for (int k = 0; k < H1; ++k) {
            const int p = s_perm[k], t = s_idx[k];
            s_idx[k] = s_idx[p];
            s_idx[p] = t;
          }
        }
        __syncthreads();
        const double* Yc = a.Y + (int64_t)c * H1 * D;
        for (int d = tid; d < D; d += blockDim.x) {
          double b[HM];
#pragma unroll
          for (int i = 0; i < HM; ++i) b[i] = i < H1 ? Yc[(int64_t)s_idx[i] * D + d] : 0.0;  // P b
#pragma unroll
          for (int i = 0; i < HM; ++i)  // L^-1
            if (i < H1) {
              double t = b[i];
#pragma unroll
              for (int j = 0; j < i; ++j) t -= sF[j * H1 + i] * b[j];
              b[i] = t;
            }
#pragma unroll
          for (int i = 0; i < HM; ++i)  // D^+ (reciprocals formed once per component)
            if (i < H1) b[i] *= s_dinv[i];
#pragma unroll
          for (int i = HM - 1; i >= 0; --i)  // L^-T
            if (i < H1) {
              double t = b[i];
#pragma unroll
              for (int j = i + 1; j < HM; ++j)
                if (j < H1) t -= sF[i * H1 + j] * b[j];
              b[i] = t;
            }
#pragma unroll
          for (int i = 0; i < HM; ++i)  // P^T
            if (i < H1) s_x[s_idx[i] * blockDim.x + tid] = b[i];
          bool fin = true;
          double fitted = 0.0;
#pragma unroll
          for (int h = 0; h < HM; ++h)
            if (h < H1) {
              const double x = s_x[h * blockDim.x + tid];
              fin &= isfinite(x);
              fitted += Yc[(int64_t)h * D + d] * x;
              if (h < H) a.lam[(int64_t)c * D * H + (int64_t)h * D + d] = x;
              else a.mu[(int64_t)c * D + d] = x;
            }
          if (!fin) s_fin = 0;
          a.psi[(int64_t)c * D + d] = fmax((a.sq[(int64_t)c * D + d] - fitted) / nc, a.floor[d]);
        }
      } else
      for (int d = tid; d < D; d += blockDim.x) {
        double b[kMaxH1];
        for (int h = 0; h < H1; ++h) b[h] = a.Y[((int64_t)c * H1 + h) * D + d];
        ldlt_solve_thread(sF, s_perm, b, H1);
        bool fin = true;
        for (int h = 0; h < H1; ++h) fin &= isfinite(b[h]);
        if (!fin) s_fin = 0;
        double fitted = 0.0;
        for (int h = 0; h < H1; ++h) fitted += a.Y[((int64_t)c * H1 + h) * D + d] * b[h];
        for (int h = 0; h < H; ++h) a.lam[(int64_t)c * D * H + (int64_t)h * D + d] = b[h];
        a.mu[(int64_t)c * D + d] = b[H];
        a.psi[(int64_t)c * D + d] = fmax((a.sq[(int64_t)c * D + d] - fitted) / nc, a.floor[d]);
      }
      __syncthreads();
      solved = s_fin != 0;
    }
    if (tid == 0) {
      if (!solved) set_status(a.status, c, 5 /* SingularEc */);
      a.pi[c] = nc / static_cast<double>(dm.Ntot);
    }
    __syncthreads();
  }
}

// pi /= sum(pi) (mstep.cpp:156-160); deterministic single-CTA reduction.
__global__ void __launch_bounds__(1024) k_renorm(Dims dm, double* pi, unsigned long long* status) {
  __shared__ double red[1024];
  double s = 0.0;
  for (int c = threadIdx.x; c < dm.C; c += 1024) s += pi[c];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  const double live = red[0];
  if (live <= 0.0) {
    if (threadIdx.x == 0) set_status(status, 0xffffff, 5);
    return;
  }
  for (int c = threadIdx.x; c < dm.C; c += 1024) pi[c] /= live;
}

// ---------------------------------------------------------------- K8: precompute
// CTA per component (model.cpp:43-73) in fp64: L = I + Lambda^T Psi^-1 Lambda
// (symmetrised), Cholesky L = R R^T (+1e-10 I retry, else CholeskyFailure),
// Sigma_z = L^-1, log|Sigma| = 2 sum log R_hh + sum log psi, log pi; fp32
// scoring rows W = U R^-T (| W^T v |^2 = (U^T v).(V v)), V32 = R^-T R^-1 U^T.
constexpr int kPreFastH = 8;  // precompute's register-blocked M for H <= 8
constexpr int kPreDC = 32;    // dimensions per staged chunk of the general-H path

template <int HM>
__global__ void __launch_bounds__(128) k_precompute(PrecompArgs a) {
  extern __shared__ __align__(16) double s_pre[];
  __shared__ double red[128];
  __shared__ double s_mpart[4][kPreFastH * (kPreFastH + 1) / 2];
  __shared__ int s_ok;
  const Dims dm = a.dm;
  const int H = dm.H, D = dm.D;
  double* sL = s_pre;
  double* sR = s_pre + H * H;
  // H > kPreFastH: staged chunks of kPreDC dimensions (H4 x kPreDC each) and
  // the per-slice partial 4x4 tiles of M
  const int H4 = (H + 3) & ~3;
  double* sA = s_pre + 2 * H * H;
  double* sB = sA + H4 * kPreDC;
  double* s_ip = sA;  // Psi^-1 of the component (M stage; overlays sA / sB)
  double* sP = sA + max(2 * H4 * kPreDC, D);
  const int NT = H4 / 4, ntile = NT * (NT + 1) / 2;
  const int nsl = max(1, static_cast<int>(blockDim.x) / ntile);  // dimension slices per tile
  const int tid = threadIdx.x;
  for (int c = blockIdx.x; c < dm.C; c += gridDim.x) {
    const double* lam = a.lam + (int64_t)c * D * H;
    const double* psi = a.psi + (int64_t)c * D;
    // M = Lambda^T Psi^-1 Lambda (+I), symmetrised (model.cpp:51-53): every
    // thread sums its dimensions for all upper entries (H <= kPreFastH), then
    // a warp-shuffle + fixed-order cross-warp reduction; else 4x4 register
    // tiles of the upper triangle, each tile's dimensions split over nsl
    // threads (slices), the slice partials summed in a fixed order
    if constexpr (HM == kPreFastH) {
      const int np = H * (H + 1) / 2;
      double acc[kPreFastH * (kPreFastH + 1) / 2];
#pragma unroll
      for (int p = 0; p < kPreFastH * (kPreFastH + 1) / 2; ++p) acc[p] = 0.0;
      for (int d = tid; d < D; d += blockDim.x) {
        const double w = 1.0 / psi[d];
        double u[kPreFastH];
#pragma unroll
        for (int i = 0; i < kPreFastH; ++i) u[i] = i < H ? lam[(int64_t)i * D + d] : 0.0;
        int p = 0;
#pragma unroll
        for (int j = 0; j < kPreFastH; ++j)
#pragma unroll
          for (int i = 0; i <= j; ++i, ++p) acc[p] += u[i] * (u[j] * w);
      }
      const int lane = tid & 31, warp = tid >> 5;
      int p = 0;
#pragma unroll
      for (int j = 0; j < kPreFastH; ++j)
#pragma unroll
        for (int i = 0; i <= j; ++i, ++p) {
          double v = acc[p];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
          if (lane == 0 && j < H) s_mpart[warp][p] = v;
        }
      __syncthreads();
      for (int q = tid; q < np; q += blockDim.x) {
        // q -> (i, j) with the same packing as above
        int jj = 0, off = 0;
        while (off + jj + 1 <= q) off += ++jj;
        const int ii = q - off;
        double v = 0.0;
        for (int w2 = 0; w2 < static_cast<int>(blockDim.x >> 5); ++w2) v += s_mpart[w2][q];
        sL[jj * H + ii] = v;
      }
    } else {
      const int nwork = ntile * nsl;
      for (int d = tid; d < D; d += blockDim.x) s_ip[d] = 1.0 / psi[d];
      __syncthreads();
      for (int t0 = 0; t0 < nwork; t0 += blockDim.x) {
        const int t = t0 + tid;
        const bool act = t < nwork;
        const int sl = t % nsl, tile = t / nsl;  // a tile's slices adjacent: neighbouring dimensions per warp
        int bi = 0, bj = 0;
        {
          int r = act ? tile : 0;
          while (r >= NT - bi) r -= NT - bi, ++bi;
          bj = bi + r;
        }
        double acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
        if (act) {
          // straight from global memory (no staging barriers), 2 dimensions in flight
          const double* la = lam + (int64_t)(4 * bi) * D;
          const double* lb = lam + (int64_t)(4 * bj) * D;
          int d = sl;
          for (; d + nsl < D; d += 2 * nsl) {
            double av[2][4], bv[2][4];
#pragma unroll
            for (int e = 0; e < 2; ++e)
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const int dd = d + e * nsl;
                av[e][k] = 4 * bi + k < H ? la[(int64_t)k * D + dd] : 0.0;
                bv[e][k] = 4 * bj + k < H ? lb[(int64_t)k * D + dd] * s_ip[dd] : 0.0;
              }
#pragma unroll
            for (int e = 0; e < 2; ++e)
#pragma unroll
              for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[e][i], bv[e][j], acc[i][j]);
          }
          for (; d < D; d += nsl) {
            double av[4], bv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              av[k] = 4 * bi + k < H ? la[(int64_t)k * D + d] : 0.0;
              bv[k] = 4 * bj + k < H ? lb[(int64_t)k * D + d] * s_ip[d] : 0.0;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
          }
        }
        if (act)
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) sP[((int64_t)sl * ntile + tile) * 16 + i * 4 + j] = acc[i][j];
        __syncthreads();
        // this round's tiles: all of them (nsl > 1: one round) or [t0, t0 + blockDim)
        const int tlo = nsl > 1 ? 0 : t0, thi = nsl > 1 ? ntile : min(ntile, t0 + static_cast<int>(blockDim.x));
        for (int e = tid; e < (thi - tlo) * 16; e += blockDim.x) {
          const int tl = tlo + e / 16, ij = e % 16;
          double v = 0.0;
          for (int s2 = 0; s2 < nsl; ++s2) v += sP[((int64_t)s2 * ntile + tl) * 16 + ij];
          int ti = 0, r = tl;
          while (r >= NT - ti) r -= NT - ti, ++ti;
          const int ii = 4 * ti + ij / 4, jj = 4 * (ti + r) + ij % 4;
          if (ii < H && jj < H && ii <= jj) sL[jj * H + ii] = v;
        }
        __syncthreads();
      }
    }
    __syncthreads();
    for (int p = tid; p < H * H; p += blockDim.x) {
      const int i = p % H, j = p / H;
      if (i <= j) continue;
      sL[j * H + i] = sL[i * H + j];  // lower from upper
    }
    __syncthreads();
    for (int p = tid; p < H * H; p += blockDim.x) {
      const int i = p % H, j = p / H;
      // (M + I) symmetrised: 0.5 (M_ij + M_ji) with exact symmetry already
      double v = sL[p] + (i == j ? 1.0 : 0.0);
      a.Lmat[(int64_t)c * H * H + p] = v;
    }
    __syncthreads();
    for (int p = tid; p < H * H; p += blockDim.x) sL[p] = a.Lmat[(int64_t)c * H * H + p];
    __syncthreads();
    if (tid < 32) warp_cholesky(sL, sR, H, &s_ok);
    __syncthreads();
    if (!s_ok) {  // model.cpp:55-63
      if (tid == 0)
        for (int i = 0; i < H; ++i) sL[i * H + i] += 1e-10;
      __syncthreads();
      if (tid < 32) warp_cholesky(sL, sR, H, &s_ok);
      __syncthreads();
      if (!s_ok) {
        if (tid == 0) set_status(a.status, c, 2 /* CholeskyFailure */);
        continue;
      }
      for (int p = tid; p < H * H; p += blockDim.x) a.Lmat[(int64_t)c * H * H + p] = sL[p];
    }
    for (int p = tid; p < H * H; p += blockDim.x) a.R[(int64_t)c * H * H + p] = sR[p];
    // Sigma_z = L^-1 (model.cpp:65)
    for (int j = tid; j < H; j += blockDim.x) {
      if constexpr (HM != 0) {
        double b[HM];
#pragma unroll
        for (int h = 0; h < HM; ++h) b[h] = h == j ? 1.0 : 0.0;
        chol_solve_thread_t<HM>(sR, b, H);
#pragma unroll
        for (int h = 0; h < HM; ++h)
          if (h < H) a.Sz[(int64_t)c * H * H + j * H + h] = b[h];
      } else {
        double b[kMaxH1];
        for (int h = 0; h < H; ++h) b[h] = h == j ? 1.0 : 0.0;
        chol_solve_thread(sR, b, H);
        for (int h = 0; h < H; ++h) a.Sz[(int64_t)c * H * H + j * H + h] = b[h];
      }
    }
    // log|Sigma| (model.cpp:67-70): deterministic block reduction of sum log psi
    double s = 0.0;
    for (int d = tid; d < D; d += blockDim.x) s += log(psi[d]);
    red[tid] = s;
    __syncthreads();
    for (int o = 64; o > 0; o >>= 1) {
      if (tid < o) red[tid] += red[tid + o];
      __syncthreads();
    }
    if (tid == 0) {
      double ld = 0.0;
      for (int h = 0; h < H; ++h) ld += log(sR[h * H + h]);
      const double logdet = 2.0 * ld + red[0];
      const double p = a.pi[c];
      const double lp = p > 0.0 ? log(p) : -INFINITY;  // model.cpp:71
      a.logdet[c] = logdet;
      a.logpi[c] = lp;
      a.kconst[c] = lp - 0.5 * (D * kLog2Pi + logdet);
    }
    // fp32 scoring rows: W = U R^-T (P, WT) and V = R^-T W (V32) per dimension
    const int HP = a.L.HP, Hc = a.L.Hc;
    if constexpr (HM != 0) {
      // the per-dimension rows: k_precompute_rows (fully parallel over (c, d))
    } else {
      // W^T = R^-1 U^T and V = Sigma_z U^T (= L^-1 U^T, model.cpp:64) as
      // register-tiled products over staged chunks of U^T = (Psi^-1 Lambda)^T:
      // R^-1 (lower, one column per thread) into sL, Sigma_z into sR
      __syncthreads();
      for (int p = tid; p < H * H; p += blockDim.x) sL[p] = 0.0;
      __syncthreads();
      for (int j = tid; j < H; j += blockDim.x)
        for (int i = j; i < H; ++i) {
          double t = i == j ? 1.0 : 0.0;
          for (int k = j; k < i; ++k) t -= sR[i * H + k] * sL[k * H + j];
          sL[i * H + j] = t / sR[i * H + i];
        }
      __syncthreads();
      for (int p = tid; p < H * H; p += blockDim.x) sR[p] = a.Sz[(int64_t)c * H * H + p];
      const int TD = kPreDC / 4, ntile = (H4 / 4) * TD;
      for (int d0 = 0; d0 < D; d0 += kPreDC) {
        __syncthreads();
        for (int i = tid; i < H4 * kPreDC; i += blockDim.x) {
          const int h = i / kPreDC, d = d0 + (i - h * kPreDC);
          sA[i] = (h < H && d < D) ? lam[(int64_t)h * D + d] * (1.0 / psi[d]) : 0.0;  // U = Psi^-1 Lambda
        }
        __syncthreads();
        for (int t = tid; t < ntile; t += blockDim.x) {
          const int h0 = 4 * (t / TD), dd0 = 4 * (t - (t / TD) * TD);
          double w[4][4], v[4][4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) w[i][j] = v[i][j] = 0.0;
          for (int k = 0; k < H; ++k) {
            double ri[4], si[4], uk[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int h = h0 + i;
              ri[i] = (h < H && k <= h) ? sL[h * H + k] : 0.0;
              si[i] = h < H ? sR[h * H + k] : 0.0;  // Sigma_z (symmetric): row h
              uk[i] = sA[k * kPreDC + dd0 + i];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                w[i][j] = fma(ri[i], uk[j], w[i][j]);
                v[i][j] = fma(si[i], uk[j], v[i][j]);
              }
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int d = d0 + dd0 + j;
            if (d >= D) continue;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int h = h0 + i;
              if (h >= H) continue;
              if (a.P) a.P[((int64_t)c * D + d) * HP + h] = static_cast<float>(w[i][j]);
              a.WT[((int64_t)c * a.Hp + h) * D + d] = static_cast<float>(w[i][j]);
              if (a.W64) a.W64[((int64_t)c * H + h) * D + d] = w[i][j];
              a.V32[((int64_t)c * D + d) * H + h] = static_cast<float>(v[i][j]);
            }
          }
        }
        // the per-dimension tail of the rows: zero padding, mean, Psi^-1
        for (int dd = tid; dd < kPreDC; dd += blockDim.x) {
          const int d = d0 + dd;
          if (d >= D) continue;
          const double ip = 1.0 / psi[d];
          if (a.P) {
            float* row = a.P + ((int64_t)c * D + d) * HP;
            for (int h = H; h < Hc; ++h) row[h] = 0.f;
            row[Hc] = static_cast<float>(a.mu[(int64_t)c * D + d]);
            row[Hc + 1] = static_cast<float>(ip);
            row[Hc + 2] = 0.f;
            row[Hc + 3] = 0.f;
          }
          for (int h = H; h < a.Hp; ++h) a.WT[((int64_t)c * a.Hp + h) * D + d] = 0.f;
          a.ipsi32[(int64_t)c * D + d] = static_cast<float>(ip);
          a.mu32[(int64_t)c * D + d] = static_cast<float>(a.mu[(int64_t)c * D + d]);
        }
      }
    }
    __syncthreads();
  }
}

// k_precompute for H <= 16 with a WARP per component (no block barriers, 8
// components in flight per CTA): M = Lambda^T Psi^-1 Lambda by fp64 DMMA
// m8n8k4 (the upper 8x8 tiles, k = 4 dimensions; A(g, t) = Lambda[8 mi + g][d],
// B(t, g) = Lambda[8 ni + g][d] / psi_d), symmetrised from the upper
// triangle, + I; Cholesky by the warp (+1e-10 retry -> CholeskyFailure),
// Sigma_z by lanes 0..H-1, log|Sigma| by a warp reduction (model.cpp:43-73).
// The per-dimension scoring rows follow in k_precompute_rows.
constexpr int kPreWarps = 8;
__global__ void __launch_bounds__(kPreWarps * 32) k_precompute_w(PrecompArgs a) {
  __shared__ double s_L[kPreWarps][16 * 16], s_R[kPreWarps][16 * 16];
  __shared__ int s_ok[kPreWarps];
  const Dims dm = a.dm;
  const int H = dm.H, D = dm.D;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double* sL = s_L[warp];
  double* sR = s_R[warp];
  const int nt = (H + 7) / 8;  // 8 x 8 tiles per side (1 or 2)
  for (int c = blockIdx.x * kPreWarps + warp; c < dm.C; c += gridDim.x * kPreWarps) {
    const double* lam = a.lam + (int64_t)c * D * H;
    const double* psi = a.psi + (int64_t)c * D;
    double acc[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};  // tiles (0,0), (0,1), (1,1)
    double lsum = 0.0;  // sum log psi over this lane's dimensions
#pragma unroll 4
    for (int d0 = 0; d0 < D; d0 += 4) {
      const int d = d0 + t;
      const bool dv = d < D;
      const double ip = dv ? 1.0 / psi[d] : 0.0;
      if (dv && g == 0) lsum += log(psi[d]);
      double av[2], bv[2];
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int h = 8 * m + g;
        av[m] = (m < nt && h < H && dv) ? lam[(int64_t)h * D + d] : 0.0;
        bv[m] = av[m] * ip;
      }
      dmma_f64_pre(acc[0], av[0], bv[0]);
      if (nt > 1) {
        dmma_f64_pre(acc[1], av[0], bv[1]);
        dmma_f64_pre(acc[2], av[1], bv[1]);
      }
    }
    // M tiles -> sL (upper, then mirrored), + I
    {
      const int tmi[3] = {0, 0, 1}, tni[3] = {0, 1, 1};
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        if (i > 0 && nt < 2) break;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int r = 8 * tmi[i] + g, cc = 8 * tni[i] + 2 * t + u;
          if (r < H && cc < H && r <= cc) {
            sL[r * H + cc] = acc[i][u];
            sL[cc * H + r] = acc[i][u];
          }
        }
      }
    }
    __syncwarp();
    for (int p = lane; p < H * H; p += 32) {
      const int i = p % H, j = p / H;
      const double v = sL[p] + (i == j ? 1.0 : 0.0);
      sL[p] = v;
      a.Lmat[(int64_t)c * H * H + p] = v;
    }
    __syncwarp();
    warp_cholesky(sL, sR, H, &s_ok[warp]);
    __syncwarp();
    if (!s_ok[warp]) {  // model.cpp:55-63
      if (lane < H) sL[lane * H + lane] += 1e-10;
      __syncwarp();
      warp_cholesky(sL, sR, H, &s_ok[warp]);
      __syncwarp();
      if (!s_ok[warp]) {
        if (lane == 0) set_status(a.status, c, 2 /* CholeskyFailure */);
        continue;
      }
      for (int p = lane; p < H * H; p += 32) a.Lmat[(int64_t)c * H * H + p] = sL[p];
    }
    for (int p = lane; p < H * H; p += 32) a.R[(int64_t)c * H * H + p] = sR[p];
    if (lane < H) {  // Sigma_z = L^-1 (model.cpp:65), column `lane`
      double b[16];
#pragma unroll
      for (int h = 0; h < 16; ++h) b[h] = h == lane ? 1.0 : 0.0;
      chol_solve_thread_t<16>(sR, b, H);
#pragma unroll
      for (int h = 0; h < 16; ++h)
        if (h < H) a.Sz[(int64_t)c * H * H + lane * H + h] = b[h];
    }
    // log|Sigma| (model.cpp:67-70): fixed-order warp reduction of sum log psi
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(kFull, lsum, o);
    if (lane == 0) {
      double ld = 0.0;
      for (int h = 0; h < H; ++h) ld += log(sR[h * H + h]);
      const double logdet = 2.0 * ld + lsum;
      const double pp = a.pi[c];
      const double lp = pp > 0.0 ? log(pp) : -INFINITY;  // model.cpp:71
      a.logdet[c] = logdet;
      a.logpi[c] = lp;
      a.kconst[c] = lp - 0.5 * (D * kLog2Pi + logdet);
    }
    __syncwarp();
  }
}

// The fp32 scoring rows of k_precompute for H <= HM, a thread per (c, d): U =
// Psi^-1 Lambda, w = R^-1 u (P, WT, W64), v = R^-T w = Sigma_z u (V32), with
// the solves in registers (reciprocal diagonals) -- the per-component kernel
// above only forms L, R, Sigma_z and the constants.
template <int HM>
__global__ void __launch_bounds__(128) k_precompute_rows(PrecompArgs a) {
  __shared__ double sR[HM * HM];
  __shared__ double s_rinv[HM];
  const Dims dm = a.dm;
  const int H = dm.H, D = dm.D, c = blockIdx.y, tid = threadIdx.x;
  const int HP = a.L.HP, Hc = a.L.Hc;
  for (int p = tid; p < H * H; p += blockDim.x) sR[p] = a.R[(int64_t)c * H * H + p];
  __syncthreads();
  if (tid < H) s_rinv[tid] = 1.0 / sR[tid * H + tid];
  __syncthreads();
  const double* lam = a.lam + (int64_t)c * D * H;
  const double* psi = a.psi + (int64_t)c * D;
  for (int d = blockIdx.x * blockDim.x + tid; d < D; d += gridDim.x * blockDim.x) {
    double u[HM];
    const double ip = 1.0 / psi[d];
#pragma unroll
    for (int h = 0; h < HM; ++h) u[h] = h < H ? lam[(int64_t)h * D + d] * ip : 0.0;  // U = Psi^-1 Lambda
#pragma unroll
    for (int i = 0; i < HM; ++i) {  // forward: w = R^-1 u
      if (i < H) {
        double t = u[i];
#pragma unroll
        for (int k = 0; k < i; ++k) t -= sR[i * H + k] * u[k];
        u[i] = t * s_rinv[i];
      }
    }
#pragma unroll
    for (int h = 0; h < HM; ++h)
      if (h < H) {
        a.WT[((int64_t)c * a.Hp + h) * D + d] = static_cast<float>(u[h]);
        if (a.W64) a.W64[((int64_t)c * H + h) * D + d] = u[h];
      }
    for (int h = H; h < a.Hp; ++h) a.WT[((int64_t)c * a.Hp + h) * D + d] = 0.f;
    const double mud = a.mu[(int64_t)c * D + d];
    a.ipsi32[(int64_t)c * D + d] = static_cast<float>(ip);
    a.mu32[(int64_t)c * D + d] = static_cast<float>(mud);
    if (a.P) {  // the FFMA scorer's packed rows (only that scorer reads them)
      float* row = a.P + ((int64_t)c * D + d) * HP;
#pragma unroll
      for (int h = 0; h < HM; ++h)
        if (h < H) row[h] = static_cast<float>(u[h]);
      for (int h = H; h < Hc; ++h) row[h] = 0.f;
      row[Hc] = static_cast<float>(mud);
      row[Hc + 1] = static_cast<float>(ip);
      row[Hc + 2] = 0.f;
      row[Hc + 3] = 0.f;
    }
#pragma unroll
    for (int i = HM - 1; i >= 0; --i) {  // backward: v = R^-T w => V column d
      if (i < H) {
        double t = u[i];
#pragma unroll
        for (int k = i + 1; k < HM; ++k)
          if (k < H) t -= sR[k * H + i] * u[k];
        u[i] = t * s_rinv[i];
      }
    }
    float* vrow = a.V32 + ((int64_t)c * D + d) * H;
    if ((H & 3) == 0) {  // 16-byte stores
#pragma unroll
      for (int h = 0; h < HM; h += 4)
        if (h < H)
          *reinterpret_cast<float4*>(vrow + h) = make_float4(static_cast<float>(u[h]), static_cast<float>(u[h + 1]),
                                                             static_cast<float>(u[h + 2]), static_cast<float>(u[h + 3]));
    } else {
#pragma unroll
      for (int h = 0; h < HM; ++h)
        if (h < H) vrow[h] = static_cast<float>(u[h]);
    }
  }
}

// Full fp64 U (D x H col-major) and V (H x D col-major) for cache downloads.
__global__ void __launch_bounds__(128) k_caches_full(Dims dm, const double* lam, const double* psi,
                                                    const double* R, double* U, double* V,
                                                    double* ipsi) {
  const int H = dm.H, D = dm.D;
  for (int c = blockIdx.x; c < dm.C; c += gridDim.x) {
    const double* Rc = R + (int64_t)c * H * H;
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
      double u[kMaxH1];
      const double ip = 1.0 / psi[(int64_t)c * D + d];
      ipsi[(int64_t)c * D + d] = ip;
      for (int h = 0; h < H; ++h) {
        u[h] = ip * lam[(int64_t)c * D * H + (int64_t)h * D + d];
        U[(int64_t)c * D * H + (int64_t)h * D + d] = u[h];
      }
      chol_solve_thread(Rc, u, H);
      for (int h = 0; h < H; ++h) V[(int64_t)c * D * H + (int64_t)d * H + h] = u[h];
    }
  }
}

// ---------------------------------------------------------------- reductions
__global__ void k_lse_rows(const float* LJK, int64_t N, int Cp, double* lse) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < N; n += (int64_t)gridDim.x * blockDim.x) {
    double mx = -INFINITY;
    for (int j = 0; j < Cp; ++j) mx = fmax(mx, static_cast<double>(LJK[n * Cp + j]));
    double l = mx;
    if (isfinite(mx)) {
      double s = 0.0;
      for (int j = 0; j < Cp; ++j) s += exp(static_cast<double>(LJK[n * Cp + j]) - mx);
      l = mx + log(s);
    }
    lse[n] = l;
  }
}

// em_full_step (mstep.cpp:164-208): full responsibilities of a row chunk
// from its dense log-joints, q(n, c) = exp(l(n, c) - LSE_n) in fp64, laid
// out as the "K-pairs" of a context whose K rows are all C components (entry
// n * C + c), plus the component-major CSR of those entries (rows ascending)
__global__ void k_em_resp(const float* LJ, int64_t R, int SL, int C, const double* lse, double* resp, int* ent,
                          int* off) {
  const int64_t total = R * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = i / C;
    const int c = static_cast<int>(i - n * C);
    resp[i] = exp(static_cast<double>(LJ[n * SL + c]) - lse[n]);  // NaN rows as the reference's (App. E.4)
    ent[(int64_t)c * R + n] = static_cast<int>(i);
    if (i <= C) off[i] = static_cast<int>(i * R);  // off[c] = c * R (c = 0..C)
  }
}
__global__ void k_add_f64(const double* a, double* acc, int64_t n, int first) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc[i] = first ? a[i] : acc[i] + a[i];
}

// ---------------------------------------------------------------- AFK-MC^2 seeding (seeding.cpp:60-121)
// The reference's default seeding (seeding.hpp:14-17). Bit-identical to the
// oracle's restatement: squared distances in fp64 by explicit fma over d in
// ascending order, the proposal q and its cdf built sequentially, the
// xoshiro256++ stream (rng.hpp:30-86) advanced in the reference's order.
// k_afk_q: distances of every row to the first center (one thread per row);
// k_afk_cdf: q normalised and its cdf (one thread, the reference's order);
// k_afk_chain: the Metropolis chains (one CTA; thread 0 draws, the block
// computes distance_to_centers as a min over centers, exact in any order).
// squared_distance by one warp: lane l sums d = l, l + 32, ... (explicit fma,
// ascending), then the xor butterfly (every lane ends with the same value:
// the halving tree v[l] += v[l + o], o = 16..1, that the oracle restates)
__device__ __forceinline__ double afk_sqd_warp(const float* X, int D, int64_t a, int64_t b, int lane) {
  const float* xa = X + a * D;
  const float* xb = X + b * D;
  double t = 0.0;
  for (int d = lane; d < D; d += 32) {
    const double v = static_cast<double>(__ldg(xa + d)) - static_cast<double>(__ldg(xb + d));
    t = fma(v, v, t);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(kFull, t, o);
  return t;
}
struct AfkState {
  unsigned long long w[4];
};
__device__ __forceinline__ unsigned long long afk_next(AfkState& s) {
  auto rotl = [](unsigned long long x, int k) { return (x << k) | (x >> (64 - k)); };
  const unsigned long long out = rotl(s.w[0] + s.w[3], 23) + s.w[0];
  const unsigned long long t = s.w[1] << 17;
  s.w[2] ^= s.w[0];
  s.w[3] ^= s.w[1];
  s.w[1] ^= s.w[2];
  s.w[0] ^= s.w[3];
  s.w[2] ^= t;
  s.w[3] = rotl(s.w[3], 45);
  return out;
}
__device__ __forceinline__ double afk_unit(AfkState& s) { return static_cast<double>(afk_next(s) >> 11) * 0x1.0p-53; }

__global__ void k_afk_q(const float* X, int64_t N, int D, const int64_t* centers, double* q) {
  const int64_t c0 = centers[0];
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < N; i += nw) {
    const double d = afk_sqd_warp(X, D, i, c0, lane);
    if (lane == 0) q[i] = d;
  }
}
__global__ void k_afk_cdf(int64_t N, double* q, double* cdf) {
  double sum = 0.0;
  for (int64_t i = 0; i < N; ++i) sum += q[i];
  const double uniform_part = 0.5 / static_cast<double>(N);
  double acc = 0.0;
  for (int64_t i = 0; i < N; ++i) {
    const double a = sum > 0.0 ? 0.5 * q[i] / sum : 0.0;
    q[i] = a + uniform_part;
    acc += q[i];
    cdf[i] = acc;
  }
}
constexpr int kAfkThreads = 1024;
__global__ void __launch_bounds__(kAfkThreads) k_afk_chain(const float* X, int64_t N, int D, int C, int m,
                                                          const double* q, const double* cdf, int64_t* centers,
                                                          unsigned long long* state, unsigned long long* count,
                                                          int* degenerate) {
  __shared__ AfkState s_rng;
  __shared__ double s_red[kAfkThreads / 32];
  __shared__ int64_t s_idx[kAfkThreads / 32];
  __shared__ int64_t s_pick;
  __shared__ int s_flag;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int k = 0; k < 4; ++k) s_rng.w[k] = state[k];
  }
  unsigned long long cnt = 0;  // thread 0's squared_distance tally
  __syncthreads();
  // distance_to_centers (seeding.cpp:41-49) of row n to the first nc centers
  auto to_centers = [&](int64_t n, int nc) -> double {
    double best = INFINITY;  // warp per center
    for (int k = warp; k < nc; k += kAfkThreads / 32) best = fmin(best, afk_sqd_warp(X, D, n, centers[k], lane));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = fmin(best, __shfl_xor_sync(kFull, best, o));
    __syncthreads();
    if (lane == 0) s_red[warp] = best;
    __syncthreads();
    best = INFINITY;
    for (int w = 0; w < kAfkThreads / 32; ++w) best = fmin(best, s_red[w]);
    if (tid == 0) cnt += nc;
    return best;
  };
  // draw_from_cdf (seeding.cpp:51-56) by thread 0, broadcast
  auto draw = [&]() -> int64_t {
    __syncthreads();
    if (tid == 0) {
      const double u = afk_unit(s_rng) * cdf[N - 1];
      int64_t lo = 0, hi = N;  // first index with cdf > u
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (cdf[mid] > u) hi = mid;
        else lo = mid + 1;
      }
      s_pick = lo < N - 1 ? lo : N - 1;
    }
    __syncthreads();
    return s_pick;
  };
  for (int nc = 1; nc < C; ++nc) {
    int64_t x = draw();
    double dx = to_centers(x, nc);
    for (int step = 1; step < m; ++step) {
      const int64_t y = draw();
      const double dy = to_centers(y, nc);
      if (dy <= 0.0) continue;  // duplicates of chosen centers never accepted
      bool accept = dx <= 0.0;
      if (!accept) {
        __syncthreads();
        if (tid == 0) s_flag = afk_unit(s_rng) < (dy * q[x]) / (dx * q[y]) ? 1 : 0;
        __syncthreads();
        accept = s_flag != 0;
      }
      if (accept) {
        x = y;
        dx = dy;
      }
    }
    if (dx <= 0.0) {  // every proposal duplicated a chosen center: farthest point (first on ties)
      double best = -1.0;  // warp per row (rows ascending within a warp: first max kept)
      int64_t bi = -1;
      for (int64_t i = warp; i < N; i += kAfkThreads / 32) {
        double d = INFINITY;
        for (int k = 0; k < nc; ++k) d = fmin(d, afk_sqd_warp(X, D, i, centers[k], lane));
        if (d > best) best = d, bi = i;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(kFull, best, o);
        const int64_t oi = __shfl_xor_sync(kFull, bi, o);
        if (ob > best || (ob == best && oi >= 0 && (bi < 0 || oi < bi))) best = ob, bi = oi;
      }
      __syncthreads();
      if (lane == 0) s_red[warp] = best, s_idx[warp] = bi;
      __syncthreads();
      if (tid == 0) {
        double b = -1.0;
        int64_t ib = -1;
        for (int w = 0; w < kAfkThreads / 32; ++w)
          if (s_red[w] > b || (s_red[w] == b && s_idx[w] >= 0 && (ib < 0 || s_idx[w] < ib))) b = s_red[w], ib = s_idx[w];
        s_pick = ib;
        cnt += static_cast<unsigned long long>(N) * nc;
        if (!(b > 0.0)) *degenerate = 1;  // fewer than C distinct rows (count_distinct_rows, :65-67)
      }
      __syncthreads();
      x = s_pick;
    }
    if (tid == 0) centers[nc] = x;
    __syncthreads();
  }
  if (tid == 0) {
    for (int k = 0; k < 4; ++k) state[k] = s_rng.w[k];
    *count = cnt;
  }
}

// per-row log-sum-exp over the C dense slots (exact_log_likelihood,
// model.cpp:101-148): warp per row, fixed-order butterflies (deterministic)
__global__ void k_lse_dense(const float* LJ, int64_t R, int SL, int C, double* lse) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t n = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; n < R; n += nw) {
    const float* l = LJ + n * SL;
    double mx = -INFINITY;
    for (int c = lane; c < C; c += 32) mx = fmax(mx, static_cast<double>(l[c]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
    double out = mx;
    if (isfinite(mx)) {
      double sum = 0.0;
      for (int c = lane; c < C; c += 32) sum += exp(static_cast<double>(l[c]) - mx);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(kFull, sum, o);
      out = mx + log(sum);
    }
    if (lane == 0) lse[n] = out;
  }
}

// LJK[n][j] = the anchor-pass log-joint of (n, K(n)[j]) under the current
// parameters: anchor c = K(n)[j] scores itself in slot j*G + pos(c in g_c)
// (mu_c centring, delta = 0 -- the same arithmetic as a one-component pass).
__global__ void k_self_slots(Dims dm, const int* K, const int* g, const int* gcnt, const float* LJ, float* LJK) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < dm.N * dm.Cp;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = i / dm.Cp;
    const int j = static_cast<int>(i - n * dm.Cp);
    const int c = K[i];
    const int* gc = g + (int64_t)c * dm.G;
    int pos = 0;
    for (int t = 0; t < gcnt[c]; ++t)
      if (gc[t] == c) pos = t;
    LJK[i] = LJ[n * dm.SL + j * dm.G + pos];
  }
}

constexpr int kSumBlocks = 296;
// Two-stage deterministic sum: fixed contiguous segments per CTA, fixed tree.
__global__ void __launch_bounds__(256) k_sum_stage1(const double* v, int64_t n, double* partials) {
  __shared__ double red[256];
  const int64_t seg = (n + gridDim.x - 1) / gridDim.x;
  const int64_t b = blockIdx.x * seg, e = (n < b + seg) ? n : b + seg;
  double s = 0.0;
  for (int64_t i = b + threadIdx.x; i < e; i += 256) s += v[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = red[0];
}
__global__ void __launch_bounds__(32) k_sum_stage2(const double* partials, int m, double* out) {
  __shared__ double s_p[kSumBlocks];
  for (int i = threadIdx.x; i < m; i += 32) s_p[i] = partials[i];  // lane-parallel loads
  __syncwarp();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += s_p[i];  // fixed order
    *out = s;
  }
}
__global__ void k_sum_i32(const int* v, int64_t n, unsigned long long* out) {
  unsigned long long s = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += static_cast<unsigned long long>(v[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}
// VarState::validate for K (estep.cpp:15-68): rows sorted, distinct, in range;
// the first offending row (smallest n) is reported through *bad (init INT_MAX)
__global__ void k_validate_K(const int* K, int64_t N, int Cp, int C, long long* bad) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < N; n += (int64_t)gridDim.x * blockDim.x) {
    bool ok = true;
    for (int j = 0; j < Cp; ++j) {
      const int v = K[n * Cp + j];
      ok &= v >= 0 && v < C && (j == 0 || v > K[n * Cp + j - 1]);
    }
    if (!ok) atomicMin(bad, static_cast<long long>(n));
  }
}

__global__ void k_count_empty(const double* pi, int C, int* out) {
  int s = 0;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) s += pi[c] == 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}
__global__ void k_logpi(const double* pi, int C, double* logpi) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x)
    logpi[c] = pi[c] > 0.0 ? log(pi[c]) : -INFINITY;
}

int grid_for(int64_t n, int threads, int cap) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<int>(g);
}

}  // namespace

cudaError_t ensure_dyn_smem(const void* kern, size_t bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, size_t>> done;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : done)
    if (e.first == kern) {
      if (e.second >= bytes) return cudaSuccess;
      const cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(bytes));
      if (r == cudaSuccess) e.second = bytes;
      return r;
    }
  const cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (r == cudaSuccess) done.emplace_back(kern, bytes);
  return r;
}

int sm_count() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (cached <= 0) cached = 148;
  }
  return cached;
}

cudaError_t launch_iota(int* v, int64_t n, cudaStream_t s) {
  k_iota<<<grid_for(n, 256, 4096), 256, 0, s>>>(v, n);
  return cudaGetLastError();
}
cudaError_t launch_fill_i32(int* v, int64_t n, int value, cudaStream_t s) {
  k_fill_i32<<<grid_for(n, 256, 4096), 256, 0, s>>>(v, n, value);
  return cudaGetLastError();
}
cudaError_t launch_keys_from_i32(const int* src, unsigned* keys, int64_t n, cudaStream_t s) {
  k_keys_from_i32<<<grid_for(n, 256, 4096), 256, 0, s>>>(src, keys, n);
  return cudaGetLastError();
}
cudaError_t launch_hist(const unsigned* keys, int64_t n, int C, int* cnt, cudaStream_t s) {
  k_hist<<<grid_for(n, 256, 4096), 256, 0, s>>>(keys, n, C, cnt);
  return cudaGetLastError();
}
cudaError_t launch_offsets_sorted(const unsigned* sorted, int64_t n, int C, int* off, cudaStream_t s) {
  k_offsets_scan<<<grid_for(n + 1, 256, 8192), 256, 0, s>>>(sorted, n, C, off);
  return cudaGetLastError();
}
cudaError_t launch_items_scan(const int* off, int C, int rows, int min1, int* items, cudaStream_t s) {
  k_items_scan<<<1, 1024, 0, s>>>(off, C, rows, min1, items);
  return cudaGetLastError();
}
cudaError_t launch_chunks(const int* cnt, int C, int rows, int* chunks, cudaStream_t s) {
  k_chunks<<<grid_for(C + 1, 256, 4096), 256, 0, s>>>(cnt, C, rows, chunks);
  return cudaGetLastError();
}
cudaError_t launch_chunks_from_off(const int* off, int C, int rows, int min1, int* chunks, cudaStream_t s) {
  k_chunks_from_off<<<grid_for(C + 1, 256, 4096), 256, 0, s>>>(off, C, rows, min1, chunks);
  return cudaGetLastError();
}
cudaError_t launch_extra(const Dims& dm, const int* K, const int* g, const int* gcnt,
                         const unsigned long long* sit, int* rx, unsigned* rkey, cudaStream_t s) {
  k_extra<<<grid_for(dm.N, 256, 8192), 256, 0, s>>>(dm, K, g, gcnt, sit, rx, rkey);
  return cudaGetLastError();
}

template <int MODE>
static cudaError_t launch_score_mode(const ScoreArgs& a, int grid, cudaStream_t s) {
  const size_t smem = static_cast<size_t>(a.dm.D) * kXsStride * sizeof(float);
  auto go = [&](auto kern) {
    ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
    kern<<<grid, kScoreThreads, smem, s>>>(a);
  };
  if (a.L.hc == 4) go(k_score<MODE, 4>);
  else if (a.L.hc == 8) go(k_score<MODE, 8>);
  else go(k_score<MODE, 16>);
  return cudaGetLastError();
}
cudaError_t launch_score(int mode, const ScoreArgs& a, int grid, cudaStream_t s) {
  if (mode == kModeAnchor) return launch_score_mode<kModeAnchor>(a, grid, s);
  if (mode == kModeExtra) return launch_score_mode<kModeExtra>(a, grid, s);
  return launch_score_mode<kModeTruncF>(a, grid, s);
}

cudaError_t launch_select(const SelectArgs& a, cudaStream_t s) {
  const int ns = (a.dm.SL + 31) / 32;
  const int grid = grid_for(a.dm.N * 32, 256, sm_count() * 32);  // (16 per SM: 1.01 ms at config 3, 32: 0.98)
  // 8 warps' bitmaps + their anchor log-joints and ranks
  const size_t hs = ns <= 2 ? 0 : ns <= 4 ? 256 : 512;  // k_select's per-warp hash (key + value), NS > 2 only
  const size_t smem = static_cast<size_t>((a.dm.C + 31) / 32) * 8 * sizeof(unsigned) +
                      64 * (sizeof(float) + sizeof(int)) + 8 * hs * 8;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  auto go = [&](auto kern) {
    ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
    kern<<<grid, 256, smem, s>>>(a);
  };
  switch (ns) {
    case 1: go(k_select<1>); break;
    case 2: go(k_select<2>); break;
    case 3: go(k_select<3>); break;
    case 4: go(k_select<4>); break;
    case 5: go(k_select<5>); break;
    case 6: go(k_select<6>); break;
    case 7: go(k_select<7>); break;
    case 8: go(k_select<8>); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

int gupd_capmax(const Dims& dm, int pts_per_item) {
  const long long bound = std::min<long long>((long long)dm.C - 1, (long long)pts_per_item * (dm.stride - 1));
  int cap = 32;
  while (cap < 2 * bound && cap < kGupdCap) cap <<= 1;
  return cap;
}
cudaError_t launch_gupdate(const GupdArgs& a, int grid, cudaStream_t s) {
  int capmax = gupd_capmax(a.dm, a.pts_per_item);
  if (a.force_rows) capmax = std::min(capmax, kGupdRowsCap);
  size_t smem = static_cast<size_t>(capmax) * (2 * sizeof(long long) + 2 * sizeof(int));
  // small C: a dense (cnt, hi, lo) row per CTA in shared memory -- no hash
  // probing, and 24 C bytes instead of 24 cap (config 3: 96 KB, two CTAs per SM)
  if (a.dm.C <= kGupdDenseMax && !a.dump) {
    capmax = -1;
    smem = static_cast<size_t>(a.dm.C) * (2 * sizeof(long long) + sizeof(unsigned));
  }
  ensure_dyn_smem(reinterpret_cast<const void*>(k_gupdate), smem);
  k_gupdate<<<grid, kGupdThreads, smem, s>>>(a, capmax);
  return cudaGetLastError();
}
cudaError_t launch_cooc_heads(const CoocArgs& a, cudaStream_t s) {
  if (a.n > 0) k_cooc_heads<<<grid_for(a.n, 256, sm_count() * 8), 256, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_cooc_sums(const CoocArgs& a, cudaStream_t s) {
  if (a.n > 0) k_cooc_sums<<<grid_for(a.n, 256, sm_count() * 8), 256, 0, s>>>(a);
  k_cooc_offsets<<<grid_for(a.dm.C + 1, 256, sm_count() * 4), 256, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_cooc_select(const CoocArgs& a, int c0, int c1, int zero_others, int* g_new, int* gcnt_new,
                               cudaStream_t s) {
  k_cooc_select<<<grid_for(a.dm.C, 8, sm_count() * 8), 256, 0, s>>>(a, c0, c1, zero_others, g_new, gcnt_new);
  return cudaGetLastError();
}
cudaError_t launch_gselect_dense(const Dims& dm, long long* xc, const int* itemoff, int all,
                                 int* g_new, int* gcnt_new, cudaStream_t s) {
  k_gselect_dense<<<min(dm.C, sm_count() * 8), kGupdThreads, 0, s>>>(dm, xc, itemoff, all, g_new, gcnt_new);
  return cudaGetLastError();
}

template <int NH1>
static void stats_pass(const StatsArgs& a, const int* itemoff, int rpi, int grid, int col0,
                       double* part, int64_t ps, cudaStream_t s) {
  const int D = a.dm.D;
  constexpr int NZ = NH1 == kStatsMaxH1 ? NH1 : NH1 - 1;
  constexpr int VS = (NZ + 3) / 4 * 4, ZS = (NH1 + 3) / 4 * 4;
  const size_t XS = (D + 3) / 4 * 4 + kXPad;
  const size_t fixed = (static_cast<size_t>(D) * VS + (D + 3) / 4 * 4 + 4 + 8 * kStatsBatch * NZ +
                        kStatsBatch * ZS + 8) * sizeof(float) + kStatsBatch * ZS * sizeof(double);
  const size_t per_buf = static_cast<size_t>(kStatsBatch) * XS * sizeof(float);
  // the row-group reduction reuses the row buffers: RG-1 slices of GD*4*(NH1+1) doubles
  const int GD = (D + 3) / 4;
  const int RG = std::max(1, kStatsThreads / GD);
  const size_t red = static_cast<size_t>(std::max(RG - 1, 0)) * GD * 4 * (NH1 + 1) * sizeof(double);
  static const int want = [] {
    const char* v = std::getenv("VMFA_STATS_NBUF");
    return v ? std::atoi(v) : 0;
  }();
  int nbuf = (2 * per_buf + fixed <= 200 * 1024) ? 2 : 1;
  if (static_cast<size_t>(nbuf) * per_buf < red) nbuf = 2;
  if (want > 2)  // deeper ring when it fits
    for (int nb = std::min(kStatsMaxBuf, want > 0 ? want : 2); nb > nbuf; --nb)
      if (nb * per_buf + fixed <= 200 * 1024) {
        nbuf = nb;
        break;
      }
  const size_t smem = std::max(static_cast<size_t>(nbuf) * per_buf, red) + fixed;
  auto go = [&](auto kern) {
    ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
    kern<<<grid, kStatsThreads, smem, s>>>(a, itemoff, rpi, col0, part, ps, nbuf);
  };
  if (GD <= kStatsThreads) go(k_stats<NH1, 1>);
  else go(k_stats<NH1, 2>);
}
int64_t stats_part_stride(const Dims& dm) {
  const int H1 = dm.H + 1;
  const int nh1 = H1 <= 5 ? 5 : (H1 <= 9 ? 9 : kStatsMaxH1);
  return static_cast<int64_t>(nh1) * dm.D + dm.D + static_cast<int64_t>(H1) * H1 + 1;
}
// the tensor-core statistics kernel covers H + 1 <= 17 (one m16 tile of
// [zhat; 1], the 17th column by FFMA) and D % 8 == 0, D <= 1024;
// VMFA_STATS=ffma selects k_stats (the cross-check in the parity tests)
bool stats_mma_ok(const Dims& dm) {
  const char* v = std::getenv("VMFA_STATS");
  const bool ffma = v && std::strcmp(v, "ffma") == 0;
  return !ffma && dm.D % 8 == 0 && ((dm.H + 1 <= 16 && dm.D <= 512) || (dm.H + 1 <= 17 && dm.D <= 1024));
}
// BIG variant: 16-row batches, one CTA per SM (D > 256: the 2-CTA variant
// would spill its 8 dimension tiles per warp; or H + 1 = 17)
static bool stats_mma_big(const Dims& dm) { return dm.D > 256 || dm.H + 1 > 16; }
// the tcgen05 statistics kernel (vmfa_stats_tc.cu) is opt-in (VMFA_STATS=tc):
// parity-tested, but measured 2-3x slower than k_stats_mma on configs 1-3
// (GEMM ii reduces over rows, so every row chunk is produced twice and the
// synchronous cooperative fills stay latency-bound)
// K-pairs per statistics item, at most: with the BIG tensor-core variant most
// components are a single item (written directly, no partial rows to reduce)
int stats_rows_cap(const Dims& dm) {
  return stats_mma_ok(dm) && stats_mma_big(dm) && dm.D <= 832 && !stats_use_tc(dm) ? kStatsMaxRowsBig : kStatsMaxRows;
}
bool stats_use_tc(const Dims& dm) {
  const char* v = std::getenv("VMFA_STATS");
  return v && std::strcmp(v, "tc") == 0 && stats_tc_ok(dm);
}
cudaError_t launch_stats(const StatsArgs& a, const int* itemoff, int rows_per_item, double* part,
                         cudaStream_t s) {
  if (a.dm.D > 4 * kStatsThreads) return cudaErrorInvalidValue;
  const int grid = sm_count() * 4;
  const int H1 = a.dm.H + 1;
  const int nh1 = H1 <= 5 ? 5 : (H1 <= 9 ? 9 : kStatsMaxH1);
  const int64_t ps = stats_part_stride(a.dm);
  if (a.xmax && a.mumax && a.zbuf && a.qctr && rows_per_item == stats_tc_rows() && stats_use_tc(a.dm)) {
    cudaError_t e = launch_stats_tc(a, a.xmax, a.mumax, itemoff, nh1, part, ps, s);
    if (e != cudaSuccess) return e;
    k_stats_reduce<<<sm_count() * 8, 256, 0, s>>>(a.dm, itemoff, part, ps, 0, 0, nh1, 1, a.Nc, a.E, a.Y, a.sq);
    k_stats_uncenter<<<grid_for((int64_t)a.dm.C * a.dm.D, 256, 8192), 256, 0, s>>>(a.dm, a.mu32, a.Nc, a.E, a.Y,
                                                                                  a.sq);
    k_stats_sz<<<grid_for((int64_t)a.dm.C * a.dm.H * a.dm.H, 256, 4096), 256, 0, s>>>(a.dm, a.Nc, a.Sz, a.E);
    return cudaGetLastError();
  }
  if (stats_mma_ok(a.dm)) {
    if (a.qctr) {
      cudaError_t e = cudaMemsetAsync(a.qctr, 0, sizeof(int), s);
      if (e != cudaSuccess) return e;
    }
    const bool big = stats_mma_big(a.dm);
    const int KS = a.dm.D / 8, NTH = (big || a.dm.H > 8) ? 2 : 1;
    const int ntw = (KS + 7) / 8;
    const int BR = big ? 16 : kSmBatch;
    const size_t per_buf = static_cast<size_t>(BR) * (a.dm.D + 4) * sizeof(float);
    const size_t fixed = static_cast<size_t>(KS) * NTH * 32 * (big ? 8 : 16) + a.dm.D * sizeof(float);
    // row-batch ring: 2 deep at 2 CTAs per SM (deeper rings at 1 CTA per SM
    // measured slower: 0.93 vs 0.67 ms on config 2); BIG: 1 CTA per SM
    static const int want = [] {
      const char* v = std::getenv("VMFA_STATS_NBUF");
      return v ? std::atoi(v) : 0;
    }();
    const size_t budget = 200 * 1024 - 32 * 1024;  // minus the static smem
    int nbuf = want > 0 ? std::min(want, kStatsMaxBuf) : 2;
    while (nbuf > 2 && nbuf * per_buf + fixed > budget) --nbuf;
    const int per_sm = (!big && nbuf <= 2) ? 2 : 1;  // 2 x (66.5 + 17 KB dynamic + 30 KB static) fits at D = 256
    const size_t smem = nbuf * per_buf + fixed;
    auto go = [&](auto kern) {
      ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
      kern<<<sm_count() * per_sm, kStatsThreads, smem, s>>>(a, itemoff, rows_per_item, nh1, part, ps, nbuf);
    };
    if (big) {
      if (ntw <= 4) go(k_stats_mma<2, 4, true>);
      else if (ntw <= 8) go(k_stats_mma<2, 8, true>);
      else if (ntw <= 13) go(k_stats_mma<2, 13, true>);
      else go(k_stats_mma<2, 16, true>);
    } else if (NTH == 1) {
      if (ntw <= 1) go(k_stats_mma<1, 1, false>);
      else if (ntw <= 2) go(k_stats_mma<1, 2, false>);
      else go(k_stats_mma<1, 4, false>);
    } else {
      if (ntw <= 1) go(k_stats_mma<2, 1, false>);
      else if (ntw <= 2) go(k_stats_mma<2, 2, false>);
      else go(k_stats_mma<2, 4, false>);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_stats_reduce<<<sm_count() * 8, 256, 0, s>>>(a.dm, itemoff, part, ps, 0, 0, nh1, 1, a.Nc, a.E, a.Y, a.sq);
    k_stats_uncenter<<<grid_for((int64_t)a.dm.C * a.dm.D, 256, 8192), 256, 0, s>>>(a.dm, a.mu32, a.Nc, a.E, a.Y,
                                                                                  a.sq);
    k_stats_sz<<<grid_for((int64_t)a.dm.C * a.dm.H * a.dm.H, 256, 4096), 256, 0, s>>>(a.dm, a.Nc, a.Sz, a.E);
    return cudaGetLastError();
  }
  for (int col0 = 0; col0 < H1; col0 += nh1) {
    if (a.qctr) {
      cudaError_t e = cudaMemsetAsync(a.qctr, 0, sizeof(int), s);
      if (e != cudaSuccess) return e;
    }
    if (nh1 == 5) stats_pass<5>(a, itemoff, rows_per_item, grid, col0, part, ps, s);
    else if (nh1 == 9) stats_pass<9>(a, itemoff, rows_per_item, grid, col0, part, ps, s);
    else stats_pass<kStatsMaxH1>(a, itemoff, rows_per_item, grid, col0, part, ps, s);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_stats_reduce<<<sm_count() * 8, 256, 0, s>>>(a.dm, itemoff, part, ps, 0, col0, nh1, H1 <= nh1 ? 1 : 0,
                                                  a.Nc, a.E, a.Y, a.sq);
  }
  if (H1 > nh1) {
    const size_t smem = 2 * static_cast<size_t>(kStatsBatch) * kEZS * sizeof(double);
    ensure_dyn_smem(reinterpret_cast<const void*>(k_stats_E), smem);
    k_stats_E<<<grid, kStatsThreads, smem, s>>>(a, itemoff, rows_per_item, part, ps);
    k_stats_reduce<<<sm_count() * 8, 256, 0, s>>>(a.dm, itemoff, part, ps, 1, 0, nh1, 1, a.Nc, a.E, a.Y, a.sq);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  k_stats_uncenter<<<grid_for((int64_t)a.dm.C * a.dm.D, 256, 8192), 256, 0, s>>>(a.dm, a.mu32, a.Nc, a.E, a.Y, a.sq);
  k_stats_sz<<<grid_for((int64_t)a.dm.C * a.dm.H * a.dm.H, 256, 4096), 256, 0, s>>>(a.dm, a.Nc, a.Sz, a.E);
  return cudaGetLastError();
}
}  // namespace
extern "C" int vmfa_diag_stats_cycles(int enable, unsigned long long* out) {
  using namespace vmfa_b200;
  cudaMemcpyToSymbol(g_stats_prof_on, &enable, sizeof(int));
  if (out) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_stats_prof, sizeof(unsigned long long) * 16);
  }
  unsigned long long z[16] = {};
  if (out || !enable) cudaMemcpyToSymbol(g_stats_prof, z, sizeof(z));
  return 0;
}
namespace vmfa_b200 {
cudaError_t launch_update(const UpdateArgs& a, cudaStream_t s) {
  const int H1 = a.dm.H + 1;
  const size_t smem = (2 * static_cast<size_t>(H1) * H1 + static_cast<size_t>(H1) * 128) * sizeof(double);
  auto go = [&](auto kern) {
    ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
    // a block per component: 8 blocks per SM left a second wave at a third of
    // the occupancy (config 3: 0.635 -> 0.55 ms)
    kern<<<a.dm.C, 128, smem, s>>>(a);
  };
  if (H1 <= 5) go(k_update<5>);
  else if (H1 <= 9) go(k_update<9>);
  else if (H1 <= 17) go(k_update<17>);
  else if (H1 <= 33) go(k_update<33>);
  else go(k_update<0>);
  return cudaGetLastError();
}
cudaError_t launch_renorm(const Dims& dm, double* pi, unsigned long long* status, cudaStream_t s) {
  k_renorm<<<1, 1024, 0, s>>>(dm, pi, status);
  return cudaGetLastError();
}
cudaError_t launch_precompute(const PrecompArgs& a, cudaStream_t s) {
  const int H = a.dm.H;
  const size_t H4 = (static_cast<size_t>(H) + 3) & ~size_t{3};
  const size_t NT = H4 / 4, ntile = NT * (NT + 1) / 2, nsl = ntile < 128 ? 128 / ntile : 1;
  const size_t smem = (2 * static_cast<size_t>(H) * H +
                       (H > kPreFastH ? std::max<size_t>(2 * H4 * kPreDC, a.dm.D) + nsl * ntile * 16 : 0)) *
                      sizeof(double);
  const dim3 rgrid((a.dm.D + 127) / 128, a.dm.C);
  auto go = [&](auto kern, auto rows) {
    ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
    kern<<<min(a.dm.C, sm_count() * 8), 128, smem, s>>>(a);
    if (rows) rows<<<rgrid, 128, 0, s>>>(a);
  };
  using RowsK = void (*)(PrecompArgs);
  if (H <= kPreFastH) go(k_precompute<kPreFastH>, static_cast<RowsK>(k_precompute_rows<kPreFastH>));
  else if (H <= 16) {
    k_precompute_w<<<(a.dm.C + kPreWarps - 1) / kPreWarps, kPreWarps * 32, 0, s>>>(a);
    k_precompute_rows<16><<<rgrid, 128, 0, s>>>(a);
  }
  else if (H <= 32) go(k_precompute<32>, static_cast<RowsK>(k_precompute_rows<32>));
  else go(k_precompute<0>, static_cast<RowsK>(nullptr));
  return cudaGetLastError();
}
cudaError_t launch_caches_full(const Dims& dm, const double* lam, const double* psi, const double* R,
                               double* U, double* V, double* ipsi, cudaStream_t s) {
  k_caches_full<<<min(dm.C, sm_count() * 8), 128, 0, s>>>(dm, lam, psi, R, U, V, ipsi);
  return cudaGetLastError();
}
cudaError_t launch_self_slots(const Dims& dm, const int* K, const int* g, const int* gcnt, const float* LJ,
                              float* LJK, cudaStream_t s) {
  k_self_slots<<<grid_for(dm.N * dm.Cp, 256, 8192), 256, 0, s>>>(dm, K, g, gcnt, LJ, LJK);
  return cudaGetLastError();
}
cudaError_t launch_lse_rows(const float* LJK, int64_t N, int Cp, double* lse, cudaStream_t s) {
  k_lse_rows<<<grid_for(N, 256, 8192), 256, 0, s>>>(LJK, N, Cp, lse);
  return cudaGetLastError();
}
cudaError_t launch_lse_dense(const float* LJ, int64_t R, int SL, int C, double* lse, cudaStream_t s) {
  k_lse_dense<<<grid_for(R * 32, 256, 16384), 256, 0, s>>>(LJ, R, SL, C, lse);
  return cudaGetLastError();
}
cudaError_t launch_em_resp(const float* LJ, int64_t R, int SL, int C, const double* lse, double* resp, int* ent,
                           int* off, cudaStream_t s) {
  k_em_resp<<<grid_for(R * C, 256, sm_count() * 16), 256, 0, s>>>(LJ, R, SL, C, lse, resp, ent, off);
  return cudaGetLastError();
}
cudaError_t launch_add_f64(const double* a, double* acc, int64_t n, int first, cudaStream_t s) {
  k_add_f64<<<grid_for(n, 256, sm_count() * 16), 256, 0, s>>>(a, acc, n, first);
  return cudaGetLastError();
}
cudaError_t launch_afkmc2(const float* X, int64_t N, int D, int C, int m, double* q, double* cdf, int64_t* centers,
                          unsigned long long* state, unsigned long long* count, int* degenerate, cudaStream_t s) {
  k_afk_q<<<grid_for(N, 256, sm_count() * 8), 256, 0, s>>>(X, N, D, centers, q);
  k_afk_cdf<<<1, 1, 0, s>>>(N, q, cdf);
  k_afk_chain<<<1, kAfkThreads, 0, s>>>(X, N, D, C, m, q, cdf, centers, state, count, degenerate);
  return cudaGetLastError();
}
cudaError_t launch_sum_f64(const double* v, int64_t n, double* partials, double* out, cudaStream_t s) {
  k_sum_stage1<<<kSumBlocks, 256, 0, s>>>(v, n, partials);
  k_sum_stage2<<<1, 32, 0, s>>>(partials, kSumBlocks, out);
  return cudaGetLastError();
}
cudaError_t launch_sum_i32(const int* v, int64_t n, unsigned long long* out, cudaStream_t s) {
  cudaMemsetAsync(out, 0, sizeof(unsigned long long), s);
  k_sum_i32<<<grid_for(n, 256, 1024), 256, 0, s>>>(v, n, out);
  return cudaGetLastError();
}
cudaError_t launch_validate_K(const int* K, int64_t N, int Cp, int C, long long* bad, cudaStream_t s) {
  k_validate_K<<<grid_for(N, 256, 4096), 256, 0, s>>>(K, N, Cp, C, bad);
  return cudaGetLastError();
}
cudaError_t launch_count_empty(const double* pi, int C, int* out, cudaStream_t s) {
  cudaMemsetAsync(out, 0, sizeof(int), s);
  k_count_empty<<<grid_for(C, 256, 1024), 256, 0, s>>>(pi, C, out);
  return cudaGetLastError();
}
cudaError_t launch_logpi(const double* pi, int C, double* logpi, cudaStream_t s) {
  k_logpi<<<grid_for(C, 256, 1024), 256, 0, s>>>(pi, C, logpi);
  return cudaGetLastError();
}

}  // namespace vmfa_b200
