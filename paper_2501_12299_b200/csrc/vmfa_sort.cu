// vmfa_sort.cu — the K1 map inversion's stable sort and the scans, hand-written.
//
// Block 1 inverts the point -> candidate map K (N x C') into per-component
// point lists (the reference builds its partition by pushing n into
// I_{label(n)}, estep.cpp:169-172, i.e. in increasing n: the lists here keep
// that order, so the sort must be stable). The keys are component indices
// (< 2^16 for every BASELINE config), so the sort is an LSD radix sort over
// 8-bit digits, one stable counting sort per digit:
//   k_digit_hist     per tile of kSortTile entries, a 256-bin histogram,
//                    stored digit-major: hist[d * T + t]
//   scan_i32         exclusive scan of hist: entry (d, t) is where tile t's
//                    digit-d entries start in the output
//   k_digit_scatter  per tile: every warp owns a contiguous run of the tile;
//                    per-warp digit counts (__match_any_sync groups, the
//                    group leader adds its size), per-warp bases from the
//                    tile's scanned offset, then the warp walks its run again
//                    in input order, an entry's position = base + its rank
//                    among the equal-digit lanes before it.
// Traffic per pass: keys read twice, (key, value) read once and written once
// (n = 5e6 entries at config 3: ~60 MB, ~10 us at HBM rate). The first pass
// reads no values: an entry's value is its input index.
// The scans (three kernels: tile sums, one-block scan of the sums, tiles
// rescanned from their base) serve the histograms, the sparse co-occurrence
// segment heads and any int32 prefix sum.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "vmfa_kernels.cuh"

namespace vmfa_b200 {
namespace {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortSteps = 16;                            // 32-entry steps per warp
constexpr int kSortTile = kSortWarps * kSortSteps * 32;   // 4096 entries per tile
constexpr int kScanTile = 4096;                           // entries per scan block (256 threads x 16)
constexpr unsigned kAll = 0xffffffffu;

__global__ void __launch_bounds__(kSortThreads) k_digit_hist(const unsigned* __restrict__ keys, int64_t n, int shift,
                                                            int T, int* __restrict__ hist) {
  __shared__ int h[256];
  const int tid = threadIdx.x;
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    h[tid] = 0;
    __syncthreads();
    const int64_t base = (int64_t)t * kSortTile;
    for (int i = tid; i < kSortTile; i += kSortThreads) {
      const int64_t e = base + i;
      if (e < n) atomicAdd(&h[(__ldg(keys + e) >> shift) & 255u], 1);
    }
    __syncthreads();
    hist[(int64_t)tid * T + t] = h[tid];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kSortThreads) k_digit_scatter(const unsigned* __restrict__ kin,
                                                               const int* __restrict__ vin, int64_t n, int shift,
                                                               int T, const int* __restrict__ hscan,
                                                               unsigned* __restrict__ kout, int* __restrict__ vout) {
  __shared__ int s_cnt[kSortWarps][256];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned lt = (1u << lane) - 1u;
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    for (int i = tid; i < kSortWarps * 256; i += kSortThreads) (&s_cnt[0][0])[i] = 0;
    __syncthreads();
    const int64_t wbase = (int64_t)t * kSortTile + warp * (kSortSteps * 32);
    unsigned k[kSortSteps], mk[kSortSteps];
    int v[kSortSteps];
#pragma unroll
    for (int s = 0; s < kSortSteps; ++s) {
      const int64_t e = wbase + s * 32 + lane;
      const bool ok = e < n;
      k[s] = ok ? __ldg(kin + e) : 0u;
      v[s] = ok ? (vin ? __ldg(vin + e) : static_cast<int>(e)) : 0;
      const unsigned d = ok ? (k[s] >> shift) & 255u : 256u;  // past the end: its own group, skipped
      mk[s] = __match_any_sync(kAll, d);
      if (d < 256u && (mk[s] & lt) == 0u) s_cnt[warp][d] += __popc(mk[s]);
      __syncwarp();
    }
    __syncthreads();
    {  // per-warp bases of digit tid: the tile's offset plus the earlier warps' counts
      int run = hscan[(int64_t)tid * T + t];
#pragma unroll
      for (int w = 0; w < kSortWarps; ++w) {
        const int c = s_cnt[w][tid];
        s_cnt[w][tid] = run;
        run += c;
      }
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < kSortSteps; ++s) {
      const int64_t e = wbase + s * 32 + lane;
      const bool ok = e < n;
      const unsigned d = (k[s] >> shift) & 255u;
      int pos = 0;
      if (ok) pos = s_cnt[warp][d] + __popc(mk[s] & lt);
      __syncwarp();
      if (ok) {
        kout[pos] = k[s];
        vout[pos] = v[s];
        if ((mk[s] & lt) == 0u) s_cnt[warp][d] += __popc(mk[s]);
      }
      __syncwarp();
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- int32 scans
__device__ __forceinline__ int block_excl_scan(int x, int* s_w, int* total) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(kAll, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = lane < (blockDim.x >> 5) ? s_w[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kAll, w, o);
      if (lane >= o) w += y;
    }
    if (lane < (blockDim.x >> 5)) s_w[lane] = w;
  }
  __syncthreads();
  const int before = (warp > 0 ? s_w[warp - 1] : 0) + incl - x;
  *total = s_w[(blockDim.x >> 5) - 1];
  __syncthreads();
  return before;
}

// sums[b] = sum of tile b
__global__ void __launch_bounds__(256) k_scan_sums(const int* __restrict__ in, int64_t n, int* __restrict__ sums) {
  __shared__ int s_w[8];
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  int acc = 0;
  for (int i = threadIdx.x; i < kScanTile; i += 256) {
    const int64_t e = base + i;
    if (e < n) acc += in[e];
  }
  int total = 0;
  block_excl_scan(acc, s_w, &total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}
// one block: exclusive scan of m tile sums in place
__global__ void __launch_bounds__(1024) k_scan_top(int* sums, int m) {
  __shared__ int s_w[32];
  const int per = (m + 1023) / 1024;
  const int c0 = threadIdx.x * per, c1 = min(m, c0 + per);
  int acc = 0;
  for (int c = c0; c < c1; ++c) acc += sums[c];
  int total = 0;
  int run = block_excl_scan(acc, s_w, &total);
  for (int c = c0; c < c1; ++c) {
    const int x = sums[c];
    sums[c] = run;
    run += x;
  }
}
// tile b rescanned from base sums[b]: 16 consecutive entries per thread
// (in == out allowed: a thread reads its entries before the block scan)
__global__ void __launch_bounds__(256) k_scan_tiles(const int* in, int64_t n, const int* __restrict__ sums,
                                                    int inclusive, int* out) {
  __shared__ int s_w[8];
  constexpr int P = kScanTile / 256;
  const int64_t base = (int64_t)blockIdx.x * kScanTile + threadIdx.x * P;
  int x[P];
  int acc = 0;
#pragma unroll
  for (int i = 0; i < P; ++i) {
    x[i] = base + i < n ? in[base + i] : 0;
    acc += x[i];
  }
  int total = 0;
  int run = sums[blockIdx.x] + block_excl_scan(acc, s_w, &total);
#pragma unroll
  for (int i = 0; i < P; ++i) {
    if (inclusive) run += x[i];
    if (base + i < n) out[base + i] = run;
    if (!inclusive) run += x[i];
  }
}

}  // namespace

int64_t scan_tmp_ints(int64_t n) { return (n + kScanTile - 1) / kScanTile + 1; }

cudaError_t scan_i32(const int* in, int* out, int64_t n, bool inclusive, int* tmp, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int64_t m = (n + kScanTile - 1) / kScanTile;
  k_scan_sums<<<static_cast<unsigned>(m), 256, 0, s>>>(in, n, tmp);
  k_scan_top<<<1, 1024, 0, s>>>(tmp, static_cast<int>(m));
  k_scan_tiles<<<static_cast<unsigned>(m), 256, 0, s>>>(in, n, tmp, inclusive ? 1 : 0, out);
  return cudaGetLastError();
}

int64_t sort_hist_ints(int64_t n) {
  const int64_t T = (n + kSortTile - 1) / kSortTile;
  return 256 * T + scan_tmp_ints(256 * T);
}

// Per pass: the tile histograms of that pass's input (a tile's digit counts
// depend on which entries the previous pass put in it), one scan, one
// scatter: 5 launches per pass.
cudaError_t radix_sort_pairs(const unsigned* keys, const int* vals, int64_t n, int bits, unsigned* ktmp, int* vtmp,
                             unsigned* kout, int* vout, int* hist, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (bits > 32 || n > 0x7fffffff) return cudaErrorInvalidValue;
  const int passes = bits <= 8 ? 1 : (bits + 7) / 8;
  const int T = static_cast<int>((n + kSortTile - 1) / kSortTile);
  const int grid = std::min(T, sm_count() * 8);
  const int64_t nh = (int64_t)256 * T;
  const unsigned* ks = keys;
  const int* vs = vals;
  for (int p = 0; p < passes; ++p) {
    // ping-pong so that the last pass lands in (kout, vout)
    const bool to_out = ((passes - 1 - p) & 1) == 0;
    unsigned* kd = to_out ? kout : ktmp;
    int* vd = to_out ? vout : vtmp;
    k_digit_hist<<<grid, kSortThreads, 0, s>>>(ks, n, 8 * p, T, hist);
    if (cudaError_t e = scan_i32(hist, hist, nh, false, hist + nh, s); e != cudaSuccess) return e;
    k_digit_scatter<<<grid, kSortThreads, 0, s>>>(ks, vs, n, 8 * p, T, hist, kd, vd);
    ks = kd;
    vs = vd;
  }
  return cudaGetLastError();
}

}  // namespace vmfa_b200

// Diagnostic entry (include/vmfa_b200.h): sort n host keys (< 2^bits) with the
// device radix sort `reps` times on a fresh stream; returns the last result
// and the number of repetitions whose output differed from the first (0
// expected), or -1 on a CUDA error.
extern "C" int vmfa_diag_radix_sort(const uint32_t* keys, int64_t n, int bits, uint32_t* keys_out, int32_t* vals_out,
                                    int reps) {
  using namespace vmfa_b200;
  if (n <= 0 || reps < 1) return -1;
  cudaStream_t s = nullptr;
  unsigned *dk = nullptr, *dt = nullptr, *dko = nullptr;
  int *dvt = nullptr, *dvo = nullptr, *dh = nullptr;
  const size_t B = static_cast<size_t>(n) * 4;
  bool ok = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess &&
            cudaMalloc(&dk, B) == cudaSuccess && cudaMalloc(&dt, B) == cudaSuccess &&
            cudaMalloc(&dko, B) == cudaSuccess && cudaMalloc(&dvt, B) == cudaSuccess &&
            cudaMalloc(&dvo, B) == cudaSuccess &&
            cudaMalloc(&dh, static_cast<size_t>(sort_hist_ints(n)) * 4) == cudaSuccess;
  int differ = 0;
  std::vector<uint32_t> k0(n);
  std::vector<int32_t> v0(n);
  if (ok) ok = cudaMemcpyAsync(dk, keys, B, cudaMemcpyHostToDevice, s) == cudaSuccess;
  for (int r = 0; ok && r < reps; ++r) {
    ok = cudaMemsetAsync(dko, 0xff, B, s) == cudaSuccess && cudaMemsetAsync(dvo, 0xff, B, s) == cudaSuccess &&
         radix_sort_pairs(dk, nullptr, n, bits, dt, dvt, dko, dvo, dh, s) == cudaSuccess &&
         cudaMemcpyAsync(keys_out, dko, B, cudaMemcpyDeviceToHost, s) == cudaSuccess &&
         cudaMemcpyAsync(vals_out, dvo, B, cudaMemcpyDeviceToHost, s) == cudaSuccess &&
         cudaStreamSynchronize(s) == cudaSuccess;
    if (!ok) break;
    if (r == 0) {
      std::copy(keys_out, keys_out + n, k0.begin());
      std::copy(vals_out, vals_out + n, v0.begin());
    } else if (!std::equal(k0.begin(), k0.end(), keys_out) || !std::equal(v0.begin(), v0.end(), vals_out)) {
      ++differ;
    }
  }
  for (void* p : {static_cast<void*>(dk), static_cast<void*>(dt), static_cast<void*>(dko), static_cast<void*>(dvt),
                  static_cast<void*>(dvo), static_cast<void*>(dh)})
    if (p) cudaFree(p);
  if (s) cudaStreamDestroy(s);
  return ok ? differ : -1;
}
