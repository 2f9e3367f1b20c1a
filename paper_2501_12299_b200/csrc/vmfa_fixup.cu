// vmfa_fixup.cu — fp64 re-evaluation of cancelling log-joints.
//
// The tensor-core scorer evaluates the Woodbury form (model.cpp:87-94)
//   Q = sum_d v_d^2 / psi_d - |W^T v|^2,   l = kconst - Q / 2
// (around the anchor's mean: v = u - delta, u = x - mu_a) in fp32-accurate
// arithmetic (3xFP16 products, fp32 accumulation), whose error is ~1e-6 of the
// magnitude B of the terms. They cancel when the component has collapsed onto
// a few points (psi at the variance floor, L = I + Lambda^T Psi^-1 Lambda with
// trace 1e5..1e7) or the row sits far from the anchor but near the candidate;
// the scorer's epilogue flags such a score (B > kCancel max(D, |Q|)) in its
// lowest mantissa bit. The kernels here re-evaluate every flagged slot in fp64
// exactly as the reference does: v = f64(x) - mu, y = R^-1 Lambda^T (v / psi)
// (L = R R^T), Q = v^T Psi^-1 v - |y|^2. A block owns one (anchor, g-slot) or
// one component, first checks its rows' flags, and only then stages
// W_q = Psi^-1 Lambda R^-T (fp64) with mu_q and 1/psi_q in shared memory; a
// warp evaluates one flagged row at a time.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "vmfa_kernels.cuh"

namespace vmfa_b200 {
namespace {

constexpr int kFixThreads = 256;
constexpr int kFixWarps = kFixThreads / 32;
constexpr int kFixHC = 16;  // latent chunk held in registers per lane

struct FixParams {
  int D, H;
  const float* X;
  const double* mu;
  const double* psi;
  const double* lam;
  const double* R;
  const double* kconst;
  bool smem;  // W_q = Psi^-1 Lambda R^-T (D x H) staged in shared memory
};

// stage component q (fp64): mu_q, 1/psi_q and, when it fits, the whitened
// loadings W_q = Psi_q^-1 Lambda_q R_q^-T (row d: R^-1 (Lambda_d / psi_d)), so
// that |W^T v|^2 = (U^T v).(V v) needs no per-row triangular solve
__device__ void stage_component(const FixParams& p, int q, double* s_W, double* s_mu, double* s_ip, double* s_R) {
  const int D = p.D, H = p.H;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    s_mu[d] = p.mu[(int64_t)q * D + d];
    s_ip[d] = 1.0 / p.psi[(int64_t)q * D + d];
  }
  for (int i = threadIdx.x; i < H * H; i += blockDim.x) s_R[i] = p.R[(int64_t)q * H * H + i];
  __syncthreads();
  if (p.smem) {
    const double* lq = p.lam + (int64_t)q * D * H;
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
      const double ip = s_ip[d];
      for (int i = 0; i < H; ++i) {  // forward substitution, W[i * D + d] = (R^-1 u_d)_i
        double t = lq[(int64_t)i * D + d] * ip;
        for (int k = 0; k < i; ++k) t -= s_R[i * H + k] * s_W[k * D + d];
        s_W[i * D + d] = t / s_R[i * H + i];
      }
    }
  }
  __syncthreads();
}

// l(n, q) in fp64 by one warp (every lane returns the value)
__device__ double lj_f64(const FixParams& p, int q, int64_t n, const double* s_W, const double* s_mu,
                         const double* s_ip, const double* s_R, double* s_a) {
  const int D = p.D, H = p.H, lane = threadIdx.x & 31;
  const float* x = p.X + n * D;
  // staged: W (y = W^T v directly); else Lambda from global memory (a =
  // Lambda^T (v / psi)) and y = R^-1 a
  const double* B = p.smem ? s_W : p.lam + (int64_t)q * D * H;
  double m = 0.0, yy = 0.0;
  for (int h0 = 0; h0 < H; h0 += kFixHC) {
    double acc[kFixHC];
#pragma unroll
    for (int h = 0; h < kFixHC; ++h) acc[h] = 0.0;
    for (int d = lane; d < D; d += 32) {
      const double v = static_cast<double>(x[d]) - s_mu[d];
      const double w = v * s_ip[d];
      if (h0 == 0) m = fma(v, w, m);
      const double f = p.smem ? v : w;
#pragma unroll
      for (int h = 0; h < kFixHC; ++h)
        if (h0 + h < H) acc[h] = fma(B[(int64_t)(h0 + h) * D + d], f, acc[h]);
    }
#pragma unroll
    for (int h = 0; h < kFixHC; ++h) {
      double t = acc[h];
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (p.smem) {
        if (h0 + h < H) yy = fma(t, t, yy);
      } else if (lane == 0 && h0 + h < H) {
        s_a[h0 + h] = t;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
  if (!p.smem) {
    __syncwarp();
    if (lane == 0) {  // y = R^-1 a (forward substitution), |y|^2
      for (int i = 0; i < H; ++i) {
        double t = s_a[i];
        for (int k = 0; k < i; ++k) t -= s_R[i * H + k] * s_a[k];
        t /= s_R[i * H + i];
        s_a[i] = t;
        yy = fma(t, t, yy);
      }
    }
    yy = __shfl_sync(0xffffffffu, yy, 0);
    __syncwarp();
  }
  return p.kconst[q] - 0.5 * (m - yy);
}

__device__ __forceinline__ bool flagged(float v) { return (__float_as_uint(v) & 1u) && isfinite(v); }

// anchor slots: block item (a, i) -> candidate q = g_a[i]; rows = K-inverse of a
__global__ void __launch_bounds__(kFixThreads) k_fix_anchor(FixParams p, Dims dm, const int* g, const int* gcnt,
                                                            const int* kinv_off, const int* kinv_ent,
                                                            const unsigned long long* ovf, float* LJ) {
  __shared__ int s_any;
  if (!ovf[1]) return;  // (the scan serves only a list overflow)
  extern __shared__ double s_fx[];
  double* s_mu = s_fx;
  double* s_ip = s_mu + p.D;
  double* s_a = s_ip + p.D;  // kFixWarps x 64
  double* s_R = s_a + kFixWarps * 64;
  double* s_W = s_R + p.H * p.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t items = (int64_t)dm.C * dm.G;
  for (int64_t b = blockIdx.x; b < items; b += gridDim.x) {
    const int a = static_cast<int>(b / dm.G), i = static_cast<int>(b - (int64_t)a * dm.G);
    if (i >= gcnt[a]) continue;
    const int q = g[(int64_t)a * dm.G + i];
    const int e0 = kinv_off[a], e1 = kinv_off[a + 1];
    if (e0 == e1) continue;
    auto slot = [&](int e) {
      const int ent = kinv_ent[e];
      const int64_t n = ent / dm.Cp;
      return n * dm.SL + (ent - static_cast<int>(n) * dm.Cp) * dm.G + i;
    };
    if (threadIdx.x == 0) s_any = 0;
    __syncthreads();
    int any = 0;
    for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) any |= flagged(LJ[slot(e)]);
    if (any) s_any = 1;
    __syncthreads();
    if (!s_any) continue;
    stage_component(p, q, s_W, s_mu, s_ip, s_R);
    for (int e = e0 + warp; e < e1; e += kFixWarps) {
      const int64_t o = slot(e);
      if (!flagged(LJ[o])) continue;
      const double l = lj_f64(p, q, o / dm.SL, s_W, s_mu, s_ip, s_R, s_a + warp * 64);
      if (lane == 0) LJ[o] = __uint_as_float(__float_as_uint(static_cast<float>(l)) & ~1u);
    }
    __syncthreads();
  }
}

// one-component slots: rows of component q from a CSR (extras: entry = row,
// out index row * stride + col; truncated F: entry = n * Cp + j, out = entry)
__global__ void __launch_bounds__(kFixThreads) k_fix_single(FixParams p, int C, const int* off, const int* ent,
                                                            int extra_stride, int extra_col,
                                                            const unsigned long long* ovf, float* out) {
  __shared__ int s_any;
  if (!ovf[1]) return;  // (the scan serves only a list overflow)
  extern __shared__ double s_fx[];
  double* s_mu = s_fx;
  double* s_ip = s_mu + p.D;
  double* s_a = s_ip + p.D;
  double* s_R = s_a + kFixWarps * 64;
  double* s_W = s_R + p.H * p.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // extras: entry = row, slot row * stride + col; truncated F: entry = n C' + j
  // (extra_stride == 0, extra_col = C'), slot = entry
  auto slot = [&](int e) { return extra_stride ? (int64_t)ent[e] * extra_stride + extra_col : (int64_t)ent[e]; };
  for (int q = blockIdx.x; q < C; q += gridDim.x) {
    const int e0 = off[q], e1 = off[q + 1];
    if (e0 == e1) continue;
    if (threadIdx.x == 0) s_any = 0;
    __syncthreads();
    int any = 0;
    for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) any |= flagged(out[slot(e)]);
    if (any) s_any = 1;
    __syncthreads();
    if (!s_any) continue;
    stage_component(p, q, s_W, s_mu, s_ip, s_R);
    for (int e = e0 + warp; e < e1; e += kFixWarps) {
      const int64_t o = slot(e);
      if (!flagged(out[o])) continue;
      const int64_t xrow = extra_stride ? ent[e] : ent[e] / extra_col;
      const double l = lj_f64(p, q, xrow, s_W, s_mu, s_ip, s_R, s_a + warp * 64);
      if (lane == 0) out[o] = __uint_as_float(__float_as_uint(static_cast<float>(l)) & ~1u);
    }
    __syncthreads();
  }
}

// component of a listed output index. mode 0 anchor slots (n SL + j G + i:
// q = g_{K(n)[j]}[i]), 1 extras (n SL + C'G: q = rx[n]), 2 truncated F
// (n C' + j: q = K(n)[j])
__device__ __forceinline__ int list_component(const Dims& dm, int mode, const int* K, const int* g, const int* rx,
                                              long long o, int64_t* n_out) {
  if (mode == 2) {
    *n_out = o / dm.Cp;
    return K[o];
  }
  const int64_t n = o / dm.SL;
  *n_out = n;
  if (mode == 1) return rx[n];
  const int s = static_cast<int>(o - n * dm.SL);
  const int j = s / dm.G;
  return g[(int64_t)K[n * dm.Cp + j] * dm.G + (s - j * dm.G)];
}

// the flagged scores grouped by component (a counting sort of the list):
// count, exclusive scan, scatter
__global__ void k_fix_count(Dims dm, int mode, const int* K, const int* g, const int* rx, const long long* list,
                            const unsigned long long* cnt, long long cap, int* qcnt, int* qkey) {
  const long long total = min(static_cast<long long>(cnt[0]), cap);
  for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < total; w += (long long)gridDim.x * blockDim.x) {
    int64_t n;
    const int q = list_component(dm, mode, K, g, rx, list[w], &n);
    qkey[w] = q;
    atomicAdd(qcnt + q, 1);
  }
}
constexpr int kFixChunk = 128;  // listed scores per work item (a component's list may be long)
// exclusive scans of the per-component counts (qoff) and of their work items
// of kFixChunk scores (iof), one block
__global__ void __launch_bounds__(1024) k_fix_scan(const int* qcnt, int C, int* qoff, int* qfill, int* iof) {
  __shared__ int s_warp[2][32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = (C + 1023) / 1024;
  const int c0 = tid * per, c1 = min(C, c0 + per);
  int sum = 0, isum = 0;
  for (int c = c0; c < c1; ++c) {
    sum += qcnt[c];
    isum += (qcnt[c] + kFixChunk - 1) / kFixChunk;
  }
  int incl = sum, iincl = isum;
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    const int u = __shfl_up_sync(0xffffffffu, iincl, o);
    if (lane >= o) incl += t, iincl += u;
  }
  if (lane == 31) s_warp[0][warp] = incl, s_warp[1][warp] = iincl;
  __syncthreads();
  if (warp == 0) {
    int w = s_warp[0][lane], v = s_warp[1][lane];
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, w, o);
      const int u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) w += t, v += u;
    }
    s_warp[0][lane] = w;
    s_warp[1][lane] = v;
  }
  __syncthreads();
  int run = incl - sum + (warp > 0 ? s_warp[0][warp - 1] : 0);
  int irun = iincl - isum + (warp > 0 ? s_warp[1][warp - 1] : 0);
  for (int c = c0; c < c1; ++c) {
    qoff[c] = run;
    qfill[c] = run;
    iof[c] = irun;
    run += qcnt[c];
    irun += (qcnt[c] + kFixChunk - 1) / kFixChunk;
  }
  if (tid == 1023) qoff[C] = run, iof[C] = irun;
}
__global__ void k_fix_scatter(const long long* list, const unsigned long long* cnt, long long cap, const int* qkey,
                              int* qfill, int* sorted) {
  const long long total = min(static_cast<long long>(cnt[0]), cap);
  for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < total; w += (long long)gridDim.x * blockDim.x)
    sorted[atomicAdd(qfill + qkey[w], 1)] = static_cast<int>(list[w]);
}

// work items of <= kFixChunk listed scores of one component: W_q staged per
// item (shared memory when it fits), a warp per score
__global__ void __launch_bounds__(kFixThreads) k_fix_grouped(FixParams p, Dims dm, int mode, const int* qoff,
                                                             const int* iof, const int* sorted,
                                                             unsigned long long* nfix, float* out) {
  extern __shared__ double s_fx[];
  double* s_mu = s_fx;
  double* s_ip = s_mu + p.D;
  double* s_a = s_ip + p.D;
  double* s_R = s_a + kFixWarps * 64;
  double* s_W = s_R + p.H * p.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(nfix, static_cast<unsigned long long>(qoff[dm.C]));
  const int items = iof[dm.C];
  for (int t = blockIdx.x; t < items; t += gridDim.x) {
    int lo = 0, hi = dm.C;  // the component q with iof[q] <= t < iof[q + 1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (iof[mid] <= t) lo = mid;
      else hi = mid;
    }
    const int q = lo;
    const int e0 = qoff[q] + (t - iof[q]) * kFixChunk, e1 = min(qoff[q + 1], e0 + kFixChunk);
    stage_component(p, q, s_W, s_mu, s_ip, s_R);
    for (int e = e0 + warp; e < e1; e += kFixWarps) {
      const int64_t o = sorted[e];
      const int64_t n = mode == 2 ? o / dm.Cp : o / dm.SL;
      const double l = lj_f64(p, q, n, s_W, s_mu, s_ip, s_R, s_a + warp * 64);
      if (lane == 0) out[o] = __uint_as_float(__float_as_uint(static_cast<float>(l)) & ~1u);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- DMMA path
// The same fp64 re-evaluation as a grouped contraction on the fp64 tensor
// cores: per work item (<= kFixChunk listed rows of one component q) the block
// stages W_q^T (H x D, fp64, from the precompute), mu_q and 1/psi_q; each warp
// takes 16 rows (two m8 tiles) and runs Y = V W_q with
// mma.m8n8k4.f64 over k-steps of 4 dimensions, V = f64(x) - mu_q formed in
// registers from float4 row loads. Dimension k-step j of chunk k0 holds
// dimensions k0 + 4 t + j on lane (g, t), so every lane's A and B elements
// are 4 consecutive dimensions (one float4 of x, two double2 of W / mu / ip).
// m = sum v^2 / psi rides along on the FP64 pipe; Q = m - |y|^2.
__device__ __forceinline__ void dmma_f64(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

size_t fix_dmma_smem(int D, int H) { return (static_cast<size_t>(H) * (D + 2) + 2 * static_cast<size_t>(D)) * sizeof(double); }

template <int NT>
__global__ void __launch_bounds__(kFixThreads) k_fix_dmma(FixParams p, const double* __restrict__ W64, Dims dm, int mode,
                                                          const int* qoff, const int* iof, const int* sorted,
                                                          unsigned long long* nfix, float* out) {
  extern __shared__ __align__(16) double s_fx[];
  const int D = p.D, Dp = D + 2;  // padded rows: the 8 g-lanes of a quarter-warp hit distinct banks
  double* s_W = s_fx;             // (NT 8) x Dp
  double* s_mu = s_W + NT * 8 * Dp;
  double* s_ip = s_mu + D;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(nfix, static_cast<unsigned long long>(qoff[dm.C]));
  const int items = iof[dm.C];
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    int lo = 0, hi = dm.C;  // the component q with iof[q] <= it < iof[q + 1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (iof[mid] <= it) lo = mid;
      else hi = mid;
    }
    const int q = lo;
    const int e0 = qoff[q] + (it - iof[q]) * kFixChunk, e1 = min(qoff[q + 1], e0 + kFixChunk);
    __syncthreads();  // the previous item's readers are done
    const double* wq = W64 + (int64_t)q * NT * 8 * D;
    for (int i = threadIdx.x; i < NT * 8 * (D >> 1); i += blockDim.x) {
      const int h = (2 * i) / D, d = 2 * i - h * D;
      *reinterpret_cast<double2*>(s_W + h * Dp + d) = __ldg(reinterpret_cast<const double2*>(wq + (int64_t)h * D + d));
    }
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
      s_mu[d] = p.mu[(int64_t)q * D + d];
      s_ip[d] = 1.0 / p.psi[(int64_t)q * D + d];
    }
    __syncthreads();
    const int r0 = e0 + warp * 16;
    if (r0 >= e1) continue;
    int64_t o[2];
    bool ok[2];
    const float* xr[2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int r = r0 + mt * 8 + g;
      ok[mt] = r < e1;
      o[mt] = ok[mt] ? sorted[r] : 0;
      const int64_t n = mode == 2 ? o[mt] / dm.Cp : o[mt] / dm.SL;
      xr[mt] = p.X + n * D + 4 * t;
    }
    double acc[2][NT][2], m[2] = {0.0, 0.0};
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 xa[2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) xa[mt] = ok[mt] ? __ldg(reinterpret_cast<const float4*>(xr[mt])) : z4;
    for (int k0 = 0; k0 < D; k0 += 16) {
      float4 xn[2] = {z4, z4};
      if (k0 + 16 < D) {
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
          if (ok[mt]) xn[mt] = __ldg(reinterpret_cast<const float4*>(xr[mt] + k0 + 16));
      }
      const int kb = k0 + 4 * t;
      const double2 mu01 = *reinterpret_cast<const double2*>(s_mu + kb), mu23 = *reinterpret_cast<const double2*>(s_mu + kb + 2);
      const double2 ip01 = *reinterpret_cast<const double2*>(s_ip + kb), ip23 = *reinterpret_cast<const double2*>(s_ip + kb + 2);
      double v[2][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        v[mt][0] = ok[mt] ? static_cast<double>(xa[mt].x) - mu01.x : 0.0;
        v[mt][1] = ok[mt] ? static_cast<double>(xa[mt].y) - mu01.y : 0.0;
        v[mt][2] = ok[mt] ? static_cast<double>(xa[mt].z) - mu23.x : 0.0;
        v[mt][3] = ok[mt] ? static_cast<double>(xa[mt].w) - mu23.y : 0.0;
        m[mt] = fma(v[mt][0] * ip01.x, v[mt][0], m[mt]);
        m[mt] = fma(v[mt][1] * ip01.y, v[mt][1], m[mt]);
        m[mt] = fma(v[mt][2] * ip23.x, v[mt][2], m[mt]);
        m[mt] = fma(v[mt][3] * ip23.y, v[mt][3], m[mt]);
      }
      double b[NT][4];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const double* wr = s_W + (nt * 8 + g) * Dp + kb;
        const double2 b01 = *reinterpret_cast<const double2*>(wr), b23 = *reinterpret_cast<const double2*>(wr + 2);
        b[nt][0] = b01.x;
        b[nt][1] = b01.y;
        b[nt][2] = b23.x;
        b[nt][3] = b23.y;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma_f64(acc[mt][nt], v[mt][j], b[nt][j]);
      xa[0] = xn[0];
      xa[1] = xn[1];
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      double yy = 0.0;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) yy = fma(acc[mt][nt][0], acc[mt][nt][0], fma(acc[mt][nt][1], acc[mt][nt][1], yy));
      double mm = m[mt];
#pragma unroll
      for (int s = 1; s < 4; s <<= 1) {
        yy += __shfl_xor_sync(0xffffffffu, yy, s);
        mm += __shfl_xor_sync(0xffffffffu, mm, s);
      }
      if (t == 0 && ok[mt]) {
        const double l = p.kconst[q] - 0.5 * (mm - yy);
        out[o[mt]] = __uint_as_float(__float_as_uint(static_cast<float>(l)) & ~1u);
      }
    }
  }
}

size_t fix_smem(int D, int H, bool* smem) {
  const size_t base = (2 * static_cast<size_t>(D) + kFixWarps * 64 + static_cast<size_t>(H) * H) * sizeof(double);
  const size_t lam = static_cast<size_t>(D) * H * sizeof(double);
  *smem = base + lam <= 200 * 1024;
  return *smem ? base + lam : base;
}

}  // namespace

bool fix_dmma_ok(int D, int H) {
  return H % 8 == 0 && H <= 32 && D % 16 == 0 && fix_dmma_smem(D, H) <= 200 * 1024;
}

// ovf[1] |= cnt[1] (first: =): a list overflow at either stage; first also
// counts the scores listed for the one-component tensor pass (nfix[1])
__global__ void k_fix_ovf(const unsigned long long* cnt, unsigned long long* ovf, int first, unsigned long long* nfix) {
  ovf[1] = first ? cnt[1] : (ovf[1] | cnt[1]);
  if (first) nfix[1] += cnt[0];
}
cudaError_t launch_fix_ovf(const FixArgs& f, int first, cudaStream_t s) {
  k_fix_ovf<<<1, 1, 0, s>>>(f.cnt, f.ovf, first, f.nfix);
  return cudaGetLastError();
}

// group the listed scores by component (counting sort: entries in sorted,
// per-component offsets qoff and work items of 128 in iof)
cudaError_t launch_fix_group(const Dims& dm, const FixArgs& f, int mode, const int* K, const int* g, const int* rx,
                             cudaStream_t s) {
  if (cudaError_t e = cudaMemsetAsync(f.qcnt, 0, sizeof(int) * dm.C, s); e != cudaSuccess) return e;
  k_fix_count<<<sm_count() * 4, 256, 0, s>>>(dm, mode, K, g, rx, f.list, f.cnt, f.cap, f.qcnt, f.qkey);
  k_fix_scan<<<1, 1024, 0, s>>>(f.qcnt, dm.C, f.qoff, f.qfill, f.iof);
  k_fix_scatter<<<sm_count() * 4, 256, 0, s>>>(f.list, f.cnt, f.cap, f.qkey, f.qfill, f.sorted);
  return cudaGetLastError();
}

// fp64 re-evaluation of the listed (grouped) scores, then the overflow scans
cudaError_t launch_fix_f64(const Dims& dm, const FixArgs& f, int mode, const int* K, const int* g, const int* rx,
                           float* out, cudaStream_t s) {
  if (cudaError_t e = launch_fix_group(dm, f, mode, K, g, rx, s); e != cudaSuccess) return e;
  bool sm = false;
  if (f.W64 && fix_dmma_ok(dm.D, dm.H)) {
    FixParams p{dm.D, dm.H, f.X, f.mu, f.psi, f.lam, f.R, f.kconst, false};
    const size_t smem = fix_dmma_smem(dm.D, dm.H);
    auto go = [&](auto kern) {
      ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
      kern<<<sm_count() * 2, kFixThreads, smem, s>>>(p, f.W64, dm, mode, f.qoff, f.iof, f.sorted, f.nfix, out);
    };
    switch (dm.H / 8) {
      case 1: go(k_fix_dmma<1>); break;
      case 2: go(k_fix_dmma<2>); break;
      case 3: go(k_fix_dmma<3>); break;
      default: go(k_fix_dmma<4>); break;
    }
    return cudaGetLastError();
  }
  const size_t smem = fix_smem(dm.D, dm.H, &sm);
  FixParams p{dm.D, dm.H, f.X, f.mu, f.psi, f.lam, f.R, f.kconst, sm};
  ensure_dyn_smem(reinterpret_cast<const void*>(k_fix_grouped), smem);
  k_fix_grouped<<<sm_count() * 2, kFixThreads, smem, s>>>(p, dm, mode, f.qoff, f.iof, f.sorted, f.nfix, out);
  return cudaGetLastError();
}

cudaError_t launch_fix_scan_anchor(const Dims& dm, const FixArgs& f, const int* g, const int* gcnt,
                                   const int* kinv_off, const int* kinv_ent, float* LJ, cudaStream_t s) {
  bool sm = false;
  const size_t smem = fix_smem(dm.D, dm.H, &sm);
  FixParams p{dm.D, dm.H, f.X, f.mu, f.psi, f.lam, f.R, f.kconst, sm};
  ensure_dyn_smem(reinterpret_cast<const void*>(k_fix_anchor), smem);
  k_fix_anchor<<<sm_count() * 4, kFixThreads, smem, s>>>(p, dm, g, gcnt, kinv_off, kinv_ent, f.ovf, LJ);
  return cudaGetLastError();
}

cudaError_t launch_fix_scan_single(const Dims& dm, const FixArgs& f, const int* off, const int* ent, int extra_stride,
                                   int extra_col, float* out, cudaStream_t s) {
  bool sm = false;
  const size_t smem = fix_smem(dm.D, dm.H, &sm);
  FixParams p{dm.D, dm.H, f.X, f.mu, f.psi, f.lam, f.R, f.kconst, sm};
  ensure_dyn_smem(reinterpret_cast<const void*>(k_fix_single), smem);
  k_fix_single<<<sm_count() * 4, kFixThreads, smem, s>>>(p, dm.C, off, ent, extra_stride, extra_col, f.ovf, out);
  return cudaGetLastError();
}

}  // namespace vmfa_b200
