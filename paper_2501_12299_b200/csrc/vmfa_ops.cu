// vmfa_ops.cu — the reference's per-operation E-step pieces and log_joint as
// batched device kernels over a context's rows (estep.hpp:82-117,
// model.hpp:83-86). The fused E-step (k_extra, k_score_*, k_select,
// k_gupdate) computes the same quantities inside one pass; these entry points
// exist for callers of the reference API that drive the pieces themselves.
//   k_log_joint_pairs   log_joint (model.cpp:81-95) in fp64, a warp per pair
//   k_search_space      build_search_space (estep.cpp:83-101, 126-133)
//   k_update_k          update_k (estep.cpp:103-122, 135-142)
//   k_hard_labels       hard_partition's labels (estep.cpp:144-166)
//   k_responsibilities  responsibilities_row (estep.cpp:222-228, numerics.hpp:15-22)
//   k_distances         accumulate_distances (estep.cpp:175-202): a thread per
//                       component, rows in partition order, fp64 sums in the
//                       reference's per-key order (bit-identical sums)
//   k_update_g          update_g (estep.cpp:204-220)
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "vmfa_kernels.cuh"
#include "vmfa_rng.hpp"

namespace vmfa_b200 {
namespace {

constexpr double kLog2PiD = 1.8378770664093453;  // numerics.hpp:10

// log_joint: v = f64(x) - mu, a = Lambda^T (v / psi), y = R^-1 a (L = R R^T),
// l = log pi - 0.5 (D log 2pi + log|Sigma| + v^T Psi^-1 v - |y|^2)
__global__ void k_log_joint_pairs(int D, int H, const float* X, const int* comp, int64_t n, const double* mu,
                                  const double* psi, const double* lam, const double* R, const double* kconst,
                                  double* out) {
  const int lane = threadIdx.x & 31;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < n;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int q = comp[w];
    const float* x = X + w * D;
    const double* m = mu + (int64_t)q * D;
    const double* ps = psi + (int64_t)q * D;
    const double* lq = lam + (int64_t)q * D * H;
    const double* Rq = R + (int64_t)q * H * H;
    double mm = 0.0, a0 = 0.0, a1 = 0.0;
    for (int h0 = 0; h0 < H; h0 += 8) {
      double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int d = lane; d < D; d += 32) {
        const double v = static_cast<double>(x[d]) - m[d];
        const double u = v / ps[d];
        if (h0 == 0) mm = fma(v, u, mm);
#pragma unroll
        for (int h = 0; h < 8; ++h)
          if (h0 + h < H) acc[h] = fma(lq[(int64_t)(h0 + h) * D + d], u, acc[h]);
      }
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        double t = acc[h];
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        const int j = h0 + h;
        if (j < H && (j & 31) == lane) (j < 32 ? a0 : a1) = t;
      }
    }
    for (int o = 16; o > 0; o >>= 1) mm += __shfl_xor_sync(0xffffffffu, mm, o);
    double yy = 0.0;
    for (int i = 0; i < H; ++i) {  // forward substitution, a_j held by lane j % 32
      const double yi = __shfl_sync(0xffffffffu, i < 32 ? a0 : a1, i & 31) / Rq[i * H + i];
      yy = fma(yi, yi, yy);
      if (lane > i && lane < H) a0 -= Rq[lane * H + i] * yi;
      if (lane + 32 > i && lane + 32 < H) a1 -= Rq[(lane + 32) * H + i] * yi;
    }
    if (lane == 0) out[w] = kconst[q] - 0.5 * (mm - yy);
  }
}

// S(n) = dedup(U_{c in K(n)} g_c, then r_n) in insertion order (-1 padded)
__global__ void k_search_space(Dims dm, const int* K, const int* g, const int* gcnt, const int* extras,
                               uint64_t seed, uint64_t it, int* count, int* idx) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < dm.N; n += (int64_t)gridDim.x * blockDim.x) {
    int* out = idx + n * dm.stride;
    int m = 0;
    auto push = [&](int c) {
      for (int k = 0; k < m; ++k)
        if (out[k] == c) return;
      out[m++] = c;
    };
    for (int j = 0; j < dm.Cp; ++j) {
      const int a = K[n * dm.Cp + j];
      for (int i = 0; i < gcnt[a]; ++i) push(g[(int64_t)a * dm.G + i]);
    }
    push(extras ? extras[n] : extra_candidate(seed, it, static_cast<uint64_t>(dm.n0 + n), dm.C));
    count[n] = m;
    for (int k = m; k < dm.stride; ++k) out[k] = -1;
  }
}

// top-C' by (l desc, index asc), sorted ascending; status 1 if |S(n)| < C'
__global__ void k_update_k(Dims dm, const int* count, const int* idx, const double* lj, int* Kout, int* status) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < dm.N; n += (int64_t)gridDim.x * blockDim.x) {
    const int m = count[n];
    int* out = Kout + n * dm.Cp;
    if (m < dm.Cp) {
      atomicOr(status, 1);
      for (int j = 0; j < dm.Cp; ++j) out[j] = -1;
      continue;
    }
    const int* ci = idx + n * dm.stride;
    const double* l = lj + n * dm.stride;
    int prev_j = -1;
    for (int r = 0; r < dm.Cp; ++r) {  // r-th best, strictly after the (r-1)-th in (l desc, index asc)
      int best = -1;
      for (int j = 0; j < m; ++j) {
        if (prev_j >= 0) {
          const bool after = l[j] < l[prev_j] || (l[j] == l[prev_j] && ci[j] > ci[prev_j]);
          if (!after) continue;
        }
        if (best < 0 || l[j] > l[best] || (l[j] == l[best] && ci[j] < ci[best])) best = j;
      }
      out[r] = ci[best];
      prev_j = best;
    }
    for (int i = 1; i < dm.Cp; ++i)  // ascending
      for (int k = i; k > 0 && out[k - 1] > out[k]; --k) {
        const int t = out[k];
        out[k] = out[k - 1];
        out[k - 1] = t;
      }
  }
}

// label = the first K member, replaced only by a strictly larger retained l
__global__ void k_hard_labels(Dims dm, const int* K, const int* count, const int* idx, const double* lj, int* labels) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < dm.N; n += (int64_t)gridDim.x * blockDim.x) {
    int best = -1;
    double bl = -INFINITY;
    for (int j = 0; j < dm.Cp; ++j) {
      const int c = K[n * dm.Cp + j];
      for (int k = 0; k < count[n]; ++k) {
        if (idx[n * dm.stride + k] != c) continue;
        const double v = lj[n * dm.stride + k];
        if (best < 0 || v > bl) best = c, bl = v;
        break;
      }
    }
    labels[n] = best;
  }
}

__global__ void k_responsibilities(int64_t rows, int width, const double* lj, double* resp) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < rows; n += (int64_t)gridDim.x * blockDim.x) {
    const double* l = lj + n * width;
    double m = -INFINITY;
    for (int j = 0; j < width; ++j) m = fmax(m, l[j]);
    double lse = m;
    if (isfinite(m)) {
      double s = 0.0;
      for (int j = 0; j < width; ++j) s += exp(l[j] - m);
      lse = m + log(s);
    }
    for (int j = 0; j < width; ++j) resp[n * width + j] = exp(l[j] - lse);
  }
}

// accumulate_distances: component c's keys in an open-addressing table at
// tab_off[c] (capacity tab_cap[c], a power of two), then sorted by ct in place
__global__ void k_distances(Dims dm, int mode, const int* part_off, const int* part_ent, const int* count,
                            const int* idx, const double* lj, const double* pi, const int64_t* tab_off,
                            const int* tab_cap, int* key, double* sum, long long* cnt, int* nkeys) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < dm.C; c += gridDim.x * blockDim.x) {
    int* tk = key + tab_off[c];
    double* ts = sum + tab_off[c];
    long long* tc = cnt + tab_off[c];
    const int cap = tab_cap[c];
    for (int i = 0; i < cap; ++i) tk[i] = -1;
    const double lpc = pi[c] > 0.0 ? log(pi[c]) : -INFINITY;
    for (int e = part_off[c]; e < part_off[c + 1]; ++e) {
      const int64_t n = part_ent[e];
      const int* ci = idx + n * dm.stride;
      const double* l = lj + n * dm.stride;
      double lc = NAN;  // RetainedJoints::lookup (estep.cpp:70-77)
      for (int k = 0; k < count[n]; ++k)
        if (ci[k] == c) {
          lc = l[k];
          break;
        }
      const double cond_c = lc - lpc;
      for (int k = 0; k < count[n]; ++k) {
        const int ct = ci[k];
        if (ct == c || pi[ct] <= 0.0) continue;
        const double v = mode == 0 ? cond_c - (l[k] - log(pi[ct])) : -l[k];
        unsigned h = (static_cast<unsigned>(ct) * 2654435761u) & (cap - 1);
        while (tk[h] != -1 && tk[h] != ct) h = (h + 1) & (cap - 1);
        if (tk[h] == -1) {
          tk[h] = ct;
          ts[h] = 0.0;
          tc[h] = 0;
        }
        ts[h] += v;
        tc[h] += 1;
      }
    }
    int m = 0;  // compact to the front, then insertion-sort by ct
    for (int i = 0; i < cap; ++i)
      if (tk[i] != -1) {
        tk[m] = tk[i], ts[m] = ts[i], tc[m] = tc[i];
        ++m;
      }
    for (int i = 1; i < m; ++i)
      for (int k = i; k > 0 && tk[k - 1] > tk[k]; --k) {
        const int a = tk[k];
        tk[k] = tk[k - 1], tk[k - 1] = a;
        const double b = ts[k];
        ts[k] = ts[k - 1], ts[k - 1] = b;
        const long long d = tc[k];
        tc[k] = tc[k - 1], tc[k - 1] = d;
      }
    nkeys[c] = m;
  }
}

// update_g from rows (c, ct, sum, count) sorted by (c, ct) with offsets row_off
__global__ void k_update_g(int C, int G, const int64_t* row_off, const int* ct, const double* sum,
                           const long long* cnt, int* g, int* gcnt) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    const int64_t r0 = row_off[c], r1 = row_off[c + 1];
    int* out = g + (int64_t)c * G;
    int m = 0;
    out[m++] = c;
    double pv = -INFINITY;
    int pc = -1;
    const int64_t avail = r1 - r0;
    const int take = static_cast<int>(avail < G - 1 ? avail : G - 1);
    for (int t = 0; t < take; ++t) {  // next in (avg, ct) ascending after (pv, pc)
      double bv = INFINITY;
      int bc = -1;
      for (int64_t r = r0; r < r1; ++r) {
        const double v = sum[r] / static_cast<double>(cnt[r]);
        const int k = ct[r];
        const bool after = pc < 0 || v > pv || (v == pv && k > pc);
        if (!after) continue;
        if (bc < 0 || v < bv || (v == bv && k < bc)) bv = v, bc = k;
      }
      out[m++] = bc;
      pv = bv, pc = bc;
    }
    for (int i = 1; i < m; ++i)
      for (int k = i; k > 0 && out[k - 1] > out[k]; --k) {
        const int a = out[k];
        out[k] = out[k - 1], out[k - 1] = a;
      }
    gcnt[c] = m;
    for (int i = m; i < G; ++i) out[i] = -1;
  }
}

int ops_grid(int64_t n, int threads) {
  const int64_t b = (n + threads - 1) / threads;
  return static_cast<int>(b < 1 ? 1 : (b > 65535 ? 65535 : b));
}

}  // namespace

cudaError_t launch_log_joint_pairs(int D, int H, const float* X, const int* comp, int64_t n, const double* mu,
                                   const double* psi, const double* lam, const double* R, const double* kconst,
                                   double* out, cudaStream_t s) {
  if (H > 64) return cudaErrorInvalidValue;
  k_log_joint_pairs<<<ops_grid(n * 32, 256), 256, 0, s>>>(D, H, X, comp, n, mu, psi, lam, R, kconst, out);
  return cudaGetLastError();
}
cudaError_t launch_search_space(const Dims& dm, const int* K, const int* g, const int* gcnt, const int* extras,
                                uint64_t seed, uint64_t it, int* count, int* idx, cudaStream_t s) {
  k_search_space<<<ops_grid(dm.N, 128), 128, 0, s>>>(dm, K, g, gcnt, extras, seed, it, count, idx);
  return cudaGetLastError();
}
cudaError_t launch_update_k(const Dims& dm, const int* count, const int* idx, const double* lj, int* Kout,
                            int* status, cudaStream_t s) {
  k_update_k<<<ops_grid(dm.N, 128), 128, 0, s>>>(dm, count, idx, lj, Kout, status);
  return cudaGetLastError();
}
cudaError_t launch_hard_labels(const Dims& dm, const int* K, const int* count, const int* idx, const double* lj,
                               int* labels, cudaStream_t s) {
  k_hard_labels<<<ops_grid(dm.N, 128), 128, 0, s>>>(dm, K, count, idx, lj, labels);
  return cudaGetLastError();
}
cudaError_t launch_responsibilities(int64_t rows, int width, const double* lj, double* resp, cudaStream_t s) {
  k_responsibilities<<<ops_grid(rows, 128), 128, 0, s>>>(rows, width, lj, resp);
  return cudaGetLastError();
}
cudaError_t launch_distances(const Dims& dm, int mode, const int* part_off, const int* part_ent, const int* count,
                             const int* idx, const double* lj, const double* pi, const int64_t* tab_off,
                             const int* tab_cap, int* key, double* sum, long long* cnt, int* nkeys, cudaStream_t s) {
  k_distances<<<ops_grid(dm.C, 64), 64, 0, s>>>(dm, mode, part_off, part_ent, count, idx, lj, pi, tab_off, tab_cap,
                                                 key, sum, cnt, nkeys);
  return cudaGetLastError();
}
cudaError_t launch_update_g(int C, int G, const int64_t* row_off, const int* ct, const double* sum,
                            const long long* cnt, int* g, int* gcnt, cudaStream_t s) {
  k_update_g<<<ops_grid(C, 64), 64, 0, s>>>(C, G, row_off, ct, sum, cnt, g, gcnt);
  return cudaGetLastError();
}

}  // namespace vmfa_b200
