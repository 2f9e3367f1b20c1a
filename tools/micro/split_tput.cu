// Microbenchmark: SM throughput of the scorer producers' per-element operand
// split (v = (x - mu) s, q = v^2 2^-14, each split into hi / lo halves).
//   variant 0: fp16 via cvt pack + unpack (current split2)
//   variant 1: fp16 via Veltkamp split (x*(2^13+1)) + cvt pack of hi and lo
//   variant 2: tf32 split_fast (integer round + residual)
// 8 warps per SM (like the producers), 148 CTAs; reports cycles per element per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ void split_cvt(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x0, x1);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
__device__ __forceinline__ void split_vk(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const float c0 = x0 * 8193.0f, c1 = x1 * 8193.0f;
  const float h0 = c0 - (c0 - x0), h1 = c1 - (c1 - x1);
  const __half2 h = __floats2half2_rn(h0, h1);
  const __half2 l = __floats2half2_rn(x0 - h0, x1 - h1);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
__device__ __forceinline__ void split_tf(float x, uint32_t& hi, uint32_t& lo) {
  hi = (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
  lo = __float_as_uint(x - __uint_as_float(hi));
}

template <int V>
__global__ void k(const float* in, int iters, unsigned long long* cyc, uint32_t* sink) {
  float x[32], mu[32];
  for (int i = 0; i < 32; ++i) {
    x[i] = in[(threadIdx.x * 32 + i) & 1023];
    mu[i] = in[(threadIdx.x * 7 + i) & 1023];
  }
  const float sA = 64.f;
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t vh[16], vl[16], qh[16], ql[16];
    if (V == 2) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float v = (x[i] - mu[i]) * sA;
        split_tf(v, vh[i], vl[i]);
        split_tf(v * v, qh[i], ql[i]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float v0 = (x[2 * i] - mu[2 * i]) * sA, v1 = (x[2 * i + 1] - mu[2 * i + 1]) * sA;
        const float q0 = (v0 * v0) * 6.103515625e-05f, q1 = (v1 * v1) * 6.103515625e-05f;
        if (V == 0) {
          split_cvt(v0, v1, vh[i], vl[i]);
          split_cvt(q0, q1, qh[i], ql[i]);
        } else {
          split_vk(v0, v1, vh[i], vl[i]);
          split_vk(q0, q1, qh[i], ql[i]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) acc ^= vh[i] + vl[i] * 3u + qh[i] * 5u + ql[i] * 7u;
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = __uint_as_float(__float_as_uint(x[i]) ^ (acc & 1u));
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  float* in;
  cudaMalloc(&in, 4096 * 4);
  cudaMemset(in, 0, 4096 * 4);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  uint32_t* sink;
  cudaMalloc(&sink, 148 * 256 * 4);
  const int iters = 2000;
  auto run = [&](auto kern, const char* name, int per_iter) {
    kern<<<148, 256>>>(in, 10, cyc, sink);
    kern<<<148, 256>>>(in, iters, cyc, sink);
    cudaDeviceSynchronize();
    unsigned long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    // elements per SM per iteration: 256 threads x 32 (16 v + 16 q ... = 32 x values -> 32 v and 32 q)
    const double elems = 256.0 * per_iter * iters;
    printf("%-28s %8.3f cyc per x element per SM (%s)\n", name, (double)h / elems, cudaGetErrorString(cudaGetLastError()));
  };
  run(k<0>, "fp16 cvt pack+unpack", 32);
  run(k<1>, "fp16 Veltkamp + pack", 32);
  run(k<2>, "tf32 split_fast", 16);
  return 0;
}
