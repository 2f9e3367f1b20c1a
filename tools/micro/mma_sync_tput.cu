// Throughput of warp-level mma.sync on sm_100a (legacy tensor-core path):
// m16n8k8 tf32 and m16n8k16 f16, fp32 accumulate, independent accumulator
// chains per warp, W warps per SM. Prints mma/clk/SM and dense TFLOP/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_sync_tput mma_sync_tput.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void k_tf32(float* out, int iters) {
  float c[kChains][4] = {};
  uint32_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < kChains; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0.f;
  for (int j = 0; j < kChains; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 1.2345f) out[threadIdx.x] = s;
}

__global__ void k_f16(float* out, int iters) {
  float c[kChains][4] = {};
  uint32_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < kChains; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0.f;
  for (int j = 0; j < kChains; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 1.2345f) out[threadIdx.x] = s;
}

__global__ void k_ffma(float* out, int iters) {
  float c[kChains * 4];
  for (int j = 0; j < kChains * 4; ++j) c[j] = threadIdx.x * 1e-3f + j;
  const float m = 0.999f, d = 1e-4f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int j = 0; j < kChains * 4; ++j) c[j] = fmaf(c[j], m, d);
  }
  float s = 0.f;
  for (int j = 0; j < kChains * 4; ++j) s += c[j];
  if (s == 1.2345f) out[threadIdx.x] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, 4096 * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    for (int kind = 0; kind < 3; ++kind) {
      auto run = [&]() {
        if (kind == 0) k_tf32<<<sms, warps * 32>>>(out, kIters);
        else if (kind == 1) k_f16<<<sms, warps * 32>>>(out, kIters);
        else k_ffma<<<sms, warps * 32>>>(out, kIters / 16);
      };
      run();
      cudaEventRecord(e0);
      run();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ghz = clk * 1e-6;
      if (kind < 2) {
        const double mmas = (double)sms * warps * kIters * kChains;
        const double flop = mmas * (kind == 0 ? 16 * 8 * 8 : 16 * 8 * 16) * 2;
        printf("%-5s warps/SM=%2d  %.3f ms  %.3f mma/clk/SM  %.1f TFLOP/s\n", kind == 0 ? "tf32" : "f16", warps, ms,
               mmas / sms / (ms * 1e-3 * ghz * 1e9), flop / (ms * 1e-3) / 1e12);
      } else {
        const double fma = (double)sms * warps * 32 * (kIters / 16) * 16 * kChains * 4;
        printf("ffma  warps/SM=%2d  %.3f ms  %.1f FMA/clk/SM  %.1f TFLOP/s\n", warps, ms,
               fma / sms / (ms * 1e-3 * ghz * 1e9), 2 * fma / (ms * 1e-3) / 1e12);
      }
    }
  }
  printf("(clock rate attribute %.3f GHz)\n", clk * 1e-6);
  return 0;
}
