// Microbenchmark: random-row gather bandwidth (rows of `rowb` bytes from a
// 205 MB table, i.e. beyond L2), persistent grid of 148 CTAs:
//   mode 0: LDG.128, one warp per row-slice, U rows in flight per warp (registers)
//   mode 1: cp.async 16 B into a per-warp smem ring, depth U rows
//   mode 2: cp.async.bulk per row by one thread per warp, ring of U rows
// Reports aggregate GB/s of gathered bytes.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t hash(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}

template <int MODE, int U, int HH = 2>
__global__ void k(const float4* X, int64_t nrows, int rowb, int rows_per_warp, float* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar[32][U];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * nw + warp;
  const int f4 = rowb / 16;  // float4 per row
  float acc = 0.f;
  if (MODE == 0) {
    for (int r0 = 0; r0 < rows_per_warp; r0 += U) {
      float4 v[U][HH];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t row = hash(gw * 1000003 + r0 + u) % nrows;
#pragma unroll
        for (int h = 0; h < HH; ++h) {
          const int o = lane + 32 * h;
          v[u][h] = o < f4 ? __ldg(X + row * f4 + o) : make_float4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int h = 0; h < HH; ++h) acc += v[u][h].x + v[u][h].y + v[u][h].z + v[u][h].w;
    }
  } else if (MODE == 1) {
    const uint32_t base = smem_u32(sm) + warp * U * rowb;
    for (int r = 0; r < rows_per_warp + U; ++r) {
      if (r < rows_per_warp) {
        const int64_t row = hash(gw * 1000003 + r) % nrows;
        const uint32_t dst = base + (r % U) * rowb;
        for (int o = lane; o < f4; o += 32)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + o * 16), "l"(X + row * f4 + o) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      if (r >= U) {
        asm volatile("cp.async.wait_group %0;" ::"n"(U) : "memory");
        const uint32_t src = base + (r % U) * rowb;
        for (int o = lane; o < f4; o += 32) {
          float a, b, c, d;
          asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "r"(src + o * 16));
          acc += a + b + c + d;
        }
      }
    }
  } else if (MODE == 3) {
    // every lane issues one row's bulk copy: a batch of 32 rows per warp, U batches in flight
    const uint32_t base = smem_u32(sm) + warp * U * 32 * rowb;
    if (lane == 0)
      for (int u = 0; u < U; ++u) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[warp][u])));
    __syncwarp();
    const int nb = rows_per_warp / 32;
    for (int r = 0; r < nb + U; ++r) {
      if (r >= U) {
        const int u = r % U;
        const uint32_t ph = ((r - U) / U) & 1;
        uint32_t ok = 0;
        do {
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p;}"
                       : "=r"(ok) : "r"(smem_u32(&bar[warp][u])), "r"(ph));
        } while (!ok);
        const uint32_t src = base + u * 32 * rowb + lane * rowb;
        for (int o = 0; o < f4; o += 8) {
          float a, b, c, d;
          asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "r"(src + o * 16));
          acc += a + b + c + d;
        }
        __syncwarp();
      }
      if (r < nb) {
        const int u = r % U;
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[warp][u])), "r"(32 * rowb) : "memory");
        __syncwarp();
        const int64_t row = hash(gw * 1000003 + r * 32 + lane) % nrows;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(base + u * 32 * rowb + lane * rowb),
                     "l"(X + row * f4), "r"(rowb), "r"(smem_u32(&bar[warp][u])) : "memory");
      }
      __syncwarp();
    }
  } else {
    const uint32_t base = smem_u32(sm) + warp * U * rowb;
    if (lane == 0)
      for (int u = 0; u < U; ++u) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[warp][u])));
    __syncwarp();
    for (int r = 0; r < rows_per_warp + U; ++r) {
      if (r >= U) {
        const int u = r % U;
        const uint32_t ph = ((r - U) / U) & 1;
        uint32_t ok = 0;
        do {
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p;}"
                       : "=r"(ok) : "r"(smem_u32(&bar[warp][u])), "r"(ph));
        } while (!ok);
        const uint32_t src = base + u * rowb;
        for (int o = lane; o < f4; o += 32) {
          float a, b, c, d;
          asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "r"(src + o * 16));
          acc += a + b + c + d;
        }
        __syncwarp();
      }
      if (r < rows_per_warp && lane == 0) {
        const int u = r % U;
        const int64_t row = hash(gw * 1000003 + r) % nrows;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[warp][u])), "r"(rowb) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(base + u * rowb),
                     "l"(X + row * f4), "r"(rowb), "r"(smem_u32(&bar[warp][u])) : "memory");
      }
      __syncwarp();
    }
  }
  if (acc == 1234.5f) sink[0] = acc;
}

int main(int argc, char** argv) {
  const int64_t nrows = argc > 1 ? atoll(argv[1]) : 200000;
  const int rowb = argc > 2 ? atoi(argv[2]) : 1024;
  if (argc > 1) {  // large-table mode: LDG gathers of long rows only
    float4* X;
    cudaMalloc(&X, nrows * rowb);
    cudaMemset(X, 0, nrows * rowb);
    float* sink;
    cudaMalloc(&sink, 4);
    for (int rep = 0; rep < 2; ++rep)
    for (int threads : {256, 512}) {
      auto kern = rowb <= 512 ? k<0, 24, 1> : k<0, 4, 7>;
      const int rpw = 512;
      kern<<<148, threads>>>(X, nrows, rowb, 16, sink);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      kern<<<148, threads>>>(X, nrows, rowb, rpw, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("table %.2f GB rows %d B threads %d: %7.1f GB/s %s\n", nrows * (double)rowb / 1e9, rowb, threads,
             148.0 * (threads / 32) * rpw * rowb / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    // contiguous rows (same kernel, row = sequential): stream reference
    return 0;
  }
  float4* X;
  cudaMalloc(&X, nrows * rowb);
  cudaMemset(X, 0, nrows * rowb);
  float* sink;
  cudaMalloc(&sink, 4);
  const int rows_per_warp = 2048;
  auto run = [&](auto kern, int mode, int U, int threads, size_t smem) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<148, threads, smem>>>(X, nrows, rowb, 64, sink);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<148, threads, smem>>>(X, nrows, rowb, rows_per_warp, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = 148.0 * (threads / 32) * rows_per_warp * rowb;
    printf("mode %d U %2d warps %2d smem %6zu: %7.1f GB/s  %s\n", mode, U, threads / 32, smem, bytes / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  };
  run(k<0, 4>, 0, 4, 256, 0);
  run(k<0, 8>, 0, 8, 256, 0);
  run(k<0, 8>, 0, 8, 512, 0);
  run(k<0, 8>, 0, 8, 1024, 0);
  run(k<1, 4>, 1, 4, 256, 8 * 4 * 1024);
  run(k<1, 8>, 1, 8, 256, 8 * 8 * 1024);
  run(k<1, 8>, 1, 8, 512, 16 * 8 * 1024);
  run(k<1, 4>, 1, 4, 1024, 32 * 4 * 1024);
  run(k<3, 2>, 3, 2, 64, 2 * 2 * 32 * 1024);
  run(k<3, 2>, 3, 2, 96, 3 * 2 * 32 * 1024);
  run(k<3, 3>, 3, 3, 64, 2 * 3 * 32 * 1024);
  run(k<3, 1>, 3, 1, 192, 6 * 1 * 32 * 1024);
  run(k<2, 4>, 2, 4, 256, 8 * 4 * 1024);
  run(k<2, 8>, 2, 8, 256, 8 * 8 * 1024);
  run(k<2, 12>, 2, 12, 512, 16 * 12 * 1024);
  run(k<2, 6>, 2, 6, 1024, 32 * 6 * 1024);
  return 0;
}
