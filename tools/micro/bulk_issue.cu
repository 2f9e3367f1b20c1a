// Microbenchmark: issue cost of cp.async.bulk row copies (1 KB rows gathered
// from a 200 MB table) -- cycles for one warp to issue 32 copies when
//   mode 0: 32 lanes each issue one copy (one instruction, lanes serialised)
//   mode 1: lane 0 issues all 32 in a loop
//   mode 2: 4 lanes of each of 8 warps issue one each (k_stats' pattern), warp 0 timed
//   mode 3: 32 lanes each issue one 16-byte cp.async x 64 (one row's worth per lane... 2 KB/lane)
// Prints the median over CTAs of the issue-loop cycles (wait excluded).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t hash(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}

__global__ void k(const float* X, int64_t nrows, int mode, unsigned long long* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t base = smem_u32(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned long long t_acc = 0;
  for (int it = 0; it < 16; ++it) {
    __syncthreads();
    const uint32_t rowb = 1024;
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(32 * rowb) : "memory");
    __syncthreads();
    const unsigned long long t0 = clock64();
    if (mode == 0 && warp == 0) {
      const int64_t row = hash(blockIdx.x * 100003 + it * 32 + lane) % nrows;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(base + lane * rowb),
                   "l"(X + row * 256), "r"(rowb), "r"(smem_u32(&bar)) : "memory");
    } else if (mode == 1 && threadIdx.x == 0) {
      for (int r = 0; r < 32; ++r) {
        const int64_t row = hash(blockIdx.x * 100003 + it * 32 + r) % nrows;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(base + r * rowb),
                     "l"(X + row * 256), "r"(rowb), "r"(smem_u32(&bar)) : "memory");
      }
    } else if (mode == 2 && lane < 4) {
      const int r = warp * 4 + lane;
      const int64_t row = hash(blockIdx.x * 100003 + it * 32 + r) % nrows;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(base + r * rowb),
                   "l"(X + row * 256), "r"(rowb), "r"(smem_u32(&bar)) : "memory");
    } else if (mode == 3) {
      // 256 threads x 8 x 16 B = 32 KB, thread = (row slot, column)
      for (int j = 0; j < 8; ++j) {
        const int i = threadIdx.x + 256 * j;
        const int r = i >> 6, f = i & 63;
        const int64_t row = hash(blockIdx.x * 100003 + it * 32 + r) % nrows;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(base + r * rowb + f * 16), "l"(X + row * 256 + f * 4) : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    }
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) t_acc += t1 - t0;
    // wait for completion
    if (mode == 3) {
      // the barrier expects 1 arrival + 32 KB tx from expect_tx; noinc arrivals of 256 threads would
      // over-arrive -- so mode 3 waits with cp.async.wait_all instead and completes the tx by hand
      asm volatile("cp.async.wait_all;" ::: "memory");
    }
    __syncthreads();
    if (mode != 3) {
      uint32_t ok = 0;
      do {
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p;}"
                     : "=r"(ok) : "r"(smem_u32(&bar)), "r"(it & 1));
      } while (!ok);
    }
  }
  if (threadIdx.x == 0) out[blockIdx.x] = t_acc / 16;
}

int main() {
  const int64_t nrows = 200000;
  float* X;
  cudaMalloc(&X, nrows * 1024);
  cudaMemset(X, 0, nrows * 1024);
  unsigned long long* out;
  cudaMalloc(&out, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  for (int mode : {0, 1, 2}) {
    k<<<148, 256, 40 * 1024>>>(X, nrows, mode, out);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> h(148);
    cudaMemcpy(h.data(), out, 148 * 8, cudaMemcpyDeviceToHost);
    std::sort(h.begin(), h.end());
    printf("mode %d: issue cycles (thread 0 timeline) median %llu  min %llu  max %llu  %s\n", mode, h[74], h[0], h[147],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
