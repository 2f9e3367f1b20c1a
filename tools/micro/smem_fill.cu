// Microbenchmark: how fast can one SM fill shared memory from an L2-resident
// buffer? Persistent grid (1 CTA/SM), each CTA repeatedly copies `chunk`
// bytes from a 16 MB source (random 2 KB blocks) into a smem ring.
//   mode 0: cp.async.cg 16 B by `nw` warps (wait_all per chunk)
//   mode 1: cp.async.bulk of `blk` bytes per instruction by one thread
//   mode 2: ld.global.v4 + st.shared.v4 by `nw` warps
// Reports cycles per chunk (CTA 0) and aggregate GB/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_fill(const float4* src, size_t src_blocks, int mode, int chunk, int blk, int iters,
                       unsigned long long* cyc, int nw) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  const int tid = threadIdx.x;
  const uint32_t base = smem_u32(sm);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t rng = 0x9e3779b97f4a7c15ull * (blockIdx.x + 1);
  unsigned long long t0 = clock64();
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    const int nblk = chunk / 2048;
    if (mode == 3) {  // streaming LDG.128, 8 independent loads per thread in flight
      if (tid < nw * 32) {
        const size_t per = (size_t)chunk / 16;  // float4 per chunk
        const size_t cb = ((size_t)(blockIdx.x * 7919u + it * 104729u) % (src_blocks * 128 / per)) * per;
        for (size_t o = tid; o < per; o += nw * 32 * 8) {
          float4 v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = o + u * nw * 32 < per ? __ldg(src + cb + o + u * nw * 32) : make_float4(0, 0, 0, 0);
#pragma unroll
          for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
        }
      }
      __syncthreads();
      continue;
    }
    if (mode == 0 || mode == 2) {
      if (tid < nw * 32) {
        for (int b = 0; b < nblk; ++b) {
          rng = rng * 6364136223846793005ull + 1442695040888963407ull;
          const size_t sb = (rng >> 33) % src_blocks;
          const float4* s = src + sb * 128;
          for (int o = tid; o < 128; o += nw * 32) {
            const uint32_t dst = base + b * 2048 + o * 16;
            if (mode == 0) {
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(s + o) : "memory");
            } else {
              const float4 v = __ldg(s + o);
              asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "f"(v.x), "f"(v.y), "f"(v.z),
                           "f"(v.w)
                           : "memory");
            }
          }
        }
        if (mode == 0) asm volatile("cp.async.wait_all;" ::: "memory");
      }
      __syncthreads();
    } else {
      if (tid == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(chunk)
                     : "memory");
        for (int off = 0; off < chunk; off += blk) {
          rng = rng * 6364136223846793005ull + 1442695040888963407ull;
          const size_t sb = ((rng >> 33) % (src_blocks * 2048 / blk));
          const char* s = reinterpret_cast<const char*>(src) + sb * blk;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  base + off),
              "l"(s), "r"(blk), "r"(smem_u32(&bar))
              : "memory");
        }
        uint32_t ok = 0;
        do {
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p;}"
                       : "=r"(ok)
                       : "r"(smem_u32(&bar)), "r"(it & 1));
        } while (!ok);
      }
      __syncthreads();
    }
  }
  if (tid == 0) cyc[blockIdx.x] = clock64() - t0;
  if (acc == 12345.f) cyc[0] = 0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = 16u << 20;
  float4* src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sizeof(unsigned long long) * sms);
  cudaFuncSetAttribute(k_fill, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int chunk = 28 * 1024 / 2048 * 2048;  // 28 KB
  const int iters = 200;
  struct Cfg { int mode, nw, blk; };
  const Cfg cfgs[] = {{3, 2, 0}, {3, 4, 0}, {3, 8, 0}, {0, 1, 0}, {0, 2, 0}, {0, 4, 0}, {0, 8, 0}, {2, 2, 0}, {2, 4, 0}, {2, 8, 0},
                      {1, 0, 1024}, {1, 0, 2048}, {1, 0, 4096}, {1, 0, 14336}, {1, 0, 28672}};
  for (const Cfg& c : cfgs) {
    for (int grid : {1, sms}) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      k_fill<<<grid, 256, 64 * 1024>>>(src, bytes / 2048, c.mode, chunk, c.blk, 5, cyc, c.nw);
      cudaEventRecord(e0);
      k_fill<<<grid, 256, 64 * 1024>>>(src, bytes / 2048, c.mode, chunk, c.blk, iters, cyc, c.nw);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long h = 0;
      cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      const double gbs = (double)chunk * iters * grid / (ms * 1e-3) / 1e9;
      printf("mode %d nw %d blk %6d grid %3d: %8.0f cyc/chunk (CTA0)  %8.1f B/cyc/SM  agg %8.1f GB/s  %s\n", c.mode,
             c.nw, c.blk, grid, (double)h / iters, (double)chunk * iters / h, gbs, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
