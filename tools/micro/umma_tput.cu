// Microbenchmark: back-to-back tcgen05.mma kind::tf32 (SS and TS) throughput
// per shape on one SM (cycles per instruction), M = 128, cta_group::1.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16; d |= (uint64_t)(1024 >> 4) << 32; d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61;
  return d;
}
__device__ int g_amn = 0;  // 1: A MN-major (bit 15), LBO 16 KB between 64-element atoms
__device__ __forceinline__ uint32_t idesc(int N, int kind_bf16) {
  const uint32_t fmt = kind_bf16 ? 1u : 2u;
  return (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24) |
         (g_amn ? (1u << 15) : 0u);
}
template <int TS, int BF16>
__global__ void k(int N, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t s_tmem;
  __shared__ uint64_t bar;
  const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
  for (int i = threadIdx.x * 16; i < 96 * 1024; i += blockDim.x * 16)
    asm volatile("st.shared.v4.b32 [%0], {%1,%1,%1,%1};" :: "r"(base + i), "r"(0));
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar))); }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc(N, BF16);
    uint64_t a = sdesc(base);
    if (g_amn) a = (a & ~(0x3FFFull << 16)) | ((uint64_t)((16384 >> 4) & 0x3FFF) << 16);
    const uint64_t b = sdesc(base + 32 * 1024);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (TS) {
        if (BF16) asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" :: "r"(tmem), "r"(tmem + 256), "l"(b), "r"(id), "r"(1));
        else asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;}" :: "r"(tmem), "r"(tmem + 256), "l"(b), "r"(id), "r"(1));
      } else {
        if (BF16) asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" :: "r"(tmem), "l"(a), "l"(b), "r"(id), "r"(1));
        else asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;}" :: "r"(tmem), "l"(a), "l"(b), "r"(id), "r"(1));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)));
    uint32_t ok = 0;
    do {
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p;}" : "=r"(ok) : "r"(smem_u32(&bar)));
    } while (!ok);
    unsigned long long t1 = clock64();
    out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}
int main(int argc, char** argv) {
  unsigned long long* d; cudaMalloc(&d, 8);
  if (argc > 1) { int one = 1; cudaMemcpyToSymbol(g_amn, &one, sizeof one); printf("A MN-major\n"); }
  const int Ns[] = {16, 32, 64, 96, 128, 192, 256};
  for (int ts = 0; ts < 2; ++ts) for (int bf = 0; bf < 2; ++bf) for (int N : Ns) {
    auto kern = ts ? (bf ? k<1,1> : k<1,0>) : (bf ? k<0,1> : k<0,0>);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int iters = 2000;
    kern<<<1, 128, 100 * 1024>>>(N, iters, d);
    unsigned long long c = 0;
    cudaError_t e = cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    const double cyc = (double)c / iters;
    const double kdim = bf ? 16 : 8;
    printf("%s %s N=%3d  cycles/mma=%7.2f  MAC/cycle=%8.1f\n", ts ? "TS" : "SS", bf ? "bf16" : "tf32", N, cyc,
           128.0 * N * kdim / cyc);
  }
  return 0;
}
