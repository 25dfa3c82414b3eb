// Microbenchmark: cycles per tcgen05.mma.cta_group::1.kind::i8 (M=128, K=32)
// for several N, A from smem (SS) or TMEM (TS). One CTA per SM, one issuing
// thread, back-to-back MMAs into one accumulator, timed with clock64 around
// a commit+wait. Dev tool for choosing the K3 tile shape.
#include <cuda.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ uint32_t idesc(int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

template <bool TS>
__global__ void bench(int N, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 128 * 1024 / 4; i += blockDim.x) ((uint32_t*)s)[i] = i * 2654435761u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc(N);
    const uint64_t a = desc(smem_u32(s));
    const uint64_t b = desc(smem_u32(s + 65536));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t acc = i > 0;
      if (TS) {
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(tm + 256), "r"(tm + (i & 7) * 8), "l"(b), "r"(id), "r"(acc));
      } else {
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tm + 256), "l"(a + (i & 3) * 2), "l"(b), "r"(id), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)));
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  const int iters = 4096;
  for (int ts = 0; ts < 2; ++ts) {
    for (int N : {32, 64, 128, 256}) {
      if (ts && N > 256) continue;
      auto k = ts ? bench<true> : bench<false>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
      k<<<148, 128, 140 * 1024>>>(N, iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148.0 * iters;
      double macs = 128.0 * N * 32;
      printf("%s N=%3d: %6.1f cycles/MMA, %7.0f MACs/cycle/SM (%s)\n", ts ? "TS" : "SS", N, avg,
             macs / avg, cudaGetErrorString(e));
    }
  }
  return 0;
}
