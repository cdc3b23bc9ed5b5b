// Latency of tcgen05.mma chains (kind::tf32, M = 128) on this GPU: issue +
// commit + mbarrier wait, for chain lengths / N / A-operand source.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_timing umma_timing.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t dsw(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int N, bool TA>
__global__ void bench(int chain, long long* out) {
  extern __shared__ __align__(16) char raw[];
  char* sm = raw + ((1024u - (su32(raw) & 1023u)) & 1023u);
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t mbar;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&s_tmem)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((float*)sm)[i] = 0.001f * (i % 7);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = s_tmem;
  uint32_t phase = 0;
  for (int rep = 0; rep < 3; ++rep) {
    long long t0 = clock64();
    if (threadIdx.x == 0) {
      const uint64_t a = dsw(su32(sm)), b = dsw(su32(sm + 32768));
      for (int i = 0; i < chain; ++i) {
        const uint32_t o = (uint32_t)((i & 3) * 32) >> 4;
        if (TA)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tm + 256),
                       "r"(tm + (i & 15) * 8), "l"(b + o), "r"(idesc(128, N)), "r"(i > 0 ? 1u : 0u));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm + 256),
                       "l"(a + o), "l"(b + o), "r"(idesc(128, N)), "r"(i > 0 ? 1u : 0u));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar)) : "memory");
    }
    asm volatile("{\n\t.reg .pred d;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1;\n\t@!d bra W;\n\t}\n" ::"r"(su32(&mbar)), "r"(phase) : "memory");
    phase ^= 1;
    long long t1 = clock64();
    if (threadIdx.x == 0 && rep == 2) out[0] = t1 - t0;
    __syncthreads();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  long long h;
  auto run = [&](auto kern, const char* name, int chain) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    kern<<<1, 128, 80 * 1024>>>(chain, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-18s chain %3d: %7lld cycles (%6.1f / mma) %s\n", name, chain, h, (double)h / chain, e ? cudaGetErrorString(e) : "");
  };
  for (int ch : {1, 4, 16, 32, 64}) {
    run(bench<32, false>, "N=32 smem A", ch);
    run(bench<64, false>, "N=64 smem A", ch);
    run(bench<128, false>, "N=128 smem A", ch);
    run(bench<256, false>, "N=256 smem A", ch);
    run(bench<64, true>, "N=64 tmem A", ch);
    run(bench<128, true>, "N=128 tmem A", ch);
  }
  return 0;
}
