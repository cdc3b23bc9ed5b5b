// Microbenchmark (not part of the library): tcgen05.ld 32x32b.x32 (+ wait::ld)
// latency / throughput per warp, for 4 / 8 / 16 warps per CTA, one CTA per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tmem_ld_bench tmem_ld_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int X>
__global__ void bench(int iters, int batch, unsigned long long* cyc, float* sink) {
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&s_tmem)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16);
  float acc = 0.f;
  const unsigned long long c0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t r[32];
    for (int b = 0; b < batch; ++b) {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
            "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
            "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(t + 32 * (b & 3)));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int k = 0; k < 32; ++k) acc += __uint_as_float(r[k]);
  }
  const unsigned long long c1 = clock64();
  if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + warp] = c1 - c0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(128));
}
int main() {
  unsigned long long* cyc;
  float* sink;
  cudaMalloc(&cyc, 148 * 32 * 8);
  cudaMalloc(&sink, 148 * 1024 * 4);
  for (int warps : {1, 4, 8, 16})
    for (int batch : {1, 4}) {
      const int iters = 1000;
      bench<32><<<148, 32 * warps>>>(iters, batch, cyc, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      unsigned long long h[32];
      cudaMemcpy(h, cyc, 8 * 32, cudaMemcpyDeviceToHost);
      printf("warps %2d batch %d: %.1f cycles per (batch of tcgen05.ld x32 + wait), warp 0\n", warps, batch,
             (double)h[0] / iters);
    }
  return 0;
}
