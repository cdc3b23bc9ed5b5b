// Probe (not part of the library): tcgen05 kind::tf32 with MN-major
// SWIZZLE_128B operands (A and / or B), both LBO/SBO field assignments.
// MN-major SW128 (32-bit elements): element (mn, k) at
//   (mn / 32) * MNBLK + (k / 8) * 1024 + (k % 8) * 128 + ((((mn % 32) / 4) ^ (k % 8)) * 16) + (mn % 4) * 4
// K-major SW128: element (row, k) at (k / 32) * ROWS * 128 + row * 128 + (((k % 32) / 4 ^ row % 8) * 16) + (k % 4) * 4
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_mn2 umma_mn2.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t mkdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, bool amn, bool bmn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((amn ? 1u : 0u) << 15) | ((bmn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
constexpr int M = 128, K = 128, NMAX = 128;
__device__ uint32_t kmaj(int r, int k, int rows) {
  return (uint32_t)((k / 32) * rows * 128 + r * 128 + ((((k % 32) / 4) ^ (r % 8)) * 16) + (k % 4) * 4);
}
__device__ uint32_t mnmaj(int mn, int k) {
  return (uint32_t)((mn / 32) * K * 128 + (k / 8) * 1024 + (k % 8) * 128 + ((((mn % 32) / 4) ^ (k % 8)) * 16) +
                    (mn % 4) * 4);
}
__global__ void probe(int N, int amn, int bmn, int variant, const float* A, const float* B, float* D) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* sm = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  char* sa = sm;
  char* sb = sm + M * K * 4;
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t s_mbar;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&s_tmem)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&s_mbar)));
  for (int e = threadIdx.x; e < M * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    *(float*)(sa + (amn ? mnmaj(r, k) : kmaj(r, k, M))) = A[e];
  }
  for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    *(float*)(sb + (bmn ? mnmaj(r, k) : kmaj(r, k, N))) = B[e];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = s_tmem;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc(M, N, amn, bmn);
    const uint32_t blk = K * 128;  // MN block stride
    for (int k0 = 0; k0 < K; k0 += 8) {
      uint64_t ad, bd;
      if (amn) {
        const uint32_t s = su32(sa) + (k0 / 8) * 1024;
        ad = variant == 0 ? mkdesc(s, blk, 1024) : mkdesc(s, 1024, blk);
      } else {
        ad = mkdesc(su32(sa) + (k0 / 32) * M * 128 + (k0 % 32) * 4, 16, 1024);
      }
      if (bmn) {
        const uint32_t s = su32(sb) + (k0 / 8) * 1024;
        bd = variant == 0 ? mkdesc(s, blk, 1024) : mkdesc(s, 1024, blk);
      } else {
        bd = mkdesc(su32(sb) + (k0 / 32) * N * 128 + (k0 % 32) * 4, 16, 1024);
      }
      const uint32_t acc = k0 > 0 ? 1u : 0u;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm),
                   "l"(ad), "l"(bd), "r"(id), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&s_mbar))
                 : "memory");
  }
  asm volatile("{\n\t.reg .pred d;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 d, [%0], 0;\n\t@!d bra W;\n\t}\n" ::"r"(
                   su32(&s_mbar))
               : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    const int row = warp * 32 + lane;
    for (int c = 0; c < N; ++c) {
      uint32_t v;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tm + ((uint32_t)(warp * 32) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      D[row * N + c] = __uint_as_float(v);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(128));
}
int main() {
  std::vector<float> A(M * K), B(NMAX * K), D(M * NMAX);
  srand(1);
  for (auto& v : A) v = (float)(rand() % 33 - 16) / 8.f;  // exact in tf32
  for (auto& v : B) v = (float)(rand() % 33 - 16) / 8.f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  for (int amn = 0; amn < 2; ++amn)
    for (int bmn = 0; bmn < 2; ++bmn)
      for (int N : {32, 64, 128})
        for (int variant = 0; variant < 2; ++variant) {
          if (!amn && !bmn && variant) continue;
          cudaMemset(dD, 0, D.size() * 4);
          probe<<<1, 128, (M + NMAX) * K * 4 + 1024>>>(N, amn, bmn, variant, dA, dB, dD);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) {
            printf("amn=%d bmn=%d N=%d variant=%d CUDA error %s\n", amn, bmn, N, variant, cudaGetErrorString(e));
            return 1;
          }
          cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
          double maxerr = 0, maxref = 0, maxd = 0;
          for (int i = 0; i < M; ++i)
            for (int j = 0; j < N; ++j) {
              double s = 0;
              for (int k = 0; k < K; ++k) s += (double)A[i * K + k] * B[j * K + k];
              maxerr = fmax(maxerr, fabs(s - D[i * N + j]));
              maxref = fmax(maxref, fabs(s));
              maxd = fmax(maxd, fabs(D[i * N + j]));
            }
          printf("A %s B %s N=%3d variant=%d (%s): max|err| %.3g max|ref| %.3g max|D| %.3g %s\n", amn ? "MN" : "K ",
                 bmn ? "MN" : "K ", N, variant, variant == 0 ? "LBO=MN blk,SBO=1024" : "LBO=1024,SBO=MN blk", maxerr,
                 maxref, maxd, maxerr == 0 ? "EXACT" : "MISMATCH");
        }
  return 0;
}
