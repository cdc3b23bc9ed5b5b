// Probe of tcgen05 kind::tf32 operand layouts on this GPU (not part of the
// library): K-major interleave / SW128, MN-major interleave, A from TMEM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_probe umma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t mkdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)(layout & 7u) << 61;
  return d;
}

__host__ __device__ constexpr uint32_t idesc(int M, int N, bool amn, bool bmn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((amn ? 1u : 0u) << 15) | ((bmn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

enum Mode { KNONE = 0, KSW128 = 1, MNNONE = 2, TMEM_A = 3, MNNONE_SWAP = 4 };

constexpr int M = 128, N = 64;

// byte offset of element (r, k) in an operand image with R rows and K cols
__device__ uint32_t img_off(int mode, int r, int k, int R, int K) {
  switch (mode) {
    case KNONE: return (uint32_t)(((k / 4) * R + r) * 16 + (k % 4) * 4);
    case KSW128: {
      const int kb = k / 32, kk = k % 32;
      return (uint32_t)(kb * R * 128 + r * 128 + (((kk / 4) ^ (r % 8)) * 16) + (kk % 4) * 4);
    }
    case MNNONE:
    case MNNONE_SWAP:
      return (uint32_t)(((r / 4) * (K / 8) + k / 8) * 128 + (k % 8) * 16 + (r % 4) * 4);
  }
  return 0;
}

__device__ uint64_t step_desc(int mode, const float* base, int k0, int R, int K) {
  const uint32_t a = su32(base);
  switch (mode) {
    case KNONE: return mkdesc(a + (k0 / 4) * R * 16, R * 16, 128, 0);
    case KSW128: return mkdesc(a + (k0 / 32) * R * 128 + (k0 % 32) * 4, 16, 1024, 2);
    case MNNONE: return mkdesc(a + (k0 / 8) * 128, 128, (K / 8) * 128, 0);
    case MNNONE_SWAP: return mkdesc(a + (k0 / 8) * 128, (K / 8) * 128, 128, 0);
  }
  return 0;
}

__global__ void probe(int amode, int bmode, int K, const float* A, const float* B, float* D) {
  extern __shared__ __align__(1024) float smem[];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t s_mbar;
  float* sa = smem;               // M x K
  float* sb = smem + M * K;       // N x K (1024-aligned: M*K*4 multiple of 1024)
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&s_tmem)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&s_mbar)));
  for (int e = threadIdx.x; e < M * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    if (amode != TMEM_A) *(float*)((char*)sa + img_off(amode, r, k, M, K)) = A[e];
  }
  for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    *(float*)((char*)sb + img_off(bmode, r, k, N, K)) = B[e];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = s_tmem;
  const uint32_t ta = tm + 128;  // A operand columns
  if (amode == TMEM_A && warp < 4) {
    const int row = warp * 32 + lane;
    for (int k = 0; k < K; k += 4) {
      uint32_t r0 = __float_as_uint(A[row * K + k]), r1 = __float_as_uint(A[row * K + k + 1]);
      uint32_t r2 = __float_as_uint(A[row * K + k + 2]), r3 = __float_as_uint(A[row * K + k + 3]);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(ta + ((uint32_t)(warp * 32) << 16) + k),
                   "r"(r0), "r"(r1), "r"(r2), "r"(r3));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    const uint32_t id = idesc(M, N, amode == MNNONE || amode == MNNONE_SWAP, bmode == MNNONE || bmode == MNNONE_SWAP);
    for (int k0 = 0; k0 < K; k0 += 8) {
      const uint64_t bd = step_desc(bmode, sb, k0, N, K);
      const uint32_t acc = k0 > 0 ? 1u : 0u;
      if (amode == TMEM_A) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tm),
                     "r"(ta + k0), "l"(bd), "r"(id), "r"(acc));
      } else {
        const uint64_t ad = step_desc(amode, sa, k0, M, K);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm),
                     "l"(ad), "l"(bd), "r"(id), "r"(acc));
      }
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
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}

int main() {
  const char* names[] = {"K-none", "K-sw128", "MN-none", "tmem", "MN-none-swap"};
  int cases[][3] = {{KNONE, KNONE, 32},  {KSW128, KSW128, 32}, {KSW128, KSW128, 128}, {MNNONE, KNONE, 32},
                    {KNONE, MNNONE, 32}, {MNNONE_SWAP, KNONE, 32}, {KNONE, MNNONE_SWAP, 32}, {TMEM_A, KNONE, 32},
                    {TMEM_A, KSW128, 128}, {MNNONE, MNNONE, 64}, {TMEM_A, MNNONE, 64}};
  const int Kmax = 128;
  std::vector<float> A(M * Kmax), B(N * Kmax), D(M * N);
  srand(1);
  for (auto& v : A) v = (float)(rand() % 33 - 16) / 8.f;
  for (auto& v : B) v = (float)(rand() % 33 - 16) / 8.f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (auto& cs : cases) {
    const int K = cs[2];
    // A is M x K, B is N x K (row-major, dense for this K)
    std::vector<float> a(M * K), b(N * K);
    for (int i = 0; i < M * K; ++i) a[i] = A[i];
    for (int i = 0; i < N * K; ++i) b[i] = B[i];
    cudaMemcpy(dA, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, D.size() * 4);
    const size_t sm = (size_t)(M + N) * K * 4 + 1024;
    probe<<<1, 256, sm>>>(cs[0], cs[1], K, dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("A=%-12s B=%-12s K=%3d  CUDA error %s\n", names[cs[0]], names[cs[1]], K, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double s = 0;
        for (int k = 0; k < K; ++k) s += (double)a[i * K + k] * b[j * K + k];
        maxerr = fmax(maxerr, fabs(s - D[i * N + j]));
        maxref = fmax(maxref, fabs(s));
      }
    printf("A=%-12s B=%-12s K=%3d  max|err| %.3g  (max|ref| %.3g)  %s\n", names[cs[0]], names[cs[1]], K, maxerr,
           maxref, maxerr == 0 ? "EXACT" : "MISMATCH");
  }
  return 0;
}
