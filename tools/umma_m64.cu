// Where do the rows of an M=64 kind::tf32 accumulator land in TMEM?
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "ttb_umma.cuh"
using namespace ttb;
constexpr int M = 64, N = 32, K = 16;
__global__ void k(const float* A, const float* B, float* D) {
  extern __shared__ __align__(128) unsigned char sm[];
  float* a = (float*)sm; float* b = a + M * K;
  __shared__ uint64_t mbar; __shared__ uint32_t tbase;
  for (int e = threadIdx.x; e < M * K; e += blockDim.x) { int m = e / K, kk = e % K; *(float*)((char*)a + umma::kmaj_off(m, kk, M)) = A[e]; }
  for (int e = threadIdx.x; e < K * N; e += blockDim.x) { int kk = e / N, n = e % N; *(float*)((char*)b + umma::kmaj_off(n, kk, N)) = B[e]; }
  umma::fence_smem_to_async();
  if (threadIdx.x < 32) umma::tmem_alloc(&tbase, 32);
  if (threadIdx.x == 0) umma::mbar_init(&mbar, 1);
  umma::fence_before_sync(); __syncthreads(); umma::fence_after_sync();
  const uint32_t tb = tbase;
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma::idesc_tf32(M, N, false, false);
    for (int s = 0; s < K / 8; ++s) {
      uint64_t ad = umma::desc(umma::smem_u32(a) + s * 2 * M * 16, M * 16, 128);
      uint64_t bd = umma::desc(umma::smem_u32(b) + s * 2 * N * 16, N * 16, 128);
      umma::mma_tf32(tb, ad, bd, idesc, s > 0);
    }
    umma::commit(&mbar);
  }
  umma::mbar_wait(&mbar, 0); umma::fence_after_sync();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float v[32];
  umma::tmem_ld32(tb + ((uint32_t)(32 * w) << 16), v);
  for (int i = 0; i < 32; ++i) D[(32 * w + lane) * 32 + i] = v[i];
  umma::fence_before_sync(); __syncthreads();
  if (threadIdx.x < 32) umma::tmem_free(tb, 32);
}
int main() {
  std::vector<float> A(M * K), B(K * N), D(128 * 32);
  srand(2);
  for (auto& x : A) x = (rand() % 7) - 3; for (auto& x : B) x = (rand() % 5) - 2;
  float *dA, *dB, *dD; cudaMalloc(&dA, A.size()*4); cudaMalloc(&dB, B.size()*4); cudaMalloc(&dD, D.size()*4);
  cudaMemcpy(dA, A.data(), A.size()*4, cudaMemcpyHostToDevice); cudaMemcpy(dB, B.data(), B.size()*4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, D.size()*4);
  k<<<1, 128, (M*K + K*N)*4>>>(dA, dB, dD);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  cudaMemcpy(D.data(), dD, D.size()*4, cudaMemcpyDeviceToHost);
  // for every TMEM lane, find the reference row (if any) it matches on all 32 columns
  for (int lane = 0; lane < 128; ++lane) {
    int found = -1;
    for (int m = 0; m < M && found < 0; ++m) {
      bool ok = true;
      for (int n = 0; n < N && ok; ++n) { double r = 0; for (int kk = 0; kk < K; ++kk) r += A[m*K+kk]*B[kk*N+n]; ok = fabs(r - D[lane*32+n]) < 1e-3; }
      if (ok) found = m;
    }
    printf("%d:%d ", lane, found);
  }
  printf("\n");
}
