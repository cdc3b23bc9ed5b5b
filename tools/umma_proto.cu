// Prototype check of the tcgen05 kind::tf32 helpers (descriptors, TMEM, 3xTF32).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2507_14668_b200/csrc tools/umma_proto.cu -o /tmp/umma_proto
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "ttb_umma.cuh"
using namespace ttb;

constexpr int M = 128, N = 128, K = 32;

__global__ void proto(const float* A, const float* B, float* D, int a_mn, int b_mn, int nsplit, int swap) {
  extern __shared__ __align__(128) unsigned char sm[];
  float* a_hi = (float*)sm;
  float* a_lo = a_hi + M * K;
  float* b_hi = a_lo + M * K;
  float* b_lo = b_hi + K * N;
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  for (int e = threadIdx.x; e < M * K; e += blockDim.x) {
    int m = e / K, k = e % K;
    float h, l;
    umma::split3(A[e], h, l);
    uint32_t off = a_mn ? (uint32_t)((((m >> 2) * K + k) * 16) + (m & 3) * 4) : umma::kmaj_off(m, k, M);
    *(float*)((char*)a_hi + off) = h;
    *(float*)((char*)a_lo + off) = l;
  }
  for (int e = threadIdx.x; e < K * N; e += blockDim.x) {
    int k = e / N, n = e % N;
    float h, l;
    umma::split3(B[e], h, l);
    uint32_t off = b_mn ? (uint32_t)((((n >> 2) * K + k) * 16) + (n & 3) * 4) : umma::kmaj_off(n, k, N);
    *(float*)((char*)b_hi + off) = h;
    *(float*)((char*)b_lo + off) = l;
  }
  umma::fence_smem_to_async();
  if (threadIdx.x < 32) umma::tmem_alloc(&tbase, 128);
  if (threadIdx.x == 0) umma::mbar_init(&mbar, 1);
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tb = tbase;
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma::idesc_tf32(M, N, a_mn, b_mn);
    const float* as[3] = {a_hi, a_hi, a_lo};
    const float* bs[3] = {b_hi, b_lo, b_hi};
    for (int s = 0; s < K / 8; ++s)
      for (int v = 0; v < nsplit; ++v) {
        uint64_t ad, bd;
        if (a_mn) ad = swap ? umma::desc(umma::smem_u32(as[v]) + s * 8 * 16, K * 16, 128) : umma::desc(umma::smem_u32(as[v]) + s * 8 * 16, 128, K * 16);
        else ad = umma::desc(umma::smem_u32(as[v]) + s * 2 * M * 16, M * 16, 128);
        if (b_mn) bd = swap ? umma::desc(umma::smem_u32(bs[v]) + s * 8 * 16, K * 16, 128) : umma::desc(umma::smem_u32(bs[v]) + s * 8 * 16, 128, K * 16);
        else bd = umma::desc(umma::smem_u32(bs[v]) + s * 2 * N * 16, N * 16, 128);
        umma::mma_tf32(tb, ad, bd, idesc, (s > 0 || v > 0) ? 1u : 0u);
      }
    umma::commit(&mbar);
  }
  umma::mbar_wait(&mbar, 0);
  umma::fence_after_sync();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    umma::tmem_ld32(tb + ((uint32_t)(32 * w) << 16) + c0, v);
    for (int i = 0; i < 32; ++i) D[(32 * w + lane) * N + c0 + i] = v[i];
  }
  umma::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) umma::tmem_free(tb, 128);
}

int main() {
  std::vector<float> A(M * K), B(K * N), D(M * N);
  srand(1);
  for (auto& x : A) x = (rand() / (float)RAND_MAX - 0.5f) * 2.f;
  for (auto& x : B) x = (rand() / (float)RAND_MAX - 0.5f) * 2.f;
  std::vector<double> R(M * N, 0.0);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double acc = 0;
      for (int k = 0; k < K; ++k) acc += (double)A[m * K + k] * B[k * N + n];
      R[m * N + n] = acc;
    }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  size_t smem = (2 * M * K + 2 * K * N) * 4;
  cudaFuncSetAttribute(proto, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int sw = 0; sw < 2; ++sw)
  for (int am = 0; am < 2; ++am)
    for (int bm = 0; bm < 2; ++bm)
      for (int ns : {3}) {
        cudaMemset(dD, 0, D.size() * 4);
        proto<<<1, 128, smem>>>(dA, dB, dD, am, bm, ns, sw);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double maxe = 0, maxr = 0;
        for (int i = 0; i < M * N; ++i) { maxe = fmax(maxe, fabs(D[i] - R[i])); maxr = fmax(maxr, fabs(R[i])); }
        printf("swap=%d a_mn=%d b_mn=%d nsplit=%d  err=%s  rel=%.3e  D[0]=%f R[0]=%f\n", sw, am, bm, ns, cudaGetErrorString(e), maxe / maxr, D[0], R[0]);
      }
  return 0;
}
