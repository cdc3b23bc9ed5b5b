// Microbenchmark (not part of the library): the backward's Z / dG3 phase loop
// in isolation (8 warps, warp per item, lane <-> c), with ablations.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o zphase_bench zphase_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void red_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
__device__ __forceinline__ int xs_idx(int it, int a, int b, int c) { return it * 512 + (4 * a + b) * 32 + (c ^ (b << 3)); }
template <int MODE, int NT = 256>
__global__ void __launch_bounds__(NT, 1) zb(int reps, int npos_per_item, float* dG3, unsigned m3, float* sink,
                                            unsigned long long* cyc) {
  extern __shared__ float4 sm4[];
  float* xs = reinterpret_cast<float*>(sm4);              // 32 items x 512
  float4* st_g = sm4 + 32 * 128;                            // 128 pos x 16
  float4* st_g3 = st_g + 128 * 16;                          // 128 pos x 32
  int2* st_sbi = reinterpret_cast<int2*>(st_g3 + 128 * 32);  // 128
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < 32 * 512; e += NT) xs[e] = 0.001f * (e % 97);
  for (int e = threadIdx.x; e < 128 * 16; e += NT) st_g[e] = make_float4(0.01f, 0.02f, 0.03f, 0.04f);
  for (int e = threadIdx.x; e < 128 * 32; e += NT) st_g3[e] = make_float4(0.5f, 0.25f, 0.125f, 0.1f);
  for (int e = threadIdx.x; e < 128; e += NT) st_sbi[e] = make_int2(e, (e * 37) % m3);
  __syncthreads();
  const unsigned long long c0 = clock64();
  float bad = 0.f;
  for (int r = 0; r < reps; ++r) {
    for (int it = warp; it < 32; it += NT / 32) {
      float x[16], z[16];
#pragma unroll
      for (int ab = 0; ab < 16; ++ab) {
        x[ab] = xs[xs_idx(it, ab >> 2, ab & 3, lane)];
        z[ab] = 0.f;
      }
      const int s1 = (it + 1) * npos_per_item;
      int qq = it * npos_per_item;
      while (qq < s1) {
        const int bag = st_sbi[qq].x;
        float gv[64];
        if (MODE == 2) {
          const float* sg = reinterpret_cast<const float*>(st_g + qq * 16);
#pragma unroll
          for (int k = 0; k < 64; ++k) gv[k] = sg[k];
        } else if (MODE == 3) {
#pragma unroll
          for (int k = 0; k < 64; ++k) gv[k] = x[k & 15] * (float)(qq + k);
        } else {
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const float4 v = st_g[qq * 16 + k];
            gv[4 * k] = v.x; gv[4 * k + 1] = v.y; gv[4 * k + 2] = v.z; gv[4 * k + 3] = v.w;
          }
        }
        float dh[4] = {0.f, 0.f, 0.f, 0.f};
        if (MODE == 7) {
        } else if (MODE == 4) {  // 16 independent chains of 4, then a 4-way add per j
          float p4[4][4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int j = 0; j < 4; ++j) p4[q][j] = 0.f;
#pragma unroll
          for (int ab = 0; ab < 16; ++ab)
#pragma unroll
            for (int j = 0; j < 4; ++j) p4[ab & 3][j] = fmaf(x[ab], gv[4 * ab + j], p4[ab & 3][j]);
#pragma unroll
          for (int j = 0; j < 4; ++j) dh[j] = (p4[0][j] + p4[1][j]) + (p4[2][j] + p4[3][j]);
        } else {
#pragma unroll
          for (int ab = 0; ab < 16; ++ab)
#pragma unroll
            for (int j = 0; j < 4; ++j) dh[j] = fmaf(x[ab], gv[4 * ab + j], dh[j]);
        }
        float gs[4] = {0.f, 0.f, 0.f, 0.f};
        int e = qq;
        if (MODE == 8) {
          const float4 h3 = st_g3[e * 32 + lane];
          gs[0] = h3.x; gs[1] = h3.y; gs[2] = h3.z; gs[3] = h3.w;
          red_v4(dG3 + ((size_t)lane * m3 + st_sbi[e].y) * 4, dh[0], dh[1], dh[2], dh[3]);
          ++e;
        } else
        for (; e < s1; ++e) {
          const int2 pr = st_sbi[e];
          if (pr.x != bag) break;
          const float4 h3 = st_g3[e * 32 + lane];
          gs[0] += h3.x; gs[1] += h3.y; gs[2] += h3.z; gs[3] += h3.w;
          if (MODE != 1) red_v4(dG3 + ((size_t)lane * m3 + pr.y) * 4, dh[0], dh[1], dh[2], dh[3]);
          else bad += dh[0] + dh[1] + dh[2] + dh[3];
        }
        if (MODE == 6) {
          bad += gs[0] + gs[1] + gs[2] + gs[3] + gv[0];
        } else if (MODE == 5) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int ab = 0; ab < 16; ++ab) z[ab] = fmaf(gv[4 * ab + j], gs[j], z[ab]);
        } else {
#pragma unroll
          for (int ab = 0; ab < 16; ++ab)
#pragma unroll
            for (int j = 0; j < 4; ++j) z[ab] = fmaf(gv[4 * ab + j], gs[j], z[ab]);
        }
        qq = e;
      }
#pragma unroll
      for (int ab = 0; ab < 16; ++ab) xs[xs_idx(it, ab >> 2, ab & 3, lane)] = z[ab];
    }
    __syncthreads();
  }
  const unsigned long long c1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
  sink[blockIdx.x * NT + threadIdx.x] = bad;
}
template <int NT = 256>
__global__ void __launch_bounds__(NT, 1) zb2(int reps, int npos_per_item, float* dG3, unsigned m3, float* sink,
                                             unsigned long long* cyc) {
  extern __shared__ float4 sm4[];
  float* xs = reinterpret_cast<float*>(sm4);
  float4* st_g = sm4 + 32 * 128;
  float4* st_g3 = st_g + 128 * 16;
  int2* st_sbi = reinterpret_cast<int2*>(st_g3 + 128 * 32);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < 32 * 512; e += NT) xs[e] = 0.001f * (e % 97);
  for (int e = threadIdx.x; e < 128 * 16; e += NT) st_g[e] = make_float4(0.01f, 0.02f, 0.03f, 0.04f);
  for (int e = threadIdx.x; e < 128 * 32; e += NT) st_g3[e] = make_float4(0.5f, 0.25f, 0.125f, 0.1f);
  for (int e = threadIdx.x; e < 128; e += NT) st_sbi[e] = make_int2(e, (e * 37) % m3);
  __syncthreads();
  const unsigned long long c0 = clock64();
  const int cb2 = 2 * (lane & 15), abh = lane >> 4;
  for (int r = 0; r < reps; ++r) {
    for (int it = warp; it < 32; it += NT / 32) {
      float x[8][2], z[8][2];
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int ab = 8 * abh + u;
          x[u][cc] = xs[xs_idx(it, ab >> 2, ab & 3, cb2 + cc)];
          z[u][cc] = 0.f;
        }
      const int s1 = (it + 1) * npos_per_item;
      int qq = it * npos_per_item;
      while (qq < s1) {
        const int bag = st_sbi[qq].x;
        float4 gv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) gv[u] = st_g[qq * 16 + 8 * abh + u];
        float dh[2][4];
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          dh[cc][0] = dh[cc][1] = dh[cc][2] = dh[cc][3] = 0.f;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            dh[cc][0] = fmaf(x[u][cc], gv[u].x, dh[cc][0]);
            dh[cc][1] = fmaf(x[u][cc], gv[u].y, dh[cc][1]);
            dh[cc][2] = fmaf(x[u][cc], gv[u].z, dh[cc][2]);
            dh[cc][3] = fmaf(x[u][cc], gv[u].w, dh[cc][3]);
          }
        }
        float rr[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float send = abh ? dh[0][j] : dh[1][j];
          const float keep = abh ? dh[1][j] : dh[0][j];
          rr[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
        }
        const int cme = cb2 + abh;
        float gs[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        int e = qq;
        for (; e < s1; ++e) {
          const int2 pr = st_sbi[e];
          if (pr.x != bag) break;
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const float4 h3 = st_g3[e * 32 + cb2 + cc];
            gs[cc][0] += h3.x; gs[cc][1] += h3.y; gs[cc][2] += h3.z; gs[cc][3] += h3.w;
          }
          red_v4(dG3 + ((size_t)cme * m3 + pr.y) * 4, rr[0], rr[1], rr[2], rr[3]);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            z[u][cc] = fmaf(gv[u].x, gs[cc][0], z[u][cc]);
            z[u][cc] = fmaf(gv[u].y, gs[cc][1], z[u][cc]);
            z[u][cc] = fmaf(gv[u].z, gs[cc][2], z[u][cc]);
            z[u][cc] = fmaf(gv[u].w, gs[cc][3], z[u][cc]);
          }
        qq = e;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int ab = 8 * abh + u;
          xs[xs_idx(it, ab >> 2, ab & 3, cb2 + cc)] = z[u][cc];
        }
    }
    __syncthreads();
  }
  const unsigned long long c1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
  sink[blockIdx.x * NT + threadIdx.x] = 0.f;
}
int main() {
  float *dG3, *sink;
  unsigned long long* cyc;
  cudaMalloc(&dG3, 32 * 256 * 4 * 4);
  cudaMalloc(&sink, 148 * 256 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int smem = 32 * 512 * 4 + 128 * 16 * 16 + 128 * 32 * 16 + 128 * 8;
  cudaFuncSetAttribute(zb<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(zb<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(zb<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(zb<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(zb<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(zb<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(zb<0, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(zb<0, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int nt : {128, 512}) {
    const int reps = 200;
    if (nt == 512) zb<0, 512><<<148, 512, smem>>>(reps, 2, dG3, 250, sink, cyc);
    else zb<0, 128><<<148, 128, smem>>>(reps, 2, dG3, 250, sink, cyc);
    cudaDeviceSynchronize();
    unsigned long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%d threads: %.0f cycles per tile\n", nt, (double)h / reps);
  }
  cudaFuncSetAttribute(zb2<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(zb2<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int nt : {256, 512}) {
    const int reps = 200;
    if (nt == 512) zb2<512><<<148, 512, smem>>>(reps, 2, dG3, 250, sink, cyc);
    else zb2<256><<<148, 256, smem>>>(reps, 2, dG3, 250, sink, cyc);
    cudaDeviceSynchronize();
    unsigned long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("(2c, 8ab) mapping, %d threads: %.0f cycles per tile\n", nt, (double)h / reps);
  }
  float* big;
  cudaMalloc(&big, 148 * 1024 * 4);
  cudaFuncSetAttribute(zb<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(zb<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(zb<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int npi : {2})
    for (int mode = 0; mode < 9; ++mode) {
      const int reps = 200;
      if (mode == 0) zb<0><<<148, 256, smem>>>(reps, npi, dG3, 250, sink, cyc);
      else if (mode == 1) zb<1><<<148, 256, smem>>>(reps, npi, dG3, 250, sink, cyc);
      else if (mode == 2) zb<2><<<148, 256, smem>>>(reps, npi, dG3, 250, sink, cyc);
      else if (mode == 3) zb<3><<<148, 256, smem>>>(reps, npi, dG3, 250, sink, cyc);
      else if (mode == 4) zb<4><<<148, 256, smem>>>(reps, npi, dG3, 250, sink, cyc);
      else if (mode == 5) zb<5><<<148, 256, smem>>>(reps, npi, dG3, 250, sink, cyc);
      else if (mode == 6) zb<6><<<148, 256, smem>>>(reps, npi, dG3, 250, sink, cyc);
      else if (mode == 7) zb<7><<<148, 256, smem>>>(reps, npi, dG3, 250, sink, cyc);
      else zb<8><<<148, 256, smem>>>(reps, npi, dG3, 250, sink, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      unsigned long long h;
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      const double per_tile = (double)h / reps;
      printf("positions/item %d %s: %.0f cycles per tile of 32 items (%.0f per position per warp-slot)\n", npi,
             mode == 0 ? "LDS.128 bcast" : mode == 1 ? "no red       " : mode == 2 ? "LDS.32 bcast " : mode == 3 ? "gv in regs   " : mode == 4 ? "dh 16 chains " : mode == 5 ? "z j-outer    " : mode == 6 ? "no z         " : mode == 7 ? "no dh        " : "no bag loop  ", per_tile, per_tile / (4.0 * npi));
    }
  return 0;
}
