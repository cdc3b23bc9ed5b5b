// Pooling-scatter micro-benchmark: 256-B bag rows added into random rows of
// `out` by (A) per-thread red.global.add.v4.f32 in the forward epilogue's
// pattern (lane (item, a) adds 16 B at a * 64 + 16 b, 8 bags per warp
// instruction) and (B) one cp.reduce.async.bulk (TMA, 256 B from shared
// memory) per row. nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_bench red_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) k_red(float* out, const int* bag, int n) {
  const int lane = threadIdx.x & 31, gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const int it = lane >> 2, a = lane & 3;
  float v = 1.f + lane;
  for (int base = gw * 8; base < n; base += nw * 8) {
    const int l = base + it;
    if (l < n) {
      float* o = out + (size_t)bag[l] * 64 + a * 16;
#pragma unroll
      for (int b = 0; b < 4; ++b)
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(o + 4 * b), "f"(v), "f"(v), "f"(v), "f"(v) : "memory");
    }
  }
}

// (C) the same rows with lanes laid out along the row: 16 lanes cover one
// bag row's 256 contiguous bytes, a warp instruction two rows
__global__ void __launch_bounds__(512) k_red_rows(float* out, const int* bag, int n) {
  const int lane = threadIdx.x & 31, gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  float v = 1.f + lane;
  for (int base = gw * 8; base < n; base += nw * 8) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int l = base + 2 * r + (lane >> 4);
      if (l < n) {
        float* o = out + (size_t)bag[l] * 64 + 4 * (lane & 15);
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(o), "f"(v), "f"(v), "f"(v), "f"(v) : "memory");
      }
    }
  }
}

__global__ void __launch_bounds__(512) k_bulk(float* out, const int* bag, int n) {
  __shared__ __align__(128) float buf[16][2][4][64];  // per warp: two stages of 4 rows (static smem limit)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = lane; i < 2 * 4 * 64; i += 32) (&buf[w][0][0][0])[i] = 1.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  int st = 0;
  for (int base = gw * 4; base < n; base += nw * 4, st ^= 1) {
    // (a real epilogue would write the stage here after wait_group.read)
    if (lane < 4 && base + lane < n) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(&buf[w][st][lane][0]);
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 256;" ::"l"(out + (size_t)bag[base + lane] * 64), "r"(sa) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    }
    __syncwarp();
  }
  if (lane < 4) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const int n = 1310720;
  for (int rows : {65536, 65536 * 26}) {
    std::vector<int> hb(n);
    srand(1);
    for (int i = 0; i < n; ++i) hb[i] = (int)(((unsigned)rand() * 2654435761u) % (unsigned)rows);
    float* out; int* bag;
    cudaMalloc(&out, (size_t)rows * 256);
    cudaMalloc(&bag, n * 4);
    cudaMemset(out, 0, (size_t)rows * 256);
    cudaMemcpy(bag, hb.data(), n * 4, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int kind = 0; kind < 3; ++kind) {
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        if (kind == 0) k_red<<<148, 512>>>(out, bag, n);
        else if (kind == 1) k_bulk<<<148, 512>>>(out, bag, n);
        else k_red_rows<<<148, 512>>>(out, bag, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("rows %d %s: %.1f us for %d rows of 256 B (%.0f GB/s of added data) err=%s\n", rows, kind == 0 ? "red.v4 (epilogue lanes)" : kind == 1 ? "bulk" : "red.v4 (lanes along the row)",
             best * 1e3, n, n * 256.0 / best / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(out); cudaFree(bag);
  }
  return 0;
}
