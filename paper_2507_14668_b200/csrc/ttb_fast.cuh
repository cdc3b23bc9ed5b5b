// Device helpers of the tensor-core pipeline (ttb_fast.cu):
// tile constants, fp32 reductions, cp.async, the per-tile
// metadata ring.
#pragma once
#include "ttb_internal.h"
#include "ttb_umma.cuh"

namespace ttb {
namespace fast {

constexpr int kItemLen = 32;    // max lookups per work item
constexpr int kTileItems = 32;  // items per tile: M = 32 * n1 = 128
constexpr int kSortItems = 256; // full items per row-sort chunk (k_rowsort, pooled batches)
constexpr int R1 = 32, C = 128, NOUT = 64;
constexpr int kImg = 16384;     // bytes of one 128 x 32 / 32 x 128 fp32 image

__device__ __forceinline__ void red_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
__device__ __forceinline__ void red_f32(float* p, float a) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(a) : "memory");
}

// fast_hdr word set by the backward when some gradient contribution is
// non-finite or >= 2^95 in magnitude. Without one, every final gradient is
// finite: each element sums < 2^31 contributions from 0, and a rounded sum
// moves by at most twice the addend (|fl(s + x) - s| <= 2|x|), so it stays
// below 2^127. The finiteness scan before the fused update runs only if set.
constexpr int kHdrSuspect = 6;
constexpr int kHdrChunks = 7;  // fast_hdr word: number of row-sort chunks (f_chunks) of the plan
constexpr int kHdrNextTile = 5;  // fast_hdr word: the pooled backward's tile counter (reset per launch)
__device__ __forceinline__ bool suspicious(float v) { return !(fabsf(v) < 0x1p95f); }

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------ async copies
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(umma::smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(umma::smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(umma::smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void sync_for_mma() {
  umma::fence_smem_to_async();
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
}

struct TileMeta {
  int i2, n, item0, pad;
  unsigned key[kTileItems];
  int start[kTileItems + 1];
};

struct MetaPrefetch {
  int4 next;  // tile table entry of the tile after the one being fetched
};

// lanes 0..31 of the calling warp: slot <- tile `info`
__device__ inline void fetch_meta_async(const int4& info, const int* __restrict__ item_start,
                                        const unsigned* __restrict__ item_key, TileMeta* m) {
  const int l = threadIdx.x & 31, n = info.z, item0 = info.y;
  if (l == 0) {
    m->i2 = info.x;
    m->n = n;
    m->item0 = item0;
    cp_async4(&m->start[n], item_start + item0 + n);
  }
  if (l < n) {
    cp_async4(&m->key[l], item_key + item0 + l);
    cp_async4(&m->start[l], item_start + item0 + l);
  }
}

// G1 row (image index) of item `it`: its table's block (tables are stacked
// at M1 rows, M2 slices) plus the key's i1 digit
// (one table: no division — these run per staged element)
__device__ __forceinline__ int item_i1(const TileMeta* m, int it, KGeom g) {
  const unsigned base = m->key[it] - (unsigned)m->i2 * g.m1;
  return (int)(g.nt == 1 ? base : base + ((unsigned)m->i2 / g.tm2) * g.m1);
}
// G3 slice offset of a tile's table (its lookups' i3 digits are table-local)
__device__ __forceinline__ unsigned tile_i3_base(const TileMeta* m, KGeom g) {
  return g.nt == 1 ? 0u : ((unsigned)m->i2 / g.tm2) * g.tm3;
}

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// per-i1 G1 images written by the update kernel (floats): for item parity
// p = 0, 1 the rows image [256 p: hi, 256 p + 128: lo], rows a = 0..3 already
// SWIZZLE_128B-permuted for smem lines 4 p + a (an item's 512 bytes of the
// tile's rows image are one bulk copy); then t_hi[k][a] (512), t_lo[k][a] (640)
constexpr int kG1Img = 768;
constexpr int kG1T = 512;
__host__ __device__ constexpr int g1_rows_off(int parity) { return 256 * parity; }

}  // namespace fast
}  // namespace ttb
