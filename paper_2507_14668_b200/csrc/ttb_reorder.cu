// Offline index-reordering passes on the GPU (reference reorder.py):
//   count_frequencies  reorder.py:90-104  per-row access counts over all
//                      batches, rows ranked by (count desc, id asc)
//   apply_bijection    reorder.py:286-296 relabel every index through a
//                      permutation (with the reference's range check)
// Community detection (reorder.py:176-236, O(n E) Python) stays on the host.
#include "ttb_internal.h"

namespace ttb {

__global__ void __launch_bounds__(kBlock) k_count(const int64_t* __restrict__ idx, int64_t n, int64_t table_len,
                                                  unsigned long long* __restrict__ counts, int* __restrict__ err) {
  pdl_enter();
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = idx[i];
    if (v < 0 || v >= table_len) {
      bad = true;
      continue;
    }
    // warp-aggregated: hot rows repeat within a warp
    const unsigned peers = __match_any_sync(__activemask(), (unsigned long long)v);
    if ((peers & lanemask_lt()) == 0) atomicAdd(&counts[v], (unsigned long long)__popc(peers));
  }
  if (bad) atomicOr(err, 1);
}

// sort key: complement of the (u32-saturated) count -> ascending key order is
// descending count, and the stable LSD sort keeps ascending row id on ties
__global__ void k_rank_keys(const unsigned long long* __restrict__ counts, int64_t n, unsigned* __restrict__ keys) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long c = counts[i];
    keys[i] = ~(unsigned)(c > 0xFFFFFFFFull ? 0xFFFFFFFFull : c);
  }
}

__global__ void k_rank_out(const unsigned* __restrict__ rows_sorted, int64_t n, int64_t* __restrict__ row_of_rank,
                           int64_t* __restrict__ rank_of) {
  pdl_enter();
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const unsigned row = rows_sorted[r];
    if (row_of_rank) row_of_rank[r] = row;
    if (rank_of) rank_of[row] = r;
  }
}

__global__ void k_gather(const int64_t* __restrict__ forward, int64_t table_len, const int64_t* __restrict__ in,
                         int64_t* __restrict__ out, int64_t n, int* __restrict__ err) {
  pdl_enter();
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = in[i];
    if (v < 0 || v >= table_len) {
      bad = true;
      out[i] = -1;
    } else {
      out[i] = forward[v];
    }
  }
  if (bad) atomicOr(err, 1);
}

static int grid_for(int64_t n) {
  int64_t g = (n + kBlock - 1) / kBlock;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

struct RankLayout {
  size_t keys, vals, kA, vA, kB, vB, hist, status, ctr, total;
  int tiles;
};

static RankLayout rank_layout(int64_t n) {
  RankLayout L{};
  L.tiles = (int)((n + kSortTile - 1) / kSortTile) + 1;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    off = (off + 255) & ~(size_t)255;
    size_t at = off;
    off += bytes;
    return at;
  };
  L.keys = take(4 * (size_t)n);
  L.vals = take(4 * (size_t)n);
  L.kA = take(4 * (size_t)n);
  L.vA = take(4 * (size_t)n);
  L.kB = take(4 * (size_t)n);
  L.vB = take(4 * (size_t)n);
  L.hist = take(4 * 4 * 256);
  L.status = take((size_t)4 * 4 * L.tiles * 256);
  L.ctr = take(4 * 8);
  L.total = off + 256;
  return L;
}

}  // namespace ttb

using namespace ttb;

extern "C" {

int ttb_count_frequencies(const int64_t* indices, int64_t n, int64_t table_len, uint64_t* counts, int* err,
                          ttb_stream stream) {
  if (!counts || !err || table_len < 1 || n < 0 || (n > 0 && !indices)) return TTB_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(counts, 0, sizeof(uint64_t) * table_len, s) != cudaSuccess) return TTB_ECUDA;
  if (cudaMemsetAsync(err, 0, sizeof(int), s) != cudaSuccess) return TTB_ECUDA;
  if (n == 0) return TTB_OK;
  cudaError_t e = launch_pdl(k_count, dim3(grid_for(n)), dim3(kBlock), 0, s, indices, n, table_len,
                             (unsigned long long*)counts, err);
  count_launch();
  return e == cudaSuccess ? TTB_OK : TTB_ECUDA;
}

int ttb_rank_workspace_bytes(int64_t table_len, size_t* bytes) {
  if (!bytes || table_len < 1 || table_len >= (1ll << 29)) return TTB_EINVAL;
  *bytes = rank_layout(table_len).total;
  return TTB_OK;
}

int ttb_rank_rows(const uint64_t* counts, int64_t table_len, int64_t* row_of_rank, int64_t* rank_of, void* workspace,
                  size_t bytes, ttb_stream stream) {
  if (!counts || !workspace || table_len < 1 || table_len >= (1ll << 29)) return TTB_EINVAL;
  RankLayout L = rank_layout(table_len);
  if (bytes < L.total) return TTB_EINVAL;
  char* base = (char*)(((uintptr_t)workspace + 255) & ~(uintptr_t)255);
  cudaStream_t s = (cudaStream_t)stream;
  const int n = (int)table_len;
  if (cudaMemsetAsync(base + L.hist, 0, L.ctr + 32 - L.hist, s) != cudaSuccess) return TTB_ECUDA;
  launch_pdl(k_rank_keys, dim3(grid_for(n)), dim3(kBlock), 0, s, (const unsigned long long*)counts, table_len,
             (unsigned*)(base + L.keys));
  count_launch();
  unsigned *ko, *vo;
  cudaError_t e = launch_sort_raw((const unsigned*)(base + L.keys), nullptr, (unsigned*)(base + L.kA),
                                  (unsigned*)(base + L.vA), (unsigned*)(base + L.kB), (unsigned*)(base + L.vB), n, 32,
                                  (unsigned*)(base + L.hist), (unsigned*)(base + L.status), L.tiles,
                                  (unsigned*)(base + L.ctr), &ko, &vo, s);
  if (e != cudaSuccess) return TTB_ECUDA;
  launch_pdl(k_rank_out, dim3(grid_for(n)), dim3(kBlock), 0, s, (const unsigned*)vo, table_len, row_of_rank, rank_of);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? TTB_OK : TTB_ECUDA;
}

int ttb_apply_bijection(const int64_t* forward, int64_t table_len, const int64_t* in, int64_t* out, int64_t n,
                        int* err, ttb_stream stream) {
  if (!forward || !err || table_len < 1 || n < 0 || (n > 0 && (!in || !out))) return TTB_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(err, 0, sizeof(int), s) != cudaSuccess) return TTB_ECUDA;
  if (n == 0) return TTB_OK;
  cudaError_t e = launch_pdl(k_gather, dim3(grid_for(n)), dim3(kBlock), 0, s, forward, table_len, in, out, n, err);
  count_launch();
  return e == cudaSuccess ? TTB_OK : TTB_ECUDA;
}

}  // extern "C"
