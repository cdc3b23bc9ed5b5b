// Stable LSD radix sort of (u32 key, u32 value) pairs, 8-bit digits, one
// kernel per digit pass ("onesweep": per-digit decoupled look-back across
// tiles instead of a separate histogram/scan/scatter trio per pass).
//
// Used by the backward to order the batch's indices by row (so every row's
// occurrences, and every prefix's rows, become contiguous runs — the GPU form
// of unique_aggregate's np.unique, backward.py:81-87), and to order the
// distinct rows by their last digit i3 for the deterministic G3 reduction.
// The item count may live on the device (graph capture: no host read-back).
#include "ttb_internal.h"

namespace ttb {

constexpr int kRadix = 256;
constexpr unsigned kSFlagAgg = 1u << 30;
constexpr unsigned kSFlagInc = 2u << 30;
constexpr unsigned kSValMask = (1u << 30) - 1;

__device__ __forceinline__ int sort_count(const int* d_count, int max_n) {
  return d_count ? *d_count : max_n;
}

// global digit histograms for every pass at once
__global__ void __launch_bounds__(kBlock) k_sort_hist(const unsigned* __restrict__ keys, const int* d_count,
                                                      int max_n, int passes, unsigned* __restrict__ hist) {
  pdl_enter();
  __shared__ unsigned sh[4][kRadix];
  for (int i = threadIdx.x; i < 4 * kRadix; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  const int n = sort_count(d_count, max_n);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned k = keys[i];
    for (int p = 0; p < passes; ++p) atomicAdd(&sh[p][(k >> (8 * p)) & 255u], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x) {
    const unsigned v = (&sh[0][0])[i];
    if (v) atomicAdd(&hist[i], v);
  }
}

// one digit pass; items of a tile are laid out warp-blocked so that
// (warp, round, lane) order equals input order (stability)
__global__ void __launch_bounds__(kBlock) k_sort_pass(const unsigned* __restrict__ kin,
                                                      const unsigned* __restrict__ vin, unsigned* __restrict__ kout,
                                                      unsigned* __restrict__ vout, const int* d_count, int max_n,
                                                      int shift, const unsigned* __restrict__ goff,
                                                      unsigned* status, unsigned* ctr) {
  pdl_enter();
  constexpr int NW = kBlock / 32;
  __shared__ int s_tile;
  __shared__ unsigned whist[NW][kRadix];
  __shared__ unsigned s_goff[kRadix];
  const int n = sort_count(d_count, max_n);
  const int tile = claim_tile(ctr, &s_tile);
  const int base = tile * kSortTile;
  if (base >= n) return;
  // global digit offsets: exclusive scan of this pass's 256-bin histogram
  // (every tile recomputes it: 256 values, no extra kernel)
  {
    __shared__ unsigned s_wsum[NW];
    const unsigned v = goff[threadIdx.x];
    unsigned incl = v;
    const int ln = threadIdx.x & 31, wi = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
      if (ln >= o) incl += y;
    }
    if (ln == 31) s_wsum[wi] = incl;
    __syncthreads();
    unsigned wbase = 0;
    for (int i = 0; i < wi; ++i) wbase += s_wsum[i];
    s_goff[threadIdx.x] = wbase + incl - v;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = lanemask_lt();
  for (int i = threadIdx.x; i < NW * kRadix; i += kBlock) (&whist[0][0])[i] = 0;
  __syncthreads();


  unsigned key[kSortItems], val[kSortItems];
  int rank[kSortItems];
#pragma unroll
  for (int k = 0; k < kSortItems; ++k) {
    const int pos = base + w * (32 * kSortItems) + k * 32 + lane;
    const bool ok = pos < n;
    key[k] = ok ? kin[pos] : 0u;
    val[k] = ok ? (vin ? vin[pos] : (unsigned)pos) : 0u;
    const unsigned d = ok ? ((key[k] >> shift) & 255u) : 256u;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    unsigned prior = 0;
    if (ok) prior = whist[w][d];
    __syncwarp();
    rank[k] = (int)(prior + __popc(peers & lt));
    if (ok && (peers & lt) == 0) whist[w][d] = prior + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {
    const int d = threadIdx.x;  // kBlock == kRadix
    unsigned run = 0;
#pragma unroll
    for (int ww = 0; ww < NW; ++ww) {
      const unsigned c = whist[ww][d];
      whist[ww][d] = run;
      run += c;
    }
    unsigned* st = status + (size_t)tile * kRadix + d;
    unsigned excl = 0;
    if (tile == 0) {
      st_relaxed_u32(st, kSFlagInc | run);
    } else {
      st_relaxed_u32(st, kSFlagAgg | run);
      // windowed look-back: 8 predecessors per round trip instead of 1
      int j = tile - 1;
      while (j >= 0) {
        unsigned sv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) sv[i] = (j - i >= 0) ? ld_relaxed_u32(status + (size_t)(j - i) * kRadix + d) : 0u;
        bool done = false;
        int used = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (done || used < i || j - i < 0) continue;
          const unsigned f = sv[i] & ~kSValMask;
          if (f == 0) continue;
          excl += sv[i] & kSValMask;
          used = i + 1;
          if (f == kSFlagInc) done = true;
        }
        if (done) break;
        j -= used;
      }
      st_relaxed_u32(st, kSFlagInc | (excl + run));
    }
    s_goff[d] += excl;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kSortItems; ++k) {
    const int pos = base + w * (32 * kSortItems) + k * 32 + lane;
    if (pos < n) {
      const unsigned d = (key[k] >> shift) & 255u;
      const unsigned o = s_goff[d] + whist[w][d] + (unsigned)rank[k];
      kout[o] = key[k];
      vout[o] = val[k];
    }
  }
}

// region r uses hist/status/counters block r (the idx sort and the i3 sort
// of one backward own different regions, so one memset clears both).
cudaError_t launch_sort(ttb_handle* h, const unsigned* keys_in, const unsigned* vals_in, unsigned* kA, unsigned* vA,
                        unsigned* kB, unsigned* vB, const int* d_count, int max_n, int bits, int region,
                        unsigned** keys_out, unsigned** vals_out, cudaStream_t s) {
  Workspace& w = h->w;
  int passes = (bits + 7) / 8;
  if (passes < 1) passes = 1;
  if (passes > 4) return cudaErrorInvalidValue;
  unsigned* hist = w.sort_hist + (size_t)region * 4 * kRadix;
  unsigned* status = w.sort_status + (size_t)region * 4 * h->sort_tiles * kRadix;
  unsigned* ctr = w.sort_ctr + region * 4;
  // hist / status / counters live in zero block B, cleared before the backward
  cudaError_t e;
  int hgrid = (max_n + kBlock * 4 - 1) / (kBlock * 4);
  if (hgrid > 148 * 4) hgrid = 148 * 4;
  if (hgrid < 1) hgrid = 1;
  {
    ProfScope _ps(h, s, region ? "sort_i3_hist" : "sort_rows_hist");
    e = launch_pdl(k_sort_hist, dim3(hgrid), dim3(kBlock), 0, s, keys_in, d_count, max_n, passes, hist);
    if (e) return e;
  }
  count_launch(1);
  const int tiles = (max_n + kSortTile - 1) / kSortTile;
  const unsigned* ki = keys_in;
  const unsigned* vi = vals_in;
  for (int p = 0; p < passes; ++p) {
    unsigned* ko = (p & 1) ? kB : kA;
    unsigned* vo = (p & 1) ? vB : vA;
    {
      ProfScope _ps(h, s, region ? "sort_i3_pass" : "sort_rows_pass");
      e = launch_pdl(k_sort_pass, dim3(tiles), dim3(kBlock), 0, s, ki, vi, ko, vo, d_count, max_n, 8 * p,
                     (const unsigned*)(hist + p * kRadix), status + (size_t)p * h->sort_tiles * kRadix, ctr + p);
      if (e) return e;
    }
    count_launch();
    ki = ko;
    vi = vo;
  }
  *keys_out = const_cast<unsigned*>(ki);
  *vals_out = const_cast<unsigned*>(vi);
  return cudaGetLastError();
}

// Sort with caller-provided state (no handle): used by the offline reorder
// passes. status: 4 x tiles x 256 u32, hist: 4 x 256 u32, ctr: 4 u32, all
// zero on entry.
cudaError_t launch_sort_raw(const unsigned* keys_in, const unsigned* vals_in, unsigned* kA, unsigned* vA, unsigned* kB,
                            unsigned* vB, int n, int bits, unsigned* hist, unsigned* status, int tiles_cap,
                            unsigned* ctr, unsigned** keys_out, unsigned** vals_out, cudaStream_t s) {
  int passes = (bits + 7) / 8;
  if (passes < 1) passes = 1;
  if (passes > 4) return cudaErrorInvalidValue;
  cudaError_t e;
  int hgrid = (n + kBlock * 4 - 1) / (kBlock * 4);
  if (hgrid > 148 * 4) hgrid = 148 * 4;
  if (hgrid < 1) hgrid = 1;
  if ((e = launch_pdl(k_sort_hist, dim3(hgrid), dim3(kBlock), 0, s, keys_in, (const int*)nullptr, n, passes, hist)))
    return e;
  count_launch();
  const int tiles = (n + kSortTile - 1) / kSortTile;
  const unsigned* ki = keys_in;
  const unsigned* vi = vals_in;
  for (int p = 0; p < passes; ++p) {
    unsigned* ko = (p & 1) ? kB : kA;
    unsigned* vo = (p & 1) ? vB : vA;
    if ((e = launch_pdl(k_sort_pass, dim3(tiles), dim3(kBlock), 0, s, ki, vi, ko, vo, (const int*)nullptr, n, 8 * p,
                        (const unsigned*)(hist + p * kRadix), status + (size_t)p * tiles_cap * kRadix, ctr + p)))
      return e;
    count_launch();
    ki = ko;
    vi = vo;
  }
  *keys_out = const_cast<unsigned*>(ki);
  *vals_out = const_cast<unsigned*>(vi);
  return cudaGetLastError();
}

}  // namespace ttb
