// K1: per-batch plan — digits, first-occurrence prefix slots, (bag, slot)
// segments. Reference: lookup.py:88-124 (prepare_reuse_plan, _check_bag),
// lookup.py:254-260 and 280-284 (bag ids, np.unique of bag*P + slot).
//
// First-occurrence order without a sort: every index does an atomicMin of
// its position into a dense table over the m1*m2 prefix keys; the index that
// wins is the first occurrence, and an exclusive scan of the "I won" flags in
// index order numbers the slots exactly as the reference's sequential
// dictionary walk does (lookup.py:115-119).
#include "ttb_internal.h"

namespace ttb {

// ---------------------------------------------------------------- P1: mark
template <typename IdxT>
__global__ void __launch_bounds__(kBlock) k_plan_mark(const IdxT* __restrict__ idx,
                                                      const int64_t* __restrict__ offsets, int T, int B,
                                                      KGeom g, unsigned* __restrict__ pmap,
                                                      unsigned* __restrict__ keys32, int* __restrict__ bag_of,
                                                      int* __restrict__ bag_off, int* __restrict__ err,
                                                      int allow_empty) {
  pdl_enter();
  const int stride = gridDim.x * blockDim.x;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  int bits = 0, multi = 0;
  for (int b = tid; b <= B; b += stride) {
    const int64_t ob = offsets[b];
    bag_off[b] = (int)(ob < 0 ? 0 : (ob > T ? T : ob));
    if (b == 0 && ob != 0) bits |= 4;
    if (b == B && ob != (int64_t)T) bits |= 4;
    if (b < B) {
      const int64_t on = offsets[b + 1];
      if (on == ob) bits |= allow_empty ? 0 : 2;
      else if (on < ob) bits |= 4;
      // bag id of each index (clamped so malformed offsets cannot write out of range)
      const int lo = (int)(ob < 0 ? 0 : (ob > T ? T : ob)), hi = (int)(on < lo ? lo : (on > T ? T : on));
      for (int t = lo; t < hi; ++t) bag_of[t] = b;
      if (hi - lo > 1) multi = 1;
    }
  }
  for (int t = tid; t < T; t += stride) {
    long long v = (long long)idx[t];
    if (v < 0 || v >= (long long)g.rows) {
      bits |= 1;
      v = 0;
    }
    const unsigned i = (unsigned)v;
    keys32[t] = i;
    // warp-aggregated: one atomic per distinct prefix per warp (hot Zipf
    // prefixes would otherwise serialise thousands of atomics on one word);
    // the lowest lane of a peer group holds the smallest position
    const unsigned key = i / g.m3;
    const unsigned peers = __match_any_sync(__activemask(), key);
    // (a plain read first: once a hot prefix holds a small position most
    // later candidates see it and skip the atomic entirely)
    if ((peers & lanemask_lt()) == 0 && pmap[key] > (unsigned)t) atomicMin(&pmap[key], (unsigned)t);
  }
  if (bits) atomicOr(err, bits);
  if (multi) err[4] = 1;  // counts[4]: some bag holds more than one index
}

// ---------------------------------------------------------------- P2: slots
__global__ void __launch_bounds__(kBlock) k_plan_slots(const unsigned* __restrict__ keys32, int T, KGeom g,
                                                       const unsigned* __restrict__ pmap, int* __restrict__ pslot,
                                                       unsigned* __restrict__ work_key, int* __restrict__ counts,
                                                       unsigned long long* status, unsigned* ctr) {
  pdl_enter();
  __shared__ int s_tile;
  __shared__ int s_tmp[kItems * (kBlock / 32) + 2];
  const int tile = claim_tile(ctr, &s_tile);
  const int base = tile * kTile;
  bool f[kItems];
  unsigned key[kItems];
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int t = base + k * kBlock + threadIdx.x;
    f[k] = false;
    key[k] = 0;
    if (t < T) {
      key[k] = keys32[t] / g.m3;
      f[k] = (pmap[key[k]] == (unsigned)t);
    }
  }
  int rank[kItems];
  long long incl;
  tile_flag_scan(f, rank, status, tile, s_tmp, &incl);
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    if (f[k]) {
      work_key[rank[k]] = key[k];
      pslot[key[k]] = rank[k];
    }
  }
  if (tile == (int)((T + kTile - 1) / kTile) - 1 && threadIdx.x == 0) counts[1] = (int)incl;
}

// ---------------------------------------------------------------- P3: segments
// A tile is 256 consecutive bags, one thread each. The distinct slots of a
// bag, in ascending order, are its segments (np.unique sorts bag * P + slot).
// Bags of <= kShortBag indices are ranked in registers by their thread; longer
// bags are handed to whole warps (O(L^2 / 32) through global scratch). The
// bag's segment base comes from a look-back scan of the per-bag counts.
constexpr int kShortBag = 8;
constexpr int kBagsPerTile = kBlock;

__device__ inline void long_bag_rank(int o0, int o1, const unsigned* __restrict__ keys32, unsigned m3,
                                     const int* __restrict__ pslot, int* __restrict__ occ_slot,
                                     int* __restrict__ occ_tmp, int* __restrict__ seg_inv, int* cnt_out) {
  const int lane = threadIdx.x & 31;
  for (int t = o0 + lane; t < o1; t += 32) occ_slot[t] = pslot[keys32[t] / m3];
  __syncwarp();
  for (int t = o0 + lane; t < o1; t += 32) {
    const int sl = occ_slot[t];
    int first = 1;
    for (int u = o0; u < t; ++u)
      if (occ_slot[u] == sl) {
        first = 0;
        break;
      }
    occ_tmp[t] = first;
  }
  __syncwarp();
  int c = 0;
  for (int t = o0 + lane; t < o1; t += 32) {
    const int sl = occ_slot[t];
    int r = 0;
    for (int u = o0; u < o1; ++u) r += (occ_tmp[u] && occ_slot[u] < sl) ? 1 : 0;
    seg_inv[t] = r;  // local rank for now
    c += occ_tmp[t];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) *cnt_out = c;
  __syncwarp();
}

__global__ void __launch_bounds__(kBlock) k_plan_segs(const unsigned* __restrict__ keys32,
                                                      const int* __restrict__ bag_off, int T, int B, KGeom g,
                                                      const int* __restrict__ pslot, int* __restrict__ occ_slot,
                                                      int* __restrict__ occ_tmp, int* __restrict__ seg_inv,
                                                      int* __restrict__ seg_slot, int* __restrict__ seg_bag,
                                                      int* __restrict__ bag_seg, int* __restrict__ counts,
                                                      unsigned long long* status, unsigned* ctr) {
  pdl_enter();
  constexpr int NW = kBlock / 32;
  __shared__ int s_tile;
  __shared__ int s_cnt[kBagsPerTile];
  __shared__ int s_long[kBagsPerTile];
  __shared__ int s_nlong, s_base, s_wsum[NW];
  const int tile = claim_tile(ctr, &s_tile);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_nlong = 0;
  __syncthreads();
  const int b = tile * kBagsPerTile + threadIdx.x;
  int o0 = 0, L = 0;
  int sl[kShortBag], rk[kShortBag];
  unsigned firstm = 0;
  int cnt = 0;
  if (b < B) {
    o0 = bag_off[b];
    const int o1 = bag_off[b + 1];
    L = o1 > o0 ? o1 - o0 : 0;
    if (L <= kShortBag) {
#pragma unroll
      for (int i = 0; i < kShortBag; ++i) {
        sl[i] = 0x7fffffff;
        if (i < L) {
          sl[i] = pslot[keys32[o0 + i] / g.m3];
          occ_slot[o0 + i] = sl[i];
        }
      }
#pragma unroll
      for (int i = 0; i < kShortBag; ++i) {
        bool first = i < L;
#pragma unroll
        for (int j = 0; j < i; ++j) first = first && (sl[j] != sl[i]);
        if (first) firstm |= 1u << i;
      }
      cnt = __popc(firstm);
#pragma unroll
      for (int i = 0; i < kShortBag; ++i) {
        int r = 0;
#pragma unroll
        for (int j = 0; j < kShortBag; ++j) r += ((firstm >> j) & 1u) && sl[j] < sl[i] ? 1 : 0;
        rk[i] = r;
      }
    } else {
      s_long[atomicAdd(&s_nlong, 1)] = threadIdx.x;
    }
  }
  s_cnt[threadIdx.x] = cnt;
  __syncthreads();
  for (int i = w; i < s_nlong; i += NW) {
    const int tb = s_long[i];
    const int bb = tile * kBagsPerTile + tb;
    const int lo = bag_off[bb], hi = bag_off[bb + 1];
    if (hi - lo <= 32) {
      // one index per lane: first occurrences by match_any, ranks by shuffles
      const bool act = lane < hi - lo;
      int sl = 0x7fffffff;
      if (act) {
        sl = pslot[keys32[lo + lane] / g.m3];
        occ_slot[lo + lane] = sl;
      }
      const unsigned peers = __match_any_sync(0xffffffffu, sl);
      const bool first = act && ((peers & lanemask_lt()) == 0);
      int r = 0;
      for (int j = 0; j < 32; ++j) {
        const int sj = __shfl_sync(0xffffffffu, sl, j);
        const bool fj = __shfl_sync(0xffffffffu, first, j);
        r += (fj && sj < sl) ? 1 : 0;
      }
      if (act) {
        seg_inv[lo + lane] = r;  // local rank for now
        occ_tmp[lo + lane] = first ? 1 : 0;
      }
      const int c = __popc(__ballot_sync(0xffffffffu, first));
      if (lane == 0) s_cnt[tb] = c;
    } else {
      long_bag_rank(lo, hi, keys32, g.m3, pslot, occ_slot, occ_tmp, seg_inv, &s_cnt[tb]);
    }
  }
  __syncthreads();
  // block exclusive scan of the 256 counts + look-back across tiles
  const int v = s_cnt[threadIdx.x];
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_wsum[w] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int i = 0; i < NW; ++i) {
      const int c = s_wsum[i];
      s_wsum[i] = acc;
      acc += c;
    }
    s_base = (int)lookback_exclusive(status, tile, acc);
    const int ntiles = (B + kBagsPerTile - 1) / kBagsPerTile;
    if (tile == ntiles - 1) {
      bag_seg[B] = s_base + acc;
      counts[2] = s_base + acc;
    }
  }
  __syncthreads();
  const int base = s_base + s_wsum[w] + incl - v;
  if (b < B) {
    bag_seg[b] = base;
    if (L <= kShortBag) {
#pragma unroll
      for (int i = 0; i < kShortBag; ++i) {
        if (i < L) {
          const int sg = base + rk[i];
          seg_inv[o0 + i] = sg;
          if ((firstm >> i) & 1u) {
            seg_slot[sg] = sl[i];
            seg_bag[sg] = b;
          }
        }
      }
    }
  }
  // long bags: finish with their local ranks (warp per bag)
  for (int i = w; i < s_nlong; i += NW) {
    const int tb = s_long[i];
    const int bb = tile * kBagsPerTile + tb;
    // base of bag tb = its exclusive prefix within the tile, from s_cnt
    int pre = 0;
    for (int j = lane; j < tb; j += 32) pre += s_cnt[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
    const int bbase = s_base + pre;
    for (int t = bag_off[bb] + lane; t < bag_off[bb + 1]; t += 32) {
      const int sg = bbase + seg_inv[t];
      seg_inv[t] = sg;
      if (occ_tmp[t]) {
        seg_slot[sg] = occ_slot[t];
        seg_bag[sg] = bb;
      }
    }
  }
}

// ---------------------------------------------------------------- launcher
cudaError_t launch_plan(ttb_handle* h, const void* idx, int idx64, const int64_t* offsets, cudaStream_t s) {
  Workspace& w = h->w;
  const int T = (int)h->T, B = (int)h->B;
  cudaError_t e;
  // fresh prefix table, error word/counters and look-back state
  // one memset for all per-batch state (zero blocks A and B are contiguous);
  // the prefix table is reset by the previous backward unless it was skipped
  if (!h->pmap_clean && (e = cudaMemsetAsync(w.pmap, 0xFF, sizeof(unsigned) * h->kg.m1m2, s))) return e;
  h->pmap_clean = 0;
  if ((e = cudaMemsetAsync(w.zeroA, 0, w.zeroA_bytes + w.zeroB_bytes, s))) return e;
  h->bwd_zeroed = 1;

  const int work = T > B + 1 ? T : B + 1;
  int grid = (work + kBlock - 1) / kBlock;
  if (grid > 148 * 16) grid = 148 * 16;
  {
  ProfScope _ps(h, s, "plan_mark");
  if (idx64)
    launch_pdl(k_plan_mark<long long>, dim3(grid), dim3(kBlock), 0, s, (const long long*)idx, offsets, T, B, h->kg, w.pmap, w.keys32,
                                                   w.bag_of, w.bag_off, w.err, h->allow_empty);
  else
    launch_pdl(k_plan_mark<int>, dim3(grid), dim3(kBlock), 0, s, (const int*)idx, offsets, T, B, h->kg, w.pmap, w.keys32, w.bag_of,
                                             w.bag_off, w.err, h->allow_empty);
  }
  count_launch();
  const int tiles = (T + kTile - 1) / kTile;
  { ProfScope _ps(h, s, "plan_slots");
  launch_pdl(k_plan_slots, dim3(tiles), dim3(kBlock), 0, s, w.keys32, T, h->kg, w.pmap, w.pslot, w.work_key, w.counts,
                                        w.scan_status + kScanSlots * h->scan_tiles, w.scan_ctr + kScanSlots);
  }
  count_launch();
  const int btiles = (B + kBagsPerTile - 1) / kBagsPerTile;
  { ProfScope _ps(h, s, "plan_segs");
  launch_pdl(k_plan_segs, dim3(btiles), dim3(kBlock), 0, s, w.keys32, w.bag_off, T, B, h->kg, w.pslot, w.occ_slot, w.occ_tmp, w.seg_inv,
                                        w.seg_slot, w.seg_bag, w.bag_seg, w.counts,
                                        w.scan_status + kScanSegs * h->scan_tiles, w.scan_ctr + kScanSegs);
  }
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------- export
__global__ void k_export_plan(const Workspace w, KGeom g, int T, int64_t* work, int64_t* slot_occ, int64_t* seg_ids,
                              int64_t* seg_invo, int64_t* digits) {
  pdl_enter();
  const int P = w.counts[1], S = w.counts[2];
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < T; i += stride) {
    if (work && i < P) {
      const unsigned key = w.work_key[i];
      work[4 * i + 0] = key;
      work[4 * i + 1] = key / g.m2;
      work[4 * i + 2] = key % g.m2;
      work[4 * i + 3] = i;
    }
    if (slot_occ) slot_occ[i] = w.occ_slot[i];
    if (seg_invo) seg_invo[i] = w.seg_inv[i];
    if (seg_ids && i < S) seg_ids[i] = (int64_t)w.seg_bag[i] * P + w.seg_slot[i];
    if (digits) {
      const unsigned r = w.keys32[i];
      const unsigned key = r / g.m3;
      digits[3 * i + 0] = key / g.m2;
      digits[3 * i + 1] = key % g.m2;
      digits[3 * i + 2] = r % g.m3;
    }
  }
}

cudaError_t launch_export_plan(ttb_handle* h, int64_t* work, int64_t* slot_occ, int64_t* seg_ids, int64_t* seg_inv,
                               int64_t* digits, cudaStream_t s) {
  const int T = (int)h->T;
  int grid = (T + kBlock - 1) / kBlock;
  if (grid > 148 * 8) grid = 148 * 8;
  k_export_plan<<<grid, kBlock, 0, s>>>(h->w, h->kg, T, work, slot_occ, seg_ids, seg_inv, digits);
  count_launch();
  return cudaGetLastError();
}

}  // namespace ttb
