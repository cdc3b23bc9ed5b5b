// Tensor-core step pipeline ("fast path") for the production geometry
// n = (4, 4, 4), ranks (1, 32, 32, 1) — BASELINE configs 2 and 3.
//
// Same operator semantics as the plan/forward/backward of ttb_plan.cu /
// ttb_backward.cu (reference lookup.py:236-296, backward.py:131-200), but
// organised around the i2 digit so every contraction with a G2 slice is a
// 128-row tcgen05 GEMM (3xTF32, fp32-level accuracy):
//
//   plan     keys (i2 m1 + i1, i3, bag) -> stable radix sort by prefix key ->
//            work items (<= 32 lookups of one prefix) -> tiles (<= 32 items
//            of one i2 = 128 accumulator rows (item, a))
//   forward  X[(item, a), (c, b)] = G1[i1] . G2[:, i2]  in TMEM; each lookup
//            closes X with its G3 slice in registers and pools into its bag
//   backward X^T recomputed in TMEM (cheaper than storing it); per segment
//            (lookups of one bag under one prefix) Z += g (x) sum G3 and
//            dG3 += X^T g (SIMT, lane <-> (c, b)); then on the tensor core
//            dG2 += Z^T . G1 (Z^T from TMEM) and dG1 += Z . G2^T
//
// Reuse of the partial products across duplicate prefixes (the paper's reuse
// buffer) is the item grouping: X is formed once per item for all its
// lookups. Gradient accumulation into the cores uses fp32 reductions in L2
// (red.global.add), so summation order — unlike the legacy path — is not
// fixed; results agree with the reference within the north-star tolerances.
#include <stdio.h>
#include <stdlib.h>

#include "ttb_fast.cuh"

namespace ttb {
namespace fast {

constexpr int kThreads = 512;  // backward: 16 warps, four per TMEM lane quadrant

// ------------------------------------------------------------ plan
// One persistent kernel (grid <= SM count, all CTAs co-resident) in three
// phases separated by grid barriers — a counting sort over the m1 m2 prefix
// keys instead of a radix sort of the positions:
//   0  per index: digits, i2-major prefix key, rank within its key from a
//      warp-aggregated atomicAdd on the key's counter; per bag: bag ids
//   A  per i2 group (warp): totals, then the group's exclusive offsets
//      (positions, work items, tiles); the group's items are laid out by
//      descending length (counting sort by length), with their item / tile
//      tables and each key's item positions; counters reset
//   B  per index: (bag, i3) scattered to its item's position + rank
// Order inside a prefix is arbitrary (summation order of fp32 reductions
// only); items are runs of <= kItemLen positions of one prefix, tiles runs of
// <= kTileItems items of one i2 of similar lengths.
constexpr int kPlanThreads = 512;
constexpr int kTileCost = 32;
constexpr int kA2Regs = 8;
constexpr int kPlanUnroll = 8;  // lookups per thread per round in phases 0 and B
constexpr int kPlanRegs = 4;   // lookups per thread whose plan fields stay in registers (phase 0 -> B)     // per-lane registers caching an i2 group's prefix counters (m1 <= 256)  // per-tile fixed cost in lookup units (CTA range balancing)

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ inline void grid_barrier(unsigned* bar, unsigned& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    while (ld_acquire_u32(bar) < target) __nanosleep(32);
  }
  __syncthreads();
}


template <typename IdxT, bool kMany>  // kMany: more than two lookups per thread (phases 0 / B unrolled)
__global__ void __launch_bounds__(kPlanThreads) k_fplan(const IdxT* __restrict__ idx,
                                                        const int64_t* __restrict__ offsets, int T, int B, KGeom g,
                                                        unsigned* __restrict__ key, unsigned* __restrict__ i3o,
                                                        int* __restrict__ rk, int* __restrict__ bag_of,
                                                        int* __restrict__ cnt, int* __restrict__ start,
                                                        int* __restrict__ rstart, int* __restrict__ split,
                                                        int4* __restrict__ gtot, int* __restrict__ item_start,
                                                        int* __restrict__ cta_tiles, int ctas,
                                                        unsigned* __restrict__ item_key, int4* __restrict__ tile_info,
                                                        int2* __restrict__ sbi, int* __restrict__ hdr, int dbg,
                                                        int allow_empty, const uint4* __restrict__ tgeom,
                                                        int2* __restrict__ chunks, float4* __restrict__ zgrad,
                                                        int64_t nzgrad4) {
  pdl_enter();
  // the backward's flat gradient buffer cleared here, off the step's
  // critical path (a memset node between the forward and the backward would
  // also break their programmatic overlap); fast_backward skips its memset
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nzgrad4; i += (int64_t)gridDim.x * blockDim.x)
    zgrad[i] = make_float4(0.f, 0.f, 0.f, 0.f);
#define PSTAMP(i)                                                                                          \
  do {                                                                                                     \
    if (dbg && threadIdx.x == 0 && blockIdx.x == 0) {                                                      \
      unsigned long long _t;                                                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                                               \
      reinterpret_cast<unsigned long long*>(hdr + 16)[i] = _t;                                             \
    }                                                                                                      \
  } while (0)
  PSTAMP(0);
  __shared__ int s_hist[kPlanThreads / 32][2 * (kItemLen + 1)];
  __shared__ int s_poff[kPlanThreads / 32][kItemLen + 1];
  unsigned* bar = reinterpret_cast<unsigned*>(hdr + 12);  // [0] barrier arrivals, [1] CTAs done (reset by the last)
  unsigned target = 0;
  // the plan's header words (errors, counts, the backward's tile counter and
  // suspect flag) are cleared here instead of by a memset node before the
  // launch; every other write to them comes after the first grid barrier
  if (blockIdx.x == 0 && threadIdx.x < 12) hdr[threadIdx.x] = 0;
  const int nthr = gridDim.x * blockDim.x, tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  // tables (one unless the handle is batched): table f's lookups are
  // [offsets[f bpt], offsets[(f + 1) bpt]) and its digits use its own factors
  __shared__ int s_toff[TTB_MAX_TABLES + 1];
  __shared__ uint4 s_tg[TTB_MAX_TABLES];
  const int nt = (int)g.nt;
  for (int f = threadIdx.x; f <= nt; f += blockDim.x) {
    if (f < nt) s_tg[f] = tgeom[f];
    const int64_t b = nt > 1 ? (int64_t)f * g.bpt : (f ? B : 0);
    const int64_t o = b >= B ? (int64_t)T : offsets[b];
    s_toff[f] = (int)(o < 0 ? 0 : (o > T ? T : o));
  }
  __syncthreads();
  // ---- phase 0
  int bits = 0, multi = 0;
  for (int b = tid; b < B; b += nthr) {
    const int64_t ob = offsets[b], on = offsets[b + 1];
    if (b == 0 && ob != 0) bits |= 4;
    if (b == B - 1 && on != (int64_t)T) bits |= 4;
    if (on == ob) bits |= allow_empty ? 0 : 2;
    else if (on < ob) bits |= 4;
    const int lo = (int)(ob < 0 ? 0 : (ob > T ? T : ob)), hi = (int)(on < lo ? lo : (on > T ? T : on));
    for (int t = lo; t < hi; ++t) bag_of[t] = b;
    if (hi - lo > 1) multi = 1;
  }
  // the first kPlanRegs lookups of this thread keep (key, rank, i3) in
  // registers for phase B (same thread <-> lookup mapping there)
  unsigned rkey[kPlanRegs], ri3[kPlanRegs];
  int rrk[kPlanRegs];
  if constexpr (!kMany) {  // at most two lookups per thread (config 2): one lookup per round
    int iter = 0;
    for (int t0 = blockIdx.x * blockDim.x; t0 < T; t0 += nthr, ++iter) {  // warp-uniform trip count
      const int t = t0 + threadIdx.x;
      const bool ok = t < T;
      unsigned k = 0xFFFFFFFFu, i3 = 0;
      if (ok) {
        int f = 0;  // the lookup's table: the last f with s_toff[f] <= t
        for (int lo2 = 1, hi2 = nt - 1; lo2 <= hi2;) {
          const int mid = (lo2 + hi2) >> 1;
          if (s_toff[mid] <= t) f = mid, lo2 = mid + 1;
          else hi2 = mid - 1;
        }
        const uint4 tg = s_tg[f];  // (m2, m3, rows) of the table
        long long v = (long long)idx[t];
        if (v < 0 || v >= (long long)tg.z) {
          bits |= 1;
          v = 0;
        }
        const unsigned m2m3 = tg.x * tg.y;
        const unsigned i = (unsigned)v, i1 = i / m2m3, r = i - i1 * m2m3, i2 = r / tg.y;
        k = ((unsigned)f * g.tm2 + i2) * g.m1 + i1;
        i3 = r - i2 * tg.y;
        if (iter >= kPlanRegs) {
          key[t] = k;
          i3o[t] = i3;
        }
      }
      const unsigned peers = __match_any_sync(0xffffffffu, k);
      const int leader = __ffs(peers) - 1;
      int base = 0;
      if (ok && lane == leader) base = atomicAdd(&cnt[k], __popc(peers));
      base = __shfl_sync(0xffffffffu, base, leader);
      const int rank = base + __popc(peers & lanemask_lt());
#pragma unroll
      for (int q = 0; q < kPlanRegs; ++q)
        if (q == iter) {
          rkey[q] = k;
          ri3[q] = i3;
          rrk[q] = rank;
        }
      if (ok && iter >= kPlanRegs) rk[t] = rank;
    }
  } else {
    // kPlanUnroll lookups per thread per round: their index loads, then their
    // counter atomics, are in flight together (one round trip per round
    // instead of one per lookup when a thread has many lookups)
    for (int g0 = blockIdx.x * blockDim.x; g0 < T; g0 += kPlanUnroll * nthr) {
      unsigned kk[kPlanUnroll], ii3[kPlanUnroll];
#pragma unroll
      for (int u = 0; u < kPlanUnroll; ++u) {
        const int t = g0 + u * nthr + threadIdx.x;
        kk[u] = 0xFFFFFFFFu;
        ii3[u] = 0;
        if (t < T) {
          int f = 0;  // the lookup's table: the last f with s_toff[f] <= t
          for (int lo2 = 1, hi2 = nt - 1; lo2 <= hi2;) {
            const int mid = (lo2 + hi2) >> 1;
            if (s_toff[mid] <= t) f = mid, lo2 = mid + 1;
            else hi2 = mid - 1;
          }
          const uint4 tg = s_tg[f];  // (m2, m3, rows) of the table
          long long v = (long long)idx[t];
          if (v < 0 || v >= (long long)tg.z) {
            bits |= 1;
            v = 0;
          }
          const unsigned m2m3 = tg.x * tg.y;
          const unsigned i = (unsigned)v, i1 = i / m2m3, r = i - i1 * m2m3, i2 = r / tg.y;
          kk[u] = ((unsigned)f * g.tm2 + i2) * g.m1 + i1;
          ii3[u] = r - i2 * tg.y;
          key[t] = kk[u];  // (many lookups per thread: none kept in registers)
          i3o[t] = ii3[u];
        }
      }
      unsigned peers[kPlanUnroll];
      int base[kPlanUnroll];
#pragma unroll
      for (int u = 0; u < kPlanUnroll; ++u) {  // (warp-uniform: every lane takes part in every match)
        peers[u] = __match_any_sync(0xffffffffu, kk[u]);
        base[u] = 0;
        if (g0 + u * nthr + threadIdx.x < T && lane == __ffs(peers[u]) - 1)
          base[u] = atomicAdd(&cnt[kk[u]], __popc(peers[u]));
      }
#pragma unroll
      for (int u = 0; u < kPlanUnroll; ++u) {
        const int t = g0 + u * nthr + threadIdx.x;
        const int rank = __shfl_sync(0xffffffffu, base[u], __ffs(peers[u]) - 1) + __popc(peers[u] & lanemask_lt());
        if (t < T) rk[t] = rank;
      }
    }
  }
  grid_barrier(bar, target);
  if (bits) atomicOr(&hdr[0], bits);  // (after the first barrier: block 0 has cleared the words)
  if (multi) hdr[1] = 1;
  PSTAMP(1);
  // ---- phase A1: per-i2 totals (positions, items, present prefixes)
  // group i2 -> CTA i2 % grid, warp i2 / grid: the groups spread over every SM
  const int gw = (threadIdx.x >> 5) * gridDim.x + blockIdx.x, nw = nthr >> 5;
  for (unsigned i2 = gw; i2 < g.m2; i2 += nw) {
    int c = 0, it = 0, p = 0;
    for (unsigned i1 = lane; i1 < g.m1; i1 += 32) {
      const int v = cnt[i2 * g.m1 + i1];
      c += v;
      it += (v + kItemLen - 1) / kItemLen;
      p += v > 0;
    }
    c = warp_sum(c);
    it = warp_sum(it);
    p = warp_sum(p);
    if (lane == 0) gtot[i2] = make_int4(c, it, p, 0);
  }
  grid_barrier(bar, target);
  PSTAMP(2);
  // ---- phase A2: group offsets, key starts, item and tile tables
  const bool pooled = hdr[1] != 0;  // some bag holds several lookups: row-sort chunks for the backward
  for (unsigned i2 = gw; i2 < g.m2; i2 += nw) {
    int pc = 0, pi = 0, pt = 0;
    for (unsigned j = lane; j < i2; j += 32) {
      const int4 q = gtot[j];
      pc += q.x;
      pi += q.y;
      pt += (q.y + kTileItems - 1) / kTileItems;
    }
    pc = warp_sum(pc);
    pi = warp_sum(pi);
    pt = warp_sum(pt);
    const int4 mine = gtot[i2];
    const int ntile = (mine.y + kTileItems - 1) / kTileItems;
    // items in descending length inside the group: full items (kItemLen
    // lookups) first, then each key's remainder item by length, so the items
    // of a tile have similar lengths (balanced epilogue / Z-phase work).
    // Item i's lookups are [item_start[i], item_start[i + 1]) as before.
    int* hist = s_hist[threadIdx.x >> 5];  // [L] items of length L, then cursors
    int* ioff = hist + kItemLen + 1;       // [L] first item (group-relative) of length L
    for (int L = lane; L <= kItemLen; L += 32) hist[L] = 0;
    // the group's counters: the first 32 kA2Regs in registers (one round of
    // loads for both passes), the rest re-read
    int cv[kA2Regs];
#pragma unroll
    for (int r = 0; r < kA2Regs; ++r) {
      const unsigned i1 = 32 * r + lane;
      cv[r] = i1 < g.m1 ? cnt[i2 * g.m1 + i1] : 0;
    }
    __syncwarp();
    auto pass1 = [&](int v) {
      if (v >= kItemLen) atomicAdd(&hist[kItemLen], v / kItemLen);
      if (v % kItemLen) atomicAdd(&hist[v % kItemLen], 1);
    };
#pragma unroll
    for (int r = 0; r < kA2Regs; ++r) pass1(cv[r]);
    for (unsigned i1b = 32 * kA2Regs; i1b < g.m1; i1b += 32) {
      const unsigned i1 = i1b + lane;
      pass1(i1 < g.m1 ? cnt[i2 * g.m1 + i1] : 0);
    }
    __syncwarp();
    {  // lane l <-> length L = kItemLen - l (descending); exclusive scans of items and lookups
      const int L = kItemLen - lane, h = hist[L];
      int si = h, sp = h * L;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int a2 = __shfl_up_sync(0xffffffffu, si, o), b2 = __shfl_up_sync(0xffffffffu, sp, o);
        if (lane >= o) si += a2, sp += b2;
      }
      ioff[L] = si - h;
      hist[L] = si - h;  // cursor
      hist[0] = 0;
      // lookup offset of length L's first item, kept in the key loop below via ioff
      s_poff[threadIdx.x >> 5][L] = sp - h * L;
    }
    __syncwarp();
    const int* poff = s_poff[threadIdx.x >> 5];
    auto pass2 = [&](unsigned i1, int v) {
      const unsigned k = i2 * g.m1 + i1;
      const int nf = v / kItemLen, r = v % kItemLen;
      int f = 0, fp = 0, rp = 0;
      if (nf) {
        f = atomicAdd(&hist[kItemLen], nf);
        fp = pc + poff[kItemLen] + (f - ioff[kItemLen]) * kItemLen;
      }
      // full items: the whole warp writes each key's run (hot keys own
      // thousands of items — one lane alone would serialise on them)
      unsigned many = __ballot_sync(0xffffffffu, nf > 0);
      while (many) {
        const int src = __ffs(many) - 1;
        many &= many - 1;
        const int sf = __shfl_sync(0xffffffffu, f, src), sfp = __shfl_sync(0xffffffffu, fp, src);
        const int snf = __shfl_sync(0xffffffffu, nf, src);
        const unsigned sk = __shfl_sync(0xffffffffu, k, src);
        for (int j = lane; j < snf; j += 32) {
          item_start[pi + sf + j] = sfp + kItemLen * j;
          item_key[pi + sf + j] = sk;
        }
        if (pooled && snf >= 2) {  // the key's full items in runs of <= kSortItems (k_rowsort)
          const int nch = (snf + kSortItems - 1) / kSortItems;
          int cb = 0;
          if (lane == 0) cb = atomicAdd(&hdr[kHdrChunks], nch);
          cb = __shfl_sync(0xffffffffu, cb, 0);
          for (int j = lane; j < nch; j += 32)
            chunks[cb + j] = make_int2(sfp + j * kSortItems * kItemLen,
                                       min(kSortItems, snf - j * kSortItems) * kItemLen);
        }
      }
      if (r) {
        const int q = atomicAdd(&hist[r], 1);
        rp = pc + poff[r] + (q - ioff[r]) * r;
        item_start[pi + q] = rp;
        item_key[pi + q] = k;
      }
      if (v > 0) {
        start[k] = fp;                   // lookups with rank < nf * kItemLen: start + rank
        rstart[k] = rp - nf * kItemLen;  // the rest: rstart + rank
        split[k] = nf * kItemLen;
        cnt[k] = 0;                      // counters reset for the next plan
      }
    };
#pragma unroll
    for (int r = 0; r < kA2Regs; ++r) pass2(32 * r + lane, cv[r]);  // (zero counts past m1 are no-ops)
    for (unsigned i1b = 32 * kA2Regs; i1b < g.m1; i1b += 32) {
      const unsigned i1 = i1b + lane;
      pass2(i1, i1 < g.m1 ? cnt[i2 * g.m1 + i1] : 0);
    }
    __syncwarp();
    // tiles: (i2, first item, items, first lookup position); the position of
    // the tile's first item from the length buckets (items [ioff[L], hist[L])
    // have length L), not re-read from global memory
    for (int j = lane; j < ntile; j += 32) {
      const int left = mine.y - kTileItems * j, f = kTileItems * j;
      int L = kItemLen;
      while (L > 1 && hist[L] <= f) --L;
      tile_info[pt + j] = make_int4((int)i2, pi + f, left < kTileItems ? left : kTileItems,
                                    pc + poff[L] + (f - ioff[L]) * L);
    }
    if (lane == 0) {
      atomicAdd(&hdr[3], mine.z);
      if (i2 == g.m2 - 1) {
        hdr[2] = pi + mine.y;
        hdr[4] = pt + ntile;
        item_start[pi + mine.y] = T;
      }
    }
  }
  grid_barrier(bar, target);
  PSTAMP(3);
  // ---- phase B: per-CTA tile ranges for the step kernels (grid = ctas):
  // contiguous tile runs of equal weight (lookups + kTileCost per tile)
  // cta_tiles[b] = #{tiles t : W_t < wtot b / ctas} with W_t = position of t
  // + kTileCost t (increasing): thread t writes it for every b whose target
  // lies in (W_{t-1}, W_t] — one load per tile instead of a dependent
  // binary search per CTA boundary
  {
    const int nt = hdr[4];
    const long long wtot = (long long)T + (long long)kTileCost * nt;
    for (int t = tid; t <= nt; t += nthr) {
      const long long lo_w = t == 0 ? -1 : (long long)tile_info[t - 1].w + (long long)kTileCost * (t - 1);
      const long long hi_w = t == nt ? wtot : (long long)tile_info[t].w + (long long)kTileCost * t;
      // first b with wtot b / ctas > lo_w, i.e. b >= ceil((lo_w + 1) ctas / wtot)
      long long b = lo_w < 0 ? 0 : ((lo_w + 1) * ctas + wtot - 1) / wtot;
      for (; b <= ctas && wtot * b / ctas <= hi_w; ++b)
        if (wtot * b / ctas > lo_w) cta_tiles[b] = t;
    }
  }
  // ---- phase B: scatter (bag, i3) into item order
  {
    const bool one = hdr[1] == 0 && T == B;  // one lookup per bag: bag id = lookup index
    if constexpr (!kMany) {
      int it2 = 0;
      for (int t = tid; t < T; t += nthr, ++it2) {
        unsigned k, i3;
        int r;
        if (it2 < kPlanRegs) {
#pragma unroll
          for (int q = 0; q < kPlanRegs; ++q)
            if (q == it2) {
              k = rkey[q];
              i3 = ri3[q];
              r = rrk[q];
            }
        } else {
          k = key[t];
          i3 = i3o[t];
          r = rk[t];
        }
        sbi[(r < split[k] ? start[k] : rstart[k]) + r] = make_int2(one ? t : bag_of[t], (int)i3);
      }
    } else {
      for (int t0 = tid; t0 < T; t0 += kPlanUnroll * nthr) {
        unsigned k[kPlanUnroll], i3[kPlanUnroll];
        int r[kPlanUnroll], bg[kPlanUnroll];
#pragma unroll
        for (int u = 0; u < kPlanUnroll; ++u) {  // every load of the round first
          const int t = t0 + u * nthr;
          k[u] = 0;
          i3[u] = 0;
          r[u] = 0;
          bg[u] = 0;
          if (t < T) {
            k[u] = key[t];
            i3[u] = i3o[t];
            r[u] = rk[t];
            bg[u] = one ? t : bag_of[t];
          }
        }
        int pos[kPlanUnroll];
#pragma unroll
        for (int u = 0; u < kPlanUnroll; ++u) {  // (the key's three words loaded together)
          const int sp = split[k[u]], st = start[k[u]], rs = rstart[k[u]];
          pos[u] = (r[u] < sp ? st : rs) + r[u];
        }
#pragma unroll
        for (int u = 0; u < kPlanUnroll; ++u)
          if (t0 + u * nthr < T) sbi[pos[u]] = make_int2(bg[u], (int)i3[u]);
      }
    }
  }
  __syncthreads();
  // the last CTA out (every CTA is past every barrier) resets the barrier
  // words for the next plan
  if (threadIdx.x == 0 && atomicAdd(&bar[1], 1u) == gridDim.x - 1) {
    bar[0] = 0u;
    bar[1] = 0u;
  }
  PSTAMP(4);
#undef PSTAMP
}

// ------------------------------------------------------------ core images
// Split (hi / lo) tf32 forms of the cores, built once per step (the cores
// change every step) and copied verbatim into shared memory by the step
// kernels (cp.async, no register staging):
//   per i2 (4 x 16 KB, the exact K-major SWIZZLE_128B smem images)
//     [0] cb_hi  [1] cb_lo : rows (c, b) = 4 c + b (128), K = k (32)
//     [2..3] k      : rows k (hi 0..31, lo 32..63), K = (c, b) (128)
//   per i1 (512 floats): rows_hi[a][k], rows_lo[a][k], t_hi[k][a], t_lo[k][a]
constexpr int kImgThreads = 512;

// Optional SGD(+momentum) step applied to each element before it is imaged:
// the fused update of the previous backward writes the next step's images.
struct SgdArgs {
  const float* grad;  // flat |G1| + |G2| + |G3| gradients
  double *v0, *v1, *v2;
  float* p2;
  double lr, mu;       // Adagrad: mu carries eps
  int mask, on;
  const int* err;     // device error word: any bit set -> no update (cores untouched)
  int adagrad;        // 0: SGD(+momentum), v = velocity; 1: Adagrad, v = squared-gradient sums
  float* g3t;         // G3 written slice-major (i3, c, n3) after the update (step kernels' bulk copies)
  const int* suspect;  // backward's kHdrSuspect word: set -> exact finiteness scan before updating
  int64_t ngrad;       // |G1| + |G2| + |G3| (the scan's extent)
};

// ------------------------------------------------------------ row sort
// Pooled batches, at the end of the plan: every run of <= kSortItems full
// items of one prefix (a plan chunk) is counting-sorted by i3 in shared
// memory, so the lookups of one row sit together and an item of a hot prefix
// holds one or two rows instead of a scatter of them: the forward closes each
// row once per item and pools it into every lookup's bag, and the row-grouped
// backward does X^T g, the dG3 reduction and the Z update once per (item, row)
// with the row's gradient rows summed first (the reference's unique_aggregate,
// backward.py:72-87, applied inside each chunk). Item boundaries, keys and
// tiles are unchanged.
constexpr int kSortMax = kSortItems * kItemLen;  // positions per chunk
constexpr int kSortThreads = 512;
constexpr int kSortPer = kSortMax / kSortThreads;  // positions per thread (CTA-wide chunks), in registers
constexpr int kSortSmall = 1024;                    // chunks up to this size: one warp each
constexpr int kSortHist = 320;                      // >= m3 of any tensor-core table (kFwdMaxM3 = 288)
constexpr int kSortSmem = (kSortMax > (kSortThreads / 32) * kSortSmall ? kSortMax : (kSortThreads / 32) * kSortSmall) *
                          (int)sizeof(int2);
__device__ __forceinline__ void warp_exclusive_scan(int* hist, unsigned n, int lane) {
  int carry = 0;
  for (unsigned b0 = 0; b0 < n; b0 += 32) {
    const unsigned bi = b0 + lane;
    const int h = bi < n ? hist[bi] : 0;
    int x = h;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (bi < n) hist[bi] = carry + x - h;
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
}
__global__ void __launch_bounds__(kSortThreads) k_rowsort(int2* __restrict__ sbi, const int2* __restrict__ chunks,
                                                         const int* __restrict__ hdr, unsigned tm3) {
  pdl_enter();
  extern __shared__ __align__(16) char smem_raw[];
  int2* o = reinterpret_cast<int2*>(smem_raw);  // CTA-wide chunk output; per warp 1024 entries for small chunks
  __shared__ int hist[kSortThreads / 32][kSortHist];  // per warp; warp 0's row is the CTA-wide histogram
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = hdr[kHdrChunks];
  // large chunks: the whole CTA, every load of the chunk in flight at once
  for (int ci = blockIdx.x; ci < nch; ci += gridDim.x) {
    const int2 cd = chunks[ci];
    const int p0 = cd.x, L = cd.y;
    if (L <= kSortSmall) continue;  // (uniform)
    // per-warp histograms (no atomics: a bin's count is updated by its
    // match leader only), combined into per-warp cursors
    int2 v[kSortPer];
#pragma unroll
    for (int r = 0; r < kSortPer; ++r) {
      const int i = r * kSortThreads + threadIdx.x;
      v[r] = i < L ? sbi[p0 + i] : make_int2(0, -1 - lane);
    }
    constexpr int NW = kSortThreads / 32;
    for (int i = threadIdx.x; i < NW * kSortHist; i += kSortThreads) (&hist[0][0])[i] = 0;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kSortPer; ++r) {
      if (r * kSortThreads >= L) break;  // (uniform)
      const unsigned peers = __match_any_sync(0xffffffffu, v[r].y);
      if (v[r].y >= 0 && (__ffs(peers) - 1) == lane) hist[warp][v[r].y] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    // bin b: warp w's cursor = start_b + (counts of warps < w); bin totals in
    // hist[NW - 1] (scanned by warp 0), then added back
    __shared__ int s_tot[kSortHist];
    for (int b = threadIdx.x; b < (int)tm3; b += kSortThreads) {
      int run = 0;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const int h = hist[w][b];
        hist[w][b] = run;
        run += h;
      }
      s_tot[b] = run;
    }
    __syncthreads();
    if (warp == 0) warp_exclusive_scan(s_tot, tm3, lane);
    __syncthreads();
    for (int b = threadIdx.x; b < (int)tm3; b += kSortThreads) {
      const int st = s_tot[b];
#pragma unroll
      for (int w = 0; w < NW; ++w) hist[w][b] += st;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kSortPer; ++r) {
      if (r * kSortThreads >= L) break;
      const unsigned peers = __match_any_sync(0xffffffffu, v[r].y);
      const int ld = __ffs(peers) - 1;
      int base = 0;
      if (v[r].y >= 0 && ld == lane) {
        base = hist[warp][v[r].y];
        hist[warp][v[r].y] = base + __popc(peers);
      }
      base = __shfl_sync(0xffffffffu, base, ld);
      if (v[r].y >= 0) o[base + __popc(peers & lanemask_lt())] = v[r];
      __syncwarp();
    }
    __syncthreads();
    for (int i = threadIdx.x; i < L; i += kSortThreads) sbi[p0 + i] = o[i];
    __syncthreads();
  }
  // small chunks (most keys): one warp each, no CTA barriers
  int* hw = hist[warp];
  int2* ow = o + warp * kSortSmall;
  const int gw = blockIdx.x * (kSortThreads / 32) + warp, nw = gridDim.x * (kSortThreads / 32);
  for (int ci = gw; ci < nch; ci += nw) {
    const int2 cd = chunks[ci];
    const int p0 = cd.x, L = cd.y;
    if (L > kSortSmall) continue;
    int2 v[kSortSmall / 32];
#pragma unroll
    for (int r = 0; r < kSortSmall / 32; ++r) {
      const int i = r * 32 + lane;
      v[r] = i < L ? sbi[p0 + i] : make_int2(0, -1 - lane);
    }
    for (int i = lane; i < (int)tm3; i += 32) hw[i] = 0;
    __syncwarp();
#pragma unroll
    for (int r = 0; r < kSortSmall / 32; ++r) {
      if (r * 32 >= L) break;
      const unsigned peers = __match_any_sync(0xffffffffu, v[r].y);
      if (v[r].y >= 0 && (__ffs(peers) - 1) == lane) hw[v[r].y] += __popc(peers);
      __syncwarp();
    }
    warp_exclusive_scan(hw, tm3, lane);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < kSortSmall / 32; ++r) {
      if (r * 32 >= L) break;
      const unsigned peers = __match_any_sync(0xffffffffu, v[r].y);
      const int ld = __ffs(peers) - 1;
      int base = 0;
      if (v[r].y >= 0 && ld == lane) {
        base = hw[v[r].y];
        hw[v[r].y] = base + __popc(peers);
      }
      base = __shfl_sync(0xffffffffu, base, ld);
      if (v[r].y >= 0) ow[base + __popc(peers & lanemask_lt())] = v[r];
      __syncwarp();
    }
    for (int i = lane; i < L; i += 32) sbi[p0 + i] = ow[i];
    __syncwarp();
  }
}

// Finiteness pre-pass over the final gradients (fused_update rejects a
// non-finite gradient before touching any core, backward.py:190-194): sets
// TTB_ERRBIT_NONFINITE in *err; the update kernel that follows reads it.
__global__ void __launch_bounds__(256) k_gradcheck(const float* __restrict__ g, int64_t n, int* __restrict__ err,
                                                   const int* __restrict__ suspect) {
  pdl_enter();
  // the backward flags any contribution that is non-finite or >= 2^95 in
  // magnitude; without one, every final sum (< 2^31 terms) is finite
  if (suspect && *(volatile const int*)suspect == 0) return;
  bool bad = false;
  const int64_t n4 = (reinterpret_cast<uintptr_t>(g) & 15) ? 0 : n >> 2;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = g4[i];
    bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
  }
  for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(g[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, TTB_ERRBIT_NONFINITE);
}

// dG3 slice-major (i3, c, n3) -> the reference layout (c, i3, n3)
__global__ void __launch_bounds__(256) k_g3_unslice(const float* __restrict__ src, float* __restrict__ dst,
                                                    unsigned m3) {
  pdl_enter();
  const unsigned n = 128 * m3;
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const unsigned c = e / (4 * m3), r = e - c * 4 * m3;
    dst[e] = src[((size_t)(r >> 2) * 32 + c) * 4 + (r & 3)];
  }
}

__device__ __forceinline__ float maybe_sgd(float p, const SgdArgs& u, int core, size_t flat, size_t j, double* v) {
  if (!u.on || !((u.mask >> core) & 1)) return p;
  if (u.adagrad) return adagrad_apply(p, u.grad[flat], v + j, u.lr, u.mu);
  return sgd_apply(p, u.grad[flat], v ? v + j : nullptr, u.lr, u.mu);
}

__global__ void __launch_bounds__(kImgThreads, 2) k_coreimg(float* __restrict__ G1, float* __restrict__ G2, KGeom g,
                                                         float* __restrict__ img, float* __restrict__ g1img,
                                                         SgdArgs u) {
  pdl_enter();
  // an error latched by the plan or the backward (range, empty bag,
  // non-finite gradient) cancels the update: the images are rebuilt from the
  // unchanged cores and velocities
  __shared__ int s_gate;  // one read of the words per CTA: every thread takes the same branch
  if (threadIdx.x == 0)
    s_gate = !(u.on && u.err) ? 0
             : *(volatile const int*)u.err != 0 ? 1
             : (u.suspect && *(volatile const int*)u.suspect != 0) ? 2 : 0;
  __syncthreads();
  {
    const int gate = s_gate;
    if (gate == 1) {
      u.on = 0;
    } else if (gate == 2) {
      // rare: the backward saw a contribution that is non-finite or >= 2^95.
      // Every CTA scans every gradient, so all reach the same all-or-nothing
      // decision without a grid-wide barrier (fused_update rejects a
      // non-finite gradient before touching any core, backward.py:190-194)
      bool bad = false;
      for (int64_t i = threadIdx.x; i < u.ngrad; i += blockDim.x) bad |= !isfinite(u.grad[i]);
      if (__syncthreads_or(bad)) {
        if (threadIdx.x == 0) atomicOr(const_cast<int*>(u.err), TTB_ERRBIT_NONFINITE);
        u.on = 0;
      }
    }
  }
  const size_t n0 = (size_t)g.g1rows * 4 * R1, n1 = (size_t)R1 * g.m2 * C;
  const unsigned nb12 = g.m2 + (g.g1rows + 3) / 4;
  if (blockIdx.x >= nb12) {  // G3: update, and its slice-major copy
    const size_t n2 = (size_t)32 * g.m3 * 4, stride = (size_t)(gridDim.x - nb12) * kImgThreads;
    const bool upd = u.on && (u.mask & 4), has_v = u.adagrad || u.v2 != nullptr;
    constexpr int kU = 4;  // elements per thread in flight
    for (size_t j0 = (size_t)(blockIdx.x - nb12) * kImgThreads + threadIdx.x; j0 < n2; j0 += kU * stride) {
      float pv[kU], gr[kU];
      double st[kU];
      unsigned jt[kU];
#pragma unroll
      for (int q = 0; q < kU; ++q) {
        const size_t j = j0 + q * stride;
        // the backward accumulates dG3 slice-major, (i3, c, n3), as the copy
        const unsigned jj = (unsigned)j, c = jj / (g.m3 * 4), r = jj - c * g.m3 * 4;  // n2 < 2^32
        jt[q] = ((r >> 2) * 32 + c) * 4 + (r & 3);
        if (j < n2) {
          pv[q] = u.p2[j];
          gr[q] = upd ? u.grad[n0 + n1 + jt[q]] : 0.f;
          st[q] = upd && has_v ? u.v2[j] : 0.0;
        }
      }
#pragma unroll
      for (int q = 0; q < kU; ++q) {
        const size_t j = j0 + q * stride;
        if (j >= n2) break;
        float w = pv[q];
        if (upd) {
          double ns;
          w = u.adagrad ? adagrad_step(w, gr[q], st[q], &ns, u.lr, u.mu)
                        : sgd_step(w, gr[q], st[q], &ns, has_v, u.lr, u.mu);
          if (has_v) u.v2[j] = ns;
          u.p2[j] = w;
        }
        u.g3t[jt[q]] = w;
      }
    }
    return;
  }
  if (blockIdx.x >= g.m2) {  // G1 images: 4 i1 per block (128 elements each)
    const unsigned i1 = (blockIdx.x - g.m2) * 4 + (threadIdx.x >> 7);
    const int e = threadIdx.x & 127, a = e >> 5, k = e & 31;
    if (i1 < g.g1rows) {
      const size_t j = (size_t)i1 * 128 + e;
      float v = G1[j];
      if (u.on && (u.mask & 1)) {
        v = maybe_sgd(v, u, 0, j, j, u.v0);
        G1[j] = v;
      }
      float hi, lo;
      umma::split3(v, hi, lo);
      float* d = g1img + (size_t)i1 * kG1Img;
#pragma unroll
      for (int p = 0; p < 2; ++p) {  // row a at smem line 4 p + a: 16-byte chunk k / 4 -> (k / 4) ^ (4 p + a)
        const int o = g1_rows_off(p) + a * 32 + ((((k >> 2) ^ (4 * p + a)) & 7) << 2) + (k & 3);
        d[o] = hi;
        d[128 + o] = lo;
      }
      d[kG1T + k * 4 + a] = hi;
      d[kG1T + 128 + k * 4 + a] = lo;
    }
    return;
  }
  extern __shared__ __align__(16) char smem_raw[];
  char* sm = smem_raw + ((1024u - (umma::smem_u32(smem_raw) & 1023u)) & 1023u);
  const unsigned i2 = blockIdx.x;
  constexpr int kPer = R1 * C / kImgThreads;  // 8
  float vals[kPer];
#pragma unroll
  for (int r = 0; r < kPer; ++r) {
    const int e = threadIdx.x + r * kImgThreads, k = e >> 7;
    vals[r] = G2[((size_t)k * g.m2 + i2) * C + (e & 127)];
  }
  if (u.on && (u.mask & 2)) {
    // every load of the slice's gradients and optimizer state first (one
    // round trip), then the updates and stores
    float gr[kPer];
    double st[kPer];
    const bool has_v = u.adagrad || u.v1 != nullptr;
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
      const int e = threadIdx.x + r * kImgThreads, k = e >> 7;
      const size_t j = ((size_t)k * g.m2 + i2) * C + (e & 127);
      gr[r] = u.grad[n0 + j];
      st[r] = has_v ? u.v1[j] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
      const int e = threadIdx.x + r * kImgThreads, k = e >> 7;
      const size_t j = ((size_t)k * g.m2 + i2) * C + (e & 127);
      double ns;
      vals[r] = u.adagrad ? adagrad_step(vals[r], gr[r], st[r], &ns, u.lr, u.mu)
                          : sgd_step(vals[r], gr[r], st[r], &ns, has_v, u.lr, u.mu);
      if (has_v) u.v1[j] = ns;
      G2[j] = vals[r];
    }
  }
  // the slice in shared memory first (row k padded to 129 floats), then each
  // image row written by one warp — 32 consecutive K of one 128-byte row, no
  // bank conflicts (a direct scatter from the load layout is 16-way)
  float* raw = reinterpret_cast<float*>(sm);
#pragma unroll
  for (int r = 0; r < kPer; ++r) {
    const int e = threadIdx.x + r * kImgThreads;
    raw[(e >> 7) * 129 + (e & 127)] = vals[r];
  }
  __syncthreads();
  // image rows go straight to global memory: each warp store is one whole
  // (swizzled) 128-byte row, and the CTA needs only the 16.5 KB slice buffer
  char* gi = reinterpret_cast<char*>(img + (size_t)i2 * (4 * kImg / 4));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r < 128 / (kImgThreads / 32); ++r) {  // cb images: row cb = 4 c + b, K = k = lane
    const int cb = warp + r * (kImgThreads / 32), b = cb & 3, c = cb >> 2;
    float hi, lo;
    umma::split3(raw[lane * 129 + b * 32 + c], hi, lo);
    const uint32_t o1 = umma::sw128_off(cb, lane, 128);
    *(float*)(gi + o1) = hi;
    *(float*)(gi + kImg + o1) = lo;
  }
#pragma unroll
  for (int r = 0; r < 128 / (kImgThreads / 32); ++r) {  // k images: row k, K = cb (block of 32)
    const int unit = warp + r * (kImgThreads / 32), k = unit >> 2, cb = 32 * (unit & 3) + lane;
    float hi, lo;
    umma::split3(raw[k * 129 + (cb & 3) * 32 + (cb >> 2)], hi, lo);
    *(float*)(gi + 2 * kImg + umma::sw128_off(k, cb, 64)) = hi;
    *(float*)(gi + 2 * kImg + umma::sw128_off(32 + k, cb, 64)) = lo;
  }
}


__device__ inline void copy_img_async(char* dst, const float* __restrict__ src, int bytes) {
  for (int e = threadIdx.x; e < bytes / 16; e += kThreads) cp_async16(dst + 16 * e, src + 4 * e);
}


// 3xTF32 product of two smem images over K (k-steps of 8)
__device__ inline void mma3_ss(uint32_t d, uint32_t a_hi, uint32_t a_lo, int a_rows, uint32_t b_hi, uint32_t b_lo,
                               int b_rows, int K, uint32_t idesc) {
  for (int k0 = 0; k0 < K; k0 += 8) {
    const uint64_t ah = umma::sw128_desc_at(a_hi, k0, a_rows), al = umma::sw128_desc_at(a_lo, k0, a_rows);
    const uint64_t bh = umma::sw128_desc_at(b_hi, k0, b_rows), bl = umma::sw128_desc_at(b_lo, k0, b_rows);
    umma::mma_tf32(d, ah, bh, idesc, k0 > 0 ? 1u : 0u);
    umma::mma_tf32(d, ah, bl, idesc, 1u);
    umma::mma_tf32(d, al, bh, idesc, 1u);
  }
}

// ------------------------------------------------------------ tile bookkeeping
// Tile metadata lives in a two-slot ring: while tile t is processed, the
// last warp fetches tile t + grid's (cp.async) and the tile table entry of
// t + 2 grid (a register load, consumed an iteration later).

// G1^T image of the tile's items (rows k, K = (item, a)); zero columns past n
// (one 64-row image: rows k = hi, rows 32 + k = lo). Only the first item of
// each run of one key is copied from global memory: a hot key fills whole
// tiles with items of one i1, and thousands of copies of the same 512 bytes
// from every CTA serialise in the memory system; the run's other items are
// filled from the first one by g1_t_replicate once the copies landed.
__device__ __forceinline__ unsigned tile_run_heads(const TileMeta* m, int lane) {
  const unsigned kl = lane < m->n ? m->key[lane] : 0xFFFFFFFFu;
  const unsigned kp = __shfl_up_sync(0xffffffffu, kl, 1);
  return __ballot_sync(0xffffffffu, lane == 0 || kl != kp);
}
__device__ inline void stage_g1_t_async(const TileMeta* m, KGeom g, const float* __restrict__ g1img, char* img) {
  const unsigned heads = tile_run_heads(m, threadIdx.x & 31);
#pragma unroll
  for (int i = 0; i < 1024 / kThreads; ++i) {
    const int e = threadIdx.x + i * kThreads, it = e >> 5, k = e & 31;
    const uint32_t oh = umma::sw128_off(k, 4 * it, 64), ol = umma::sw128_off(32 + k, 4 * it, 64);
    if (it < m->n) {
      if ((heads >> it) & 1u) {
        const float* src = g1img + (size_t)item_i1(m, it, g) * kG1Img + kG1T + 4 * k;
        cp_async16(img + oh, src);
        cp_async16(img + ol, src + 128);
      }
    } else {
      *reinterpret_cast<float4*>(img + oh) = make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(img + ol) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}
// after the copies landed and a barrier: each run's other items from its first
__device__ inline void g1_t_replicate(const TileMeta* m, char* img) {
  const unsigned heads = tile_run_heads(m, threadIdx.x & 31);
  if (m->n == 32 ? heads == 0xFFFFFFFFu : (~heads & ((1u << m->n) - 1u)) == 0u) return;  // distinct keys (uniform)
#pragma unroll
  for (int i = 0; i < 1024 / kThreads; ++i) {
    const int e = threadIdx.x + i * kThreads, it = e >> 5, k = e & 31;
    if (it < m->n && !((heads >> it) & 1u)) {
      const int src = 31 - __clz(heads & (0xFFFFFFFFu >> (31 - it)));  // the run's first item
      *reinterpret_cast<float4*>(img + umma::sw128_off(k, 4 * it, 64)) =
          *reinterpret_cast<const float4*>(img + umma::sw128_off(k, 4 * src, 64));
      *reinterpret_cast<float4*>(img + umma::sw128_off(32 + k, 4 * it, 64)) =
          *reinterpret_cast<const float4*>(img + umma::sw128_off(32 + k, 4 * src, 64));
    }
  }
}

// ------------------------------------------------------------ forward
// Persistent: one 512-thread CTA per SM loops over a contiguous range of
// tiles (consecutive tiles mostly share i2: the G2 image is reloaded only when
// it changes). G3 stays resident in shared memory; each tile's operands and
// (bag, i3) list arrive by one round of cp.async and one thread issues the
// 3xTF32 X MMA. Epilogue thread <-> accumulator row (item, a): the four warps
// of a lane quadrant take every fourth segment of the item, reading the X row
// from TMEM in two halves of c (64 registers).
constexpr int kMaxTilePos = kTileItems * kItemLen;  // 1024

constexpr int kFwdMaxM3 = 288;                       // G3 (32 x m3 x 4 fp32) kept in smem
constexpr int kFwdThreads = 512;

// G3 region sized by the table's m3 (the (bag, i3) stages follow it)
__host__ __device__ constexpr int fwd_g3_bytes(unsigned m3) { return (int)(32 * m3 * 16 + 1023) & ~1023; }
__host__ __device__ constexpr int fwd_smem_bytes(unsigned m3) { return 4 * kImg + fwd_g3_bytes(m3) + 2 * kMaxTilePos * 8 + 1024; }

template <bool kPooled>
__global__ void __launch_bounds__(kFwdThreads, 1) k_fwd(KGeom g, const float* __restrict__ g1img,
                                                        const float* __restrict__ G3, const float* __restrict__ img,
                                                        const int* __restrict__ hdr, const int4* __restrict__ tile_info,
                                                        const int* __restrict__ item_start,
                                                        const unsigned* __restrict__ item_key,
                                                        const int2* __restrict__ sbi, float* __restrict__ out,
                                                        const int* __restrict__ cta_tiles, int direct, int dbg) {
  pdl_enter();
  extern __shared__ __align__(16) char smem_raw[];
  char* sm = smem_raw + ((1024u - (umma::smem_u32(smem_raw) & 1023u)) & 1023u);
#define FSTAMP(k)                                                                                     \
  do {                                                                                                \
    if ((dbg & 16) && threadIdx.x == 0 && blockIdx.x == 0 && t - tb < 4) {                           \
      unsigned long long _t;                                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                                          \
      reinterpret_cast<unsigned long long*>(const_cast<int*>(hdr) + 16)[(k) * 4 + (t - tb)] = _t;     \
    }                                                                                                 \
  } while (0)
  char* a_hi = sm;             // G1 rows image
  char* a_lo = sm + kImg;
  char* b_hi = sm + 2 * kImg;  // G2 cb image
  char* b_lo = sm + 3 * kImg;
  float4* s_g3 = reinterpret_cast<float4*>(sm + 4 * kImg);
  int2* s_sbi2 = reinterpret_cast<int2*>(sm + 4 * kImg + fwd_g3_bytes(g.tm3));  // two (bag, i3) stages
  __shared__ TileMeta s_m[3];
  __shared__ uint64_t s_mbar;
  __shared__ uint32_t s_tmem;
  __shared__ unsigned s_segm[kTileItems];  // per item of the tile: its segments' first positions (bit mask)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned m3 = g.tm3;  // the resident G3 block: one table's slices (m3 <= kFwdMaxM3, fast_supported)
  const int ntiles = hdr[4];
  const int tb = cta_tiles[blockIdx.x], te = cta_tiles[blockIdx.x + 1];  // weight-balanced (k_fplan)
  (void)ntiles;
  if (warp == 0) umma::tmem_alloc(&s_tmem, 128);  // X
  if (threadIdx.x == 32) umma::mbar_init(&s_mbar, 1);
  // table f's G3 slices [f M3, (f + 1) M3) of every row c (rows are g.m3 slices long)
  auto stage_g3 = [&](unsigned f) {
    const float4* src = reinterpret_cast<const float4*>(G3) + (size_t)f * m3;
    for (int e = threadIdx.x; e < 32 * (int)m3; e += kFwdThreads) {
      const int c = e / (int)m3, j = e - c * (int)m3;
      cp_async16(s_g3 + e, src + (size_t)c * g.m3 + j);
    }
  };
  unsigned g3_table = tb < te ? (unsigned)tile_info[tb].x / g.tm2 : 0u;
  stage_g3(g3_table);
  int4 pf = make_int4(0, 0, 0, 0);
  if (warp == 15 && tb < te) {
    fetch_meta_async(tile_info[tb], item_start, item_key, &s_m[0]);
    if (tb + 1 < te) pf = tile_info[tb + 1];
  }
  cp_async_wait_all();
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = s_tmem;
  int last_i2 = -1;
  // all threads: tile u's (bag, i3) list and X operands (cp.async), and the
  // metadata of tile u+1 (warp 15)
  auto stage = [&](int u) {
    const TileMeta* mu = &s_m[(u - tb) % 3];
    const int q0 = mu->start[0], nq = mu->start[mu->n] - q0;
    int2* st = s_sbi2 + ((u - tb) & 1) * kMaxTilePos;
    for (int e = threadIdx.x; e < nq; e += kFwdThreads) cp_async8(st + e, sbi + q0 + e);
    if (mu->i2 != last_i2) {  // cb_hi, cb_lo
      const float* src = img + (size_t)mu->i2 * kImg;
      for (int e = threadIdx.x; e < 2 * kImg / 16; e += kFwdThreads) cp_async16(b_hi + 16 * e, src + 4 * e);
      last_i2 = mu->i2;
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {  // the items' G1 rows (hi, lo): 512 pre-swizzled bytes per item
      const int e = threadIdx.x + i * kFwdThreads, iu = e >> 5, q = e & 31;
      if (iu < mu->n) {
        const float* src = g1img + (size_t)item_i1(mu, iu, g) * kG1Img + g1_rows_off(iu & 1) + 4 * q;
        cp_async16(a_hi + iu * 512 + 16 * q, src);
        cp_async16(a_lo + iu * 512 + 16 * q, src + 128);
      }
    }
    if (warp == 15 && u + 1 < te) {
      fetch_meta_async(pf, item_start, item_key, &s_m[(u + 1 - tb) % 3]);
      if (u + 2 < te) pf = tile_info[u + 2];
    }
  };
  auto issue_mma = [&]() {
    if (threadIdx.x == 0) {
      constexpr uint32_t id = umma::idesc_tf32(128, 128, false, false);
      mma3_ss(tmem, umma::smem_u32(a_hi), umma::smem_u32(a_lo), 128, umma::smem_u32(b_hi), umma::smem_u32(b_lo),
              128, R1, id);
      umma::commit(&s_mbar);
    }
  };
  if (tb < te) {
    stage(tb);
    cp_async_wait_all();
    sync_for_mma();
    issue_mma();
  }
  const int q4 = warp & 3, quarter = warp >> 2;
  const int row = 32 * q4 + lane, it = row >> 2, a = row & 3;
  const uint32_t trow = tmem + ((uint32_t)(32 * q4) << 16);
  uint32_t phase = 0;
  for (int t = tb; t < te; ++t) {
    const TileMeta* m = &s_m[(t - tb) % 3];
    const int2* s_sbi = s_sbi2 + ((t - tb) & 1) * kMaxTilePos;
    FSTAMP(0);
    umma::mbar_wait(&s_mbar, phase);  // X of tile t; its operands are free again
    phase ^= 1u;
    umma::fence_after_sync();
    FSTAMP(1);
    const int p0 = m->start[0];
    // segments (runs of one bag) of each item as a bit mask of their first
    // positions: one ballot per item instead of every epilogue thread
    // re-scanning its item's (bag, i3) list
    // (one lookup per bag: every position starts a segment). Pooled bags:
    // a segment is a run of one ROW (equal i3; the plan's row sort groups a
    // hot prefix's lookups by row), closed once and pooled into each of its
    // lookups' bags
    if (!direct) {
      for (int j = warp; j < m->n; j += kFwdThreads / 32) {
        const int j0 = m->start[j] - p0, len = m->start[j + 1] - m->start[j];
        const int bg = lane < len ? (kPooled ? s_sbi[j0 + lane].y : s_sbi[j0 + lane].x) : -1;
        const int pv = __shfl_up_sync(0xffffffffu, bg, 1);
        const unsigned mk = __ballot_sync(0xffffffffu, lane < len && (lane == 0 || bg != pv));
        if (lane == 0) s_segm[j] = mk;
      }
      __syncthreads();
    }
    if (t + 1 < te) stage(t + 1);  // lands while this tile is closed
    FSTAMP(2);
    // ---- epilogue. The four warps of a lane quadrant share its 32 rows
    // (item, a) and take alternate segments of each row (quarter q: segments
    // q, q + 4, ...), each closing all 32 values of c from the X row in TMEM.
    // (Splitting each segment's contraction over c across the quarters, with
    // the partial sums exchanged through TMEM, measured slower at every
    // segment count: 40.0 -> 37.5 us at config 2, 287 -> 278 us at config 3.)
    const bool live = it < m->n;
    const int q0 = live ? m->start[it] - p0 : 0, len = live ? m->start[it + 1] - p0 - q0 : 0;
    const unsigned smask = !live ? 0u : direct ? (len >= 32 ? 0xffffffffu : (1u << len) - 1u) : s_segm[it];
    // segment [qq, e) of the row from the remaining start bits
    auto seg_next = [&](unsigned& rem, int& qq, int& e) {
      qq = q0 + __ffs(rem) - 1;
      rem &= rem - 1;
      e = q0 + (rem ? __ffs(rem) - 1 : len);
    };
    unsigned rem = smask;  // quarter q takes segments q, q + 4, ...
    for (int k = 0; k < quarter && rem; ++k) rem &= rem - 1;
    for (;;) {
      const bool have = rem != 0;
      int bag = 0, qq = 0, e = 0;
      if (have) {
        seg_next(rem, qq, e);
        bag = s_sbi[qq].x;
        for (int k = 0; k < 3 && rem; ++k) rem &= rem - 1;
      }
      if (!__any_sync(0xffffffffu, have)) break;
      float acc[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = 0.f;
      if (kPooled) {
        // per quarter of c: the run's row closed once (a rank-8 update of
        // the 16 outputs per quarter), then pooled into each lookup's bag
#pragma unroll
        for (int cq = 0; cq < 4; ++cq) {
          float xq[32];  // xq[4 c' + b] = X[item][a][b][8 cq + c']
          umma::tmem_ld32(trow + 32 * cq, xq);
          if (have) {
            float4 gs[8];  // the run's row: one G3 slice
            {
              const float4* g3 = s_g3 + (unsigned)s_sbi[qq].y + 8 * cq * m3;
#pragma unroll
              for (int c = 0; c < 8; ++c) gs[c] = g3[c * m3];
            }
#pragma unroll
            for (int c = 0; c < 8; ++c)
#pragma unroll
              for (int b = 0; b < 4; ++b) {
                const float xv = xq[4 * c + b];
                acc[4 * b + 0] = fmaf(xv, gs[c].x, acc[4 * b + 0]);
                acc[4 * b + 1] = fmaf(xv, gs[c].y, acc[4 * b + 1]);
                acc[4 * b + 2] = fmaf(xv, gs[c].z, acc[4 * b + 2]);
                acc[4 * b + 3] = fmaf(xv, gs[c].w, acc[4 * b + 3]);
              }
          }
        }
      } else {
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          float xh[64];  // xh[4 c' + b] = X[item][a][b][16 ch + c']
          umma::tmem_ld32(trow + 64 * ch, *(float(*)[32])(xh));
          umma::tmem_ld32(trow + 64 * ch + 32, *(float(*)[32])(xh + 32));
          if (have) {
            for (int l = qq; l < e; ++l) {
              const float4* g3 = s_g3 + (unsigned)s_sbi[l].y + 16 * ch * m3;
#pragma unroll
              for (int c = 0; c < 16; ++c) {
                const float4 gv = g3[c * m3];
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                  const float xv = xh[4 * c + b];
                  acc[4 * b + 0] = fmaf(xv, gv.x, acc[4 * b + 0]);
                  acc[4 * b + 1] = fmaf(xv, gv.y, acc[4 * b + 1]);
                  acc[4 * b + 2] = fmaf(xv, gv.z, acc[4 * b + 2]);
                  acc[4 * b + 3] = fmaf(xv, gv.w, acc[4 * b + 3]);
                }
              }
            }
          }
        }
      }
      if (have) {
        float* o = out + (size_t)bag * NOUT + a * 16;
        if (direct) {
#pragma unroll
          for (int b = 0; b < 4; ++b)
            reinterpret_cast<float4*>(o)[b] = make_float4(acc[4 * b], acc[4 * b + 1], acc[4 * b + 2], acc[4 * b + 3]);
        } else {
          for (int l = qq; l < (kPooled ? e : qq + 1); ++l) {  // (pooled: the row into each lookup's bag)
            float* ol = kPooled ? out + (size_t)s_sbi[l].x * NOUT + a * 16 : o;
#pragma unroll
            for (int b = 0; b < 4; ++b)
              red_v4(ol + 4 * b, acc[4 * b], acc[4 * b + 1], acc[4 * b + 2], acc[4 * b + 3]);
          }
        }
      }
    }
    FSTAMP(4);
    FSTAMP(4);
    cp_async_wait_all();  // the next tile's operands, list and metadata
    sync_for_mma();       // TMEM read by every epilogue thread; operands visible to the tensor core
    if (t + 1 < te) {
      issue_mma();
      const unsigned fn = (unsigned)s_m[(t + 1 - tb) % 3].i2 / g.tm2;
      if (fn != g3_table) {  // batched handle: the next tile belongs to another table
        stage_g3(fn);
        cp_async_wait_all();
        __syncthreads();
        g3_table = fn;
      }
    }
    FSTAMP(3);
  }
  if (warp == 0) umma::tmem_free(tmem, 128);
#undef FSTAMP
}

// ------------------------------------------------------------ backward
// Persistent, one CTA per SM, all 512 TMEM columns:
//   TMEM   [0,128) X^T (lanes (c, b), cols (item, a))   [128,256) Z^T hi
//          [256,384) Z^T lo   [384,448) dG2 tile (x G1 hi | x G1 lo)
//          [448,512) E tile (x G2 hi | x G2 lo)
//   smem   R12 64 KB: X operands (G2 cb image, G1 rows image), then the
//                     64-row G2 k image and the 64-row G1^T image
//          XZ  64 KB: per item a 512-float slot holding X (dumped from TMEM),
//                     overwritten by Z; finally the Z hi image (rows (item, a),
//                     K = (c, b)) the E GEMM reads
//          ST  97 KB: per chunk of positions: (bag, i3), the bag's gradient
//                     row and (bag-run path) the lookup's G3 slice (c, j); the
//                     row path adds a per-warp 256 B row scratch. Once the Z
//                     phase is done it holds the Z lo image (at 4 KB, past the
//                     next tile's (bag, i3) list)
// Z / dG3 phase: one warp per item, lane <-> c: every lane holds the item's
// X[., ., c] and accumulates Z[., ., c] in registers, so a position costs
// 128 FMAs per lane and no cross-lane reduction (k_bwd<true>: per distinct
// row of the item instead). The next tile's X operands and first-chunk rows
// are fetched after the E GEMM, during the dG1 / dG2 reductions.
// per-phase SM cycles (thread 0, summed over block 0's tiles) into hdr[16..]
// as 9 u64 + the tile count (TTB_DBG & 8); phase k = TSTAMP(k-1) .. TSTAMP(k)
#define TSTAMP(k)                                                                                      \
  do {                                                                                                 \
    if ((dbg & 8) && threadIdx.x == 0 && blockIdx.x == 0) {                                            \
      const long long _t = clock64();                                                                  \
      if ((k) > 0) s_tacc[(k)] += _t - s_tacc[0];                                                       \
      s_tacc[0] = _t;                                                                                  \
    }                                                                                                  \
  } while (0)

constexpr int kChunkPos = 128;
constexpr int kStSbi = kChunkPos * 8, kStG = kChunkPos * 256, kStG3 = kChunkPos * 512;
constexpr int kBwdSmem = 4 * kImg + 4 * kImg + kStSbi + kStG + kStG3 + 1024;
// row-grouped backward (pooled batches): G3 slices are read per distinct row
// from L2 instead of staged per position, so a chunk holds 3x the positions
// warps per TMEM lane quadrant, and the columns each takes of a 128- / 32-column operand
// row path: per-warp ring of row slots in the Z lo image's region (dead
// during the Z phase): gradient row (256 B) + G3 slice (512 B) per slot
constexpr int kRing = 4, kRingSlot = 768;
static_assert((kThreads / 32) * kRing * kRingSlot <= 4 * kImg, "ring exceeds the Z lo image's region");
constexpr int kQuadWarps = kThreads / 128, kSpan = 128 / kQuadWarps, kRedCols = 32 / kQuadWarps;
static_assert(kSpan == 32 && kRedCols == 8, "column split below assumes 16 warps");

// X / Z slot element (item, a, b, c); the XOR keeps both the (c, b)-lane
// dump and the c-lane reads free of bank conflicts
__device__ __forceinline__ int xs_idx(int it, int a, int b, int c) { return it * 512 + (4 * a + b) * 32 + (c ^ (b << 3)); }

// chunks of whole items with <= cap positions each (thread 0)
__device__ inline void make_chunks(const TileMeta* m, int* ch, int cap, int round = kThreads / 32) {
  int nc = 0, it = 0;
  const int n = m->n;
  ch[0] = 0;
  if (m->start[n] - m->start[0] <= cap) {  // the common case: one chunk
    ch[1] = n;
    ch[kTileItems + 1] = 1;
    return;
  }
  while (it < n) {
    const int first = it, base = m->start[it];
    while (it < n && m->start[it + 1] - base <= cap) ++it;
    // whole rounds of one item per warp where possible (items have similar
    // lengths inside a tile, so the warps finish a chunk together)
    if (it < n && it - first > round) it = first + (it - first) / round * round;
    ch[++nc] = it;
  }
  ch[kTileItems + 1] = nc;
}


// one gradient row g (16 float4, (a, b) major) against the item's X^T column
// x[(a, b)] (lane c): dH[c, :] = sum_ab x[ab] g[ab, :] and Z[ab, c] += g[ab, :] . h3
__device__ __forceinline__ void lookup_update(const float4* src, const float (&x)[16], float (&z)[16], float4 h3,
                                              float (&dh)[4]) {
#pragma unroll
  for (int ab = 0; ab < 16; ++ab) {
    const float4 v = src[ab];
    dh[0] = fmaf(x[ab], v.x, dh[0]);
    dh[1] = fmaf(x[ab], v.y, dh[1]);
    dh[2] = fmaf(x[ab], v.z, dh[2]);
    dh[3] = fmaf(x[ab], v.w, dh[3]);
    z[ab] = fmaf(v.x, h3.x, z[ab]);
    z[ab] = fmaf(v.y, h3.y, z[ab]);
    z[ab] = fmaf(v.z, h3.z, z[ab]);
    z[ab] = fmaf(v.w, h3.w, z[ab]);
  }
}

// Warp roles: warps 0-15 (kThreads) do the SIMT work and synchronise among
// themselves with named barrier 1; warp 16 issues every tcgen05.mma of the
// CTA (X, dG2, E) when the SIMT warps signal that its operands are ready, so
// no SIMT warp blocks in a long MMA issue and the next tile's X GEMM runs
// under the current tile's dG1 / dG2 reductions.
constexpr int kBwdThreads = kThreads + 32;
__device__ __forceinline__ void simt_sync() { named_sync(1, kThreads); }
__device__ __forceinline__ void simt_sync_for_mma() {
  umma::fence_smem_to_async();
  umma::fence_before_sync();
  simt_sync();
  umma::fence_after_sync();
}

template <bool kRows>
__global__ void __launch_bounds__(kBwdThreads, 1) k_bwd(KGeom g, const float* __restrict__ g1img,
                                                        const float* __restrict__ g3t, const float* __restrict__ img,
                                                        const int4* __restrict__ tile_info,
                                                        const int* __restrict__ item_start,
                                                        const unsigned* __restrict__ item_key,
                                                        const int2* __restrict__ sbi, const float* __restrict__ gout,
                                                        float* __restrict__ dG1, float* __restrict__ dG2,
                                                        float* __restrict__ dG3, int* __restrict__ hdr,
                                                        const int* __restrict__ cta_tiles, int dbg) {
  pdl_enter();
  extern __shared__ __align__(16) char smem_raw[];
  char* sm = smem_raw + ((1024u - (umma::smem_u32(smem_raw) & 1023u)) & 1023u);
  char* r1_hi = sm;  // X: G2 cb hi / lo; later the 64-row G2 k image
  char* r1_lo = sm + kImg;
  char* r2_hi = sm + 2 * kImg;  // X: G1 rows hi / lo; later the 64-row G1^T image
  char* r2_lo = sm + 3 * kImg;
  char* zi = sm + 4 * kImg;  // X / Z slots, then the Z image
  float* xs = reinterpret_cast<float*>(zi);
  // staged per chunk: the (bag, i3) list and, one lookup per bag, the
  // gradient rows and G3 slices. The row path stages the whole tile's list
  // only: a row's gradient rows are summed straight from L2 (after the plan's
  // row sort an item holds one or two rows, so few sums per item)
  constexpr int kCap = kRows ? kMaxTilePos : kChunkPos;  // positions per staged chunk
  int2* st_sbi = reinterpret_cast<int2*>(sm + 8 * kImg);
  float4* st_g = reinterpret_cast<float4*>(sm + 8 * kImg + kCap * 8);
  float4* st_g3 = st_g + kCap * 16;  // per-position G3 slices (bag-run path only)
  float4* st_acc = st_g;             // row path: per-warp summed gradient row (16 x 256 B)
  // Z lo image: the dead staging past the next tile's (bag, i3) list (bag-run
  // path: exactly the G3-slice staging, so the next tile's gradient rows can
  // stream in while the E GEMM runs; row path: past the row scratch)
  char* zlo = sm + 8 * kImg + (kRows ? kMaxTilePos * 8 + 4096 : kChunkPos * 8 + kChunkPos * 256);
  __shared__ TileMeta s_m[2];
  __shared__ int s_chunk[2][kTileItems + 2];
  // SIMT -> MMA warp: G1 rows staged / Z^T in TMEM + G1^T staged / Z images
  // written; MMA warp -> SIMT: X done / dG2 + E done; bulk copies of the G2
  // cb / k images (issued and waited for by the MMA warp)
  __shared__ uint64_t s_mb_xop, s_mb_z, s_mb_zi, s_mb_x, s_mb_d2, s_mb_e, s_mb_xtma, s_mb_ktma;
  __shared__ int s_acc2;
  // row path: the Z phase's next item of the tile in each slot (warps take
  // items dynamically: an item's cost follows its distinct rows, not its length)
  __shared__ int s_itc[2];
  // tile of each metadata slot (-1: none). Pooled batches take tiles from a
  // global counter (hdr[kHdrNextTile]): after the row sort, a tile's cost no
  // longer follows its lookup count, so the plan's static ranges would leave
  // CTAs idle; one lookup per bag keeps the static, i2-contiguous ranges
  __shared__ int s_tile[2];
  __shared__ long long s_tacc[12];
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tb = cta_tiles[blockIdx.x], te = cta_tiles[blockIdx.x + 1];  // weight-balanced (k_fplan)
  if (threadIdx.x < 12) s_tacc[threadIdx.x] = 0;
  if (threadIdx.x < 2) s_itc[threadIdx.x] = 0;
  if (warp == 0) umma::tmem_alloc(&s_tmem, 512);
  if (threadIdx.x == 32) {
    umma::mbar_init(&s_mb_xop, 1);
    umma::mbar_init(&s_mb_z, 1);
    umma::mbar_init(&s_mb_xtma, 1);
    umma::mbar_init(&s_mb_ktma, 1);
    umma::mbar_init(&s_mb_zi, 1);
    umma::mbar_init(&s_mb_x, 1);
    umma::mbar_init(&s_mb_d2, 1);
    umma::mbar_init(&s_mb_e, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int ntiles = hdr[4];
  // the tile after `t` (this CTA's next): -1 when there is none
  auto next_tile = [&](int t) -> int {
    if (kRows) {
      const int u = atomicAdd(&hdr[kHdrNextTile], 1);
      return u < ntiles ? u : -1;
    }
    return t + 1 < te ? t + 1 : -1;
  };
  if (warp == kThreads / 32 - 1) {
    int t0 = 0;
    if (lane == 0) t0 = kRows ? next_tile(-1) : (tb < te ? tb : -1);
    t0 = __shfl_sync(0xffffffffu, t0, 0);
    if (lane == 0) s_tile[0] = t0;
    if (t0 >= 0) fetch_meta_async(tile_info[t0], item_start, item_key, &s_m[0]);
  }
  cp_async_wait_all();
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = s_tmem;
  // smem descriptors (start addresses are fixed for the kernel)
  const uint64_t d_r1h = umma::desc_sw128(umma::smem_u32(r1_hi)), d_r1l = umma::desc_sw128(umma::smem_u32(r1_lo));
  const uint64_t d_r2h = umma::desc_sw128(umma::smem_u32(r2_hi)), d_r2l = umma::desc_sw128(umma::smem_u32(r2_lo));
  const uint64_t d_zi = umma::desc_sw128(umma::smem_u32(zi)), d_zl = umma::desc_sw128(umma::smem_u32(zlo));

  if (warp == kThreads / 32) {
    // ---------------- MMA warp: also the bulk-copy producer of the G2 images
    // (one 32 KB copy each: the cb image (hi, lo) for X, the k image for E)
    auto load_cb = [&](const TileMeta* mt) {
      if (lane == 0) {
        umma::mbar_expect_tx(&s_mb_xtma, 2 * kImg);
        umma::bulk_g2s(r1_hi, img + (size_t)mt->i2 * kImg, 2 * kImg, &s_mb_xtma);
      }
      __syncwarp();
    };
    uint32_t ph = 0;
    if (s_tile[0] >= 0) load_cb(&s_m[0]);
    for (int k = 0; s_tile[k & 1] >= 0; ++k, ph ^= 1u) {
      const TileMeta* mt = &s_m[k & 1];
      umma::mbar_wait(&s_mb_xtma, ph);  // the G2 cb image of tile t
      umma::mbar_wait(&s_mb_xop, ph);   // its items' G1 rows (SIMT cp.async)
      umma::fence_after_sync();
      if (lane == 0) {
        constexpr uint32_t id = umma::idesc_tf32(128, 128, false, false);
#pragma unroll
        for (int k0 = 0; k0 < R1; k0 += 8) {
          const uint32_t o = (uint32_t)((k0 & 31) * 4) >> 4;
          umma::mma_tf32(tmem, d_r1h + o, d_r2h + o, id, k0 > 0 ? 1u : 0u);
          umma::mma_tf32(tmem, d_r1h + o, d_r2l + o, id, 1u);
          umma::mma_tf32(tmem, d_r1l + o, d_r2h + o, id, 1u);
        }
        umma::commit(&s_mb_x);
      }
      __syncwarp();
      umma::mbar_wait(&s_mb_x, ph);  // X read its operands: the G2 k image replaces the cb image
      if (lane == 0) {
        umma::mbar_expect_tx(&s_mb_ktma, 2 * kImg);
        umma::bulk_g2s(r1_hi, img + (size_t)mt->i2 * kImg + 2 * kImg / 4, 2 * kImg, &s_mb_ktma);
      }
      __syncwarp();
      umma::mbar_wait(&s_mb_z, ph);  // Z^T hi / lo in TMEM, G1^T image in R12
      umma::mbar_wait(&s_mb_ktma, ph);
      umma::fence_after_sync();
      if (lane == 0) {
        constexpr uint32_t id64 = umma::idesc_tf32(128, 64, false, false);
        constexpr uint32_t id32 = umma::idesc_tf32(128, 32, false, false);  // B rows 0-31: the hi half
        const bool acc2 = s_acc2 != 0;  // same i2 as the previous tile: keep accumulating dG2 in TMEM
        // dG2 tile [(c, b), (hi | lo) k] = sum_(item, a) (Z^T hi + Z^T lo) . G1^T (A from TMEM)
#pragma unroll
        for (int k0 = 0; k0 < 128; k0 += 8) {
          const uint32_t o = (uint32_t)((k0 >> 5) * 64 * 128 + (k0 & 31) * 4) >> 4;
          umma::mma_tf32_ta(tmem + 384, tmem + 128 + k0, d_r2h + o, id64, (acc2 || k0 > 0) ? 1u : 0u);
          umma::mma_tf32_ta(tmem + 384, tmem + 256 + k0, d_r2h + o, id32, 1u);  // Z lo . G1 hi only
        }
        umma::commit(&s_mb_d2);  // -> SIMT: the G1^T image is free for the next tile's G1 rows
      }
      __syncwarp();
      umma::mbar_wait(&s_mb_zi, ph);  // Z images (hi, lo) in shared memory
      umma::fence_after_sync();
      if (lane == 0) {
        constexpr uint32_t id64 = umma::idesc_tf32(128, 64, false, false);
        constexpr uint32_t id32 = umma::idesc_tf32(128, 32, false, false);
        // E tile [(item, a), (hi | lo) k] = sum_(c, b) (Z hi . G2^T + Z lo . G2 hi^T)
#pragma unroll
        for (int k0 = 0; k0 < 128; k0 += 8) {
          const uint32_t oa = (uint32_t)((k0 >> 5) * 128 * 128 + (k0 & 31) * 4) >> 4;
          const uint32_t ob = (uint32_t)((k0 >> 5) * 64 * 128 + (k0 & 31) * 4) >> 4;
          umma::mma_tf32(tmem + 448, d_zi + oa, d_r1h + ob, id64, k0 > 0 ? 1u : 0u);
        }
#pragma unroll
        for (int k0 = 0; k0 < 128; k0 += 8) {
          const uint32_t oa = (uint32_t)((k0 >> 5) * 128 * 128 + (k0 & 31) * 4) >> 4;
          const uint32_t ob = (uint32_t)((k0 >> 5) * 64 * 128 + (k0 & 31) * 4) >> 4;
          umma::mma_tf32(tmem + 448, d_zl + oa, d_r1h + ob, id32, 1u);  // Z lo . G2 hi only
        }
        umma::commit(&s_mb_e);  // tracks the dG2 MMAs too
      }
      __syncwarp();
      if (s_tile[(k + 1) & 1] >= 0) {  // R12 free once E is done: the next tile's cb image
        umma::mbar_wait(&s_mb_e, ph);
        load_cb(&s_m[(k + 1) & 1]);  // (its slot and metadata: visible since the Z signal)
      } else {
        break;
      }
    }
  } else {
  // ---------------- SIMT warps
  // a chunk's per-position rows (cp.async): the bag's gradient row and, one
  // lookup per bag, the lookup's slice-major G3 slice (512 contiguous bytes)
  auto stage_rows = [&](int np, unsigned i3base) {
    if (kRows) return;  // (row path: gradient rows read from L2 when summed)
    for (int e = threadIdx.x; e < np * 16; e += kThreads)
      cp_async16(st_g + e, gout + (size_t)st_sbi[e >> 4].x * NOUT + 4 * (e & 15));
    if (!kRows)
      for (int e = threadIdx.x; e < np * 32; e += kThreads)
        cp_async16(st_g3 + e, g3t + (size_t)(i3base + st_sbi[e >> 5].y) * 128 + 4 * (e & 31));
  };
  // the items' pre-swizzled G1 rows (hi, lo): 512 contiguous bytes per item
  auto stage_g1_rows = [&](const TileMeta* mt) {
#pragma unroll
    for (int i = 0; i < 1024 / kThreads; ++i) {
      const int e = threadIdx.x + i * kThreads, it = e >> 5, q = e & 31;
      if (it < mt->n) {
        const float* src = g1img + (size_t)item_i1(mt, it, g) * kG1Img + g1_rows_off(it & 1) + 4 * q;
        cp_async16(r2_hi + 512 * it + 16 * q, src);
        cp_async16(r2_lo + 512 * it + 16 * q, src + 128);
      }
    }
  };
  const int q4 = warp & 3, qw = warp >> 2;  // lane quadrant, and this warp's share of its columns
  const int row = 32 * q4 + lane;  // TMEM lane of this thread: (c, b) = (row / 4, row % 4)
  const int c = row >> 2, b = row & 3;
  const uint32_t tl = tmem + ((uint32_t)(32 * q4) << 16);
  // prologue: the first tile's first chunk and X operands
  if (s_tile[0] >= 0) {
    const TileMeta* m = &s_m[0];
    if (threadIdx.x == 0) make_chunks(m, s_chunk[0], kCap);
    simt_sync();
    const int np = m->start[s_chunk[0][1]] - m->start[0];
    for (int e = threadIdx.x; e < np; e += kThreads) cp_async8(st_sbi + e, sbi + m->start[0] + e);
    stage_g1_rows(m);
    cp_async_wait_all();
    simt_sync_for_mma();
    if (threadIdx.x == 0) umma::mbar_arrive(&s_mb_xop);  // X of the first tile
    stage_rows(np, tile_i3_base(m, g));
  }
  uint32_t phase = 0;
  bool bad = false;
  int slot = 0;
  int prev_i2 = -1;
  int ntile_done = 0;
  for (; s_tile[slot] >= 0; slot ^= 1, phase ^= 1u, ++ntile_done) {
    const int t = s_tile[slot];
    const TileMeta* m = &s_m[slot];
    const int* chunk = s_chunk[slot];
    const int n = m->n, nchunk = chunk[kTileItems + 1];
    const unsigned i3b = tile_i3_base(m, g);          // the tile's table's G3 slices (batched handles)
    TSTAMP(0);
    TSTAMP(1);
    umma::mbar_wait(&s_mb_x, phase);  // X of tile t (its operands in R12 are free again)
    umma::fence_after_sync();
    TSTAMP(2);
    // X^T -> item slots (this warp's 32 columns)
    {
      uint32_t v0[kSpan];
      umma::tmem_ld32_nw(tl + kSpan * qw, v0);
      umma::tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < kSpan; ++i) {
        const int col = kSpan * qw + i;
        xs[xs_idx(col >> 2, col & 3, b, c)] = __uint_as_float(v0[i]);
      }
    }
    cp_async_wait_all();  // chunk 0's gradient rows and G3 slices (staged by the previous tile)
    // the dG2 GEMM's G1^T image streams in during the Z phase (the MMA warp
    // loads the G2 k image)
    stage_g1_t_async(m, g, g1img, r2_hi);
    cp_async_commit();
    umma::fence_before_sync();
    simt_sync();  // (every warp is past the previous tile: its metadata slot is free)
    if (warp == kThreads / 32 - 1) {  // next tile and its metadata into the other slot
      int tn = 0;
      if (lane == 0) tn = next_tile(t);
      tn = __shfl_sync(0xffffffffu, tn, 0);
      if (lane == 0) s_tile[slot ^ 1] = tn;  // (read by everyone after the Z^T barrier)
      if (tn >= 0) fetch_meta_async(tile_info[tn], item_start, item_key, &s_m[slot ^ 1]);  // (waited for before make_chunks)
    }
    TSTAMP(3);
    for (int ch = 0; ch < nchunk; ++ch) {
      const int it0 = chunk[ch], it1 = chunk[ch + 1];
      const int p0 = m->start[it0];
      if (ch > 0) {
        const long long _c0 = clock64();
        const int np = m->start[it1] - p0;
        for (int e = threadIdx.x; e < np; e += kThreads) cp_async8(st_sbi + e, sbi + p0 + e);
        cp_async_wait_all();
        simt_sync();
        stage_rows(np, i3b);
        cp_async_wait_all();
        simt_sync();
        if ((dbg & 8) && threadIdx.x == 0 && blockIdx.x == 0) s_tacc[10] += clock64() - _c0;
      }
      // ---- Z / dG3 phase: warp <-> item, lane <-> c
      auto take_item = [&](int prev) -> int {
        if (!kRows) return prev < 0 ? it0 + warp : prev + kThreads / 32;
        int v = 0;
        if (lane == 0) v = atomicAdd(&s_itc[slot], 1);
        return it0 + __shfl_sync(0xffffffffu, v, 0);
      };
      for (int it = take_item(-1); it < it1; it = take_item(it)) {
        float x[16], z[16];
#pragma unroll
        for (int ab = 0; ab < 16; ++ab) {
          x[ab] = xs[xs_idx(it, ab >> 2, ab & 3, lane)];
          z[ab] = 0.f;
        }
        if (kRows) {
          // the item's (<= kItemLen) positions, one per lane, grouped by row
          // (equal i3): a row's gradient rows are summed first, so dG3 gets one
          // reduction and Z one rank-4 update per distinct row of the item
          const int s0 = m->start[it] - p0, nq = m->start[it + 1] - p0 - s0;
          const int my_i3 = lane < nq ? (int)i3b + st_sbi[s0 + lane].y : -1;
          const int my_bag = lane < nq ? st_sbi[s0 + lane].x : 0;
          const unsigned grp = __match_any_sync(0xffffffffu, lane < nq ? my_i3 : (int)(0x80000000u | lane));
          unsigned lead = __ballot_sync(0xffffffffu, lane < nq && (__ffs(grp) - 1) == lane);
          // rows stream through this warp's ring of kRing slots (cp.async):
          // the G3 slice of every row and the gradient row of a one-lookup
          // row land kRing - 1 rows ahead of their use, so a warp keeps
          // several rows' L2 / HBM reads in flight instead of one
          char* ring = zlo + warp * (kRing * kRingSlot);
          unsigned lead_iss = lead;
          auto issue = [&](int sl) {
            if (lead_iss) {
              const int ld = __ffs(lead_iss) - 1;
              lead_iss &= lead_iss - 1;
              const unsigned mem = __shfl_sync(0xffffffffu, grp, ld);
              const int i3 = __shfl_sync(0xffffffffu, my_i3, ld);
              const int bg = __shfl_sync(0xffffffffu, my_bag, ld);
              char* d = ring + sl * kRingSlot;
              cp_async16(d + 256 + 16 * lane, g3t + ((size_t)i3 * 32 + lane) * 4);
              if ((mem & (mem - 1)) == 0 && lane < 16) cp_async16(d + 16 * lane, gout + (size_t)bg * NOUT + 4 * lane);
            }
            cp_async_commit();
          };
#pragma unroll
          for (int j = 0; j < kRing - 1; ++j) issue(j);
          int sl = 0;
          while (lead) {
            issue(sl == 0 ? kRing - 1 : sl - 1);
            cp_async_wait_group<kRing - 1>();
            __syncwarp();
            const int ld = __ffs(lead) - 1;
            lead &= lead - 1;
            unsigned mem = __shfl_sync(0xffffffffu, grp, ld);
            const int i3 = __shfl_sync(0xffffffffu, my_i3, ld);
            const char* d = ring + sl * kRingSlot;
            sl = sl == kRing - 1 ? 0 : sl + 1;
            const float4 h3 = reinterpret_cast<const float4*>(d + 256)[lane];
            const float4* src = reinterpret_cast<const float4*>(d);
            // a row of several lookups: its lookups' bag rows summed from L2
            // (two floats per lane per member, eight members in flight) into
            // the warp's scratch, then broadcast reads
            if (mem & (mem - 1)) {
              // the member lanes publish their bags in the warp's scratch (by
              // rank), so the eight loads of a batch issue without a chain of
              // shuffles
              int* mb = reinterpret_cast<int*>(st_acc + warp * 16);
              if ((mem >> lane) & 1u) mb[__popc(mem & lanemask_lt())] = my_bag;
              __syncwarp();
              const int nm = __popc(mem);
              float2 acc = make_float2(0.f, 0.f);
              for (int q0 = 0; q0 < nm; q0 += 8) {
                float2 w[8];
#pragma unroll
                for (int q = 0; q < 8; ++q)
                  w[q] = q0 + q < nm ? __ldg(reinterpret_cast<const float2*>(gout + (size_t)mb[q0 + q] * NOUT) + lane)
                                     : make_float2(0.f, 0.f);
                acc.x += ((w[0].x + w[1].x) + (w[2].x + w[3].x)) + ((w[4].x + w[5].x) + (w[6].x + w[7].x));
                acc.y += ((w[0].y + w[1].y) + (w[2].y + w[3].y)) + ((w[4].y + w[5].y) + (w[6].y + w[7].y));
              }
              __syncwarp();  // every bag read before the sum overwrites the scratch
              reinterpret_cast<float2*>(st_acc + warp * 16)[lane] = acc;
              __syncwarp();
              src = st_acc + warp * 16;
            }
            float dh[4] = {0.f, 0.f, 0.f, 0.f};
            lookup_update(src, x, z, h3, dh);
            __syncwarp();  // the scratch and the slot are rewritten by later rows
            if (!(dbg & 1)) red_v4(dG3 + ((size_t)i3 * 32 + lane) * 4, dh[0], dh[1], dh[2], dh[3]);
            bad |= suspicious(dh[0]) | suspicious(dh[1]) | suspicious(dh[2]) | suspicious(dh[3]);
          }
        } else {
          // one lookup per bag (T = B): every position is its own bag, so a
          // position is one gradient row, one dG3 reduction and one Z update
          const int s1 = (dbg & 64) ? 0 : m->start[it + 1] - p0;  // (ablations: TTB_DBG 64 / 32)
          for (int qq = m->start[it] - p0; qq < s1; ++qq) {
            const unsigned i3 = i3b + st_sbi[qq].y;
            const float4 h3 = st_g3[qq * 32 + lane];
            float dh[4] = {0.f, 0.f, 0.f, 0.f};
            if (!(dbg & 32)) lookup_update(st_g + qq * 16, x, z, h3, dh);
            if (!(dbg & 1)) red_v4(dG3 + ((size_t)i3 * 32 + lane) * 4, dh[0], dh[1], dh[2], dh[3]);
            bad |= suspicious(dh[0]) | suspicious(dh[1]) | suspicious(dh[2]) | suspicious(dh[3]);
          }
        }
#pragma unroll
        for (int ab = 0; ab < 16; ++ab) xs[xs_idx(it, ab >> 2, ab & 3, lane)] = z[ab];
      }
      if (ch == nchunk - 1) {  // slots past the tile's items hold zeros
        for (int it = n + warp; it < kTileItems; it += kThreads / 32)
#pragma unroll
          for (int ab = 0; ab < 16; ++ab) xs[xs_idx(it, ab >> 2, ab & 3, lane)] = 0.f;
      }
      if (ch == nchunk - 1) cp_async_wait_all();  // the G1^T image's copies (replicated after the barrier)
      {
        const long long _c0 = clock64();
        simt_sync();  // staging reused by the next chunk / tile
        if ((dbg & 8) && threadIdx.x == 0 && blockIdx.x == 0) s_tacc[11] += clock64() - _c0;
      }
    }
    TSTAMP(4);
    const bool has_next = s_tile[slot ^ 1] >= 0;  // (written before the Z phase's barriers)
    const TileMeta* mn = &s_m[slot ^ 1];
    int npn = 0;
    // ---- Z^T into TMEM (hi / lo) and the Z image (hi) for the E GEMM
    // (one split serves both: Z^T hi / lo to TMEM now, the Z images after the barrier)
    float zh[kSpan], zl[kSpan];
#pragma unroll
    for (int i = 0; i < kSpan; ++i) {
      const int ia = kSpan * qw + i;
      umma::split2(xs[xs_idx(ia >> 2, ia & 3, b, c)], zh[i], zl[i]);
    }
    umma::tmem_st32(tl + 128 + kSpan * qw, zh);
    umma::tmem_st32(tl + 256 + kSpan * qw, zl);
    g1_t_replicate(m, r2_hi);
    umma::tmem_wait_st();
    cp_async_wait_all();  // G1^T image (issued before the Z phase), next tile's metadata (warp 15)
    if (threadIdx.x == 0) {
      s_acc2 = m->i2 == prev_i2;
      s_itc[slot] = 0;  // (every warp is past this tile's Z phase; the slot's next tile is two away)
    }
    if (warp == kThreads / 32 - 1 && has_next) {  // the next tile's chunk list, from the metadata this warp fetched
      __syncwarp();
      if (lane == 0) make_chunks(mn, s_chunk[slot ^ 1], kCap);
    }
    simt_sync_for_mma();  // every slot read before the image overwrites them; Z^T is in TMEM
    if (threadIdx.x == 0) umma::mbar_arrive(&s_mb_z);  // -> dG2 MMAs
    // ---- next tile: first chunk's positions
    if (has_next) {
      npn = mn->start[s_chunk[slot ^ 1][1]] - mn->start[0];
      for (int e = threadIdx.x; e < npn; e += kThreads) cp_async8(st_sbi + e, sbi + mn->start[0] + e);
      cp_async_commit();
    }
    // Z image hi (the slots' region) and lo (the dead staging rows) for the E GEMM
#pragma unroll
    for (int i = 0; i < kSpan; ++i) {
      const uint32_t o = umma::sw128_off(kSpan * qw + i, row, 128);
      *(float*)(zi + o) = zh[i];
      *(float*)(zlo + o) = zl[i];
    }
    cp_async_wait_all();  // next tile's positions
    simt_sync_for_mma();
    if (threadIdx.x == 0) umma::mbar_arrive(&s_mb_zi);  // -> E MMAs
    TSTAMP(5);
    if (!kRows && has_next) {  // one lookup per bag: the gradient rows' region is not the Z lo image's
      for (int e = threadIdx.x; e < npn * 16; e += kThreads)
        cp_async16(st_g + e, gout + (size_t)st_sbi[e >> 4].x * NOUT + 4 * (e & 15));
      cp_async_commit();
    }
    // the next tile's G1 rows as soon as dG2 has read the G1^T image (R2),
    // the rest of its first chunk once E has read the Z lo image
    umma::mbar_wait(&s_mb_d2, phase);
    umma::fence_after_sync();
    if (has_next) {
      stage_g1_rows(mn);
      cp_async_commit();
    }
    umma::mbar_wait(&s_mb_e, phase);  // E of tile t
    umma::fence_after_sync();
    TSTAMP(6);
    if (has_next) {
      if (kRows) {
        stage_rows(npn, tile_i3_base(mn, g));
      } else {
        const unsigned i3n = tile_i3_base(mn, g);
        for (int e = threadIdx.x; e < npn * 32; e += kThreads)
          cp_async16(st_g3 + e, g3t + (size_t)(i3n + st_sbi[e >> 5].y) * 128 + 4 * (e & 31));
      }
      cp_async_commit();
    }
    TSTAMP(7);
    // the next X GEMM is released before this tile's dG2 / dG1 reductions: the
    // proxy fence of the release would otherwise wait for them to drain (the
    // dG2 / E columns are rewritten only after the next tile's Z phase)
    if (has_next) {  // the next G1 rows landed: with the cb image, the MMA warp starts the next X GEMM
      asm volatile("cp.async.wait_group 1;" ::: "memory");
      simt_sync_for_mma();
      if (threadIdx.x == 0) umma::mbar_arrive(&s_mb_xop);
    }
    if (!(dbg & 4)) {
      float v[kRedCols], w2[kRedCols];
      // dG2[k][i2][b][c] = D[:, k] + D[:, 32 + k], once per run of tiles of one i2
      if (!has_next || mn->i2 != m->i2) {
        umma::tmem_ld8(tl + 384 + kRedCols * qw, v);
        umma::tmem_ld8(tl + 384 + 32 + kRedCols * qw, w2);
        float* d2 = dG2 + ((size_t)m->i2 * 4 + b) * 32 + c;
        const size_t ks = (size_t)g.m2 * C;
#pragma unroll
        for (int i = 0; i < kRedCols; ++i) {
          bad |= suspicious(v[i] + w2[i]);
          red_f32(d2 + (size_t)(kRedCols * qw + i) * ks, v[i] + w2[i]);
        }
      }
      // dG1[i1][a][k]
      umma::tmem_ld8(tl + 448 + kRedCols * qw, v);
      umma::tmem_ld8(tl + 448 + 32 + kRedCols * qw, w2);
      const int it = row >> 2, a = row & 3;
      // a key's full items are contiguous in its tile (and one i2 per tile
      // makes equal i1 mean equal key): each run of equal i1 is summed inside
      // the warp (8 items, segmented suffix sums over item offsets 1, 2, 4)
      // and its first item reduces it, so a hot key's dG1 rows get one
      // reduction per warp instead of one per item (all CTAs of a hot key hit
      // the same 512 B)
      const unsigned i1v = it < n ? item_i1(m, it, g) : 0xFFFFFFFFu;
      const unsigned prev_i1 = __shfl_up_sync(0xffffffffu, i1v, 4);  // (every lane: full-mask shuffles)
      const bool head = lane < 4 || prev_i1 != i1v;
#pragma unroll
      for (int i = 0; i < kRedCols; ++i) v[i] += w2[i];
      if (__any_sync(0xffffffffu, !head && it < n)) {  // (warp-uniform; distinct keys only: no sums)
        int rs = head ? lane >> 2 : -1;  // first item of this item's run (a key may also recur later in the tile)
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, rs, o);
          if (lane >= o) rs = max(rs, t);
        }
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          const int nrs = __shfl_down_sync(0xffffffffu, rs, o);
          const bool take = nrs == rs && lane + o < 32;
#pragma unroll
          for (int i = 0; i < kRedCols; ++i) {
            const float t = __shfl_down_sync(0xffffffffu, v[i], o);
            if (take) v[i] += t;
          }
        }
      }
      if (it < n && head) {
        float* d1 = dG1 + ((size_t)i1v * 4 + a) * R1 + kRedCols * qw;
#pragma unroll
        for (int i = 0; i < kRedCols; i += 4) {
          bad |= suspicious(v[i]) | suspicious(v[i + 1]) | suspicious(v[i + 2]) | suspicious(v[i + 3]);
          red_v4(d1 + i, v[i], v[i + 1], v[i + 2], v[i + 3]);
        }
      }
    }
    TSTAMP(8);
    prev_i2 = m->i2;
    // TMEM reads done before the next dG2 / E MMAs (issued after the next
    // tile's barriers); slots free for the next dump (the E GEMM is done)
    umma::fence_before_sync();
  }
  if (bad) hdr[kHdrSuspect] = 1;
  if ((dbg & 8) && threadIdx.x == 0 && blockIdx.x == 0) {
    s_tacc[0] = ntile_done;
    for (int q = 0; q < 12; ++q) reinterpret_cast<long long*>(hdr + 16)[q] = s_tacc[q];
  }
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  if (warp == 0) umma::tmem_free(tmem, 512);
}



}  // namespace fast

using namespace fast;

// ------------------------------------------------------------ counters S, U
// The reference's counters (lookup.py:294-295 segments S = bag-prefix pairs;
// backward.py:218-222 distinct rows U) for the current plan, on demand (the
// step kernels never need them). U: test-and-set of one bit per row. S: per
// bag (one warp), the number of distinct prefix keys among its lookups.
template <typename IdxT>
__global__ void __launch_bounds__(256) k_count_su(const IdxT* __restrict__ idx, const int64_t* __restrict__ offsets,
                                                  int T, int B, KGeom g, unsigned* __restrict__ rowbits,
                                                  int* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  int u = 0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
    long long v = (long long)idx[t];
    if (v < 0 || v >= (long long)g.rows) continue;
    const unsigned bit = 1u << (v & 31);
    u += (atomicOr(&rowbits[v >> 5], bit) & bit) == 0;
  }
  int sseg = 0;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int b = warp; b < B; b += nwarps) {
    const int lo = (int)offsets[b], hi = (int)offsets[b + 1];
    for (int p0 = lo; p0 < hi; p0 += 32) {
      const int p = p0 + lane;
      const bool ok = p < hi;
      const unsigned key = ok ? (unsigned)((unsigned long long)idx[p] / g.m3) : 0xFFFFFFFFu;
      // first occurrence inside this chunk of 32 ...
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      bool first = ok && (__ffs(peers) - 1) == lane;
      // ... and not seen in an earlier chunk of the bag
      for (int q = lo; first && q < p0; ++q) first = (unsigned)((unsigned long long)idx[q] / g.m3) != key;
      sseg += first;
    }
  }
  u = warp_sum(u);
  sseg = warp_sum(sseg);
  if (lane == 0) {
    if (u) atomicAdd(&counts[1], u);
    if (sseg) atomicAdd(&counts[0], sseg);
  }
}

cudaError_t fast_count_su(ttb_handle* h, const void* idx, int idx64, const int64_t* offsets, int64_t su[2],
                          cudaStream_t s) {
  Workspace& w = h->w;
  cudaError_t e;
  if ((e = cudaMemsetAsync(w.f_rowbits, 0, sizeof(unsigned) * ((size_t)h->kg.rows / 32 + 1), s))) return e;
  if ((e = cudaMemsetAsync(w.fast_hdr + 8, 0, 2 * sizeof(int), s))) return e;
  const int grid = 4 * h->num_sms;
  if (idx64)
    k_count_su<long long><<<grid, 256, 0, s>>>((const long long*)idx, offsets, (int)h->T, (int)h->B, h->kg,
                                               w.f_rowbits, w.fast_hdr + 8);
  else
    k_count_su<int><<<grid, 256, 0, s>>>((const int*)idx, offsets, (int)h->T, (int)h->B, h->kg, w.f_rowbits,
                                         w.fast_hdr + 8);
  count_launch();
  if ((e = cudaGetLastError())) return e;
  int c[2];
  if ((e = cudaMemcpyAsync(c, w.fast_hdr + 8, sizeof(c), cudaMemcpyDeviceToHost, s))) return e;
  if ((e = cudaStreamSynchronize(s))) return e;
  su[0] = c[0];
  su[1] = c[1];
  return cudaSuccess;
}

cudaError_t launch_gradcheck(const float* g, int64_t n, int* err, int num_sms, cudaStream_t s, const int* suspect) {
  if (n <= 0) return cudaSuccess;
  int64_t gb = (n / 4 + 255) / 256;
  if (gb < 1) gb = 1;
  if (gb > 2 * num_sms) gb = 2 * num_sms;
  cudaError_t e = launch_pdl(k_gradcheck, dim3((int)gb), dim3(256), 0, s, g, n, err, suspect);
  if (e == cudaSuccess) count_launch();
  return e;
}

bool fast_supported(const ttb_handle* h) {
  const DynDims& d = h->dims;
  // G3 (32 x m3 x 4 fp32) stays resident in the forward kernel's shared memory
  return d.n1 == 4 && d.n2 == 4 && d.n3 == 4 && d.r1 == 32 && d.r2 == 32 && h->kg.tm3 <= (unsigned)kFwdMaxM3;
}

cudaError_t fast_plan(ttb_handle* h, const void* idx, int idx64, const int64_t* offsets, cudaStream_t s) {
  Workspace& w = h->w;
  const int T = (int)h->T, B = (int)h->B;
  cudaError_t e;
  // (no memset: k_fplan clears its header words itself; the other pipeline's
  // backward clears its zero block B when it runs)
  h->bwd_zeroed = 0;
  int work = T > B ? T : B;
  if ((int)h->kg.m1m2 > work) work = (int)h->kg.m1m2;
  int grid = (work + kPlanThreads - 1) / kPlanThreads;
  if (grid > h->num_sms) grid = h->num_sms;  // co-resident: grid barriers
  const bool many = T > 2 * grid * kPlanThreads;  // (the kernel's own test, T > 2 nthr)
  {
    // the grid barriers need every CTA resident at once: bound the grid by
    // the occupancy of this device and launch cooperatively (an SM partition
    // too small for the grid then fails the launch instead of hanging)
    int occ = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
             &occ, idx64 ? (const void*)k_fplan<long long, true> : (const void*)k_fplan<int, true>, kPlanThreads, 0)))
      return e;
    if (occ < 1) return cudaErrorCooperativeLaunchTooLarge;
  }
  // |G1| + |G2| + |G3| gradients (multiples of 4: every core has n = 4)
  const int64_t ngrad4 = ((int64_t)h->kg.g1rows * 4 * R1 + (int64_t)R1 * h->kg.m2 * C + (int64_t)32 * h->kg.m3 * 4) / 4;
  {
  ProfScope _ps(h, s, "f_plan");
  if (idx64)
    e = launch_pdl_coop(many ? k_fplan<long long, true> : k_fplan<long long, false>, dim3(grid), dim3(kPlanThreads), 0, s, (const long long*)idx, offsets, T, B,
                   h->kg, w.f_key, w.f_i3, w.f_rk, w.bag_of, w.f_cnt, w.f_start, w.f_rstart, w.f_split, w.f_gtot, w.f_item_start, w.f_cta, h->num_sms,
                   w.f_item_key, w.f_tile_info, w.f_sbi, w.fast_hdr, getenv("TTB_DBG") ? 1 : 0, h->allow_empty,
                   (const uint4*)w.f_tgeom, w.f_chunks, (float4*)w.f_grad, ngrad4);
  else
    e = launch_pdl_coop(many ? k_fplan<int, true> : k_fplan<int, false>, dim3(grid), dim3(kPlanThreads), 0, s, (const int*)idx, offsets, T, B, h->kg,
                   w.f_key, w.f_i3, w.f_rk, w.bag_of, w.f_cnt, w.f_start, w.f_rstart, w.f_split, w.f_gtot, w.f_item_start, w.f_cta, h->num_sms,
                   w.f_item_key,
                   w.f_tile_info, w.f_sbi, w.fast_hdr, getenv("TTB_DBG") ? 1 : 0, h->allow_empty,
                   (const uint4*)w.f_tgeom, w.f_chunks, (float4*)w.f_grad, ngrad4);
  }
  if (e) return e;
  h->fgrad_zeroed = 1;
  h->tilectr_zeroed = 1;
  count_launch();
  if (T > B) {  // pooled: each multi-item prefix's lookups grouped by row (forward and backward use it)
    constexpr int sort_smem = kSortSmem;
    if ((e = ensure_kernel_smem((const void*)k_rowsort, sort_smem))) return e;
    ProfScope _pr(h, s, "f_rowsort");
    if ((e = launch_pdl(k_rowsort, dim3(h->num_sms), dim3(kSortThreads), sort_smem, s, w.f_sbi,
                        (const int2*)w.f_chunks, (const int*)w.fast_hdr, h->kg.tm3)))
      return e;
    count_launch();
  }
  return cudaGetLastError();
}

cudaError_t fast_forward(ttb_handle* h, const float* c0, const float* c1, const float* c2, float* out,
                         cudaStream_t s) {
  Workspace& w = h->w;
  cudaError_t e;
  const int img_smem = 32 * 129 * 4 + 1024;
  if ((e = ensure_kernel_smem((const void*)k_coreimg, img_smem))) return e;
  if ((e = ensure_kernel_smem((const void*)k_fwd<false>, fwd_smem_bytes(kFwdMaxM3)))) return e;
  if ((e = ensure_kernel_smem((const void*)k_fwd<true>, fwd_smem_bytes(kFwdMaxM3)))) return e;
  if ((e = ensure_kernel_smem((const void*)k_bwd<false>, kBwdSmem))) return e;
  if ((e = ensure_kernel_smem((const void*)k_bwd<true>, kBwdSmem))) return e;
  if (!(h->img_valid && h->img_c0 == c0 && h->img_c1 == c1 && h->img_c2 == c2)) {
    // split tf32 images of the cores (skipped while the images written by the
    // last fused update, or the last forward, still describe these cores)
    ProfScope _ps(h, s, "f_coreimg");
    SgdArgs u = {};
    u.p2 = const_cast<float*>(c2);
    u.g3t = w.f_g3t;
    const int ng3 = (int)(((int64_t)128 * h->kg.m3 + kImgThreads - 1) / kImgThreads);
    if ((e = launch_pdl(k_coreimg, dim3(h->kg.m2 + (h->kg.g1rows + 3) / 4 + (ng3 < 64 ? ng3 : 64)),
                        dim3(kImgThreads), img_smem, s, const_cast<float*>(c0), const_cast<float*>(c1), h->kg,
                        w.f_img, w.f_g1img, u)))
      return e;
    count_launch();
    h->img_valid = 1;
    h->img_c0 = c0;
    h->img_c1 = c1;
    h->img_c2 = c2;
  }
  // one store per lookup into its bag's row; with empty bags allowed, T = B
  // no longer means one lookup per bag (and empty rows must read zero)
  const int direct = h->T == h->B && !h->allow_empty;
  if (!direct && (e = cudaMemsetAsync(out, 0, sizeof(float) * (size_t)h->B * NOUT, s))) return e;
  const int grid = h->num_sms;  // = the plan's CTA ranges (k_fplan cta_tiles)
  {
    ProfScope _ps(h, s, "f_fwd");
    // pooled bags: segments of several lookups (G3 slices summed before the product)
    if ((e = launch_pdl(h->T > h->B ? k_fwd<true> : k_fwd<false>, dim3(grid), dim3(kFwdThreads), fwd_smem_bytes(h->kg.tm3), s, h->kg, (const float*)w.f_g1img, c2,
                        (const float*)w.f_img, (const int*)w.fast_hdr, (const int4*)w.f_tile_info,
                        (const int*)w.f_item_start, (const unsigned*)w.f_item_key, (const int2*)w.f_sbi, out,
                        (const int*)w.f_cta, direct, getenv("TTB_DBG") ? atoi(getenv("TTB_DBG")) : 0)))
      return e;
  }
  count_launch();
  return cudaGetLastError();
}

// mode 0: gradients into g0..g2; mode 1: SGD(+momentum) on the cores (mask)
cudaError_t fast_backward(ttb_handle* h, const float* c0, const float* c1, const float* c2, const float* gout,
                          float* g0, float* g1, float* g2, float* p0, float* p1, float* p2, double* v0, double* v1,
                          double* v2, double lr, double mu, int mask, int mode, cudaStream_t s, int adagrad) {
  Workspace& w = h->w;
  cudaError_t e;
  const int64_t n0 = (int64_t)h->kg.g1rows * 4 * R1, n1 = (int64_t)R1 * h->kg.m2 * C, n2 = (int64_t)32 * h->kg.m3 * 4;
  if (mode == 1) {
    g0 = w.f_grad;
    g1 = w.f_grad + n0;
    g2 = w.f_grad + n0 + n1;
    if (!h->fgrad_zeroed && (e = cudaMemsetAsync(w.f_grad, 0, sizeof(float) * (size_t)(n0 + n1 + n2), s))) return e;
  } else {
    if ((e = cudaMemsetAsync(g0, 0, sizeof(float) * (size_t)n0, s))) return e;
    if ((e = cudaMemsetAsync(g1, 0, sizeof(float) * (size_t)n1, s))) return e;
    if (!h->fgrad_zeroed && (e = cudaMemsetAsync(w.f_grad + n0 + n1, 0, sizeof(float) * (size_t)n2, s))) return e;
  }
  h->fgrad_zeroed = 0;  // this backward accumulates into it
  // dG3 accumulates slice-major, (i3, c, n3): one lookup's 128 contributions
  // are 512 contiguous bytes (4 L2 lines instead of 32); the update kernel
  // reads it in that order, the caller's buffer gets the reference layout
  float* g3s = w.f_grad + n0 + n1;
  const int grid = h->num_sms;  // = the plan's CTA ranges (k_fplan cta_tiles)
  if (h->T > h->B && !h->tilectr_zeroed)  // pooled: the backward's tile counter (cleared by the plan)
    if ((e = cudaMemsetAsync(w.fast_hdr + kHdrNextTile, 0, sizeof(int), s))) return e;
  h->tilectr_zeroed = 0;
  {
    ProfScope _ps(h, s, "f_bwd");
    // pooled bags (more lookups than bags) repeat rows inside a prefix: group
    // by row; otherwise (T = B, bags are single lookups) position by position
    if ((e = launch_pdl(h->T > h->B ? k_bwd<true> : k_bwd<false>, dim3(grid), dim3(kBwdThreads), kBwdSmem, s, h->kg, (const float*)w.f_g1img, (const float*)w.f_g3t,
                        (const float*)w.f_img, (const int4*)w.f_tile_info, (const int*)w.f_item_start,
                        (const unsigned*)w.f_item_key, (const int2*)w.f_sbi, gout, g0, g1, g3s, w.fast_hdr,
                        (const int*)w.f_cta, getenv("TTB_DBG") ? atoi(getenv("TTB_DBG")) : 0)))
      return e;
  }
  count_launch();
  if (mode == 1) {
    // SGD(+momentum) on all three cores, writing the next step's G1 / G2
    // images from the updated values
    const int img_smem = 32 * 129 * 4 + 1024;
    const int ng3 = (int)((n2 + kImgThreads - 1) / kImgThreads);
    // (the finiteness gate runs inside the update kernel, see k_coreimg)
    SgdArgs u = {w.f_grad, v0, v1, v2, p2, lr, mu, mask, 1, w.fast_hdr, adagrad, w.f_g3t,
                 w.fast_hdr + kHdrSuspect, n0 + n1 + n2};
    ProfScope _ps(h, s, "f_sgd");
    if ((e = launch_pdl(k_coreimg, dim3(h->kg.m2 + (h->kg.g1rows + 3) / 4 + (ng3 < 16 ? ng3 : 16)), dim3(kImgThreads),
                        img_smem, s, p0, p1, h->kg, w.f_img, w.f_g1img, u)))
      return e;
    count_launch();
    h->img_valid = 1;
    h->img_c0 = p0;
    h->img_c1 = p1;
    h->img_c2 = p2;
  } else {
    // the caller's gradients: a suspect contribution (see kHdrSuspect) gets
    // the exact scan, which latches TTB_ERRBIT_NONFINITE (tt_core_grads
    // rejects non-finite gradients, backward.py:119-128)
    {
      const unsigned m3 = h->kg.m3;
      if ((e = launch_pdl(k_g3_unslice, dim3((128 * m3 + 255) / 256), dim3(256), 0, s, (const float*)g3s, g2, m3)))
        return e;
      count_launch();
    }
    ProfScope _pc(h, s, "f_gradcheck");
    if ((e = launch_gradcheck(g0, n0, w.fast_hdr, h->num_sms, s, w.fast_hdr + kHdrSuspect))) return e;
    if ((e = launch_gradcheck(g1, n1, w.fast_hdr, h->num_sms, s, w.fast_hdr + kHdrSuspect))) return e;
    if ((e = launch_gradcheck(g2, n2, w.fast_hdr, h->num_sms, s, w.fast_hdr + kHdrSuspect))) return e;
    h->img_valid = 0;  // the caller applies its own update to the cores
  }
  return cudaGetLastError();
}

}  // namespace ttb
