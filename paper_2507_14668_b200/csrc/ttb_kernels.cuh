// Forward / backward contraction kernels, templated on the core dims D
// (FixDims for the common shapes -> fully unrolled; DynDims otherwise).
#pragma once
#include <type_traits>

#include "ttb_internal.h"

namespace ttb {

template <class D> struct IsFixed : std::false_type {};
template <int A, int B, int C, int E, int F> struct IsFixed<FixDims<A, B, C, E, F>> : std::true_type {};

// Enumerate the present prefixes of one group, in ascending order of the
// free digit, and keep those whose ordinal falls in [chunk*CH, chunk*CH+CH).
// by_i2: group = i2, free digit i1 (keys i1*m2 + i2); else group = i1, free
// digit i2 (keys i1*m2 + i2, contiguous). Returns the group's total count;
// *n_chunk = entries written to s_free / s_slot. s_w: NW + 2 ints.
__device__ inline int collect_chunk(const unsigned* __restrict__ pmap, const int* __restrict__ pslot, KGeom g,
                                    bool by_i2, unsigned group, int chunk, int CH, int* s_free, int* s_slot,
                                    int* s_w, int* n_chunk) {
  constexpr int NW = kBlock / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = lanemask_lt();
  const int len = by_i2 ? (int)g.m1 : (int)g.m2;
  const int lo = chunk * CH, hi = lo + CH;
  int running = 0;
  for (int b0 = 0; b0 < len; b0 += kBlock) {
    const int j = b0 + threadIdx.x;
    unsigned key = 0;
    bool present = false;
    if (j < len) {
      key = by_i2 ? (unsigned)j * g.m2 + group : group * g.m2 + (unsigned)j;
      present = pmap[key] != kEmpty;
    }
    const unsigned m = __ballot_sync(0xffffffffu, present);
    if (lane == 0) s_w[w] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int i = 0; i < NW; ++i) {
        const int c = s_w[i];
        s_w[i] = acc;
        acc += c;
      }
      s_w[NW] = acc;
    }
    __syncthreads();
    const int ord = running + s_w[w] + __popc(m & lt);
    if (present && ord >= lo && ord < hi) {
      s_free[ord - lo] = j;
      s_slot[ord - lo] = pslot[key];
    }
    running += s_w[NW];
    __syncthreads();
  }
  int nc = running - lo;
  nc = nc < 0 ? 0 : (nc > CH ? CH : nc);
  *n_chunk = nc;
  return running;
}

// ------------------------------------------------------------ K2: prefix products
// slots[s] (n1 n2 x r2) = G1[i1] (n1 x r1) . G2[:, i2] (r1 x n2 r2), one CTA per
// (i2, chunk of present prefixes): the G2 slice is read once per CTA.
// Reference: lookup.py:138-146 (einsum "bxr,brys->bxys").
template <class D>
__global__ void __launch_bounds__(kBlock) k_prefix_products(D d, KGeom g, const float* __restrict__ G1,
                                                            const float* __restrict__ G2,
                                                            const unsigned* __restrict__ pmap,
                                                            const int* __restrict__ pslot, float* __restrict__ slots) {
  extern __shared__ float smem[];
  __shared__ int s_free[kPrefixChunk], s_slot[kPrefixChunk], s_w[kBlock / 32 + 2];
  const int C = dC(d), R1 = d.r1, N1 = d.n1;
  const unsigned i2 = blockIdx.x;
  int np;
  collect_chunk(pmap, pslot, g, true, i2, blockIdx.y, kPrefixChunk, s_free, s_slot, s_w, &np);
  if (np == 0) return;
  float* s_g2 = smem;            // R1 x C
  float* s_g1 = smem + R1 * C;   // np x R1 x N1 (transposed: [p][r][a])
  for (int e = threadIdx.x; e < R1 * C; e += kBlock) {
    const int r = e / C, c = e - r * C;
    s_g2[e] = G2[((size_t)r * g.m2 + i2) * C + c];
  }
  for (int e = threadIdx.x; e < np * R1 * N1; e += kBlock) {
    const int p = e / (R1 * N1), rem = e - p * (R1 * N1);
    const int a = rem / R1, r = rem - a * R1;
    s_g1[(p * R1 + r) * N1 + a] = G1[((size_t)s_free[p] * N1 + a) * R1 + r];
  }
  __syncthreads();
  const int SL = dSlot(d);
  // outputs (p, a, c): thread -> c fastest so the slot store is coalesced
  for (int e = threadIdx.x; e < np * N1 * C; e += kBlock) {
    const int p = e / (N1 * C), rem = e - p * (N1 * C);
    const int a = rem / C, c = rem - a * C;
    const float* g1 = s_g1 + p * R1 * N1 + a;
    float acc = 0.f;
#pragma unroll 8
    for (int r = 0; r < R1; ++r) acc = fmaf(g1[r * N1], s_g2[r * C + c], acc);
    slots[(size_t)s_slot[p] * SL + a * C + c] = acc;
  }
}

// ------------------------------------------------------------ K3: close + pool
// One warp per bag: for each segment (distinct prefix, ascending slot) sum the
// G3 slices of its indices in index order, multiply by the slot, and add the
// result to the bag in segment order. Reference: lookup.py:280-293.
template <class D>
__global__ void __launch_bounds__(kBlock) k_close_pool(D d, KGeom g, const float* __restrict__ G3,
                                                       const float* __restrict__ slots, const int* __restrict__ bag_off,
                                                       const int* __restrict__ bag_seg, const int* __restrict__ seg_slot,
                                                       const int* __restrict__ occ_slot,
                                                       const unsigned* __restrict__ keys32, int B,
                                                       float* __restrict__ out) {
  extern __shared__ float smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int X = dX(d), R2 = d.r2, N3 = d.n3, N = dN(d), SL = dSlot(d), G3S = dG3s(d);
  const int RS = R2 + 1;  // padded slot row stride (bank-conflict free)
  float* s_sb = smem + w * (X * RS + G3S + N);
  float* s_h = s_sb + X * RS;
  float* s_o = s_h + G3S;
  const unsigned m3n3 = g.m3 * (unsigned)N3;
  for (int b = blockIdx.x * (kBlock / 32) + w; b < B; b += gridDim.x * (kBlock / 32)) {
    const int o0 = bag_off[b], o1 = bag_off[b + 1];
    for (int o = lane; o < N; o += 32) s_o[o] = 0.f;
    for (int sg = bag_seg[b]; sg < bag_seg[b + 1]; ++sg) {
      const int slot = seg_slot[sg];
      for (int e = lane; e < G3S; e += 32) s_h[e] = 0.f;
      for (int t = o0; t < o1; ++t) {
        if (occ_slot[t] != slot) continue;
        const unsigned i3 = keys32[t] % g.m3;
        for (int e = lane; e < G3S; e += 32) {
          const int r = e / N3, j = e - r * N3;
          s_h[e] += __ldg(&G3[(size_t)r * m3n3 + i3 * N3 + j]);
        }
      }
      const float* sb = slots + (size_t)slot * SL;
      for (int e = lane; e < SL; e += 32) {
        const int x = e / R2, r = e - x * R2;
        s_sb[x * RS + r] = sb[e];
      }
      __syncwarp();
      for (int o = lane; o < N; o += 32) {
        const int x = o / N3, j = o - x * N3;
        float acc = 0.f;
#pragma unroll 8
        for (int r = 0; r < R2; ++r) acc = fmaf(s_sb[x * RS + r], s_h[r * N3 + j], acc);
        s_o[o] += acc;
      }
      __syncwarp();
    }
    for (int o = lane; o < N; o += 32) out[(size_t)b * N + o] = s_o[o];
    __syncwarp();
  }
}

// ------------------------------------------------------------ backward: rows
// Aggregated row gradient g_u = sum of the bag gradients of the row's
// occurrences, left to right in index order (backward.py:81-85 sums in the
// gradient dtype in occurrence order; the stable sort preserves that order).
template <class D>
__global__ void __launch_bounds__(kBlock) k_row_agg(D d, const int* __restrict__ counts,
                                                    const int* __restrict__ urow_start,
                                                    const unsigned* __restrict__ svals, const int* __restrict__ bag_of,
                                                    const float* __restrict__ gout, float* __restrict__ gU,
                                                    int* __restrict__ err) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int N = dN(d);
  const int U = counts[3];
  bool bad = false;
  for (int u = blockIdx.x * (kBlock / 32) + w; u < U; u += gridDim.x * (kBlock / 32)) {
    const int q0 = urow_start[u], q1 = urow_start[u + 1];
    for (int o0 = 0; o0 < N; o0 += 32) {
      const int o = o0 + lane;
      float acc = 0.f;
      if (o < N) {
        for (int q = q0; q < q1; ++q) {
          const float v = __ldg(&gout[(size_t)bag_of[svals[q]] * N + o]);
          acc += v;
        }
        if (!isfinite(acc)) bad = true;
        gU[(size_t)u * N + o] = acc;
      }
    }
  }
  if (bad) atomicOr(err, 8);
}

// ------------------------------------------------------------ backward: prefixes
// One CTA per (i2, chunk). For each prefix p = (i1, i2) and each of its rows
// u (contiguous in the row order):
//   Z_p   += g_u (n1n2 x n3) . G3[i3_u]^T (n3 x r2)       -> dL/dslot_p
//   dH_u   = slot_p^T (r2 x n1n2) . g_u                  -> G3 gradient block
// then  dG2[:, i2] += G1[i1]^T . Z_p   (accumulated in the CTA)
//       E_p         = Z_p . G2[:, i2]^T                  -> G1 gradient block
// This regroups backward.py:152-178 (per-row left/right chains) so the two
// r1 x n2 r2 products run once per distinct prefix instead of once per
// distinct row; the sums are the same.
constexpr int kRowBatch = 8;

template <class D>
__global__ void __launch_bounds__(kBlock) k_bwd_prefix(D d, KGeom g, const float* __restrict__ G1,
                                                       const float* __restrict__ G2, const float* __restrict__ G3,
                                                       const unsigned* __restrict__ pmap, const int* __restrict__ pslot,
                                                       const float* __restrict__ slots,
                                                       const int* __restrict__ prow_begin,
                                                       const int* __restrict__ prow_end,
                                                       const unsigned* __restrict__ urow_i3,
                                                       const float* __restrict__ gU, float* __restrict__ dH,
                                                       float* __restrict__ E, float* __restrict__ dG2part,
                                                       int* __restrict__ grp_cnt, int cmax) {
  extern __shared__ float smem[];
  __shared__ int s_free[kPrefixChunk], s_slot[kPrefixChunk], s_w[kBlock / 32 + 2];
  const int C = dC(d), R1 = d.r1, R2 = d.r2, N1 = d.n1, N3 = d.n3, X = dX(d), N = dN(d);
  const int SL = dSlot(d), G3S = dG3s(d), G2S = dG2s(d), G1S = dG1s(d);
  const unsigned i2 = blockIdx.x;
  int np;
  const int total = collect_chunk(pmap, pslot, g, true, i2, blockIdx.y, kPrefixChunk, s_free, s_slot, s_w, &np);
  if (blockIdx.y == 0 && threadIdx.x == 0) grp_cnt[i2] = total;
  if (np == 0) return;
  const int RS = R2 + 1;
  float* s_g2 = smem;                    // R1 x C
  float* s_acc = s_g2 + G2S;             // R1 x C  (dG2 accumulator)
  float* s_g1 = s_acc + G2S;             // N1 x R1
  float* s_sb = s_g1 + G1S;              // X x RS
  float* s_z = s_sb + X * RS;            // X x R2 == N1 x C
  float* s_g = s_z + SL;                 // kRowBatch x N
  float* s_g3 = s_g + kRowBatch * N;     // kRowBatch x G3S
  for (int e = threadIdx.x; e < G2S; e += kBlock) {
    const int r = e / C, c = e - r * C;
    s_g2[e] = G2[((size_t)r * g.m2 + i2) * C + c];
    s_acc[e] = 0.f;
  }
  const unsigned m3n3 = g.m3 * (unsigned)N3;
  for (int pi = 0; pi < np; ++pi) {
    const int slot = s_slot[pi];
    const unsigned i1 = s_free[pi];
    __syncthreads();
    for (int e = threadIdx.x; e < G1S; e += kBlock) s_g1[e] = G1[(size_t)i1 * G1S + e];
    const float* sb = slots + (size_t)slot * SL;
    for (int e = threadIdx.x; e < SL; e += kBlock) {
      const int x = e / R2, r = e - x * R2;
      s_sb[x * RS + r] = sb[e];
      s_z[e] = 0.f;
    }
    const int u0 = prow_begin[slot], u1 = prow_end[slot];
    for (int ub = u0; ub < u1; ub += kRowBatch) {
      const int nb = (u1 - ub) < kRowBatch ? (u1 - ub) : kRowBatch;
      __syncthreads();
      for (int e = threadIdx.x; e < nb * N; e += kBlock) s_g[e] = gU[(size_t)ub * N + e];
      for (int e = threadIdx.x; e < nb * G3S; e += kBlock) {
        const int k = e / G3S, rem = e - k * G3S;
        const int r = rem / N3, j = rem - r * N3;
        s_g3[e] = __ldg(&G3[(size_t)r * m3n3 + urow_i3[ub + k] * N3 + j]);
      }
      __syncthreads();
      // Z (X x R2) += sum_k g_k (X x N3) . G3_k^T
      for (int e = threadIdx.x; e < SL; e += kBlock) {
        const int x = e / R2, r = e - x * R2;
        float acc = s_z[e];
        for (int k = 0; k < nb; ++k) {
          const float* gk = s_g + k * N + x * N3;
          const float* hk = s_g3 + k * G3S + r * N3;
#pragma unroll
          for (int j = 0; j < N3; ++j) acc = fmaf(gk[j], hk[j], acc);
        }
        s_z[e] = acc;
      }
      // dH_k (R2 x N3) = slot^T . g_k
      for (int e = threadIdx.x; e < nb * G3S; e += kBlock) {
        const int k = e / G3S, rem = e - k * G3S;
        const int r = rem / N3, j = rem - r * N3;
        const float* gk = s_g + k * N + j;
        float acc = 0.f;
#pragma unroll 4
        for (int x = 0; x < X; ++x) acc = fmaf(s_sb[x * RS + r], gk[x * N3], acc);
        dH[(size_t)(ub + k) * G3S + rem] = acc;
      }
    }
    __syncthreads();
    // dG2 slice += G1^T . Z  (Z viewed as N1 x C)
    for (int e = threadIdx.x; e < G2S; e += kBlock) {
      const int r = e / C, c = e - r * C;
      float acc = s_acc[e];
#pragma unroll
      for (int a = 0; a < N1; ++a) acc = fmaf(s_g1[a * R1 + r], s_z[a * C + c], acc);
      s_acc[e] = acc;
    }
    // E_p (N1 x R1) = Z . G2_slice^T
    for (int e = threadIdx.x; e < G1S; e += kBlock) {
      const int a = e / R1, r = e - a * R1;
      const float* z = s_z + a * C;
      const float* g2 = s_g2 + r * C;
      float acc = 0.f;
#pragma unroll 8
      for (int c = 0; c < C; ++c) acc = fmaf(z[c], g2[c], acc);
      E[(size_t)slot * G1S + e] = acc;
    }
  }
  __syncthreads();
  float* part = dG2part + ((size_t)i2 * cmax + blockIdx.y) * G2S;
  for (int e = threadIdx.x; e < G2S; e += kBlock) part[e] = s_acc[e];
}

}  // namespace ttb
