// Forward / backward contraction kernels, templated on the core dims D
// (FixDims for the common shapes -> fully unrolled; DynDims otherwise).
#pragma once
#include <type_traits>

#include "ttb_internal.h"
#include "ttb_umma.cuh"

namespace ttb {

constexpr int kMaxChunk = 64;

template <class D> struct IsFixed : std::false_type {};
template <int A, int B, int C, int E, int F> struct IsFixed<FixDims<A, B, C, E, F>> : std::true_type {};
// compile-time dims (zeros for run-time dims)
template <class D> struct FixT { static constexpr int n1 = 0, n2 = 0, n3 = 0, r1 = 0, r2 = 0; };
template <int A, int B, int C, int E, int F> struct FixT<FixDims<A, B, C, E, F>> {
  static constexpr int n1 = A, n2 = B, n3 = C, r1 = E, r2 = F;
};
// warp-per-prefix backward fast path: lane <-> r2, float4 G3 slices
template <class D> constexpr bool kFastRows = FixT<D>::r2 == 32 && FixT<D>::n3 == 4 &&
                                              FixT<D>::n1 * FixT<D>::n2 * 4 <= 128;
// vectorised operand staging: row lengths multiple of 4 floats
template <class D> constexpr bool kVecStage = FixT<D>::r1 % 4 == 0 && FixT<D>::r1 > 0 &&
                                              (FixT<D>::n2 * FixT<D>::r2) % 4 == 0;
// slot size n1 n2 r2 as a compile-time constant (1 for run-time dims)
template <class D> struct FixSlot { static constexpr int value = 1; };
template <int A, int B, int C, int E, int F> struct FixSlot<FixDims<A, B, C, E, F>> {
  static constexpr int value = A * B * F;
};

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

// ------------------------------------------------------------ block GEMM helpers
template <int V>
__device__ __forceinline__ void lds_vec(float (&r)[V], const float* p) {
  if constexpr (V % 4 == 0) {
#pragma unroll
    for (int i = 0; i < V; i += 4) {
      const float4 v = *reinterpret_cast<const float4*>(p + i);
      r[i] = v.x; r[i + 1] = v.y; r[i + 2] = v.z; r[i + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) r[i] = p[i];
  }
}

// C[m][n] = sum_k At[k*lda + m] * B[k*ldb + n]   (both operands k-major in smem)
// Thread tiles TM x TN, handed out n-fastest so a warp's B loads are one
// contiguous run and its A loads broadcast. M % TM == 0, N % TN == 0.
// A TM or TN of 8 is split into two float4 groups half the extent apart
// (rows m0.., m0 + M/2..), which keeps a warp's 16-byte loads contiguous and
// bank-conflict free; out() receives the row / column of each element.
template <int V>
__device__ __forceinline__ int split_index(int base, int half, int i) {
  if constexpr (V == 8) return base + (i < 4 ? i : half + i - 4);
  else return base + i;
}
template <int V>
__device__ __forceinline__ void lds_split(float (&r)[V], const float* p, int half) {
  if constexpr (V == 8) {
    const float4 u = *reinterpret_cast<const float4*>(p);
    const float4 v = *reinterpret_cast<const float4*>(p + half);
    r[0] = u.x; r[1] = u.y; r[2] = u.z; r[3] = u.w;
    r[4] = v.x; r[5] = v.y; r[6] = v.z; r[7] = v.w;
  } else {
    lds_vec<V>(r, p);
  }
}

template <int TM, int TN, class Out>
__device__ __forceinline__ void gemm_kk(int M, int N, int K, const float* At, int lda, const float* B, int ldb,
                                        Out&& out) {
  const int tn = N / TN, tiles = (M / TM) * tn;
  const int hm = M / 2, hn = N / 2;
  for (int t = threadIdx.x; t < tiles; t += blockDim.x) {
    const int m0 = (t / tn) * (TM == 8 ? 4 : TM), n0 = (t % tn) * (TN == 8 ? 4 : TN);
    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
#pragma unroll 4
    for (int k = 0; k < K; ++k) {
      float a[TM], b[TN];
      lds_split<TM>(a, At + k * lda + m0, hm);
      lds_split<TN>(b, B + k * ldb + n0, hn);
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    out(m0, n0, hm, hn, acc);
  }
}

// One thread tile of gemm_kk accumulated into a caller-held register array
// (used when the tile grid equals the block: acc persists across sub-batches).
template <int TM, int TN>
__device__ __forceinline__ void gemm_kk_tile(int K, const float* At, int lda, const float* B, int ldb, int m0,
                                             int n0, int hm, int hn, float (&acc)[TM][TN]) {
#pragma unroll 4
  for (int k = 0; k < K; ++k) {
    float a[TM], b[TN];
    lds_split<TM>(a, At + k * lda + m0, hm);
    lds_split<TN>(b, B + k * ldb + n0, hn);
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
  }
}

// C[m][n] = sum_k A[m*lda + k] * Bt[n*ldb + k]   (contraction contiguous in both)
// K stepped by 4 with float4 loads when VEC (K % 4 == 0, 16-byte rows).
template <int TM, int TN, bool VEC, class Out>
__device__ __forceinline__ void gemm_nt(int M, int N, int K, const float* A, int lda, const float* Bt, int ldb,
                                        Out&& out) {
  const int tn = N / TN, tiles = (M / TM) * tn;
  for (int t = threadIdx.x; t < tiles; t += blockDim.x) {
    const int m0 = (t / tn) * TM, n0 = (t % tn) * TN;
    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
    if constexpr (VEC) {
#pragma unroll 2
      for (int k = 0; k < K; k += 4) {
        float4 a[TM], b[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i) a[i] = *reinterpret_cast<const float4*>(A + (m0 + i) * lda + k);
#pragma unroll
        for (int j = 0; j < TN; ++j) b[j] = *reinterpret_cast<const float4*>(Bt + (n0 + j) * ldb + k);
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) {
            float c = acc[i][j];
            c = fmaf(a[i].x, b[j].x, c);
            c = fmaf(a[i].y, b[j].y, c);
            c = fmaf(a[i].z, b[j].z, c);
            acc[i][j] = fmaf(a[i].w, b[j].w, c);
          }
      }
    } else {
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(A[(m0 + i) * lda + k], Bt[(n0 + j) * ldb + k], acc[i][j]);
    }
    out(m0, n0, acc);
  }
}

template <class D> struct Tiles {
  // run-time dims: scalar tiles (always divisible)
  static constexpr int FM = 1, FN = 1, BM = 1, BN = 1, CM = 1;
  static constexpr bool VEC = false;
};
template <int A, int B_, int C_, int R1, int R2> struct Tiles<FixDims<A, B_, C_, R1, R2>> {
  static constexpr int Cc = B_ * R2;
  static constexpr int FM = 8;                                               // chunk rows (ch % 8 == 0)
  static constexpr int FN = Cc % 8 == 0 ? 8 : (Cc % 4 == 0 ? 4 : 1);
  static constexpr int BM = R1 % 4 == 0 ? 4 : 1;
  static constexpr int BN = Cc % 4 == 0 ? 4 : 1;
  static constexpr int CM = 8;
  static constexpr bool VEC = Cc % 4 == 0;
};

// the phase-B tile grid of k_bwd_prefix equals the block: the dG2 partial
// can live in registers across the CTA's chunks
template <class D> struct RegAcc {
  static constexpr bool value = IsFixed<D>::value && FixT<D>::r1 > 0 &&
                                (FixT<D>::r1 / Tiles<D>::BM) * (FixT<D>::n2 * FixT<D>::r2 / Tiles<D>::BN) == kBlock;
};

template <class D> __host__ __device__ inline int pad_ld(const D& d) {
  return dC(d) % 4 == 0 ? dC(d) + 4 : dC(d);
}

// ------------------------------------------------------------ K2: prefix products
// slots[s] (n1 n2 x r2) = G1[i1] (n1 x r1) . G2[:, i2] (r1 x n2 r2). One CTA per
// (i2, chunk of <= ch present prefixes): a (ch n1) x (n2 r2) x r1 GEMM with the
// G2 slice read once per CTA. Reference: lookup.py:138-146.
template <class D>
__global__ void __launch_bounds__(kBlock) k_prefix_products(D d, KGeom g, int ch, const float* __restrict__ G1,
                                                            const float* __restrict__ G2,
                                                            const unsigned* __restrict__ pmap,
                                                            const int* __restrict__ pslot, float* __restrict__ slots) {
  pdl_enter();
  extern __shared__ __align__(16) float smem[];
  __shared__ int s_free[kMaxChunk], s_slot[kMaxChunk], s_w[kBlock / 32 + 2];
  const int C = dC(d), R1 = d.r1, N1 = d.n1;
  const unsigned i2 = blockIdx.x;
  const int split = blockIdx.y, nsplit = gridDim.y;
  int np;
  const int total = collect_chunk(pmap, pslot, g, true, i2, split, ch, s_free, s_slot, s_w, &np);
  const int nchunks = (total + ch - 1) / ch;
  if (split >= nchunks) return;
  const int M = ch * N1;   // padded rows (prefix, a)
  float* s_g2 = smem;      // R1 x C   (k-major: [r1][c])
  float* s_g1t = smem + R1 * C;  // R1 x M (k-major: [r1][p*N1 + a])
  // the G2 slice is staged once per CTA and reused by all its chunks
  if constexpr (kVecStage<D>) {
    constexpr int C4 = FixT<D>::n2 * FixT<D>::r2 / 4, R1c = FixT<D>::r1;
#pragma unroll 4
    for (int e = threadIdx.x; e < R1c * C4; e += kBlock) {
      const int r = e / C4, c4 = e - r * C4;
      reinterpret_cast<float4*>(s_g2)[e] =
          __ldg(reinterpret_cast<const float4*>(G2 + ((size_t)r * g.m2 + i2) * C) + c4);
    }
  } else {
    for (int e = threadIdx.x; e < R1 * C; e += kBlock) {
      const int r = e / C, c = e - r * C;
      s_g2[e] = G2[((size_t)r * g.m2 + i2) * C + c];
    }
  }
  using Tl = Tiles<D>;
  const int SL = dSlot(d);
  for (int chunk = split; chunk < nchunks; chunk += nsplit) {
    if (chunk != split) {
      __syncthreads();  // previous chunk's GEMM done with s_g1t / s_slot
      collect_chunk(pmap, pslot, g, true, i2, chunk, ch, s_free, s_slot, s_w, &np);
    }
    if constexpr (kVecStage<D>) {
      constexpr int R1c = FixT<D>::r1, N1c = FixT<D>::n1, RQ = R1c / 4;  // float4 per G1 row
#pragma unroll 4
      for (int e = threadIdx.x; e < M * RQ; e += kBlock) {
        const int row = e / RQ, q = e - row * RQ;
        const int p = row / N1c, a = row - p * N1c;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (p < np) v = __ldg(reinterpret_cast<const float4*>(G1 + ((size_t)s_free[p] * N1c + a) * R1c) + q);
        s_g1t[(4 * q + 0) * M + row] = v.x;
        s_g1t[(4 * q + 1) * M + row] = v.y;
        s_g1t[(4 * q + 2) * M + row] = v.z;
        s_g1t[(4 * q + 3) * M + row] = v.w;
      }
    } else {
      for (int e = threadIdx.x; e < M * R1; e += kBlock) {
        const int row = e / R1, r = e - row * R1;
        const int p = row / N1, a = row - p * N1;
        s_g1t[r * M + row] = p < np ? G1[((size_t)s_free[p] * N1 + a) * R1 + r] : 0.f;
      }
    }
    __syncthreads();
    gemm_kk<Tl::FM, Tl::FN>(M, C, R1, s_g1t, M, s_g2, C,
                            [&](int m0, int n0, int hm, int hn, float (&acc)[Tl::FM][Tl::FN]) {
#pragma unroll
      for (int i = 0; i < Tl::FM; ++i) {
        const int row = split_index<Tl::FM>(m0, hm, i), p = row / N1, a = row - p * N1;
        if (p >= np) continue;
        float* dst = slots + (size_t)s_slot[p] * SL + a * C;
        if constexpr (Tl::FN % 4 == 0) {
#pragma unroll
          for (int j = 0; j < Tl::FN; j += 4)
            *reinterpret_cast<float4*>(dst + split_index<Tl::FN>(n0, hn, j)) =
                make_float4(acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < Tl::FN; ++j) dst[n0 + j] = acc[i][j];
        }
      }
    });
  }
}

// ------------------------------------------------------------ K2 on the tensor cores
// Same product as k_prefix_products, issued as tcgen05.mma kind::tf32 with a
// 3xTF32 split (a = hi + lo, a.b ~ hi.hi + hi.lo + lo.hi in fp32 TMEM
// accumulators; measured 4e-7 relative vs 3e-4 for plain TF32), so the slots
// keep fp32-level accuracy. One CTA per (i2, chunk of 32 prefixes): the
// (32 n1 = 128) x (n2 r2) x r1 GEMM is one M=128 UMMA tile. Operands are
// staged K-major (SWIZZLE_NONE core matrices) by all threads, one thread issues
// the 3 * r1/8 MMAs, and the accumulator is read back by 8 warps (lane quarter
// = warp % 4, column half = warp / 4) and written through smem as full rows.
template <class D> constexpr bool kTcPrefix = FixT<D>::n1 == 4 && FixT<D>::r1 % 8 == 0 && FixT<D>::r1 >= 8 &&
                                              (FixT<D>::n2 * FixT<D>::r2) % 64 == 0 &&
                                              FixT<D>::n2 * FixT<D>::r2 <= 256;
constexpr int kTcChunk = 32;  // prefixes per CTA: M = 32 * n1 = 128

template <class D>
__global__ void __launch_bounds__(kBlock) k_prefix_products_tc(D d, KGeom g, const float* __restrict__ G1,
                                                               const float* __restrict__ G2,
                                                               const unsigned* __restrict__ pmap,
                                                               const int* __restrict__ pslot,
                                                               float* __restrict__ slots) {
  pdl_enter();
  if constexpr (kTcPrefix<D>) {
    constexpr int R1 = FixT<D>::r1, C = FixT<D>::n2 * FixT<D>::r2, M = 128, N1 = 4;
    extern __shared__ __align__(16) float smem[];
    __shared__ int s_free[kMaxChunk], s_slot[kMaxChunk], s_w[kBlock / 32 + 2];
    __shared__ uint64_t s_mbar;
    __shared__ uint32_t s_tmem;
    const unsigned i2 = blockIdx.x;
    int np;
    collect_chunk(pmap, pslot, g, true, i2, blockIdx.y, kTcChunk, s_free, s_slot, s_w, &np);
    if (np == 0) return;
    float* a_hi = smem;             // K-major [(r1/4)][row][4], M rows
    float* a_lo = a_hi + M * R1;
    float* b_hi = a_lo + M * R1;    // K-major [(r1/4)][c][4], C rows
    float* b_lo = b_hi + C * R1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) umma::tmem_alloc(&s_tmem, C <= 128 ? 128 : 256);
    if (threadIdx.x == 32) umma::mbar_init(&s_mbar, 1);
    // Operand staging. All global loads of this thread are issued first (so
    // they are in flight together), then split into hi / lo and stored.
    // A: G1 rows (prefix, a) hold r1 contiguous: one float4 = one 16-byte unit.
    // B: G2 slice [r1][c] -> K-major over r1: 4 consecutive r1 of one c.
    constexpr int NA = M * (R1 / 4) / kBlock, NB = C * (R1 / 4) / kBlock;
    static_assert(NA * kBlock == M * (R1 / 4) && NB * kBlock == C * (R1 / 4), "staging split");
    float4 va[NA], vb[NB];
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const int e = threadIdx.x + i * kBlock, row = e % M, q = e / M;
      const int p = row / N1, a = row - p * N1;
      va[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (p < np) va[i] = __ldg(reinterpret_cast<const float4*>(G1 + ((size_t)s_free[p] * N1 + a) * R1) + q);
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const int e = threadIdx.x + i * kBlock, c = e % C, q = e / C;
      const float* src = G2 + ((size_t)(4 * q) * g.m2 + i2) * C + c;
      const size_t rs = (size_t)g.m2 * C;
      vb[i].x = __ldg(src);
      vb[i].y = __ldg(src + rs);
      vb[i].z = __ldg(src + 2 * rs);
      vb[i].w = __ldg(src + 3 * rs);
    }
    auto split4 = [](const float4& v, float4& h, float4& l) {
      umma::split3(v.x, h.x, l.x);
      umma::split3(v.y, h.y, l.y);
      umma::split3(v.z, h.z, l.z);
      umma::split3(v.w, h.w, l.w);
    };
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const int e = threadIdx.x + i * kBlock, row = e % M, q = e / M;
      float4 h, l;
      split4(va[i], h, l);
      reinterpret_cast<float4*>(a_hi)[q * M + row] = h;
      reinterpret_cast<float4*>(a_lo)[q * M + row] = l;
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const int e = threadIdx.x + i * kBlock, c = e % C, q = e / C;
      float4 h, l;
      split4(vb[i], h, l);
      reinterpret_cast<float4*>(b_hi)[q * C + c] = h;
      reinterpret_cast<float4*>(b_lo)[q * C + c] = l;
    }
    umma::fence_smem_to_async();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = s_tmem;
    if (threadIdx.x == 0) {
      constexpr uint32_t idesc = umma::idesc_tf32(M, C, false, false);
      const float* as[3] = {a_hi, a_hi, a_lo};
      const float* bs[3] = {b_hi, b_lo, b_hi};
#pragma unroll
      for (int s = 0; s < R1 / 8; ++s)
#pragma unroll
        for (int v = 0; v < 3; ++v) {
          const uint64_t ad = umma::desc(umma::smem_u32(as[v]) + s * 2 * M * 16, M * 16, 128);
          const uint64_t bd = umma::desc(umma::smem_u32(bs[v]) + s * 2 * C * 16, C * 16, 128);
          umma::mma_tf32(tmem, ad, bd, idesc, (s > 0 || v > 0) ? 1u : 0u);
        }
      umma::commit(&s_mbar);
    }
    umma::mbar_wait(&s_mbar, 0);
    umma::fence_after_sync();
    // epilogue: warp -> (lane quarter, column half); rows staged in smem (the
    // operand buffers are free now) then written out as whole slot rows
    float* stage = smem;  // M x (C + 4) floats
    constexpr int LS = C + 4;
    {
      const int quarter = warp & 3, half = warp >> 2;
      const int row = 32 * quarter + lane;
#pragma unroll
      for (int c0 = 0; c0 < C / 2; c0 += 32) {
        float v[32];
        umma::tmem_ld32(tmem + ((uint32_t)(32 * quarter) << 16) + half * (C / 2) + c0, v);
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4*>(stage + row * LS + half * (C / 2) + c0 + i) =
              make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      }
    }
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_free(tmem, C <= 128 ? 128 : 256);
    constexpr int SL = N1 * C;  // slot = n1 rows (a) x C
    for (int row = warp; row < np * N1; row += kBlock / 32) {
      const int p = row / N1, a = row - p * N1;
      float* dst = slots + (size_t)s_slot[p] * SL + a * C;
      for (int c = 4 * lane; c < C; c += 128)
        *reinterpret_cast<float4*>(dst + c) = *reinterpret_cast<const float4*>(stage + row * LS + c);
    }
  }
}

// ------------------------------------------------------------ K3: close + pool
// For each segment (distinct prefix of a bag, ascending slot) sum the G3
// slices of its indices in index order, multiply by the slot, and add the
// result to the bag in segment order. Reference: lookup.py:280-293.
template <class D>
__device__ __forceinline__ void close_bag_generic(const D& d, KGeom g, const float* __restrict__ G3,
                                                  const float* __restrict__ slots, int b, int o0, int o1, int sg0,
                                                  int sg1, const int* __restrict__ seg_slot,
                                                  const int* __restrict__ occ_slot,
                                                  const unsigned* __restrict__ keys32, float* s_sb, float* s_h,
                                                  float* s_o, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int X = dX(d), R2 = d.r2, N3 = d.n3, N = dN(d), SL = dSlot(d), G3S = dG3s(d);
  const int RS = R2 + 1;
  const unsigned m3n3 = g.m3 * (unsigned)N3;
  for (int o = lane; o < N; o += 32) s_o[o] = 0.f;
  for (int sg = sg0; sg < sg1; ++sg) {
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

constexpr int kMultiSeg = 32;  // segments per bag handled by the register close path
constexpr int kSegGroup = 8;   // segments whose H sums are staged at once (smem per warp)

template <class D>
__host__ __device__ constexpr int close_warp_floats(const D& d) {
  return dX(d) * (d.r2 + 1) + dG3s(d) + dN(d);
}

template <class D>
__global__ void __launch_bounds__(kBlock) k_close_pool(D d, KGeom g, const float* __restrict__ G3,
                                                       const float* __restrict__ slots, const int* __restrict__ bag_off,
                                                       const int* __restrict__ bag_seg, const int* __restrict__ seg_slot,
                                                       const int* __restrict__ seg_inv,
                                                       const int* __restrict__ occ_slot,
                                                       const unsigned* __restrict__ keys32, int B,
                                                       float* __restrict__ out) {
  pdl_enter();
  extern __shared__ __align__(16) float smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // per-warp smem stride: the fast path also keeps per-segment H sums
  const int WF = kFastRows<D> ? max(close_warp_floats(d), 136 + kSegGroup * 128) : close_warp_floats(d);
  float* s_sb = smem + w * WF;
  float* s_h = s_sb + dX(d) * (d.r2 + 1);
  float* s_o = s_h + dG3s(d);
  const int gw = blockIdx.x * (kBlock / 32) + w, nw = gridDim.x * (kBlock / 32);
  if constexpr (kFastRows<D> && FixT<D>::n1 * FixT<D>::n2 == 16) {
    // Single-index bags (pooling 1): out[x][j] = sum_r slot[x][r] G3[r][j].
    // Lane pair (x, h) owns slot row x, half h of r: its 16 slot values come
    // straight from global (2 KB per bag, one coalesced sweep), the 32 x 4 G3
    // slice is staged once in smem and read as broadcast float4s, and the two
    // halves are combined with one shuffle. Bag metadata is fetched 32 bags at
    // a time and the next bag's operands are prefetched.
    float* f_h = s_sb;  // 32 r x 4 j, the r >= 16 half shifted by 4 floats (bank split)
    const unsigned m3n3 = g.m3 * 4u;
    const int x = lane >> 1, hf = lane & 1;
    constexpr int kGrp = 8;  // bags per warp iteration: many warps in flight
    for (int b0 = gw * kGrp; b0 < B; b0 += nw * kGrp) {
      const int b = b0 + lane;
      int o0 = 0, o1 = 0, sg0 = 0, sg1 = 0, slot = 0;
      unsigned i3 = 0;
      if (lane < kGrp && b < B) {
        o0 = bag_off[b];
        o1 = bag_off[b + 1];
        sg0 = bag_seg[b];
        sg1 = bag_seg[b + 1];
        if (o1 - o0 == 1) {
          slot = occ_slot[o0];
          i3 = keys32[o0] % g.m3;
        }
      }
      const int nb = min(kGrp, B - b0);
      const unsigned simple = __ballot_sync(0xffffffffu, lane < kGrp && b < B && o1 - o0 == 1);
      float4 psb[4], ph;
      auto fetch = [&](int i) {
        const int sl = __shfl_sync(0xffffffffu, slot, i);
        const unsigned ii3 = __shfl_sync(0xffffffffu, i3, i);
        const float4* src = reinterpret_cast<const float4*>(slots + (size_t)sl * 512 + x * 32 + hf * 16);
#pragma unroll
        for (int k = 0; k < 4; ++k) psb[k] = src[k];
        ph = __ldg(reinterpret_cast<const float4*>(G3 + (size_t)lane * m3n3 + ii3 * 4u));
      };
      int next = simple ? __ffs(simple) - 1 : 32;
      if (next < nb) fetch(next);
      for (int i = 0; i < nb; ++i) {
        if (!((simple >> i) & 1u)) continue;  // multi-index bags: k_close_multi
        float sv[16];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          sv[4 * k] = psb[k].x;
          sv[4 * k + 1] = psb[k].y;
          sv[4 * k + 2] = psb[k].z;
          sv[4 * k + 3] = psb[k].w;
        }
        // lane r2 = lane stages its G3 row
        *reinterpret_cast<float4*>(f_h + lane * 4 + (lane >= 16 ? 4 : 0)) = ph;
        const unsigned rest = simple & ~((2u << i) - 1u);
        next = rest ? __ffs(rest) - 1 : 32;
        if (next < nb) fetch(next);
        __syncwarp();
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int r = hf * 16 + k;
          const float4 hv = *reinterpret_cast<const float4*>(f_h + r * 4 + hf * 4);
          a0 = fmaf(sv[k], hv.x, a0);
          a1 = fmaf(sv[k], hv.y, a1);
          a2 = fmaf(sv[k], hv.z, a2);
          a3 = fmaf(sv[k], hv.w, a3);
        }
        // combine the two r halves: lane h keeps outputs j = 2h, 2h + 1
        const float s0 = hf ? a0 : a2, s1 = hf ? a1 : a3;
        const float r0 = __shfl_xor_sync(0xffffffffu, s0, 1), r1 = __shfl_xor_sync(0xffffffffu, s1, 1);
        const float o_0 = (hf ? a2 : a0) + r0, o_1 = (hf ? a3 : a1) + r1;
        *reinterpret_cast<float2*>(out + (size_t)(b0 + i) * 64 + x * 4 + hf * 2) = make_float2(o_0, o_1);
        __syncwarp();
      }
    }
  } else {
    for (int b = gw; b < B; b += nw)
      close_bag_generic(d, g, G3, slots, b, bag_off[b], bag_off[b + 1], bag_seg[b], bag_seg[b + 1], seg_slot,
                        occ_slot, keys32, s_sb, s_h, s_o, out);
  }
}


// Multi-index bags (pooling > 1) of the lane <-> r2 fast shape; single-index
// bags are done by k_close_pool. One warp per bag.
template <class D>
__global__ void __launch_bounds__(kBlock) k_close_multi(D d, KGeom g, const float* __restrict__ G3,
                                                        const float* __restrict__ slots,
                                                        const int* __restrict__ bag_off,
                                                        const int* __restrict__ bag_seg,
                                                        const int* __restrict__ seg_slot,
                                                        const int* __restrict__ seg_inv,
                                                        const int* __restrict__ occ_slot,
                                                        const unsigned* __restrict__ keys32, int B,
                                                        const int* __restrict__ counts, float* __restrict__ out) {
  pdl_enter();
  if constexpr (kFastRows<D> && FixT<D>::n1 * FixT<D>::n2 == 16) {
    if (counts[4] == 0) return;  // no bag has more than one index
    extern __shared__ __align__(16) float smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int WF = max(close_warp_floats(d), 136 + kSegGroup * 128);
    float* s_sb = smem + w * WF;
    float* s_h = s_sb + dX(d) * (d.r2 + 1);
    float* s_o = s_h + dG3s(d);
    const unsigned m3n3 = g.m3 * 4u;
    const int x = lane >> 1, hf = lane & 1;
    const int gw = blockIdx.x * (kBlock / 32) + w, nw = gridDim.x * (kBlock / 32);
    for (int b = gw; b < B; b += nw) {
      const int o0 = bag_off[b], o1 = bag_off[b + 1];
      if (o1 - o0 <= 1) continue;
      const int sg0 = bag_seg[b], sg1 = bag_seg[b + 1];
        {
          const int bi = b;
          const int a0i = o0, a1i = o1, s0i = sg0, s1i = sg1;
          const int L = a1i - a0i, S = s1i - s0i;
          if (L > 32 || S > kMultiSeg) {
            close_bag_generic(d, g, G3, slots, bi, a0i, a1i, s0i, s1i, seg_slot, occ_slot, keys32, s_sb, s_h, s_o,
                              out);
            continue;
          }
          // Segments are closed in groups of kSegGroup (ascending slot). Pass 1
          // builds the group's H_s sums: lane r2 fetches its float4 of every
          // index's G3 slice (8 loads in flight) and adds those of the group's
          // segments in index order. Pass 2 closes each segment with the
          // slot's row halves (next segment's halves prefetched) and adds it
          // to the bag in segment order.
          float* f_hs = s_sb + 136;  // kSegGroup x 32 x 4 (r2-major per segment)
          const int myseg = lane < L ? seg_inv[a0i + lane] - s0i : 0;
          const unsigned myi3 = lane < L ? keys32[a0i + lane] % g.m3 : 0u;
          const int myslot = lane < S ? seg_slot[s0i + lane] : 0;
          float2 ob = make_float2(0.f, 0.f);
          float4 cur4[4], nxt4[4];
          {
            const int sl = __shfl_sync(0xffffffffu, myslot, 0);
            const float4* src = reinterpret_cast<const float4*>(slots + (size_t)sl * 512 + x * 32 + hf * 16);
#pragma unroll
            for (int k = 0; k < 4; ++k) cur4[k] = src[k];
          }
          for (int g0 = 0; g0 < S; g0 += kSegGroup) {
            const int gn = min(kSegGroup, S - g0);
#pragma unroll
            for (int e = lane; e < kSegGroup * 32; e += 32)
              reinterpret_cast<float4*>(f_hs)[e] = make_float4(0.f, 0.f, 0.f, 0.f);
            __syncwarp();
            for (int t0 = 0; t0 < L; t0 += 8) {
              float4 gv[8];
              int sj[8];
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const unsigned ii3 = __shfl_sync(0xffffffffu, myi3, (t0 + k) & 31);
                sj[k] = __shfl_sync(0xffffffffu, myseg, (t0 + k) & 31) - g0;
                if (t0 + k < L && sj[k] >= 0 && sj[k] < gn)
                  gv[k] = __ldg(reinterpret_cast<const float4*>(G3 + (size_t)lane * m3n3 + ii3 * 4u));
              }
#pragma unroll
              for (int k = 0; k < 8; ++k)
                if (t0 + k < L && sj[k] >= 0 && sj[k] < gn) {
                  float4* hp4 = reinterpret_cast<float4*>(f_hs) + sj[k] * 32 + lane;
                  float4 hv = *hp4;
                  hv.x += gv[k].x;
                  hv.y += gv[k].y;
                  hv.z += gv[k].z;
                  hv.w += gv[k].w;
                  *hp4 = hv;
                }
            }
            __syncwarp();
            for (int jj = 0; jj < gn; ++jj) {
              const int j = g0 + jj;
              const int sln = __shfl_sync(0xffffffffu, myslot, (j + 1) & 31);
              if (j + 1 < S) {
                const float4* src = reinterpret_cast<const float4*>(slots + (size_t)sln * 512 + x * 32 + hf * 16);
#pragma unroll
                for (int k = 0; k < 4; ++k) nxt4[k] = src[k];
              }
              const float* hseg = f_hs + jj * 128;  // [r2][j4]
              float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float sv4[4] = {cur4[k].x, cur4[k].y, cur4[k].z, cur4[k].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const float4 hv = *reinterpret_cast<const float4*>(hseg + (hf * 16 + 4 * k + q) * 4);
                  c0 = fmaf(sv4[q], hv.x, c0);
                  c1 = fmaf(sv4[q], hv.y, c1);
                  c2 = fmaf(sv4[q], hv.z, c2);
                  c3 = fmaf(sv4[q], hv.w, c3);
                }
              }
              const float e0 = hf ? c0 : c2, e1 = hf ? c1 : c3;
              const float r0 = __shfl_xor_sync(0xffffffffu, e0, 1), r1 = __shfl_xor_sync(0xffffffffu, e1, 1);
              ob.x += (hf ? c2 : c0) + r0;
              ob.y += (hf ? c3 : c1) + r1;
#pragma unroll
              for (int k = 0; k < 4; ++k) cur4[k] = nxt4[k];
            }
            __syncwarp();
          }
          *reinterpret_cast<float2*>(out + (size_t)bi * 64 + x * 4 + hf * 2) = ob;
          __syncwarp();
          continue;
        }
    }
  }
}

// ------------------------------------------------------------ backward: rows
// Aggregated row gradient g_u = sum of the bag gradients of the row's
// occurrences (backward.py:81-85: occurrence order, gradient dtype). The
// sorted occurrence array is cut into fixed blocks of kAggBlock positions,
// one warp each, summed strictly left to right:
//   * a row that starts and ends inside a block is final (bit-exact with the
//     reference's left-to-right sum);
//   * a row crossing block boundaries leaves a tail partial in its first
//     block and head partials in the following blocks; level 2 adds them in
//     block order (deterministic; the association differs from a single
//     left-to-right chain only for such rows).
// Work per warp is bounded, so hot Zipf rows (1e5 occurrences) cost the same
// as cold ones.
constexpr int kAggBlock = 64;
constexpr int kMaxPerLane = 16;  // N <= 512

template <class D> constexpr int agg_per_lane() {
  return IsFixed<D>::value ? (FixT<D>::n1 * FixT<D>::n2 * FixT<D>::n3 + 31) / 32 : kMaxPerLane;
}

template <class D>
__global__ void __launch_bounds__(kBlock) k_row_agg(D d, int B, int T, const int* __restrict__ counts,
                                                    const int* __restrict__ urow_start, const int* __restrict__ qrow,
                                                    const unsigned* __restrict__ svals, const int* __restrict__ bag_of,
                                                    const float* __restrict__ gout, float* __restrict__ gU,
                                                    float* __restrict__ hp, float* __restrict__ tp,
                                                    int* __restrict__ span_list, int* __restrict__ span_count,
                                                    int* __restrict__ err) {
  pdl_enter();
  constexpr int PL = agg_per_lane<D>();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int N = dN(d);
  const int nblk = (T + kAggBlock - 1) / kAggBlock;
  bool bad = false;
  for (int blk = blockIdx.x * (kBlock / 32) + w; blk < nblk; blk += gridDim.x * (kBlock / 32)) {
    const int q0 = blk * kAggBlock, q1 = min(T, q0 + kAggBlock);
    // lanes prefetch bag id and row of 2 x 32 positions
    int bq[kAggBlock / 32], uq[kAggBlock / 32], kq[kAggBlock / 32];
#pragma unroll
    for (int k = 0; k < kAggBlock / 32; ++k) {
      const int q = q0 + 32 * k + lane;
      bq[k] = 0;
      uq[k] = -1;
      kq[k] = 0;
      if (q < q1) {
        int b = bag_of[svals[q]];
        bq[k] = b < 0 ? 0 : (b >= B ? B - 1 : b);  // malformed offsets: garbage ids, never OOB
        const int u = qrow[q];
        uq[k] = u;
        // where this position's row lives: 0 inside the block, 1 entered
        // from the left (head partial), 2 starts here and leaves right (tail)
        const int head = urow_start[u], tail = urow_start[u + 1];
        kq[k] = head < q0 ? 1 : (tail > q1 ? 2 : 0);
      }
    }
    float acc[PL];
#pragma unroll
    for (int i = 0; i < PL; ++i) acc[i] = 0.f;
    int cur = __shfl_sync(0xffffffffu, uq[0], 0);
    int cur_kind = __shfl_sync(0xffffffffu, kq[0], 0);
    auto flush = [&](int u, bool at_block_end) {
      float* dst;
      if (cur_kind == 0) dst = gU + (size_t)u * N;       // whole row inside the block
      else if (cur_kind == 1) dst = hp + (size_t)blk * N;  // row entered from the left
      else dst = tp + (size_t)blk * N;                     // row starts here, leaves right
      if (cur_kind == 2 && lane == 0) span_list[atomicAdd(span_count, 1)] = u;
#pragma unroll
      for (int i = 0; i < PL; ++i) {
        const int o = lane + 32 * i;
        if (o < N) {
          if (!isfinite(acc[i])) bad = true;
          dst[o] = acc[i];
        }
        acc[i] = 0.f;
      }
      (void)at_block_end;
    };
    const int n = q1 - q0;
    for (int i0 = 0; i0 < n; i0 += 8) {
      float v[8][PL];
      int uu[8], kk[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = i0 + k;
        const int src = i & 31;
        const int b = __shfl_sync(0xffffffffu, (i >> 5) ? bq[1] : bq[0], src);
        uu[k] = __shfl_sync(0xffffffffu, (i >> 5) ? uq[1] : uq[0], src);
        kk[k] = __shfl_sync(0xffffffffu, (i >> 5) ? kq[1] : kq[0], src);
#pragma unroll
        for (int j = 0; j < PL; ++j) {
          const int o = lane + 32 * j;
          v[k][j] = (i < n && o < N) ? __ldg(&gout[(size_t)b * N + o]) : 0.f;
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (i0 + k >= n) break;
        if (uu[k] != cur) {
          flush(cur, false);
          cur = uu[k];
          cur_kind = kk[k];
        }
#pragma unroll
        for (int j = 0; j < PL; ++j) acc[j] += v[k][j];
      }
    }
    flush(cur, true);
  }
  if (bad) atomicOr(err, 8);
}

// Level 2: rows spanning blocks: g_u = tp[first block] + hp[next blocks...],
// in block order. One CTA per listed row; warps own contiguous block ranges.
template <class D>
__global__ void __launch_bounds__(kBlock) k_row_agg_span(D d, const int* __restrict__ urow_start,
                                                         const int* __restrict__ span_list,
                                                         const int* __restrict__ span_count,
                                                         const float* __restrict__ hp, const float* __restrict__ tp,
                                                         float* __restrict__ gU, int* __restrict__ err) {
  pdl_enter();
  constexpr int PL = agg_per_lane<D>();
  extern __shared__ float s_part[];  // (kBlock/32) x N
  const int N = dN(d);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nspan = *span_count;
  for (int it = blockIdx.x; it < nspan; it += gridDim.x) {
    const int u = span_list[it];
    const int head = urow_start[u], tail = urow_start[u + 1];
    const int bs = head / kAggBlock, be = (tail - 1) / kAggBlock;
    const int nmid = be - bs;  // head partials of blocks bs+1 .. be
    const int per = (nmid + kBlock / 32 - 1) / (kBlock / 32);
    const int a = bs + 1 + w * per, b = min(be + 1, a + per);
    float acc[PL];
#pragma unroll
    for (int i = 0; i < PL; ++i) acc[i] = 0.f;
    for (int k0 = a; k0 < b; k0 += 8) {
      float v[8][PL];
#pragma unroll
      for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int j = 0; j < PL; ++j) {
          const int o = lane + 32 * j;
          v[k][j] = (k0 + k < b && o < N) ? hp[(size_t)(k0 + k) * N + o] : 0.f;
        }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k0 + k < b)
#pragma unroll
          for (int j = 0; j < PL; ++j) acc[j] += v[k][j];
    }
#pragma unroll
    for (int j = 0; j < PL; ++j) {
      const int o = lane + 32 * j;
      if (o < N) s_part[w * N + o] = acc[j];
    }
    __syncthreads();
    bool bad = false;
    for (int o = threadIdx.x; o < N; o += kBlock) {
      float t = tp[(size_t)bs * N + o];
      for (int ww = 0; ww < kBlock / 32; ++ww) t += s_part[ww * N + o];
      if (!isfinite(t)) bad = true;
      gU[(size_t)u * N + o] = t;
    }
    if (bad) atomicOr(err, 8);
    __syncthreads();
  }
}

// ------------------------------------------------------------ backward: prefixes
// One CTA per (i2, chunk of <= ch present prefixes).
//  Phase A (warp per prefix): for each of the prefix's rows u (contiguous in
//    the sorted row order)
//      Z_p += g_u (n1n2 x n3) . G3[i3_u]^T      -> dL/dslot_p, kept in smem
//      dH_u = slot_p^T . g_u (r2 x n3)          -> G3 gradient block, to HBM
//  Phase B: dG2[:, i2] partial (r1 x n2r2) = G1_chunk^T . Z_chunk   (GEMM, K = np n1)
//  Phase C: E_p (n1 x r1) = Z_p . G2[:, i2]^T                     (GEMM, K = n2 r2)
// This regroups backward.py:152-178 (per-row chains) so the r1 x n2 r2
// products run per distinct prefix; the sums are identical.
template <class D>
__global__ void __launch_bounds__(kBlock, 3) k_bwd_prefix(D d, KGeom g, int ch, const float* __restrict__ G1,
                                                       const float* __restrict__ G2, const float* __restrict__ G3,
                                                       const unsigned* __restrict__ pmap, const int* __restrict__ pslot,
                                                       const float* __restrict__ slots,
                                                       const int* __restrict__ prow_begin,
                                                       const int* __restrict__ prow_end,
                                                       const unsigned* __restrict__ urow_i3,
                                                       const float* __restrict__ gU, float* __restrict__ dH,
                                                       float* __restrict__ E, float* __restrict__ dG2part,
                                                       int* __restrict__ grp_cnt, int cmax) {
  pdl_enter();
  extern __shared__ __align__(16) float smem[];
  __shared__ int s_free[kMaxChunk], s_slot[kMaxChunk], s_w[kBlock / 32 + 2];
  __shared__ int s_next;
  __shared__ int s_u0[kMaxChunk], s_u1[kMaxChunk];
  const int C = dC(d), R1 = d.r1, R2 = d.r2, N1 = d.n1, N2 = d.n2, N3 = d.n3, X = dX(d), N = dN(d);
  const int SL = dSlot(d), G3S = dG3s(d), G1S = dG1s(d), G2S = dG2s(d);
  const unsigned i2 = blockIdx.x;
  const int split = blockIdx.y, nsplit = gridDim.y;
  int np;
  const int total = collect_chunk(pmap, pslot, g, true, i2, split, ch, s_free, s_slot, s_w, &np);
  if (split == 0 && threadIdx.x == 0) grp_cnt[i2] = total;
  const int nchunks = (total + ch - 1) / ch;
  if (split >= nchunks) return;
  const int M = ch * N1;
  const int LZ = pad_ld(d);
  float* s_z = smem;                 // M x LZ      Z rows (p, a), cols c = b r2 + r
  float* s_g2 = s_z + M * LZ;        // R1 x LZ     G2 slice [r1][c]
  float* s_g1 = s_g2 + R1 * LZ;      // M x R1      G1 chunk [(p, a)][r1]  (k-major for phase B)
  float* s_wk = s_g1 + M * R1;       // per warp: g (N) + G3 slice (G3S) + slot (SL)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  using Tl = Tiles<D>;
  // G2 slice: staged once per CTA
  if constexpr (kVecStage<D>) {
    constexpr int C4 = FixT<D>::n2 * FixT<D>::r2 / 4, R1c = FixT<D>::r1;
#pragma unroll 4
    for (int e = threadIdx.x; e < R1c * C4; e += kBlock) {
      const int r = e / C4, c4 = e - r * C4;
      *reinterpret_cast<float4*>(s_g2 + r * LZ + 4 * c4) =
          __ldg(reinterpret_cast<const float4*>(G2 + ((size_t)r * g.m2 + i2) * C) + c4);
    }
  } else {
    for (int e = threadIdx.x; e < R1 * C; e += kBlock) {
      const int r = e / C, c = e - r * C;
      s_g2[r * LZ + c] = G2[((size_t)r * g.m2 + i2) * C + c];
    }
  }
  for (int chunk = split; chunk < nchunks; chunk += nsplit) {
  if (chunk != split) {
    __syncthreads();  // previous chunk's phases done with s_z / s_g1 / s_slot
    collect_chunk(pmap, pslot, g, true, i2, chunk, ch, s_free, s_slot, s_w, &np);
  }
  if (threadIdx.x == 0) s_next = 0;
  // row ranges of the chunk's prefixes, one round trip for all of them
  if (threadIdx.x < np) {
    const int sl = s_slot[threadIdx.x];
    s_u0[threadIdx.x] = prow_begin[sl];
    s_u1[threadIdx.x] = prow_end[sl];
  }
  if constexpr (kVecStage<D>) {
    constexpr int R1c = FixT<D>::r1, RQ = R1c / 4;
#pragma unroll 4
    for (int e = threadIdx.x; e < M * RQ; e += kBlock) {
      const int row = e / RQ, q = e - row * RQ;
      const int p = row / FixT<D>::n1, a = row - p * FixT<D>::n1;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (p < np) v = __ldg(reinterpret_cast<const float4*>(G1 + ((size_t)s_free[p] * FixT<D>::n1 + a) * R1c) + q);
      reinterpret_cast<float4*>(s_g1)[e] = v;
    }
  } else {
    for (int e = threadIdx.x; e < M * R1; e += kBlock) {
      const int row = e / R1, r = e - row * R1;
      const int p = row / N1, a = row - p * N1;
      s_g1[e] = p < np ? G1[((size_t)s_free[p] * N1 + a) * R1 + r] : 0.f;
    }
  }
  __syncthreads();  // s_next visible before the dynamic prefix hand-out
  // ---- phase A
  if constexpr (kFastRows<D>) {
    // lane <-> r2; the slot column, Z column and one row's G3 slice live in
    // registers; the row gradient is broadcast through a double-buffered
    // per-warp smem line; the next row's loads are issued before the math.
    constexpr int Xc = FixT<D>::n1 * FixT<D>::n2, NN = Xc * 4, N2c = FixT<D>::n2;
    float* s_gw = s_wk + w * (2 * NN);
    const unsigned m3n3 = g.m3 * 4u;
    // prefixes are handed to warps dynamically (row counts differ per prefix)
    for (;;) {
      int pi = 0;
      if (lane == 0) pi = atomicAdd(&s_next, 1);
      pi = __shfl_sync(0xffffffffu, pi, 0);
      if (pi >= np) break;
      const int slot = s_slot[pi];
      const float* sb = slots + (size_t)slot * (Xc * 32);
      float sbc[Xc], zr[Xc];
#pragma unroll
      for (int x = 0; x < Xc; ++x) {
        sbc[x] = sb[x * 32 + lane];
        zr[x] = 0.f;
      }
      const int u0 = s_u0[pi], u1 = s_u1[pi];
      float ga = 0.f, gb = 0.f;
      float4 hv = make_float4(0.f, 0.f, 0.f, 0.f);
      if (u0 < u1) {
        ga = gU[(size_t)u0 * NN + lane];
        if (NN > 32) gb = gU[(size_t)u0 * NN + 32 + lane];
        hv = __ldg(reinterpret_cast<const float4*>(G3 + (size_t)lane * m3n3 + urow_i3[u0] * 4u));
      }
      int buf = 0;
      for (int u = u0; u < u1; ++u) {
        float* sg = s_gw + buf * NN;
        if (lane < NN) sg[lane] = ga;
        if (NN > 32) sg[32 + lane] = gb;
        const float4 h = hv;
        if (u + 1 < u1) {
          ga = gU[(size_t)(u + 1) * NN + lane];
          if (NN > 32) gb = gU[(size_t)(u + 1) * NN + 32 + lane];
          hv = __ldg(reinterpret_cast<const float4*>(G3 + (size_t)lane * m3n3 + urow_i3[u + 1] * 4u));
        }
        __syncwarp();
        float d0 = 0.f, d1 = 0.f, d2 = 0.f, d3 = 0.f;
#pragma unroll
        for (int x = 0; x < Xc; ++x) {
          const float4 gx = *reinterpret_cast<const float4*>(sg + 4 * x);
          float z = zr[x];
          z = fmaf(gx.x, h.x, z);
          z = fmaf(gx.y, h.y, z);
          z = fmaf(gx.z, h.z, z);
          zr[x] = fmaf(gx.w, h.w, z);
          d0 = fmaf(sbc[x], gx.x, d0);
          d1 = fmaf(sbc[x], gx.y, d1);
          d2 = fmaf(sbc[x], gx.z, d2);
          d3 = fmaf(sbc[x], gx.w, d3);
        }
        *reinterpret_cast<float4*>(dH + (size_t)u * 128 + lane * 4) = make_float4(d0, d1, d2, d3);
        buf ^= 1;
      }
#pragma unroll
      for (int x = 0; x < Xc; ++x) {
        const int a = x / N2c, b = x - a * N2c;
        s_z[(pi * FixT<D>::n1 + a) * LZ + b * 32 + lane] = zr[x];
      }
    }
    for (int e = np * N1 * LZ + threadIdx.x; e < M * LZ; e += kBlock) s_z[e] = 0.f;
  } else {
    float* s_g = s_wk + w * (N + G3S + SL);
    float* s_h = s_g + N;
    float* s_sb = s_h + G3S;
    const unsigned m3n3 = g.m3 * (unsigned)N3;
    for (int pi = w; pi < np; pi += kBlock / 32) {
      const int slot = s_slot[pi];
      const float* sb = slots + (size_t)slot * SL;
      for (int e = lane; e < SL; e += 32) s_sb[e] = sb[e];
      constexpr int KZ = (FixSlot<D>::value + 31) / 32;
      float zr[KZ];
#pragma unroll
      for (int k = 0; k < KZ; ++k) zr[k] = 0.f;
      if constexpr (!IsFixed<D>::value) {
        for (int e = lane; e < SL; e += 32) {
          const int x = e / R2, r = e - x * R2, a = x / N2, b = x - a * N2;
          s_z[(pi * N1 + a) * LZ + b * R2 + r] = 0.f;
        }
      }
      const int u0 = prow_begin[slot], u1 = prow_end[slot];
      for (int u = u0; u < u1; ++u) {
        __syncwarp();
        const unsigned i3 = urow_i3[u];
        for (int e = lane; e < N; e += 32) s_g[e] = gU[(size_t)u * N + e];
        for (int e = lane; e < G3S; e += 32) {
          const int r = e / N3, j = e - r * N3;
          s_h[e] = __ldg(&G3[(size_t)r * m3n3 + i3 * N3 + j]);
        }
        __syncwarp();
        // Z += g . G3^T
        if constexpr (IsFixed<D>::value) {
#pragma unroll
          for (int k = 0; k < KZ; ++k) {
            const int e = lane + 32 * k;
            if (e < SL) {
              const int x = e / R2, r = e - x * R2;
              float acc = zr[k];
#pragma unroll
              for (int j = 0; j < N3; ++j) acc = fmaf(s_g[x * N3 + j], s_h[r * N3 + j], acc);
              zr[k] = acc;
            }
          }
        } else {
          for (int e = lane; e < SL; e += 32) {
            const int x = e / R2, r = e - x * R2, a = x / N2, b = x - a * N2;
            float* zp = &s_z[(pi * N1 + a) * LZ + b * R2 + r];
            float acc = *zp;
            for (int j = 0; j < N3; ++j) acc = fmaf(s_g[x * N3 + j], s_h[r * N3 + j], acc);
            *zp = acc;
          }
        }
        // dH_u = slot^T . g
        for (int e = lane; e < G3S; e += 32) {
          const int r = e / N3, j = e - r * N3;
          float acc = 0.f;
#pragma unroll 4
          for (int x = 0; x < X; ++x) acc = fmaf(s_sb[x * R2 + r], s_g[x * N3 + j], acc);
          dH[(size_t)u * G3S + e] = acc;
        }
      }
      if constexpr (IsFixed<D>::value) {
#pragma unroll
        for (int k = 0; k < KZ; ++k) {
          const int e = lane + 32 * k;
          if (e < SL) {
            const int x = e / R2, r = e - x * R2, a = x / N2, b = x - a * N2;
            s_z[(pi * N1 + a) * LZ + b * R2 + r] = zr[k];
          }
        }
      }
    }
    // rows of the padding prefixes: zero so the GEMMs stay finite
    for (int e = np * N1 * LZ + threadIdx.x; e < M * LZ; e += kBlock) s_z[e] = 0.f;
  }
  __syncthreads();
  // ---- phase B: this chunk's dG2 partial = G1_chunk^T . Z_chunk
  {
    float* part = dG2part + ((size_t)i2 * cmax + chunk) * G2S;
    gemm_kk<Tl::BM, Tl::BN>(R1, C, np * N1, s_g1, R1, s_z, LZ,
                            [&](int m0, int n0, int hm, int hn, float (&acc)[Tl::BM][Tl::BN]) {
#pragma unroll
      for (int i = 0; i < Tl::BM; ++i) {
        float* dst = part + (size_t)split_index<Tl::BM>(m0, hm, i) * C;
        if constexpr (Tl::BN % 4 == 0) {
#pragma unroll
          for (int j = 0; j < Tl::BN; j += 4)
            *reinterpret_cast<float4*>(dst + split_index<Tl::BN>(n0, hn, j)) =
                make_float4(acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < Tl::BN; ++j) dst[n0 + j] = acc[i][j];
        }
      }
    });
  }
  // ---- phase C: E = Z . G2_slice^T
  gemm_nt<Tl::CM, 1, Tl::VEC>(M, R1, C, s_z, LZ, s_g2, LZ, [&](int m0, int n0, float (&acc)[Tl::CM][1]) {
#pragma unroll
    for (int i = 0; i < Tl::CM; ++i) {
      const int row = m0 + i, p = row / N1, a = row - p * N1;
      if (p < np) E[(size_t)s_slot[p] * G1S + a * R1 + n0] = acc[i][0];
    }
  });
  }  // chunk loop
}

// ------------------------------------------------------------ backward, split form
// k_bwd_rows: one warp per distinct prefix (any order, high occupancy):
//   Z_p = sum_u g_u . G3[i3_u]^T  (kept in registers, lane <-> r2) -> Zbuf[slot]
//   dH_u = slot_p^T . g_u                                          -> dH[u]
// k_bwd_gemm: one CTA per (i2, chunk of prefixes): loads the chunk's Z rows
// and runs phases B / C of k_bwd_prefix (dG2 partial, E) without the gather
// phase, so neither kernel's occupancy is set by the other's needs.
template <class D>
__global__ void __launch_bounds__(kBlock) k_bwd_rows(D d, KGeom g, const int* __restrict__ counts,
                                                     const float* __restrict__ G3, const float* __restrict__ slots,
                                                     const int* __restrict__ prow_begin,
                                                     const int* __restrict__ prow_end,
                                                     const unsigned* __restrict__ urow_i3,
                                                     const float* __restrict__ gU, float* __restrict__ dH,
                                                     float* __restrict__ Zbuf) {
  pdl_enter();
  if constexpr (kFastRows<D>) {
    constexpr int Xc = FixT<D>::n1 * FixT<D>::n2, NN = Xc * 4;
    __shared__ __align__(16) float s_g[kBlock / 32][2 * NN];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    float* s_gw = s_g[w];
    const unsigned m3n3 = g.m3 * 4u;
    const int P = counts[1];
    for (int slot = blockIdx.x * (kBlock / 32) + w; slot < P; slot += gridDim.x * (kBlock / 32)) {
      const int u0 = prow_begin[slot], u1 = prow_end[slot];
      const float* sb = slots + (size_t)slot * (Xc * 32);
      float sbc[Xc], zr[Xc];
#pragma unroll
      for (int x = 0; x < Xc; ++x) {
        sbc[x] = sb[x * 32 + lane];
        zr[x] = 0.f;
      }
      float ga = 0.f, gb = 0.f;
      float4 hv = make_float4(0.f, 0.f, 0.f, 0.f);
      if (u0 < u1) {
        ga = gU[(size_t)u0 * NN + lane];
        if (NN > 32) gb = gU[(size_t)u0 * NN + 32 + lane];
        hv = __ldg(reinterpret_cast<const float4*>(G3 + (size_t)lane * m3n3 + urow_i3[u0] * 4u));
      }
      int buf = 0;
      for (int u = u0; u < u1; ++u) {
        float* sg = s_gw + buf * NN;
        if (lane < NN) sg[lane] = ga;
        if (NN > 32) sg[32 + lane] = gb;
        const float4 h = hv;
        if (u + 1 < u1) {
          ga = gU[(size_t)(u + 1) * NN + lane];
          if (NN > 32) gb = gU[(size_t)(u + 1) * NN + 32 + lane];
          hv = __ldg(reinterpret_cast<const float4*>(G3 + (size_t)lane * m3n3 + urow_i3[u + 1] * 4u));
        }
        __syncwarp();
        float d0 = 0.f, d1 = 0.f, d2 = 0.f, d3 = 0.f;
#pragma unroll
        for (int x = 0; x < Xc; ++x) {
          const float4 gx = *reinterpret_cast<const float4*>(sg + 4 * x);
          float z = zr[x];
          z = fmaf(gx.x, h.x, z);
          z = fmaf(gx.y, h.y, z);
          z = fmaf(gx.z, h.z, z);
          zr[x] = fmaf(gx.w, h.w, z);
          d0 = fmaf(sbc[x], gx.x, d0);
          d1 = fmaf(sbc[x], gx.y, d1);
          d2 = fmaf(sbc[x], gx.z, d2);
          d3 = fmaf(sbc[x], gx.w, d3);
        }
        *reinterpret_cast<float4*>(dH + (size_t)u * 128 + lane * 4) = make_float4(d0, d1, d2, d3);
        buf ^= 1;
      }
      // Z stored column-major per prefix: [c = b r2 + r][a] (the n1 = 4 values
      // of a column form one 16-byte unit: a K-major UMMA core-matrix row)
      float4* zo = reinterpret_cast<float4*>(Zbuf + (size_t)slot * (Xc * 32));
      constexpr int N2c = FixT<D>::n2;
      static_assert(FixT<D>::n1 == 4, "Z unit layout assumes n1 = 4");
#pragma unroll
      for (int b = 0; b < N2c; ++b)
        zo[b * 32 + lane] = make_float4(zr[0 * N2c + b], zr[1 * N2c + b], zr[2 * N2c + b], zr[3 * N2c + b]);
    }
  }
}

template <class D>
__global__ void __launch_bounds__(kBlock) k_bwd_gemm(D d, KGeom g, int ch, const float* __restrict__ G1,
                                                     const float* __restrict__ G2, const unsigned* __restrict__ pmap,
                                                     const int* __restrict__ pslot, const float* __restrict__ Zbuf,
                                                     float* __restrict__ E, float* __restrict__ dG2part,
                                                     int* __restrict__ grp_cnt, int cmax) {
  pdl_enter();
  if constexpr (kFastRows<D> && kVecStage<D> && FixT<D>::n1 == 4) {
    extern __shared__ __align__(16) float smem[];
    __shared__ int s_free[kMaxChunk], s_slot[kMaxChunk], s_w[kBlock / 32 + 2];
    constexpr int C = FixT<D>::n2 * FixT<D>::r2, R1 = FixT<D>::r1, N1 = FixT<D>::n1, G1S = N1 * R1;
    constexpr int LZ = C + 4, C4 = C / 4, RQ = R1 / 4, G2S = R1 * C;
    const unsigned i2 = blockIdx.x;
    int np;
    const int total = collect_chunk(pmap, pslot, g, true, i2, blockIdx.y, ch, s_free, s_slot, s_w, &np);
    if (blockIdx.y == 0 && threadIdx.x == 0) grp_cnt[i2] = total;
    if (np == 0) return;
    const int M = ch * N1;
    float* s_z = smem;            // M x LZ
    float* s_g2 = s_z + M * LZ;   // R1 x LZ
    float* s_g1 = s_g2 + R1 * LZ; // M x R1
#pragma unroll 4
    for (int e = threadIdx.x; e < R1 * C4; e += kBlock) {
      const int r = e / C4, c4 = e - r * C4;
      *reinterpret_cast<float4*>(s_g2 + r * LZ + 4 * c4) =
          __ldg(reinterpret_cast<const float4*>(G2 + ((size_t)r * g.m2 + i2) * C) + c4);
    }
#pragma unroll 4
    for (int e = threadIdx.x; e < M * RQ; e += kBlock) {
      const int row = e / RQ, q = e - row * RQ;
      const int p = row / N1, a = row - p * N1;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (p < np) v = __ldg(reinterpret_cast<const float4*>(G1 + ((size_t)s_free[p] * N1 + a) * R1) + q);
      reinterpret_cast<float4*>(s_g1)[e] = v;
    }
    // Z rows: Zbuf[slot] is [c][a] (16-byte unit per column)
#pragma unroll 4
    for (int e = threadIdx.x; e < ch * C; e += kBlock) {
      const int p = e / C, c = e - p * C;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (p < np) v = __ldcg(reinterpret_cast<const float4*>(Zbuf + (size_t)s_slot[p] * (N1 * C)) + c);
      s_z[(p * N1 + 0) * LZ + c] = v.x;
      s_z[(p * N1 + 1) * LZ + c] = v.y;
      s_z[(p * N1 + 2) * LZ + c] = v.z;
      s_z[(p * N1 + 3) * LZ + c] = v.w;
    }
    __syncthreads();
    using Tl = Tiles<D>;
    {
      float* part = dG2part + ((size_t)i2 * cmax + blockIdx.y) * G2S;
      gemm_kk<Tl::BM, Tl::BN>(R1, C, np * N1, s_g1, R1, s_z, LZ,
                              [&](int m0, int n0, int hm, int hn, float (&acc)[Tl::BM][Tl::BN]) {
#pragma unroll
        for (int i = 0; i < Tl::BM; ++i) {
          float* dst = part + (size_t)split_index<Tl::BM>(m0, hm, i) * C;
#pragma unroll
          for (int j = 0; j < Tl::BN; j += 4)
            *reinterpret_cast<float4*>(dst + split_index<Tl::BN>(n0, hn, j)) =
                make_float4(acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]);
        }
      });
    }
    gemm_nt<Tl::CM, 1, Tl::VEC>(M, R1, C, s_z, LZ, s_g2, LZ, [&](int m0, int n0, float (&acc)[Tl::CM][1]) {
#pragma unroll
      for (int i = 0; i < Tl::CM; ++i) {
        const int row = m0 + i, p = row / N1, a = row - p * N1;
        if (p < np) E[(size_t)s_slot[p] * G1S + a * R1 + n0] = acc[i][0];
      }
    });
  }
}

// k_bwd_gemm on the tensor cores (tcgen05 kind::tf32, 3xTF32), for the
// shape with n1 = 4, r1 = 32, n2 r2 = 128 and 16-prefix chunks (64 Z rows):
//   phase B: dG2^T (M = n2 r2 = 128, N = r1, K = 64 rows)  = Z^T . G1_chunk
//   phase C: E     (M = 64 rows,   N = r1, K = n2 r2)      = Z . G2_slice^T
// Both read Z (loaded once into registers) in a different K-major layout, so
// the operands are staged, multiplied and then re-staged in the same smem.
template <class D> constexpr bool kTcBwd = FixT<D>::n1 == 4 && FixT<D>::r1 == 32 && FixT<D>::n2 * FixT<D>::r2 == 128;
constexpr int kTcBwdChunk = 16;

template <class D>
__global__ void __launch_bounds__(kBlock) k_bwd_gemm_tc(D d, KGeom g, const float* __restrict__ G1,
                                                        const float* __restrict__ G2,
                                                        const unsigned* __restrict__ pmap,
                                                        const int* __restrict__ pslot, const float* __restrict__ Zbuf,
                                                        float* __restrict__ E, float* __restrict__ dG2part,
                                                        int* __restrict__ grp_cnt, int cmax) {
  pdl_enter();
  if constexpr (kTcBwd<D>) {
    constexpr int C = 128, R1 = 32, N1 = 4, ROWS = kTcBwdChunk * N1;  // 64
    extern __shared__ __align__(16) float smem[];
    __shared__ int s_free[kMaxChunk], s_slot[kMaxChunk], s_w[kBlock / 32 + 2];
    __shared__ uint64_t s_mbar;
    __shared__ uint32_t s_tmem;
    const unsigned i2 = blockIdx.x;
    int np;
    const int total = collect_chunk(pmap, pslot, g, true, i2, blockIdx.y, kTcBwdChunk, s_free, s_slot, s_w, &np);
    if (blockIdx.y == 0 && threadIdx.x == 0) grp_cnt[i2] = total;
    if (np == 0) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) umma::tmem_alloc(&s_tmem, 64);
    if (threadIdx.x == 32) umma::mbar_init(&s_mbar, 1);
    char* za_hi = reinterpret_cast<char*>(smem);            // Z operand (32 KB) x2
    char* za_lo = za_hi + ROWS * C * 4;
    char* ob_hi = za_lo + ROWS * C * 4;                      // G1 / G2 operand (<= 16 KB) x2
    char* ob_lo = ob_hi + R1 * C * 4;
    // ---- loads, all issued up front. A thread owns (prefix p, column group
    // cg) units: 4 consecutive columns c = 4 cg .. 4 cg + 3, each a float4 of
    // the 4 rows a of prefix p (Zbuf layout [c][a]).
    constexpr int NGZ = kTcBwdChunk * (C / 4) / kBlock;  // 2 (p, cg) groups per thread
    float4 vz[NGZ][4];
#pragma unroll
    for (int i = 0; i < NGZ; ++i) {
      const int e = threadIdx.x + i * kBlock, p = e % kTcBwdChunk, cg = e / kTcBwdChunk;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        vz[i][j] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (p < np) vz[i][j] = __ldcg(reinterpret_cast<const float4*>(Zbuf + (size_t)s_slot[p] * (N1 * C)) + 4 * cg + j);
      }
    }
    // G1 chunk: a thread owns (p, r1 group rg): 4 rows a x 4 r1
    constexpr int NG1 = kTcBwdChunk * (R1 / 4) / kBlock;  // 0.5 -> threads < 128 only
    float4 vg1[4];
    const bool own_g1 = threadIdx.x < kTcBwdChunk * (R1 / 4);
    const int g1p = threadIdx.x % kTcBwdChunk, g1r = threadIdx.x / kTcBwdChunk;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      vg1[a] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (own_g1 && g1p < np)
        vg1[a] = __ldg(reinterpret_cast<const float4*>(G1 + ((size_t)s_free[g1p] * N1 + a) * R1) + g1r);
    }
    (void)NG1;
    constexpr int NG2 = R1 * C / 4 / kBlock;  // 4 float4 of the G2 slice
    float4 vg2[NG2];
#pragma unroll
    for (int i = 0; i < NG2; ++i) {
      const int e = threadIdx.x + i * kBlock, r = e % R1, c4 = e / R1;
      vg2[i] = __ldg(reinterpret_cast<const float4*>(G2 + ((size_t)r * g.m2 + i2) * C) + c4);
    }
    auto put4 = [](char* hi, char* lo, uint32_t off, const float4& v) {
      float4 h, l;
      umma::split3(v.x, h.x, l.x);
      umma::split3(v.y, h.y, l.y);
      umma::split3(v.z, h.z, l.z);
      umma::split3(v.w, h.w, l.w);
      *reinterpret_cast<float4*>(hi + off) = h;
      *reinterpret_cast<float4*>(lo + off) = l;
    };
    // ---- phase B operands (K = Z row = 4 p + a):
    //   A[c][4p + a] : 16-byte unit (k-block p, row c) = the Zbuf unit of column c
    //   B[r][4p + a] : unit (p, r) = G1[p][0..3][r] (register transpose)
#pragma unroll
    for (int i = 0; i < NGZ; ++i) {
      const int e = threadIdx.x + i * kBlock, p = e % kTcBwdChunk, cg = e / kTcBwdChunk;
#pragma unroll
      for (int j = 0; j < 4; ++j) put4(za_hi, za_lo, (uint32_t)((p * C + 4 * cg + j) * 16), vz[i][j]);
    }
    if (own_g1) {
      const float4 t0 = make_float4(vg1[0].x, vg1[1].x, vg1[2].x, vg1[3].x);
      const float4 t1 = make_float4(vg1[0].y, vg1[1].y, vg1[2].y, vg1[3].y);
      const float4 t2 = make_float4(vg1[0].z, vg1[1].z, vg1[2].z, vg1[3].z);
      const float4 t3 = make_float4(vg1[0].w, vg1[1].w, vg1[2].w, vg1[3].w);
      put4(ob_hi, ob_lo, (uint32_t)((g1p * R1 + 4 * g1r + 0) * 16), t0);
      put4(ob_hi, ob_lo, (uint32_t)((g1p * R1 + 4 * g1r + 1) * 16), t1);
      put4(ob_hi, ob_lo, (uint32_t)((g1p * R1 + 4 * g1r + 2) * 16), t2);
      put4(ob_hi, ob_lo, (uint32_t)((g1p * R1 + 4 * g1r + 3) * 16), t3);
    }
    umma::fence_smem_to_async();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = s_tmem;
    if (threadIdx.x == 0) {
      constexpr uint32_t idB = umma::idesc_tf32(128, R1, false, false);
      const char* as[3] = {za_hi, za_hi, za_lo};
      const char* bs[3] = {ob_hi, ob_lo, ob_hi};
#pragma unroll
      for (int s = 0; s < ROWS / 8; ++s)
#pragma unroll
        for (int v = 0; v < 3; ++v)
          umma::mma_tf32(tmem, umma::desc(umma::smem_u32(as[v]) + s * 2 * C * 16, C * 16, 128),
                         umma::desc(umma::smem_u32(bs[v]) + s * 2 * R1 * 16, R1 * 16, 128), idB,
                         (s > 0 || v > 0) ? 1u : 0u);
      umma::commit(&s_mbar);
    }
    umma::mbar_wait(&s_mbar, 0);  // phase B done reading smem
    umma::fence_after_sync();
    // ---- phase C operands (K = column c):
    //   A[4p + a][c] : unit (k-block cg, row 4p + a) = Z[4p + a][4cg .. 4cg + 3]
    //   B[r][c]      : unit (cg, r) = G2[r][4cg .. 4cg + 3]
#pragma unroll
    for (int i = 0; i < NGZ; ++i) {
      const int e = threadIdx.x + i * kBlock, p = e % kTcBwdChunk, cg = e / kTcBwdChunk;
      const float4 a0 = make_float4(vz[i][0].x, vz[i][1].x, vz[i][2].x, vz[i][3].x);
      const float4 a1 = make_float4(vz[i][0].y, vz[i][1].y, vz[i][2].y, vz[i][3].y);
      const float4 a2 = make_float4(vz[i][0].z, vz[i][1].z, vz[i][2].z, vz[i][3].z);
      const float4 a3 = make_float4(vz[i][0].w, vz[i][1].w, vz[i][2].w, vz[i][3].w);
      put4(za_hi, za_lo, (uint32_t)((cg * ROWS + 4 * p + 0) * 16), a0);
      put4(za_hi, za_lo, (uint32_t)((cg * ROWS + 4 * p + 1) * 16), a1);
      put4(za_hi, za_lo, (uint32_t)((cg * ROWS + 4 * p + 2) * 16), a2);
      put4(za_hi, za_lo, (uint32_t)((cg * ROWS + 4 * p + 3) * 16), a3);
    }
#pragma unroll
    for (int i = 0; i < NG2; ++i) {
      const int e = threadIdx.x + i * kBlock, r = e % R1, c4 = e / R1;
      put4(ob_hi, ob_lo, (uint32_t)((c4 * R1 + r) * 16), vg2[i]);
    }
    umma::fence_smem_to_async();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    if (threadIdx.x == 0) {
      constexpr uint32_t idC = umma::idesc_tf32(ROWS, R1, false, false);
      const char* as[3] = {za_hi, za_hi, za_lo};
      const char* bs[3] = {ob_hi, ob_lo, ob_hi};
#pragma unroll
      for (int s = 0; s < C / 8; ++s)
#pragma unroll
        for (int v = 0; v < 3; ++v)
          umma::mma_tf32(tmem + 32, umma::desc(umma::smem_u32(as[v]) + s * 2 * ROWS * 16, ROWS * 16, 128),
                         umma::desc(umma::smem_u32(bs[v]) + s * 2 * R1 * 16, R1 * 16, 128), idC,
                         (s > 0 || v > 0) ? 1u : 0u);
      umma::commit(&s_mbar);
    }
    umma::mbar_wait(&s_mbar, 1);
    umma::fence_after_sync();
    // ---- epilogue: warps 0-3 drain dG2^T (lane = c), warps 4-7 drain E
    // (M = 64: rows 16q .. 16q + 15 sit in lanes 0..15 of lane quarter q)
    const int q = warp & 3;
    if (warp < 4) {
      float v[32];
      umma::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16), v);
      float* part = dG2part + ((size_t)i2 * cmax + blockIdx.y) * (R1 * C);
      const int c = 32 * q + lane;
#pragma unroll
      for (int r = 0; r < R1; ++r) part[r * C + c] = v[r];
    } else {
      float v[32];
      umma::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + 32, v);
      const int zrow = 16 * q + lane, p = zrow / N1, a = zrow % N1;
      if (lane < 16 && p < np) {
        float* dst = E + (size_t)s_slot[p] * (N1 * R1) + a * R1;
#pragma unroll
        for (int r = 0; r < R1; r += 4)
          *reinterpret_cast<float4*>(dst + r) = make_float4(v[r], v[r + 1], v[r + 2], v[r + 3]);
      }
    }
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_free(tmem, 64);
  }
}

// Persistent form of k_bwd_gemm_tc: one CTA per (i2, split). The group's
// present prefixes are enumerated once, the G2 slice (phase C B operand) is
// staged once, and dG2^T accumulates in TMEM over all of the CTA's chunks
// (chunks split, split + nsplit, ...), so each CTA writes ONE dG2 partial.
constexpr int kMaxGroup = 512;  // prefixes per i2 group enumerated in smem (m1 <= 512)

template <class D>
__global__ void __launch_bounds__(kBlock) k_bwd_gemm_tc2(D d, KGeom g, const float* __restrict__ G1,
                                                         const float* __restrict__ G2,
                                                         const unsigned* __restrict__ pmap,
                                                         const int* __restrict__ pslot,
                                                         const float* __restrict__ Zbuf, float* __restrict__ E,
                                                         float* __restrict__ dG2part, int* __restrict__ grp_cnt) {
  pdl_enter();
  if constexpr (kTcBwd<D>) {
    constexpr int C = 128, R1 = 32, N1 = 4, CH = kTcBwdChunk, ROWS = CH * N1;  // 64
    extern __shared__ __align__(16) float smem[];
    __shared__ int s_free[kMaxGroup], s_slot[kMaxGroup], s_w[kBlock / 32 + 2];
    __shared__ uint64_t s_mbar;
    __shared__ uint32_t s_tmem;
    const unsigned i2 = blockIdx.x;
    const int split = blockIdx.y, nsplit = gridDim.y;
    int dummy;
    const int total = collect_chunk(pmap, pslot, g, true, i2, 0, kMaxGroup, s_free, s_slot, s_w, &dummy);
    if (split == 0 && threadIdx.x == 0) grp_cnt[i2] = total;
    const int nch = (total + CH - 1) / CH;
    if (split >= nch) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) umma::tmem_alloc(&s_tmem, 64);
    if (threadIdx.x == 32) umma::mbar_init(&s_mbar, 1);
    char* za_hi = reinterpret_cast<char*>(smem);  // Z operand, 32 KB each
    char* za_lo = za_hi + ROWS * C * 4;
    char* g1_hi = za_lo + ROWS * C * 4;           // G1 chunk operand, 8 KB each
    char* g1_lo = g1_hi + ROWS * R1 * 4;
    char* g2_hi = g1_lo + ROWS * R1 * 4;          // G2 slice operand, 16 KB each
    char* g2_lo = g2_hi + R1 * C * 4;
    auto put4 = [](char* hi, char* lo, uint32_t off, const float4& v) {
      float4 h, l;
      umma::split3(v.x, h.x, l.x);
      umma::split3(v.y, h.y, l.y);
      umma::split3(v.z, h.z, l.z);
      umma::split3(v.w, h.w, l.w);
      *reinterpret_cast<float4*>(hi + off) = h;
      *reinterpret_cast<float4*>(lo + off) = l;
    };
    {  // G2 slice, once: B[r][c] unit (cg, r) = G2[r][4cg .. 4cg + 3]
      constexpr int NG2 = R1 * C / 4 / kBlock;
#pragma unroll
      for (int i = 0; i < NG2; ++i) {
        const int e = threadIdx.x + i * kBlock, r = e % R1, c4 = e / R1;
        put4(g2_hi, g2_lo, (uint32_t)((c4 * R1 + r) * 16),
             __ldg(reinterpret_cast<const float4*>(G2 + ((size_t)r * g.m2 + i2) * C) + c4));
      }
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = s_tmem;
    uint32_t phase = 0;
    constexpr int NGZ = CH * (C / 4) / kBlock;  // 2 (p, cg) groups per thread
    const bool own_g1 = threadIdx.x < CH * (R1 / 4);
    const int g1p = threadIdx.x % CH, g1r = threadIdx.x / CH;
    bool first = true;
    for (int chunk = split; chunk < nch; chunk += nsplit) {
      const int p0 = chunk * CH, np = min(CH, total - p0);
      // ---- loads for this chunk
      float4 vz[NGZ][4], vg1[4];
#pragma unroll
      for (int i = 0; i < NGZ; ++i) {
        const int e = threadIdx.x + i * kBlock, p = e % CH, cg = e / CH;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          vz[i][j] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (p < np)
            vz[i][j] = __ldcg(reinterpret_cast<const float4*>(Zbuf + (size_t)s_slot[p0 + p] * (N1 * C)) + 4 * cg + j);
        }
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        vg1[a] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (own_g1 && g1p < np)
          vg1[a] = __ldg(reinterpret_cast<const float4*>(G1 + ((size_t)s_free[p0 + g1p] * N1 + a) * R1) + g1r);
      }
      // ---- phase B operands
#pragma unroll
      for (int i = 0; i < NGZ; ++i) {
        const int e = threadIdx.x + i * kBlock, p = e % CH, cg = e / CH;
#pragma unroll
        for (int j = 0; j < 4; ++j) put4(za_hi, za_lo, (uint32_t)((p * C + 4 * cg + j) * 16), vz[i][j]);
      }
      if (own_g1) {
        put4(g1_hi, g1_lo, (uint32_t)((g1p * R1 + 4 * g1r + 0) * 16), make_float4(vg1[0].x, vg1[1].x, vg1[2].x, vg1[3].x));
        put4(g1_hi, g1_lo, (uint32_t)((g1p * R1 + 4 * g1r + 1) * 16), make_float4(vg1[0].y, vg1[1].y, vg1[2].y, vg1[3].y));
        put4(g1_hi, g1_lo, (uint32_t)((g1p * R1 + 4 * g1r + 2) * 16), make_float4(vg1[0].z, vg1[1].z, vg1[2].z, vg1[3].z));
        put4(g1_hi, g1_lo, (uint32_t)((g1p * R1 + 4 * g1r + 3) * 16), make_float4(vg1[0].w, vg1[1].w, vg1[2].w, vg1[3].w));
      }
      umma::fence_smem_to_async();
      umma::fence_before_sync();
      __syncthreads();
      umma::fence_after_sync();
      if (threadIdx.x == 0) {
        constexpr uint32_t idB = umma::idesc_tf32(128, R1, false, false);
        const char* as[3] = {za_hi, za_hi, za_lo};
        const char* bs[3] = {g1_hi, g1_lo, g1_hi};
#pragma unroll
        for (int s = 0; s < ROWS / 8; ++s)
#pragma unroll
          for (int v = 0; v < 3; ++v)
            umma::mma_tf32(tmem, umma::desc(umma::smem_u32(as[v]) + s * 2 * C * 16, C * 16, 128),
                           umma::desc(umma::smem_u32(bs[v]) + s * 2 * R1 * 16, R1 * 16, 128), idB,
                           (!first || s > 0 || v > 0) ? 1u : 0u);
        umma::commit(&s_mbar);
      }
      first = false;
      umma::mbar_wait(&s_mbar, phase);
      phase ^= 1u;
      umma::fence_after_sync();
      // ---- phase C operand (Z with K = c); G2 operand is resident
#pragma unroll
      for (int i = 0; i < NGZ; ++i) {
        const int e = threadIdx.x + i * kBlock, p = e % CH, cg = e / CH;
        put4(za_hi, za_lo, (uint32_t)((cg * ROWS + 4 * p + 0) * 16), make_float4(vz[i][0].x, vz[i][1].x, vz[i][2].x, vz[i][3].x));
        put4(za_hi, za_lo, (uint32_t)((cg * ROWS + 4 * p + 1) * 16), make_float4(vz[i][0].y, vz[i][1].y, vz[i][2].y, vz[i][3].y));
        put4(za_hi, za_lo, (uint32_t)((cg * ROWS + 4 * p + 2) * 16), make_float4(vz[i][0].z, vz[i][1].z, vz[i][2].z, vz[i][3].z));
        put4(za_hi, za_lo, (uint32_t)((cg * ROWS + 4 * p + 3) * 16), make_float4(vz[i][0].w, vz[i][1].w, vz[i][2].w, vz[i][3].w));
      }
      umma::fence_smem_to_async();
      umma::fence_before_sync();
      __syncthreads();
      umma::fence_after_sync();
      if (threadIdx.x == 0) {
        constexpr uint32_t idC = umma::idesc_tf32(ROWS, R1, false, false);
        const char* as[3] = {za_hi, za_hi, za_lo};
        const char* bs[3] = {g2_hi, g2_lo, g2_hi};
#pragma unroll
        for (int s = 0; s < C / 8; ++s)
#pragma unroll
          for (int v = 0; v < 3; ++v)
            umma::mma_tf32(tmem + 32, umma::desc(umma::smem_u32(as[v]) + s * 2 * ROWS * 16, ROWS * 16, 128),
                           umma::desc(umma::smem_u32(bs[v]) + s * 2 * R1 * 16, R1 * 16, 128), idC,
                           (s > 0 || v > 0) ? 1u : 0u);
        umma::commit(&s_mbar);
      }
      umma::mbar_wait(&s_mbar, phase);
      phase ^= 1u;
      umma::fence_after_sync();
      // ---- E rows of this chunk (M = 64: rows 16q .. 16q + 15 in lanes 0..15 of quarter q)
      if (warp >= 4) {
        const int q = warp & 3;
        float v[32];
        umma::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + 32, v);
        const int zrow = 16 * q + lane, p = zrow / N1, a = zrow % N1;
        if (lane < 16 && p < np) {
          float* dst = E + (size_t)s_slot[p0 + p] * (N1 * R1) + a * R1;
#pragma unroll
          for (int r = 0; r < R1; r += 4)
            *reinterpret_cast<float4*>(dst + r) = make_float4(v[r], v[r + 1], v[r + 2], v[r + 3]);
        }
      }
      umma::fence_before_sync();
      __syncthreads();  // E drained before the next chunk's MMA C; smem free for restaging
      umma::fence_after_sync();
    }
    // ---- this CTA's dG2 partial (accumulated over its chunks): lane = c
    if (warp < 4) {
      const int q = warp;
      float v[32];
      umma::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16), v);
      float* part = dG2part + ((size_t)i2 * nsplit + split) * (R1 * C);
      const int c = 32 * q + lane;
#pragma unroll
      for (int r = 0; r < R1; ++r) part[r * C + c] = v[r];
    }
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_free(tmem, 64);
  }
}

}  // namespace ttb
