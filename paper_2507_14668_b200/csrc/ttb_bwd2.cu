// Tensor-core pipeline backward, v2.
//
// Reference: tt_core_grads (backward.py:101-183) in the regrouped schedule of
// SURVEY.md §8a row 17, for n = (4, 4, 4), ranks (1, 32, 32, 1). Per work
// item (<= 32 lookups of one prefix p = (i1, i2)) and lookup l (bag, i3):
//   X_p      = G1[i1] . G2[:, i2]                 (a, b, s)      tensor core
//   dG3[i3] += X_p^T g_l                          (s, j)         SIMT, red
//   Z_p     += g_l (x) G3[:, i3]                  (a, b, s)      SIMT
//   dG2[i2] += G1[i1]^T Z_p,  dG1[i1] += Z_p G2[i2]^T            tensor core
// where g_l = grad_out[bag] as (a, b, j); a, b, j < 4, s < 32 (= r2).
//
// X^T is formed in TMEM with lanes (s, b) = 4 s + b and columns (item, a).
// The SIMT phase works on item QUADS: the four lanes 4 s' + c of a warp load
// the quad's 16 columns of their TMEM lanes and swap 4-value blocks (a 4 x 4
// block transpose, two butterfly shuffle stages) so that lane (s, k) holds
// X[item k][a][b][s] for all 16 (a, b) — every lookup then costs each thread
// 16 broadcast shared loads of its gradient row, 64 FMA for dG3 (complete,
// no cross-lane reduction, one red.v4) and 64 FMA for Z. At the end of the
// quad the inverse transpose turns the Z registers back into Z^T (the A
// operand of the dG2 GEMM, TMEM), and each lane writes its rows of the Z
// image (rows (item, a), K = (s, b): the A operand of E = Z G2^T) — both as
// split tf32 (hi + lo; 3 products = fp32-level accuracy).
//
// The G2 slice is staged once per i2 from the fp32 core: as the TMEM A
// operand of X^T (lanes (s, b), columns r) and as the K-major B operand of E.
// 16 warps: warp w takes TMEM lane quarter w % 4 and quads w / 4, w / 4 + 4.
#include <stdlib.h>

#include "ttb_fast.cuh"

namespace ttb {
namespace fast {
namespace bw2 {

constexpr int kThreads = 512;
// TMEM columns (512)
constexpr uint32_t kColA = 0;     // G2 slice, X^T A operand: r hi [0, 32) | r lo [32, 64)
constexpr uint32_t kColX = 64;    // X^T: (item, a) 128 columns; then E (64 columns)
constexpr uint32_t kColZH = 192;  // Z^T hi: (item, a)
constexpr uint32_t kColZL = 320;  // Z^T lo
constexpr uint32_t kColD2 = 448;  // dG2 accumulator: r hi [0, 32) | r lo [32, 64)
// shared memory (SW128 images 1024-aligned)
constexpr int kOffZH = 0;           // Z image hi: rows (item, a), K = (s, b): 4 blocks x 16 KB;
                                    // before the SIMT phase: G1 rows hi | lo (the X^T B operand)
constexpr int kOffZL = 4 * kImg;    // Z image lo
constexpr int kOffG2K = 8 * kImg;   // G2 image: rows r hi 0..31 | lo 32..63, K = (s, b): 4 blocks x 8 KB
constexpr int kOffG1T = 10 * kImg;  // G1^T image (dG2 B operand): rows r hi | lo, K = (item, a)
constexpr int kOffSt = 12 * kImg;   // staged grad_out rows, item-major
constexpr int kStCap = 128;         // positions per staged chunk (one quad of full items)
constexpr int kStBytes = kStCap * 256 + 8 * 128;  // + per-item bank offsets
constexpr int kSmem = kOffSt + kStBytes + 1024;

// staged-row byte offset of item it's first position: rows of 256 B, shifted
// so that the four items of a quad start in different 32-byte bank groups
// (their rows are read by the same load instruction)
__device__ __forceinline__ int st_item_base(int pos_rel, int it, int c_lo) {
  return pos_rel * 256 + 32 * (it & 3) + 128 * ((it - c_lo) >> 2);
}

// chunks of whole quads of <= cap positions: ch[k] = first item of chunk k (one thread)
__device__ inline int make_chunks(const TileMeta* m, int* ch, int cap) {
  int nc = 0, it = 0;
  ch[0] = 0;
  while (it < m->n) {
    const int base = m->start[it];
    int e = it;
    while (e < m->n) {
      const int nx = e + 4 < m->n ? e + 4 : m->n;
      if (m->start[nx] - base > cap) break;
      e = nx;
    }
    it = e;
    ch[++nc] = it;
  }
  return nc;
}

// items [c_lo, c_hi): each position's grad_out row into its item-major slot
// (cp.async; warp w takes items c_lo + w, c_lo + w + 16)
__device__ inline void stage_chunk(const TileMeta* m, int c_lo, int c_hi, const int2* __restrict__ sbi,
                                   const float* __restrict__ gout, char* st) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cp0 = m->start[c_lo];
  for (int it = c_lo + warp; it < c_hi; it += kThreads / 32) {
    const int p0 = m->start[it], len = m->start[it + 1] - p0;
    char* dst = st + st_item_base(p0 - cp0, it, c_lo);
#pragma unroll 4
    for (int e = lane; e < len * 16; e += 32) {
      const int p = e >> 4, k = e & 15;
      const int bag = __ldg(&sbi[p0 + p].x);
      cp_async16(dst + p * 256 + 16 * k, gout + (size_t)bag * NOUT + 4 * k);
    }
  }
}

// 4 x 4 transpose of 4-value blocks across the lanes 4 s' + c of a warp:
// v[4 k + e] of lane c  ->  v[4 c + e] of lane k
__device__ __forceinline__ void transpose4(float (&v)[16], int c) {
  const bool c0 = c & 1, c1 = (c >> 1) & 1;
#pragma unroll
  for (int k1 = 0; k1 < 2; ++k1)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float& lo = v[(2 * k1) * 4 + e];
      float& hi = v[(2 * k1 + 1) * 4 + e];
      const float r = __shfl_xor_sync(0xffffffffu, c0 ? lo : hi, 1);
      if (c0) lo = r;
      else hi = r;
    }
#pragma unroll
  for (int k0 = 0; k0 < 2; ++k0)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float& lo = v[k0 * 4 + e];
      float& hi = v[(2 + k0) * 4 + e];
      const float r = __shfl_xor_sync(0xffffffffu, c1 ? lo : hi, 2);
      if (c1) lo = r;
      else hi = r;
    }
}

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// 3xTF32 split by truncation: hi = x with the low 13 mantissa bits cleared
// (exactly representable in tf32), lo = x - hi, the exact residual (< 2^-10 x,
// itself read by the tensor core to ~2^-11 of its value), so
// hi.hi + hi.lo + lo.hi carries x to ~2^-21 relative. Two instructions per
// value instead of the two round-to-nearest conversions of umma::split3.
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
__device__ __forceinline__ float tf32_lo(float x) { return x - tf32_hi(x); }

__global__ void __launch_bounds__(kThreads, 1)
    k_bwd2(KGeom g, const float* __restrict__ g1img, const float* __restrict__ G2, const float* __restrict__ G3,
           const int4* __restrict__ tile_info, const int* __restrict__ item_start,
           const unsigned* __restrict__ item_key, const int2* __restrict__ sbi, const float* __restrict__ gout,
           float* __restrict__ dG1, float* __restrict__ dG2, float* __restrict__ dG3, int* __restrict__ hdr,
           const int* __restrict__ cta_tiles, int dbg) {
  pdl_enter();
  // per-phase SM cycles (thread 0 of block 0, summed over its tiles) into
  // hdr[16..] as u64: [0] tiles, [k] phase k (TTB_DBG & 8; tools/bwd_stamps.py)
  long long t_last = 0;
  long long t_acc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long t_q = 0;  // SIMT sub-phases: [9] quad setup, [10] lookups, [11] quad epilogue
#define QSTAMP(k)                           \
  do {                                      \
    if (stamp) {                            \
      const long long _t = clock64();       \
      if ((k) > 0) t_acc[k] += _t - t_q;    \
      t_q = _t;                             \
    }                                       \
  } while (0)
  const bool stamp = (dbg & 8) && threadIdx.x == 0 && blockIdx.x == 0;
#define BSTAMP(k)                           \
  do {                                      \
    if (stamp) {                            \
      const long long _t = clock64();       \
      if ((k) > 0) t_acc[k] += _t - t_last; \
      t_last = _t;                          \
    }                                       \
  } while (0)
  extern __shared__ __align__(16) char smem_raw[];
  char* sm = smem_raw + ((1024u - (umma::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ TileMeta s_m[2];
  __shared__ int s_chunk[2][kTileItems / 4 + 2];
  __shared__ int s_nchunk[2];
  __shared__ uint64_t s_mbar[3];
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, grp = warp >> 2;
  const int c4 = lane & 3;            // b when loading X^T, the quad item after the transpose
  const int s = 8 * q + (lane >> 2);  // TMEM lane 32 q + lane = 4 s + c4
  const unsigned m2 = g.m2, m3 = g.m3;
  const int tb = cta_tiles[blockIdx.x], te = cta_tiles[blockIdx.x + 1];
  char* zh = sm + kOffZH;
  char* zl = sm + kOffZL;
  char* g2k = sm + kOffG2K;
  char* g1t = sm + kOffG1T;
  char* st = sm + kOffSt;
  if (warp == 0) umma::tmem_alloc(&s_tmem, 512);
  if (threadIdx.x == 32) {
    umma::mbar_init(&s_mbar[0], 1);  // X^T formed
    umma::mbar_init(&s_mbar[1], 1);  // E formed
    umma::mbar_init(&s_mbar[2], 1);  // dG2 accumulated
  }
  int4 pf = make_int4(0, 0, 0, 0);
  if (warp == 15 && tb < te) {
    fetch_meta_async(tile_info[tb], item_start, item_key, &s_m[0]);
    if (tb + 1 < te) pf = tile_info[tb + 1];
    cp_async_wait_all();
    __syncwarp();
    if (lane == 0) s_nchunk[0] = make_chunks(&s_m[0], s_chunk[0], kStCap);
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const float* g3s = G3 + (size_t)s * m3 * 4;  // G3[s, ., .] / dG3[s, ., .]: this thread's s
  float* d3s = dG3 + (size_t)s * m3 * 4;
  const uint32_t tmem = s_tmem;
  const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16);  // this warp's lane quarter
  const uint64_t d_zh = umma::desc_sw128(umma::smem_u32(zh)), d_zl = umma::desc_sw128(umma::smem_u32(zl));
  const uint64_t d_g2k = umma::desc_sw128(umma::smem_u32(g2k));
  const uint64_t d_g1h = d_zh, d_g1l = umma::desc_sw128(umma::smem_u32(zh + kImg));  // G1 rows, in the Z region
  const uint64_t d_g1t = umma::desc_sw128(umma::smem_u32(g1t));
  uint32_t ph_x = 0, ph_e = 0, ph_d = 0;
  int bad = 0, slot = 0, prev_i2 = -1;
  // operands of X^T for tile mt: the G2 slice when i2 changes (TMEM A operand
  // and E's B image) and the items' G1 rows (hi | lo) in the Z region
  auto stage_x = [&](const TileMeta* mt, int prev) {
    if (mt->i2 != prev) {
      // warp (q, grp): r in [8 grp, 8 grp + 8) of lanes (s, b)
      const unsigned i2x = mt->i2;
      float hv[8], lv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int r = 8 * grp + j;
        const float v = __ldg(G2 + ((size_t)(r * m2 + i2x) * 4 + c4) * 32 + s);
        hv[j] = tf32_hi(v);
        lv[j] = v - hv[j];
        *reinterpret_cast<float*>(g2k + umma::sw128_off(r, 4 * s + c4, 64)) = hv[j];
        *reinterpret_cast<float*>(g2k + umma::sw128_off(32 + r, 4 * s + c4, 64)) = lv[j];
      }
      umma::tmem_st8(tq + kColA + 8 * grp, hv);
      umma::tmem_st8(tq + kColA + 32 + 8 * grp, lv);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {  // rows (item, a), K = r: four whole 128-byte rows per warp
      const int e = threadIdx.x + i * kThreads, ia = e >> 3, kq = e & 7, it = ia >> 2, a = ia & 3;
      if (it < mt->n) {
        const float* src = g1img + (size_t)item_i1(mt, it, g) * kG1Img + a * 32 + 4 * kq;
        const uint32_t o = umma::sw128_off(ia, 4 * kq, 128);
        cp_async16(zh + o, src);
        cp_async16(zh + kImg + o, src + 128);
      }
    }
  };
  auto issue_x = [&]() {  // X^T[(s, b), (item, a)] = sum_r G2[r, b, s] G1[i1, a, r]
    if (threadIdx.x == 0) {
      constexpr uint32_t id = umma::idesc_tf32(128, 128, false, false);
#pragma unroll
      for (int k0 = 0; k0 < R1; k0 += 8) {
        const uint32_t bo = (uint32_t)(k0 * 4) >> 4;
        umma::mma_tf32_ta(tmem + kColX, tmem + kColA + k0, d_g1h + bo, id, k0 > 0 ? 1u : 0u);
        umma::mma_tf32_ta(tmem + kColX, tmem + kColA + k0, d_g1l + bo, id, 1u);
        umma::mma_tf32_ta(tmem + kColX, tmem + kColA + 32 + k0, d_g1h + bo, id, 1u);
      }
      umma::commit(&s_mbar[0]);
    }
  };
  if (tb < te) {  // the first tile's X^T operands and first chunk of gradient rows
    stage_x(&s_m[0], -1);
    cp_async_commit();
    stage_chunk(&s_m[0], 0, s_chunk[0][1], sbi, gout, st);
    cp_async_wait_all();
    umma::tmem_wait_st();
    sync_for_mma();
    issue_x();
  }
  for (int t = tb; t < te; ++t, slot ^= 1) {
    const TileMeta* m = &s_m[slot];
    const int n = m->n, i2 = m->i2;
    BSTAMP(0);
    if (warp == 15 && t + 1 < te) {  // next tile's metadata into the other slot
      fetch_meta_async(pf, item_start, item_key, &s_m[slot ^ 1]);
      if (t + 2 < te) pf = tile_info[t + 2];
    }
    umma::mbar_wait(&s_mbar[0], ph_x);  // X^T of this tile (and the previous tile's dG2 GEMM)
    ph_x ^= 1u;
    umma::fence_after_sync();
    BSTAMP(1);
    // G1^T image (rows r hi | lo, K = (item, a)) for the dG2 GEMM; zero past n.
    // Lane <-> item: a warp writes whole 128-byte row segments.
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int e = threadIdx.x + i * kThreads, it = e & 31, k = e >> 5;
      const uint32_t oh = umma::sw128_off(k, 4 * it, 64), ol = umma::sw128_off(32 + k, 4 * it, 64);
      if (it < n) {
        const float* src = g1img + (size_t)item_i1(m, it, g) * kG1Img + 256 + 4 * k;
        cp_async16(g1t + oh, src);
        cp_async16(g1t + ol, src + 128);
      } else {
        *reinterpret_cast<float4*>(g1t + oh) = make_float4(0.f, 0.f, 0.f, 0.f);
        *reinterpret_cast<float4*>(g1t + ol) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    cp_async_commit();
    if (warp == 15 && t + 1 < te) {
      // the next tile's gradient rows into L2 now, so that their staging during
      // this tile's GEMMs does not wait on HBM
      cp_async_wait_all();
      __syncwarp();
      const TileMeta* mn = &s_m[slot ^ 1];
      const int pa = mn->start[0], pb = mn->start[mn->n];
      for (int p = pa + lane; p < pb && p < pa + kStCap; p += 32)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(gout + (size_t)__ldg(&sbi[p].x) * NOUT));
    }
    BSTAMP(2);
    // ---- SIMT phase: item quads, chunk by chunk of staged gradient rows
    // (chunk 0 was staged during the previous tile's GEMMs)
    const int* chunk = s_chunk[slot];
    const int nchunk = s_nchunk[slot];
    for (int c = 0; c < nchunk; ++c) {
      const int c_lo = chunk[c], c_hi = chunk[c + 1];
      const int cp0 = m->start[c_lo];
      if (c > 0) {
        __syncthreads();  // the previous chunk's rows are consumed
        stage_chunk(m, c_lo, c_hi, sbi, gout, st);
        cp_async_wait_all();
        __syncthreads();
      }
      // this lane's item of quad qq: positions [p_, p_ + l_)
      auto quad_item = [&](int qq, int& p_, int& l_) {
        const int it = 4 * qq + c4;
        if (it < c_hi) {
          p_ = m->start[it];
          l_ = m->start[it + 1] - p_;
        } else {
          p_ = 0;
          l_ = 0;
        }
      };
      int qd = (c_lo >> 2) + grp, ps, len;
      quad_item(qd, ps, len);
      // i3 two positions ahead and G3[s, i3, :] one ahead (L2 latency); the
      // next quad's first ones are fetched during this quad
      int i3c = len > 0 ? __ldg(&sbi[ps].y) : 0;
      int i3n = len > 1 ? __ldg(&sbi[ps + 1].y) : 0;
      float4 hn = len > 0 ? ldg4(g3s + (size_t)i3c * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
      for (; 4 * qd < c_hi; qd += 4) {
        QSTAMP(0);
        const int it0 = 4 * qd, my_it = it0 + c4;
        int ps2, len2;
        quad_item(qd + 4, ps2, len2);
        const int j3c = len2 > 0 ? __ldg(&sbi[ps2].y) : 0;
        const int j3n = len2 > 1 ? __ldg(&sbi[ps2 + 1].y) : 0;
        int maxlen = len;
        maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, 1));
        maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, 2));
        float w[16];  // after the transpose: w[4 b + a] = X[my_it][a][b][s]
        {
          uint32_t r[16];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
              "[%16];"
              : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                "=r"(r[15])
              : "r"(tq + kColX + 16 * qd));
          umma::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) w[i] = __uint_as_float(r[i]);  // w[4 k + a] = X[it0 + k][a][b = c4][s]
        }
        transpose4(w, c4);
        float z[16];  // z[4 a + b] = Z[my_it][a][b][s]
#pragma unroll
        for (int i = 0; i < 16; ++i) z[i] = 0.f;
        const char* row = st + st_item_base(ps - cp0, my_it, c_lo);
        QSTAMP(9);
        for (int stp = 0; stp < maxlen; ++stp) {
          if (stp < len) {
            const float4 h = hn;
            const int i3 = i3c;
            if (stp + 1 < len) {
              hn = ldg4(g3s + (size_t)i3n * 4);
              i3c = i3n;
              if (stp + 2 < len) i3n = __ldg(&sbi[ps + stp + 2].y);
            }
            const float4* gr = reinterpret_cast<const float4*>(row + stp * 256);
            float d0 = 0.f, d1 = 0.f, d2 = 0.f, d3 = 0.f;
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int bb = 0; bb < 4; ++bb) {
                const float4 gv = gr[4 * a + bb];  // g[a][bb][0..3]
                const float x = w[4 * bb + a];
                d0 = fmaf(x, gv.x, d0);
                d1 = fmaf(x, gv.y, d1);
                d2 = fmaf(x, gv.z, d2);
                d3 = fmaf(x, gv.w, d3);
                float& zz = z[4 * a + bb];
                zz = fmaf(gv.x, h.x, fmaf(gv.y, h.y, fmaf(gv.z, h.z, fmaf(gv.w, h.w, zz))));
              }
            red_v4(d3s + (size_t)i3 * 4, d0, d1, d2, d3);
          }
        }
        QSTAMP(10);
        const float4 jn = len2 > 0 ? ldg4(g3s + (size_t)j3c * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
        bad |= !isfinite(((z[0] + z[5]) + (z[10] + z[15])) + ((z[3] + z[6]) + (z[9] + z[12])));
        // Z image rows (my_it, a): K = (s, b) = 4 s + b, four consecutive b per row
        if (my_it < c_hi) {
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const uint32_t o = umma::sw128_off(4 * my_it + a, 4 * s, 128);
            *reinterpret_cast<float4*>(zh + o) = make_float4(tf32_hi(z[4 * a]), tf32_hi(z[4 * a + 1]),
                                                             tf32_hi(z[4 * a + 2]), tf32_hi(z[4 * a + 3]));
            *reinterpret_cast<float4*>(zl + o) = make_float4(tf32_lo(z[4 * a]), tf32_lo(z[4 * a + 1]),
                                                             tf32_lo(z[4 * a + 2]), tf32_lo(z[4 * a + 3]));
          }
        }
        // Z^T: blocks by b -> lane b holds Z[it0 + k][a][b][s] at [4 k + a]
        float th[16], tl[16];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int bb = 0; bb < 4; ++bb) th[4 * bb + a] = z[4 * a + bb];
        transpose4(th, c4);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float v = th[i];
          th[i] = tf32_hi(v);
          tl[i] = v - th[i];
        }
        umma::tmem_st16(tq + kColZH + 16 * qd, th);
        umma::tmem_st16(tq + kColZL + 16 * qd, tl);
        QSTAMP(11);
        ps = ps2;
        len = len2;
        i3c = j3c;
        i3n = j3n;
        hn = jn;
      }
    }
    // quads past the last item: zero Z^T columns (the dG2 GEMM sums over all 128)
    {
      float zero16[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) zero16[i] = 0.f;
      const int nq = (n + 3) >> 2;
      for (int qd = nq + ((grp - nq) & 3); qd < kTileItems / 4; qd += 4) {
        umma::tmem_st16(tq + kColZH + 16 * qd, zero16);
        umma::tmem_st16(tq + kColZL + 16 * qd, zero16);
      }
    }
    BSTAMP(3);
    umma::tmem_wait_st();
    cp_async_wait_all();  // the G1^T image (warp 15: the next tile's metadata)
    if (warp == 15 && t + 1 < te) {
      __syncwarp();
      if (lane == 0) s_nchunk[slot ^ 1] = make_chunks(&s_m[slot ^ 1], s_chunk[slot ^ 1], kStCap);
    }
    sync_for_mma();
    BSTAMP(4);
    if (threadIdx.x == 0) {
      constexpr uint32_t id64 = umma::idesc_tf32(128, 64, false, false);
      constexpr uint32_t id32 = umma::idesc_tf32(128, 32, false, false);  // B rows 0-31: the hi half
      // E [(item, a), r hi | r lo] = sum_(s, b) (Z hi + Z lo) . G2^T  (into the dead X^T columns)
#pragma unroll
      for (int k0 = 0; k0 < 128; k0 += 8) {
        const uint32_t ao = (uint32_t)((k0 >> 5) * 128 * 128 + (k0 & 31) * 4) >> 4;
        const uint32_t bo = (uint32_t)((k0 >> 5) * 64 * 128 + (k0 & 31) * 4) >> 4;
        umma::mma_tf32(tmem + kColX, d_zh + ao, d_g2k + bo, id64, k0 > 0 ? 1u : 0u);
        umma::mma_tf32(tmem + kColX, d_zl + ao, d_g2k + bo, id32, 1u);
      }
      umma::commit(&s_mbar[1]);
      // dG2^T tile [(s, b), r hi | r lo] += sum_(item, a) (Z^T hi + Z^T lo) . G1^T;
      // it runs on while the epilogue reads E and the next tile's X^T forms
      const bool acc2 = i2 == prev_i2;  // same i2 as the previous tile: keep accumulating
#pragma unroll
      for (int k0 = 0; k0 < 128; k0 += 8) {
        const uint32_t bo = (uint32_t)((k0 >> 5) * 64 * 128 + (k0 & 31) * 4) >> 4;
        umma::mma_tf32_ta(tmem + kColD2, tmem + kColZH + k0, d_g1t + bo, id64, (acc2 || k0 > 0) ? 1u : 0u);
        umma::mma_tf32_ta(tmem + kColD2, tmem + kColZL + k0, d_g1t + bo, id32, 1u);
      }
      umma::commit(&s_mbar[2]);
    }
    // next tile: its first chunk of gradient rows streams in (the SIMT phase
    // is done with the staging)
    if (t + 1 < te) {
      stage_chunk(&s_m[slot ^ 1], 0, s_chunk[slot ^ 1][1], sbi, gout, st);
      cp_async_commit();
    }
    BSTAMP(5);
    umma::mbar_wait(&s_mbar[1], ph_e);
    ph_e ^= 1u;
    umma::fence_after_sync();
    BSTAMP(6);
    // ---- epilogue: dG1 rows from E (lanes (item, a)); warp (q, grp) takes r in [8 grp, 8 grp + 8)
    {
      uint32_t vh[8], vl[8];
      umma::tmem_ld8_nw(tq + kColX + 8 * grp, vh);
      umma::tmem_ld8_nw(tq + kColX + 32 + 8 * grp, vl);
      umma::tmem_wait_ld();
      const int row = 32 * q + lane, it = row >> 2, a = row & 3;
      if (it < n) {
        float* d1 = dG1 + ((size_t)item_i1(m, it, g) * 4 + a) * R1 + 8 * grp;
#pragma unroll
        for (int i = 0; i < 8; i += 4)
          red_v4(d1 + i, __uint_as_float(vh[i]) + __uint_as_float(vl[i]),
                 __uint_as_float(vh[i + 1]) + __uint_as_float(vl[i + 1]),
                 __uint_as_float(vh[i + 2]) + __uint_as_float(vl[i + 2]),
                 __uint_as_float(vh[i + 3]) + __uint_as_float(vl[i + 3]));
      }
    }
    // dG2[r][i2][b][s], once per run of tiles of one i2
    const bool flush = t + 1 >= te || s_m[slot ^ 1].i2 != i2;
    if (flush) {
      umma::mbar_wait(&s_mbar[2], ph_d);
      umma::fence_after_sync();
      uint32_t vh[8], vl[8];
      umma::tmem_ld8_nw(tq + kColD2 + 8 * grp, vh);
      umma::tmem_ld8_nw(tq + kColD2 + 32 + 8 * grp, vl);
      umma::tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int r = 8 * grp + j;
        red_f32(dG2 + ((size_t)(r * m2 + i2) * 4 + c4) * 32 + s, __uint_as_float(vh[j]) + __uint_as_float(vl[j]));
      }
    }
    ph_d ^= 1u;  // one dG2 commit per tile (waited only when flushed; never two phases ahead)
    // the next tile's X^T operands (E and, on an i2 change, the dG2 GEMM are done)
    if (t + 1 < te) stage_x(&s_m[slot ^ 1], i2);
    prev_i2 = i2;
    cp_async_wait_all();
    umma::tmem_wait_st();
    sync_for_mma();  // E read; staged operands visible to the tensor core
    if (t + 1 < te) issue_x();
    BSTAMP(7);
  }
#undef BSTAMP
#undef QSTAMP
  if (stamp) {
    t_acc[0] = te - tb;
    for (int k = 0; k < 12; ++k) reinterpret_cast<long long*>(hdr + 16)[k] = t_acc[k];
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&hdr[0], TTB_ERRBIT_NONFINITE);
  if (warp == 0) umma::tmem_free(tmem, 512);
}

}  // namespace bw2
}  // namespace fast

cudaError_t launch_bwd2(ttb_handle* h, const float* c1, const float* c2, const float* gout, float* g0, float* g1,
                        float* g2, cudaStream_t s) {
  using namespace fast;
  Workspace& w = h->w;
  cudaError_t e;
  if ((e = ensure_kernel_smem((const void*)bw2::k_bwd2, bw2::kSmem))) return e;
  e = launch_pdl(bw2::k_bwd2, dim3(h->num_sms), dim3(bw2::kThreads), bw2::kSmem, s, h->kg, (const float*)w.f_g1img,
                 c1, c2, (const int4*)w.f_tile_info, (const int*)w.f_item_start, (const unsigned*)w.f_item_key,
                 (const int2*)w.f_sbi, gout, g0, g1, g2, w.fast_hdr, (const int*)w.f_cta,
                 getenv("TTB_DBG") ? atoi(getenv("TTB_DBG")) : 0);
  return e;
}

}  // namespace ttb
