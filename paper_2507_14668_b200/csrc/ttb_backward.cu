// K2/K3 forward and K4/K5 backward launchers + the deterministic reductions.
#include "ttb_kernels.cuh"

namespace ttb {

// ---------------------------------------------------------------- row runs
// Over the index positions sorted by row: row heads (-> distinct rows U, in
// ascending row order) and prefix runs (-> the rows of each slot).
__global__ void __launch_bounds__(kBlock) k_runs(const unsigned* __restrict__ skeys, int T, KGeom g,
                                                 const int* __restrict__ pslot, unsigned* __restrict__ urow,
                                                 int* __restrict__ urow_start, unsigned* __restrict__ urow_i3,
                                                 int* __restrict__ prow_begin, int* __restrict__ prow_end,
                                                 int* __restrict__ qrow, int* __restrict__ counts,
                                                 unsigned long long* status, unsigned* ctr) {
  pdl_enter();
  __shared__ int s_tile;
  __shared__ int s_tmp[kItems * (kBlock / 32) + 2];
  const int tile = claim_tile(ctr, &s_tile);
  const int base = tile * kTile;
  bool f[kItems];
  unsigned key[kItems];
  bool ph[kItems], pl[kItems];
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int q = base + k * kBlock + threadIdx.x;
    f[k] = ph[k] = pl[k] = false;
    key[k] = 0;
    if (q < T) {
      key[k] = skeys[q];
      const unsigned pk = key[k] / g.m3;
      if (q == 0) {
        f[k] = ph[k] = true;
      } else {
        const unsigned prev = skeys[q - 1];
        f[k] = prev != key[k];
        ph[k] = (prev / g.m3) != pk;
      }
      pl[k] = (q == T - 1) || (skeys[q + 1] / g.m3 != pk);
    }
  }
  int rank[kItems];
  long long incl;
  tile_flag_scan(f, rank, status, tile, s_tmp, &incl);
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int q = base + k * kBlock + threadIdx.x;
    if (q >= T) continue;
    const int u = rank[k] + (f[k] ? 1 : 0) - 1;
    qrow[q] = u;
    if (f[k]) {
      urow[u] = key[k];
      urow_start[u] = q;
      urow_i3[u] = key[k] % g.m3;
    }
    if (ph[k] || pl[k]) {
      const int slot = pslot[key[k] / g.m3];
      if (ph[k]) prow_begin[slot] = u;
      if (pl[k]) prow_end[slot] = u + 1;
    }
  }
  if (tile == (T + kTile - 1) / kTile - 1 && threadIdx.x == 0) {
    counts[3] = (int)incl;
    urow_start[incl] = T;
  }
}

// ---------------------------------------------------------------- reductions
// All three are deterministic: each output element is a sum in a fixed order
// (warps own contiguous ranges of the summands; their partials are combined
// in warp order), and the SGD(+momentum) step is applied by the thread that
// produced the final gradient.
constexpr int kRedWarps = kBlock / 32;

// i3_start[v] = first position of digit v among the i3-sorted rows: every
// boundary between consecutive sorted keys fills the digits it skips.
__global__ void k_i3_bounds(const unsigned* __restrict__ k3, const int* __restrict__ counts, int m3,
                            int* __restrict__ i3_start) {
  pdl_enter();
  const int U = counts[3];
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q <= U; q += gridDim.x * blockDim.x) {
    const int prev = q > 0 ? (int)k3[q - 1] : -1;
    const int cur = q < U ? (int)k3[q] : m3;
    for (int v = prev + 1; v <= cur; ++v) i3_start[v] = q;
  }
}


// One launch for the G1 and G3 reductions: blocks [0, m1) reduce dG1 rows,
// blocks [m1, m1 + m3) reduce dG3 columns. Warp w owns a contiguous run of
// the summands; warp partials are combined in warp order (deterministic), and
// the SGD step is applied by the thread holding the final gradient.
constexpr int kRedPerLane = 16;  // fallback: G1S, G3S <= 32 * kRedPerLane

// dG1[i1] = sum of E over the present prefixes (i1, i2), ascending i2; the
// block also resets its row of the prefix table for the next batch's plan.
__device__ inline void dg1_block(KGeom g, int G1S, unsigned i1, unsigned* __restrict__ pmap,
                                 const int* __restrict__ pslot, const float* __restrict__ E, float* s_part) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int per = ((int)g.m2 + kRedWarps - 1) / kRedWarps;
  const int a = w * per, b = min((int)g.m2, a + per);
  const bool vec = G1S == 128;
  float4 acc4 = make_float4(0.f, 0.f, 0.f, 0.f);
  float acc[kRedPerLane];
#pragma unroll
  for (int i = 0; i < kRedPerLane; ++i) acc[i] = 0.f;
  for (int base = a; base < b; base += 32) {
    const int i2 = base + lane;
    int sl = -1;
    unsigned key = 0;
    if (i2 < b) {
      key = i1 * g.m2 + (unsigned)i2;
      if (pmap[key] != kEmpty) sl = pslot[key];
    }
    unsigned m = __ballot_sync(0xffffffffu, sl >= 0);
    if (sl >= 0) pmap[key] = kEmpty;  // consumed: clean for the next plan
    while (m) {
      if (vec) {
        float4 v[8];
        int sls[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          sls[k] = -1;
          if (m) {
            const int src = __ffs(m) - 1;
            m &= m - 1;
            sls[k] = __shfl_sync(0xffffffffu, sl, src);
          }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (sls[k] >= 0) v[k] = reinterpret_cast<const float4*>(E + (size_t)sls[k] * 128)[lane];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (sls[k] >= 0) {
            acc4.x += v[k].x;
            acc4.y += v[k].y;
            acc4.z += v[k].z;
            acc4.w += v[k].w;
          }
      } else {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const int slot = __shfl_sync(0xffffffffu, sl, src);
        const float* row = E + (size_t)slot * G1S;
#pragma unroll
        for (int q = 0; q < kRedPerLane; ++q)
          if (lane + 32 * q < G1S) acc[q] += row[lane + 32 * q];
      }
    }
  }
  if (vec) {
    reinterpret_cast<float4*>(s_part + w * G1S)[lane] = acc4;
  } else {
#pragma unroll
    for (int q = 0; q < kRedPerLane; ++q)
      if (lane + 32 * q < G1S) s_part[w * G1S + lane + 32 * q] = acc[q];
  }
}

// dG3[:, i3] = sum of dH over the rows with that last digit, in row order.
__device__ inline void dg3_block(int G3S, unsigned v, const int* __restrict__ i3_start,
                                 const unsigned* __restrict__ v3, const float* __restrict__ dH, float* s_part) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int k0 = i3_start[v], k1 = i3_start[v + 1];
  const int per = (k1 - k0 + kRedWarps - 1) / kRedWarps;
  const int a = k0 + w * per, b = min(k1, a + per);
  const bool vec = G3S == 128;
  float4 acc4 = make_float4(0.f, 0.f, 0.f, 0.f);
  float acc[kRedPerLane];
#pragma unroll
  for (int i = 0; i < kRedPerLane; ++i) acc[i] = 0.f;
  for (int base = a; base < b; base += 32) {
    const int myk = base + lane;
    const unsigned myu = myk < b ? v3[myk] : 0u;
    const int cnt = min(32, b - base);
    if (vec) {
      for (int i0 = 0; i0 < cnt; i0 += 8) {
        float4 r[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const unsigned u = __shfl_sync(0xffffffffu, myu, (i0 + k) & 31);
          if (i0 + k < cnt) r[k] = reinterpret_cast<const float4*>(dH + (size_t)u * 128)[lane];
        }
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (i0 + k < cnt) {
            acc4.x += r[k].x;
            acc4.y += r[k].y;
            acc4.z += r[k].z;
            acc4.w += r[k].w;
          }
      }
    } else {
      for (int i = 0; i < cnt; ++i) {
        const unsigned u = __shfl_sync(0xffffffffu, myu, i);
        const float* row = dH + (size_t)u * G3S;
#pragma unroll
        for (int q = 0; q < kRedPerLane; ++q)
          if (lane + 32 * q < G3S) acc[q] += row[lane + 32 * q];
      }
    }
  }
  if (vec) {
    reinterpret_cast<float4*>(s_part + w * G3S)[lane] = acc4;
  } else {
#pragma unroll
    for (int q = 0; q < kRedPerLane; ++q)
      if (lane + 32 * q < G3S) s_part[w * G3S + lane + 32 * q] = acc[q];
  }
}

// dG2[:, i2] = sum of the group's chunk partials in chunk order; one thread
// per 4 consecutive slice elements (float4), kBlock*4 elements per block.
__device__ inline void dg2_part(KGeom g, int C, int G2S, int nsplit, int ch, unsigned i2, int q,
                                const float* __restrict__ part, const int* __restrict__ grp_cnt,
                                const int* __restrict__ err, float* __restrict__ grad, float* __restrict__ param,
                                double* __restrict__ vel, double lr, double mu, int do_update) {
  int nch = (grp_cnt[i2] + ch - 1) / ch;  // chunks (or CTAs) that wrote a partial
  if (nch > nsplit) nch = nsplit;
  const bool upd = do_update && ((*err & 8) == 0);
  const int e0 = (q * kBlock + threadIdx.x) * 4;
  if (e0 >= G2S) return;
  const float* base = part + (size_t)i2 * nsplit * G2S;
  if (G2S % 4 == 0 && C % 4 == 0) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int c = 0;
    for (; c + 4 <= nch; c += 4) {
      float4 v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = __ldcg(reinterpret_cast<const float4*>(base + (size_t)(c + k) * G2S + e0));
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc.x += v[k].x;
        acc.y += v[k].y;
        acc.z += v[k].z;
        acc.w += v[k].w;
      }
    }
    for (; c < nch; ++c) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(base + (size_t)c * G2S + e0));
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    const int r = e0 / C, cc = e0 - r * C;
    const size_t gi = ((size_t)r * g.m2 + i2) * C + cc;
    const float a[4] = {acc.x, acc.y, acc.z, acc.w};
    if (grad) *reinterpret_cast<float4*>(grad + gi) = acc;
    if (upd) {
      float4 p = *reinterpret_cast<const float4*>(param + gi);
      float* pp = &p.x;
#pragma unroll
      for (int k = 0; k < 4; ++k) pp[k] = sgd_apply(pp[k], a[k], vel ? vel + gi + k : nullptr, lr, mu);
      *reinterpret_cast<float4*>(param + gi) = p;
    }
  } else {
    for (int e = e0; e < e0 + 4 && e < G2S; ++e) {
      float acc = 0.f;
      for (int c = 0; c < nch; ++c) acc += base[(size_t)c * G2S + e];
      const int r = e / C, cc = e - r * C;
      const size_t gi = ((size_t)r * g.m2 + i2) * C + cc;
      if (grad) grad[gi] = acc;
      if (upd) param[gi] = sgd_apply(param[gi], acc, vel ? vel + gi : nullptr, lr, mu);
    }
  }
}

__global__ void __launch_bounds__(kBlock) k_dg13_reduce(KGeom g, int G1S, int N3, int G3S, unsigned* __restrict__ pmap,
                                                        const int* __restrict__ pslot, const float* __restrict__ E,
                                                        const int* __restrict__ i3_start,
                                                        const unsigned* __restrict__ v3, const float* __restrict__ dH,
                                                        const int* __restrict__ err, float* __restrict__ grad0,
                                                        float* __restrict__ param0, double* __restrict__ vel0,
                                                        int upd0, float* __restrict__ grad2,
                                                        float* __restrict__ param2, double* __restrict__ vel2,
                                                        int upd2, double lr, double mu, int C, int G2S, int nsplit,
                                                        int ch, const float* __restrict__ part,
                                                        const int* __restrict__ grp_cnt, float* __restrict__ grad1,
                                                        float* __restrict__ param1, double* __restrict__ vel1,
                                                        int upd1) {
  pdl_enter();
  extern __shared__ __align__(16) float s_part[];  // kRedWarps x max(G1S, G3S)
  if (blockIdx.x >= g.m1 + g.m3) {
    const int qpb = (G2S + 4 * kBlock - 1) / (4 * kBlock);
    const int k = blockIdx.x - (g.m1 + g.m3);
    dg2_part(g, C, G2S, nsplit, ch, (unsigned)(k / qpb), k % qpb, part, grp_cnt, err, grad1, param1, vel1, lr, mu,
             upd1);
    return;
  }
  const bool is1 = blockIdx.x < g.m1;
  const int G = is1 ? G1S : G3S;
  if (is1) dg1_block(g, G1S, blockIdx.x, pmap, pslot, E, s_part);
  else dg3_block(G3S, blockIdx.x - g.m1, i3_start, v3, dH, s_part);
  __syncthreads();
  const bool ok = (*err & 8) == 0;
  const unsigned v = blockIdx.x - g.m1;
  const unsigned m3n3 = g.m3 * (unsigned)N3;
  for (int e = threadIdx.x; e < G; e += kBlock) {
    float acc = 0.f;
#pragma unroll
    for (int ww = 0; ww < kRedWarps; ++ww) acc += s_part[ww * G + e];
    if (is1) {
      const size_t gi = (size_t)blockIdx.x * G1S + e;
      if (grad0) grad0[gi] = acc;
      if (upd0 && ok) param0[gi] = sgd_apply(param0[gi], acc, vel0 ? vel0 + gi : nullptr, lr, mu);
    } else {
      const int r = e / N3, j = e - r * N3;
      const size_t gi = (size_t)r * m3n3 + v * N3 + j;
      if (grad2) grad2[gi] = acc;
      if (upd2 && ok) param2[gi] = sgd_apply(param2[gi], acc, vel2 ? vel2 + gi : nullptr, lr, mu);
    }
  }
}

__global__ void k_sgd(float* __restrict__ p, const float* __restrict__ gr, double* __restrict__ v, int64_t n,
                      double lr, double mu, const int* __restrict__ err) {
  pdl_enter();
  if (err && *(volatile const int*)err != 0) return;  // a latched error cancels the update
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = sgd_apply(p[i], gr[i], v ? v + i : nullptr, lr, mu);
}

__global__ void k_adagrad(float* __restrict__ p, const float* __restrict__ gr, double* __restrict__ st, int64_t n,
                          double lr, double eps, const int* __restrict__ err) {
  pdl_enter();
  if (err && *(volatile const int*)err != 0) return;  // a latched error cancels the update
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = adagrad_apply(p[i], gr[i], st + i, lr, eps);
}

cudaError_t launch_adagrad(float* p, const float* g, double* st, int64_t n, double lr, double eps, cudaStream_t s,
                           const int* err) {
  if (n <= 0) return cudaSuccess;
  int64_t grid = (n + kBlock - 1) / kBlock;
  if (grid > 148 * 8) grid = 148 * 8;
  launch_pdl(k_adagrad, dim3((int)grid), dim3(kBlock), 0, s, p, g, st, n, lr, eps, err);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_sgd(float* p, const float* g, double* v, int64_t n, double lr, double mu, cudaStream_t s,
                       const int* err) {
  if (n <= 0) return cudaSuccess;
  int64_t grid = (n + kBlock - 1) / kBlock;
  if (grid > 148 * 8) grid = 148 * 8;
  launch_pdl(k_sgd, dim3((int)grid), dim3(kBlock), 0, s, p, g, v, n, lr, mu, err);
  count_launch();
  return cudaGetLastError();
}

// several parameters in one launch: a thread's element i of the packed range
// belongs to the last tensor whose start is <= i (<= kSgdMulti tensors)
struct SgdMulti {
  float* p[kSgdMulti];
  const float* g[kSgdMulti];
  double* v[kSgdMulti];
  int64_t start[kSgdMulti + 1];
  int count;
};
__global__ void k_sgd_multi(SgdMulti a, double lr, double mu) {
  pdl_enter();
  const int64_t total = a.start[a.count];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = a.count - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (a.start[mid] <= i) lo = mid;
      else hi = mid - 1;
    }
    const int64_t j = i - a.start[lo];
    a.p[lo][j] = sgd_apply(a.p[lo][j], a.g[lo][j], a.v[lo] ? a.v[lo] + j : nullptr, lr, mu);
  }
}

cudaError_t launch_sgd_multi(const ttb_sgd_tensor* t, int count, double lr, double mu, cudaStream_t s) {
  for (int b = 0; b < count; b += kSgdMulti) {
    SgdMulti a = {};
    a.count = count - b < kSgdMulti ? count - b : kSgdMulti;
    for (int k = 0; k < a.count; ++k) {
      a.p[k] = t[b + k].param;
      a.g[k] = t[b + k].grad;
      a.v[k] = t[b + k].velocity;
      a.start[k + 1] = a.start[k] + t[b + k].n;
    }
    if (a.start[a.count] == 0) continue;
    int64_t grid = (a.start[a.count] + kBlock - 1) / kBlock;
    if (grid > 148 * 8) grid = 148 * 8;
    cudaError_t e = launch_pdl(k_sgd_multi, dim3((int)grid), dim3(kBlock), 0, s, a, lr, mu);
    if (e) return e;
    count_launch();
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------- dispatch
template <class D>
static size_t prefix_smem(const D& d, int ch) {
  return sizeof(float) * ((size_t)d.r1 * dC(d) + (size_t)d.r1 * ch * d.n1);
}
template <class D>
static size_t close_smem(const D& d) {
  size_t per = (size_t)close_warp_floats(d);
  const size_t fast = 136 + (size_t)kSegGroup * 128;  // G3 staging + per-segment H sums (k_close_multi)
  if (kFastRows<D>) per = per > fast ? per : fast;
  return sizeof(float) * (kBlock / 32) * per;
}
template <class D>
static size_t bwd_smem(const D& d, int ch) {
  const size_t M = (size_t)ch * d.n1, LZ = pad_ld(d);
  const size_t per_warp = kFastRows<D> ? 2 * (size_t)dN(d) : (size_t)dN(d) + dG3s(d) + dSlot(d);
  return sizeof(float) * (M * LZ + (size_t)d.r1 * LZ + M * d.r1 + (kBlock / 32) * per_warp);
}

// cudaFuncSetAttribute once per (kernel, size): it is a host-side call that
// would otherwise sit on every launch path.
template <class K>
static cudaError_t ensure_smem(K kernel, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  return ensure_kernel_smem((const void*)kernel, bytes);
}

template <class D>
static cudaError_t forward_impl(ttb_handle* h, const float* c0, const float* c1, const float* c2, float* out,
                                cudaStream_t s) {
  const D d = make_dims<D>(h->dims);
  Workspace& w = h->w;
  cudaError_t e;
  if constexpr (kTcPrefix<D>) {
    // tensor-core path (tcgen05 kind::tf32, 3xTF32)
    constexpr int R1 = FixT<D>::r1, C = FixT<D>::n2 * FixT<D>::r2;
    const size_t smt = sizeof(float) * ((size_t)2 * 128 * R1 + (size_t)2 * C * R1);
    const size_t sms = sizeof(float) * (size_t)128 * (C + 4);
    const size_t smtc = smt > sms ? smt : sms;
    if ((e = ensure_smem(k_prefix_products_tc<D>, smtc))) return e;
    dim3 gt(h->kg.m2, (unsigned)((h->kg.m1 + kTcChunk - 1) / kTcChunk));
    ProfScope _ps(h, s, "prefix_products_tc");
    launch_pdl(k_prefix_products_tc<D>, dim3(gt), dim3(kBlock), smtc, s, d, h->kg, c0, c1, w.pmap, w.pslot, w.slots);
  } else
  { const size_t sm1 = prefix_smem(d, h->chf);
  if ((e = ensure_smem(k_prefix_products<D>, sm1))) return e;
  dim3 g1(h->kg.m2, (unsigned)h->nsplitf);
  ProfScope _ps(h, s, "prefix_products");
  launch_pdl(k_prefix_products<D>, dim3(g1), dim3(kBlock), sm1, s, d, h->kg, h->chf, c0, c1, w.pmap, w.pslot, w.slots);
  }
  count_launch();
  const size_t sm2 = close_smem(d);
  if ((e = ensure_smem(k_close_pool<D>, sm2))) return e;
  const int B = (int)h->B;
  int grid = (B + kBlock / 32 - 1) / (kBlock / 32);
  if (grid > 148 * 32) grid = 148 * 32;
  { ProfScope _ps(h, s, "close_pool");
  launch_pdl(k_close_pool<D>, dim3(grid), dim3(kBlock), sm2, s, d, h->kg, c2, w.slots, w.bag_off, w.bag_seg, w.seg_slot, w.seg_inv, w.occ_slot,
                                            w.keys32, B, out);
  }
  count_launch();
  if (kFastRows<D> && FixT<D>::n1 * FixT<D>::n2 == 16) {
    if ((e = ensure_smem(k_close_multi<D>, sm2))) return e;
    int gridm = (B + kBlock / 32 - 1) / (kBlock / 32);
    if (gridm > 148 * 16) gridm = 148 * 16;
    ProfScope _ps(h, s, "close_multi");
    launch_pdl(k_close_multi<D>, dim3(gridm), dim3(kBlock), sm2, s, d, h->kg, c2, w.slots, w.bag_off, w.bag_seg, w.seg_slot, w.seg_inv,
                                                w.occ_slot, w.keys32, B, w.counts, out);
    count_launch();
  }
  return cudaGetLastError();
}

template <class D>
static cudaError_t aggregate_impl(ttb_handle* h, const float* gout, cudaStream_t s) {
  const D d = make_dims<D>(h->dims);
  Workspace& w = h->w;
  const int T = (int)h->T;
  cudaError_t e;
  if (!h->bwd_zeroed && (e = cudaMemsetAsync(w.zeroB, 0, w.zeroB_bytes, s))) return e;
  h->bwd_zeroed = 0;
  // 1. order the indices by row (stable: equal rows keep index order)
  unsigned *sk, *sv;
  if ((e = launch_sort(h, w.keys32, nullptr, w.skA, w.svA, w.skB, w.svB, nullptr, T, h->idx_bits, 0, &sk, &sv, s)))
    return e;
  // 2. row / prefix runs
  const int tiles = (T + kTile - 1) / kTile;
  { ProfScope _ps(h, s, "runs");
  launch_pdl(k_runs, dim3(tiles), dim3(kBlock), 0, s, sk, T, h->kg, w.pslot, w.urow, w.urow_start, w.urow_i3, w.prow_begin, w.prow_end,
                                  w.qrow, w.counts, w.runs_status, w.runs_ctr);
  }
  count_launch();
  // 3. aggregated row gradients (two-level segmented reduction)
  {
    const int nblk = (T + kAggBlock - 1) / kAggBlock;
    int grid = (nblk + kBlock / 32 - 1) / (kBlock / 32);
    if (grid > 148 * 16) grid = 148 * 16;
    ProfScope _ps(h, s, "row_agg");
    launch_pdl(k_row_agg<D>, dim3(grid), dim3(kBlock), 0, s, d, (int)h->B, T, w.counts, w.urow_start, w.qrow, sv, w.bag_of, gout, w.gU,
                                         w.agg_hp, w.agg_tp, w.span_list, reinterpret_cast<int*>(w.runs_ctr + 8), w.err);
  }
  {
    int grid = (T / kAggBlock) + 1;
    if (grid > 148 * 8) grid = 148 * 8;
    ProfScope _ps(h, s, "row_agg_span");
    launch_pdl(k_row_agg_span<D>, dim3(grid), dim3(kBlock), sizeof(float) * (kBlock / 32) * dN(d), s, 
        d, w.urow_start, w.span_list, reinterpret_cast<int*>(w.runs_ctr + 8), w.agg_hp, w.agg_tp, w.gU, w.err);
  }
  count_launch(2);
  return cudaGetLastError();
}

template <class D>
static cudaError_t backward_impl(ttb_handle* h, const float* c0, const float* c1, const float* c2, const float* gout,
                                 float* g0, float* g1, float* g2, float* p0, float* p1, float* p2, double* v0,
                                 double* v1, double* v2, double lr, double mu, int mask, int mode, cudaStream_t s) {
  const D d = make_dims<D>(h->dims);
  Workspace& w = h->w;
  const int T = (int)h->T;
  cudaError_t e;
  if ((e = aggregate_impl<D>(h, gout, s))) return e;
  // 4. per-prefix contractions, grouped by i2
  h->dg2_slots = h->cmaxb;
  // The split form (k_bwd_rows + k_bwd_gemm[_tc2]) is kept selectable: on
  // B200 at config 2 it measured 42 + 105 us (SIMT GEMM) / 42 + 156 us
  // (tcgen05, unpipelined) against 125 us for the fused k_bwd_prefix, so the
  // fused kernel is the default until the tensor-core GEMM is pipelined.
  if (h->bwd_split && kFastRows<D> && kVecStage<D> && FixT<D>::n1 == 4) {
    // split form: warp-per-prefix Z / dH, then the i2-chunk GEMMs
    {
      int grid = (int)((h->Pmax + kBlock / 32 - 1) / (kBlock / 32));
      if (grid > 148 * 8) grid = 148 * 8;
      ProfScope _ps(h, s, "bwd_rows");
      launch_pdl(k_bwd_rows<D>, dim3(grid), dim3(kBlock), 0, s, d, h->kg, (const int*)w.counts, c2,
                 (const float*)w.slots, (const int*)w.prow_begin, (const int*)w.prow_end,
                 (const unsigned*)w.urow_i3, (const float*)w.gU, w.dH, w.zbuf);
    }
    if (kTcBwd<D> && h->chb == kTcBwdChunk && h->kg.m1 <= (unsigned)kMaxGroup) {
      // persistent tensor-core form: ~2 CTAs per SM across the i2 groups
      const size_t smt = (size_t)2 * 64 * 128 * 4 + (size_t)2 * 64 * 32 * 4 + (size_t)2 * 32 * 128 * 4;
      if ((e = ensure_smem(k_bwd_gemm_tc2<D>, smt))) return e;
      int ns = (int)((2 * 148 + h->kg.m2 - 1) / h->kg.m2);
      if (ns > h->cmaxb) ns = h->cmaxb;
      if (ns < 1) ns = 1;
      h->dg2_slots = ns;
      dim3 gp(h->kg.m2, (unsigned)ns);
      ProfScope _ps(h, s, "bwd_gemm_tc");
      launch_pdl(k_bwd_gemm_tc2<D>, gp, dim3(kBlock), smt, s, d, h->kg, c0, c1, (const unsigned*)w.pmap,
                 (const int*)w.pslot, (const float*)w.zbuf, w.E, w.dG2part, w.grp_cnt);
    } else {
      const size_t smg = sizeof(float) * ((size_t)h->chb * d.n1 * (dC(d) + 4) + (size_t)d.r1 * (dC(d) + 4) +
                                          (size_t)h->chb * d.n1 * d.r1);
      if ((e = ensure_smem(k_bwd_gemm<D>, smg))) return e;
      dim3 gp(h->kg.m2, (unsigned)h->nsplitb);
      ProfScope _ps(h, s, "bwd_gemm");
      launch_pdl(k_bwd_gemm<D>, gp, dim3(kBlock), smg, s, d, h->kg, h->chb, c0, c1, (const unsigned*)w.pmap,
                 (const int*)w.pslot, (const float*)w.zbuf, w.E, w.dG2part, w.grp_cnt, h->cmaxb);
    }
    count_launch(2);
  } else {
  const size_t sm = bwd_smem(d, h->chb);
  if ((e = ensure_smem(k_bwd_prefix<D>, sm))) return e;
  dim3 gp(h->kg.m2, (unsigned)h->nsplitb);
  { ProfScope _ps(h, s, "bwd_prefix");
  launch_pdl(k_bwd_prefix<D>, dim3(gp), dim3(kBlock), sm, s, d, h->kg, h->chb, c0, c1, c2, w.pmap, w.pslot, w.slots, w.prow_begin, w.prow_end,
                                         w.urow_i3, w.gU, w.dH, w.E, w.dG2part, w.grp_cnt,
                                         h->cmaxb);
  }
  count_launch();
  }
  // 5. rows by last digit for the G3 reduction
  unsigned *k3, *v3;
  if ((e = launch_sort(h, w.urow_i3, nullptr, w.rkA, w.rvA, w.rkB, w.rvB, w.counts + 3, T, h->i3_bits, 1, &k3, &v3,
                       s)))
    return e;
  { ProfScope _ps(h, s, "i3_bounds");
  launch_pdl(k_i3_bounds, dim3((T + kBlock) / kBlock), dim3(kBlock), 0, s, k3, w.counts, (int)h->kg.m3, w.i3_start);
  }
  count_launch();
  const bool upd = mode == 1;
  // 6. reductions (+ fused update)
  {
    ProfScope _ps(h, s, "dg123_reduce");
    const size_t smr = sizeof(float) * kRedWarps * (dG1s(d) > dG3s(d) ? dG1s(d) : dG3s(d));
    const int qpb = (dG2s(d) + 4 * kBlock - 1) / (4 * kBlock);
    launch_pdl(k_dg13_reduce, dim3(h->kg.m1 + h->kg.m3 + h->kg.m2 * qpb), dim3(kBlock), smr, s,
        h->kg, dG1s(d), d.n3, dG3s(d), w.pmap, w.pslot, w.E, w.i3_start, v3, w.dH, w.err, upd ? nullptr : g0, p0, v0,
        upd && (mask & 1), upd ? nullptr : g2, p2, v2, upd && (mask & 4), lr, mu, dC(d), dG2s(d), h->dg2_slots, h->chb,
        w.dG2part, w.grp_cnt, upd ? nullptr : g1, p1, v1, upd && (mask & 2));
  }
  count_launch(1);
  return cudaGetLastError();
}

// Shapes with compiled-in dims (n1, n2, n3, r1, r2); anything else runs the
// run-time-dims instantiation of the same kernels.
#define TTB_FOR_SHAPES(X) \
  X(4, 4, 4, 32, 32)      \
  X(2, 2, 4, 16, 16)      \
  X(4, 4, 4, 16, 16)      \
  X(2, 2, 4, 8, 8)        \
  X(4, 4, 8, 32, 32)

template <class F>
static cudaError_t dispatch(const DynDims& d, bool aligned, F&& f) {
  if (!aligned) return f(d);
#define TTB_TRY(A_, B_, C_, R1_, R2_) \
  if (d.n1 == A_ && d.n2 == B_ && d.n3 == C_ && d.r1 == R1_ && d.r2 == R2_) return f(FixDims<A_, B_, C_, R1_, R2_>{});
  TTB_FOR_SHAPES(TTB_TRY)
#undef TTB_TRY
  return f(d);
}

cudaError_t launch_forward(ttb_handle* h, const float* c0, const float* c1, const float* c2, float* out,
                           cudaStream_t s) {
  const bool al = (((uintptr_t)c0 | (uintptr_t)c1 | (uintptr_t)c2 | (uintptr_t)out) & 15) == 0;
  if (h->allow_empty) {  // rows of empty bags read zero whatever the close kernels write
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(float) * (size_t)h->B * h->dims.n1 * h->dims.n2 * h->dims.n3, s);
    if (e != cudaSuccess) return e;
  }
  return dispatch(h->dims, al, [&](auto d) { return forward_impl<decltype(d)>(h, c0, c1, c2, out, s); });
}

cudaError_t launch_aggregate(ttb_handle* h, const float* gout, cudaStream_t s) {
  const bool al = ((uintptr_t)gout & 15) == 0;
  return dispatch(h->dims, al, [&](auto d) { return aggregate_impl<decltype(d)>(h, gout, s); });
}

cudaError_t launch_backward(ttb_handle* h, const float* c0, const float* c1, const float* c2, const float* gout,
                            float* g0, float* g1, float* g2, float* p0, float* p1, float* p2, double* v0, double* v1,
                            double* v2, double lr, double mu, int mask, int mode, cudaStream_t s) {
  const bool al = (((uintptr_t)c0 | (uintptr_t)c1 | (uintptr_t)c2 | (uintptr_t)gout | (uintptr_t)g0 | (uintptr_t)g1 |
                     (uintptr_t)g2 | (uintptr_t)p0 | (uintptr_t)p1 | (uintptr_t)p2) & 15) == 0;
  return dispatch(h->dims, al, [&](auto d) {
    return backward_impl<decltype(d)>(h, c0, c1, c2, gout, g0, g1, g2, p0, p1, p2, v0, v1, v2, lr, mu, mask, mode,
                                      s);
  });
}

// ---------------------------------------------------------------- unique export
// rows in first-occurrence order (backward.py:86-87): mark each row's first
// index position, then a flag scan over positions numbers them.
__global__ void k_mark_first(const int* __restrict__ counts, const int* __restrict__ urow_start,
                             const unsigned* __restrict__ sv, int* __restrict__ first_of) {
  pdl_enter();
  const int U = counts[3];
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < U; u += gridDim.x * blockDim.x)
    first_of[sv[urow_start[u]]] = u + 1;
}

__global__ void __launch_bounds__(kBlock) k_first_scan(const int* __restrict__ first_of, int T, int N,
                                                       const unsigned* __restrict__ urow, const float* __restrict__ gU,
                                                       int64_t* __restrict__ rows, float* __restrict__ grads,
                                                       unsigned long long* status, unsigned* ctr) {
  pdl_enter();
  __shared__ int s_tile;
  __shared__ int s_tmp[kItems * (kBlock / 32) + 2];
  const int tile = claim_tile(ctr, &s_tile);
  const int base = tile * kTile;
  bool f[kItems];
  int u[kItems];
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int t = base + k * kBlock + threadIdx.x;
    u[k] = t < T ? first_of[t] - 1 : -1;
    f[k] = u[k] >= 0;
  }
  int rank[kItems];
  long long incl;
  tile_flag_scan(f, rank, status, tile, s_tmp, &incl);
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    if (!f[k]) continue;
    if (rows) rows[rank[k]] = urow[u[k]];
    if (grads)
      for (int o = 0; o < N; ++o) grads[(size_t)rank[k] * N + o] = gU[(size_t)u[k] * N + o];
  }
}

cudaError_t launch_export_unique(ttb_handle* h, int64_t* rows, float* grads, cudaStream_t s) {
  Workspace& w = h->w;
  const int T = (int)h->T;
  cudaError_t e;
  // the sorted row order lives in svA/svB depending on pass parity
  const int passes = (h->idx_bits + 7) / 8 < 1 ? 1 : (h->idx_bits + 7) / 8;
  const unsigned* sv = (passes & 1) ? w.svA : w.svB;
  if ((e = cudaMemsetAsync(w.uid_first, 0, sizeof(int) * T, s))) return e;
  if ((e = cudaMemsetAsync(w.scan_status + kScanFirst * h->scan_tiles, 0,
                           sizeof(unsigned long long) * h->scan_tiles, s)))
    return e;
  if ((e = cudaMemsetAsync(w.scan_ctr + kScanFirst, 0, sizeof(unsigned), s))) return e;
  int grid = (T + kBlock - 1) / kBlock;
  if (grid > 148 * 8) grid = 148 * 8;
  k_mark_first<<<grid, kBlock, 0, s>>>(w.counts, w.urow_start, sv, w.uid_first);
  const int tiles = (T + kTile - 1) / kTile;
  k_first_scan<<<tiles, kBlock, 0, s>>>(w.uid_first, T, h->dims.n1 * h->dims.n2 * h->dims.n3, w.urow, w.gU, rows,
                                        grads, w.scan_status + kScanFirst * h->scan_tiles, w.scan_ctr + kScanFirst);
  count_launch(2);
  return cudaGetLastError();
}

}  // namespace ttb

namespace ttb {
// Picks the prefix chunk sizes (multiples of 8, <= kMaxChunk) that fit in
// shared memory; false if even 8 does not fit.
bool choose_chunks(const DynDims& d, int* chf, int* chb) {
  const size_t cap = 227 * 1024;
  *chf = *chb = 0;
  for (int c : {32, 16, 8})
    if (!*chf && prefix_smem(d, c) <= cap) *chf = c;
  for (int c : {16, 8})
    if (!*chb && bwd_smem(d, c) <= cap) *chb = c;
  return *chf && *chb && close_smem(d) <= cap && dG1s(d) <= 32 * kRedPerLane && dG3s(d) <= 32 * kRedPerLane &&
         dN(d) <= 32 * kMaxPerLane;
}
}  // namespace ttb
