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
                                                 int* __restrict__ counts, unsigned long long* status,
                                                 unsigned* ctr) {
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

// dG2[:, i2] = sum over the chunk partials of group i2, in chunk order.
__global__ void __launch_bounds__(kBlock) k_dg2_reduce(KGeom g, int C, int G2S, int cmax, int ch,
                                                       const float* __restrict__ part, const int* __restrict__ grp_cnt,
                                                       const int* __restrict__ err, float* __restrict__ grad,
                                                       float* __restrict__ param, double* __restrict__ vel, double lr,
                                                       double mu, int do_update) {
  const unsigned i2 = blockIdx.x;
  const int nch = (grp_cnt[i2] + ch - 1) / ch;
  const bool upd = do_update && ((*err & 8) == 0);
  const int e = blockIdx.y * kBlock + threadIdx.x;
  if (e >= G2S) return;
  float acc = 0.f;
  for (int c = 0; c < nch; ++c) acc += part[((size_t)i2 * cmax + c) * G2S + e];
  const int r = e / C, cc = e - r * C;
  const size_t gi = ((size_t)r * g.m2 + i2) * C + cc;
  if (grad) grad[gi] = acc;
  if (upd) param[gi] = sgd_apply(param[gi], acc, vel ? vel + gi : nullptr, lr, mu);
}

// i3_start[v] = first position of digit v among the i3-sorted rows: every
// boundary between consecutive sorted keys fills the digits it skips.
__global__ void k_i3_bounds(const unsigned* __restrict__ k3, const int* __restrict__ counts, int m3,
                            int* __restrict__ i3_start) {
  const int U = counts[3];
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q <= U; q += gridDim.x * blockDim.x) {
    const int prev = q > 0 ? (int)k3[q - 1] : -1;
    const int cur = q < U ? (int)k3[q] : m3;
    for (int v = prev + 1; v <= cur; ++v) i3_start[v] = q;
  }
}

// dG3[:, i3] = sum of dH over the rows with that last digit, in row order.
__global__ void __launch_bounds__(kBlock) k_dg3_reduce(KGeom g, int N3, int G3S, const int* __restrict__ i3_start,
                                                       const unsigned* __restrict__ v3, const float* __restrict__ dH,
                                                       const int* __restrict__ err, float* __restrict__ grad,
                                                       float* __restrict__ param, double* __restrict__ vel, double lr,
                                                       double mu, int do_update) {
  extern __shared__ float s_part[];  // kRedWarps x G3S
  const unsigned v = blockIdx.x;
  const int k0 = i3_start[v], k1 = i3_start[v + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int per = (k1 - k0 + kRedWarps - 1) / kRedWarps;
  const int a = k0 + w * per, b = min(k1, a + per);
  for (int e = lane; e < G3S; e += 32) {
    float acc = 0.f;
    for (int k = a; k < b; ++k) acc += dH[(size_t)v3[k] * G3S + e];
    s_part[w * G3S + e] = acc;
  }
  __syncthreads();
  const bool upd = do_update && ((*err & 8) == 0);
  const unsigned m3n3 = g.m3 * (unsigned)N3;
  for (int e = threadIdx.x; e < G3S; e += kBlock) {
    float acc = 0.f;
#pragma unroll
    for (int ww = 0; ww < kRedWarps; ++ww) acc += s_part[ww * G3S + e];
    const int r = e / N3, j = e - r * N3;
    const size_t gi = (size_t)r * m3n3 + v * N3 + j;
    if (grad) grad[gi] = acc;
    if (upd) param[gi] = sgd_apply(param[gi], acc, vel ? vel + gi : nullptr, lr, mu);
  }
}

// dG1[i1] = sum of E over the present prefixes (i1, i2), ascending i2.
__global__ void __launch_bounds__(kBlock) k_dg1_reduce(KGeom g, int G1S, const unsigned* __restrict__ pmap,
                                                       const int* __restrict__ pslot, const float* __restrict__ E,
                                                       const int* __restrict__ err, float* __restrict__ grad,
                                                       float* __restrict__ param, double* __restrict__ vel, double lr,
                                                       double mu, int do_update) {
  extern __shared__ float s_part[];  // kRedWarps x G1S
  const unsigned i1 = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int per = ((int)g.m2 + kRedWarps - 1) / kRedWarps;
  const int a = w * per, b = min((int)g.m2, a + per);
  for (int e = lane; e < G1S; e += 32) {
    float acc = 0.f;
    for (int i2 = a; i2 < b; ++i2) {
      const unsigned key = i1 * g.m2 + (unsigned)i2;
      if (pmap[key] != kEmpty) acc += E[(size_t)pslot[key] * G1S + e];
    }
    s_part[w * G1S + e] = acc;
  }
  __syncthreads();
  const bool upd = do_update && ((*err & 8) == 0);
  for (int e = threadIdx.x; e < G1S; e += kBlock) {
    float acc = 0.f;
#pragma unroll
    for (int ww = 0; ww < kRedWarps; ++ww) acc += s_part[ww * G1S + e];
    const size_t gi = (size_t)i1 * G1S + e;
    if (grad) grad[gi] = acc;
    if (upd) param[gi] = sgd_apply(param[gi], acc, vel ? vel + gi : nullptr, lr, mu);
  }
}

__global__ void k_sgd(float* __restrict__ p, const float* __restrict__ gr, double* __restrict__ v, int64_t n,
                      double lr, double mu) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = sgd_apply(p[i], gr[i], v ? v + i : nullptr, lr, mu);
}

cudaError_t launch_sgd(float* p, const float* g, double* v, int64_t n, double lr, double mu, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int64_t grid = (n + kBlock - 1) / kBlock;
  if (grid > 148 * 8) grid = 148 * 8;
  k_sgd<<<(int)grid, kBlock, 0, s>>>(p, g, v, n, lr, mu);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------- dispatch
template <class D>
static size_t prefix_smem(const D& d, int ch) {
  return sizeof(float) * ((size_t)d.r1 * dC(d) + (size_t)d.r1 * ch * d.n1);
}
template <class D>
static size_t close_smem(const D& d) {
  return sizeof(float) * (kBlock / 32) * ((size_t)dX(d) * (d.r2 + 1) + dG3s(d) + dN(d));
}
template <class D>
static size_t bwd_smem(const D& d, int ch) {
  const size_t M = (size_t)ch * d.n1, LZ = pad_ld(d);
  return sizeof(float) * (M * LZ + (size_t)d.r1 * LZ + M * d.r1 + (kBlock / 32) * ((size_t)dN(d) + dG3s(d) + dSlot(d)));
}

template <class D>
static cudaError_t forward_impl(ttb_handle* h, const float* c0, const float* c1, const float* c2, float* out,
                                cudaStream_t s) {
  const D d = make_dims<D>(h->dims);
  Workspace& w = h->w;
  cudaError_t e;
  const size_t sm1 = prefix_smem(d, h->chf);
  if ((e = cudaFuncSetAttribute(k_prefix_products<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1)))
    return e;
  dim3 g1(h->kg.m2, (unsigned)h->cmaxf);
  { ProfScope _ps(h, s, "prefix_products");
  k_prefix_products<D><<<g1, kBlock, sm1, s>>>(d, h->kg, h->chf, c0, c1, w.pmap, w.pslot, w.slots);
  }
  count_launch();
  const size_t sm2 = close_smem(d);
  if ((e = cudaFuncSetAttribute(k_close_pool<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2))) return e;
  const int B = (int)h->B;
  int grid = (B + kBlock / 32 - 1) / (kBlock / 32);
  if (grid > 148 * 32) grid = 148 * 32;
  { ProfScope _ps(h, s, "close_pool");
  k_close_pool<D><<<grid, kBlock, sm2, s>>>(d, h->kg, c2, w.slots, w.bag_off, w.bag_seg, w.seg_slot, w.occ_slot,
                                            w.keys32, B, out);
  }
  count_launch();
  return cudaGetLastError();
}

template <class D>
static cudaError_t aggregate_impl(ttb_handle* h, const float* gout, cudaStream_t s) {
  const D d = make_dims<D>(h->dims);
  Workspace& w = h->w;
  const int T = (int)h->T;
  cudaError_t e;
  // 1. order the indices by row (stable: equal rows keep index order)
  unsigned *sk, *sv;
  if ((e = launch_sort(h, w.keys32, nullptr, w.skA, w.svA, w.skB, w.svB, nullptr, T, h->idx_bits, 0, &sk, &sv, s)))
    return e;
  // 2. row / prefix runs
  if ((e = cudaMemsetAsync(w.scan_status + kScanRuns * h->scan_tiles, 0,
                           sizeof(unsigned long long) * h->scan_tiles, s)))
    return e;
  if ((e = cudaMemsetAsync(w.scan_ctr + kScanRuns, 0, sizeof(unsigned), s))) return e;
  const int tiles = (T + kTile - 1) / kTile;
  { ProfScope _ps(h, s, "runs");
  k_runs<<<tiles, kBlock, 0, s>>>(sk, T, h->kg, w.pslot, w.urow, w.urow_start, w.urow_i3, w.prow_begin, w.prow_end,
                                  w.counts, w.scan_status + kScanRuns * h->scan_tiles, w.scan_ctr + kScanRuns);
  }
  count_launch();
  // 3. aggregated row gradients
  int grid = (T + kBlock / 32 - 1) / (kBlock / 32);
  if (grid > 148 * 16) grid = 148 * 16;
  { ProfScope _ps(h, s, "row_agg");
  k_row_agg<D><<<grid, kBlock, 0, s>>>(d, w.counts, w.urow_start, sv, w.bag_of, gout, w.gU, w.err);
  }
  count_launch();
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
  const size_t sm = bwd_smem(d, h->chb);
  if ((e = cudaFuncSetAttribute(k_bwd_prefix<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm))) return e;
  dim3 gp(h->kg.m2, (unsigned)h->cmaxb);
  { ProfScope _ps(h, s, "bwd_prefix");
  k_bwd_prefix<D><<<gp, kBlock, sm, s>>>(d, h->kg, h->chb, c0, c1, c2, w.pmap, w.pslot, w.slots, w.prow_begin, w.prow_end,
                                         w.urow_i3, w.gU, w.dH, w.E, w.dG2part, w.grp_cnt,
                                         h->cmaxb);
  }
  count_launch();
  // 5. rows by last digit for the G3 reduction
  unsigned *k3, *v3;
  if ((e = launch_sort(h, w.urow_i3, nullptr, w.rkA, w.rvA, w.rkB, w.rvB, w.counts + 3, T, h->i3_bits, 1, &k3, &v3,
                       s)))
    return e;
  { ProfScope _ps(h, s, "i3_bounds");
  k_i3_bounds<<<(T + kBlock) / kBlock, kBlock, 0, s>>>(k3, w.counts, (int)h->kg.m3, w.i3_start);
  }
  count_launch();
  const bool upd = mode == 1;
  // 6. reductions (+ fused update)
  { ProfScope _ps(h, s, "dg1_reduce");
  k_dg1_reduce<<<h->kg.m1, kBlock, sizeof(float) * kRedWarps * dG1s(d), s>>>(h->kg, dG1s(d), w.pmap, w.pslot, w.E, w.err,
                                           upd ? nullptr : g0, p0, v0, lr, mu, upd && (mask & 1));
  }
  { ProfScope _ps(h, s, "dg2_reduce");
  k_dg2_reduce<<<dim3(h->kg.m2, (dG2s(d) + kBlock - 1) / kBlock), kBlock, 0, s>>>(h->kg, dC(d), dG2s(d), h->cmaxb, h->chb, w.dG2part,
                                           w.grp_cnt, w.err, upd ? nullptr : g1, p1, v1, lr, mu,
                                           upd && (mask & 2));
  }
  { ProfScope _ps(h, s, "dg3_reduce");
  k_dg3_reduce<<<h->kg.m3, kBlock, sizeof(float) * kRedWarps * dG3s(d), s>>>(h->kg, d.n3, dG3s(d), w.i3_start, v3, w.dH, w.err,
                                           upd ? nullptr : g2, p2, v2, lr, mu, upd && (mask & 4));
  }
  count_launch(3);
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
static cudaError_t dispatch(const DynDims& d, F&& f) {
#define TTB_TRY(A_, B_, C_, R1_, R2_) \
  if (d.n1 == A_ && d.n2 == B_ && d.n3 == C_ && d.r1 == R1_ && d.r2 == R2_) return f(FixDims<A_, B_, C_, R1_, R2_>{});
  TTB_FOR_SHAPES(TTB_TRY)
#undef TTB_TRY
  return f(d);
}

cudaError_t launch_forward(ttb_handle* h, const float* c0, const float* c1, const float* c2, float* out,
                           cudaStream_t s) {
  return dispatch(h->dims, [&](auto d) { return forward_impl<decltype(d)>(h, c0, c1, c2, out, s); });
}

cudaError_t launch_aggregate(ttb_handle* h, const float* gout, cudaStream_t s) {
  return dispatch(h->dims, [&](auto d) { return aggregate_impl<decltype(d)>(h, gout, s); });
}

cudaError_t launch_backward(ttb_handle* h, const float* c0, const float* c1, const float* c2, const float* gout,
                            float* g0, float* g1, float* g2, float* p0, float* p1, float* p2, double* v0, double* v1,
                            double* v2, double lr, double mu, int mask, int mode, cudaStream_t s) {
  return dispatch(h->dims, [&](auto d) {
    return backward_impl<decltype(d)>(h, c0, c1, c2, gout, g0, g1, g2, p0, p1, p2, v0, v1, v2, lr, mu, mask, mode,
                                      s);
  });
}

// ---------------------------------------------------------------- unique export
// rows in first-occurrence order (backward.py:86-87): mark each row's first
// index position, then a flag scan over positions numbers them.
__global__ void k_mark_first(const int* __restrict__ counts, const int* __restrict__ urow_start,
                             const unsigned* __restrict__ sv, int* __restrict__ first_of) {
  const int U = counts[3];
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < U; u += gridDim.x * blockDim.x)
    first_of[sv[urow_start[u]]] = u + 1;
}

__global__ void __launch_bounds__(kBlock) k_first_scan(const int* __restrict__ first_of, int T, int N,
                                                       const unsigned* __restrict__ urow, const float* __restrict__ gU,
                                                       int64_t* __restrict__ rows, float* __restrict__ grads,
                                                       unsigned long long* status, unsigned* ctr) {
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
  return *chf && *chb && close_smem(d) <= cap && sizeof(float) * kRedWarps * (size_t)dG1s(d) <= 48 * 1024 &&
         sizeof(float) * kRedWarps * (size_t)dG3s(d) <= 48 * 1024;
}
}  // namespace ttb
