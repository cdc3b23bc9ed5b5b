// Shared device helpers for the TT-EmbeddingBag kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ttb {

constexpr unsigned kEmpty = 0xFFFFFFFFu;
constexpr int kBlock = 256;  // threads per CTA for the streaming kernels
constexpr int kItems = 2;    // items per thread for the scan tiles (many small tiles: latency)
constexpr int kTile = kBlock * kItems;
constexpr int kSortItems = 4;  // items per thread for the radix-sort tiles
constexpr int kSortTile = kBlock * kSortItems;

// Geometry as the kernels see it (d = 3; d = 2 tables arrive embedded).
struct KGeom {
  unsigned m1, m2, m3;  // row factors
  unsigned m1m2;        // number of prefix keys
  unsigned rows;        // padded rows m1 m2 m3 (< 2^31)
  // Table-batched handles (ttb_create_batched, tensor-core pipeline only): nt
  // tables with their own row factors, stored stacked and zero-padded to the
  // common (M1, M2, M3): m1 = M1 (prefix keys per i2 group), m2 = nt M2 (G2
  // slices = i2 groups), m3 = nt M3 (G3 slices), m1m2 = M1 nt M2. Table f owns
  // G1 rows [f M1, f M1 + m1_f), G2 slices [f M2, ...), G3 slices [f M3, ...).
  // A single table is nt = 1, tm2 = m2, tm3 = m3, g1rows = m1.
  unsigned nt;      // tables
  unsigned tm2, tm3;  // per-table slice blocks M2, M3
  unsigned g1rows;  // G1 rows (nt M1)
  unsigned bpt;     // bags per table (batched plans: table of bag b = b / bpt)
};

// Core dims. DynDims carries them at run time; FixDims bakes them into the
// instantiation so the contraction loops fully unroll.
struct DynDims {
  int n1, n2, n3, r1, r2;
};
template <int N1, int N2, int N3, int R1, int R2>
struct FixDims {
  static constexpr int n1 = N1, n2 = N2, n3 = N3, r1 = R1, r2 = R2;
};
template <class D>
__host__ __device__ inline D make_dims(const DynDims& d);
template <>
__host__ __device__ inline DynDims make_dims<DynDims>(const DynDims& d) {
  return d;
}
template <class D>
__host__ __device__ inline D make_dims(const DynDims&) {
  return D{};
}

// Derived extents (floats).
template <class D> __host__ __device__ inline int dN(const D& d) { return d.n1 * d.n2 * d.n3; }
template <class D> __host__ __device__ inline int dX(const D& d) { return d.n1 * d.n2; }          // slot rows
template <class D> __host__ __device__ inline int dSlot(const D& d) { return d.n1 * d.n2 * d.r2; }  // slot size
template <class D> __host__ __device__ inline int dC(const D& d) { return d.n2 * d.r2; }          // G2 slice cols
template <class D> __host__ __device__ inline int dG1s(const D& d) { return d.n1 * d.r1; }
template <class D> __host__ __device__ inline int dG2s(const D& d) { return d.r1 * d.n2 * d.r2; }
template <class D> __host__ __device__ inline int dG3s(const D& d) { return d.r2 * d.n3; }

// ---------------------------------------------------------------- lookback
// Decoupled look-back for single-pass scans. Status word: bits 62-63 flag
// (1 = tile aggregate, 2 = inclusive prefix), bits 0-61 value.
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagInc = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

// The look-back status words carry their own payload (flag + count), so
// relaxed gpu-scope accesses are sufficient; acquire loads would invalidate
// L1 (CCTL.IVALL) on every probe of the spin loop.
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u32(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Programmatic dependent launch: every kernel of the step waits for its
// predecessor grid (and its memory) here, and immediately allows its own
// dependent to be scheduled, so launch latency overlaps the previous tail.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

constexpr int kLookWindow = 16;  // predecessors probed per look-back round trip

// Called by ONE thread of the tile. Returns the exclusive prefix of `agg`
// over all earlier tiles and publishes this tile's inclusive prefix.
__device__ inline long long lookback_exclusive(unsigned long long* status, int tile, long long agg) {
  if (tile == 0) {
    st_relaxed_u64(&status[0], kFlagInc | (unsigned long long)agg);
    return 0;
  }
  st_relaxed_u64(&status[tile], kFlagAgg | (unsigned long long)agg);
  long long excl = 0;
  int j = tile - 1;
  while (j >= 0) {  // windowed: kLookWindow predecessors per round trip
    unsigned long long sv[kLookWindow];
#pragma unroll
    for (int i = 0; i < kLookWindow; ++i) sv[i] = (j - i >= 0) ? ld_relaxed_u64(&status[j - i]) : 0ull;
    bool done = false;
    int used = 0;
#pragma unroll
    for (int i = 0; i < kLookWindow; ++i) {
      if (done || used < i || j - i < 0) continue;
      const unsigned long long f = sv[i] & ~kValMask;
      if (f == 0) continue;
      excl += (long long)(sv[i] & kValMask);
      used = i + 1;
      if (f == kFlagInc) done = true;
    }
    if (done) break;
    j -= used;
  }
  st_relaxed_u64(&status[tile], kFlagInc | (unsigned long long)(excl + agg));
  return excl;
}

// Dynamic tile id (blocks are numbered in start order, so look-back never
// waits on a block that has not started).
__device__ __forceinline__ int claim_tile(unsigned* counter, int* s_tile) {
  if (threadIdx.x == 0) *s_tile = (int)atomicAdd(counter, 1u);
  __syncthreads();
  return *s_tile;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Exclusive scan of 0/1 flags over a striped tile: element (k, tid) sits at
// position base + k * kBlock + tid. Writes the global exclusive rank of each
// element and returns the global total up to and including this tile via
// *incl_out (valid in all threads). s_tmp: kItems * (kBlock / 32) + 2 ints.
__device__ inline void tile_flag_scan(const bool (&f)[kItems], int (&rank)[kItems],
                                      unsigned long long* status, int tile, int* s_tmp,
                                      long long* incl_out) {
  constexpr int NW = kBlock / 32;
  constexpr int NV = kItems * NW;  // values in (k, warp) order
  static_assert(NV % 32 == 0 || NV < 32, "scan layout");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = lanemask_lt();
  int within[kItems];
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    unsigned m = __ballot_sync(0xffffffffu, f[k]);
    within[k] = __popc(m & lt);
    if (lane == 0) s_tmp[k * NW + w] = __popc(m);
  }
  __syncthreads();
  if (w == 0) {
    constexpr int PER = NV >= 32 ? NV / 32 : 1;
    int v[PER];
    int sum = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      v[i] = (lane * PER + i < NV) ? s_tmp[lane * PER + i] : 0;
      sum += v[i];
    }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int run = incl - sum;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      if (lane * PER + i < NV) s_tmp[lane * PER + i] = run;
      run += v[i];
    }
    int total = __shfl_sync(0xffffffffu, incl, 31);
    if (lane == 0) {
      long long ex = lookback_exclusive(status, tile, total);
      s_tmp[NV] = (int)ex;
      s_tmp[NV + 1] = (int)(ex + total);
    }
  }
  __syncthreads();
  const int g = s_tmp[NV];
#pragma unroll
  for (int k = 0; k < kItems; ++k) rank[k] = g + s_tmp[k * NW + w] + within[k];
  *incl_out = s_tmp[NV + 1];
}

// fp64 SGD(+momentum) step matching numpy's rounding in the reference:
//   vel *= mu; vel += g; core = f32(f64(core) - lr * vel)       (backward.py:195-197)
//   core = f32(f64(core) - lr * g)                              (backward.py:200)
// __dmul_rn / __dsub_rn keep nvcc from contracting into an FMA.
__device__ __forceinline__ float sgd_apply(float p, float g, double* vel, double lr, double mu) {
  double step;
  if (vel != nullptr) {
    double v = __dadd_rn(__dmul_rn(*vel, mu), (double)g);
    *vel = v;
    step = __dmul_rn(lr, v);
  } else {
    step = __dmul_rn(lr, (double)g);
  }
  return (float)__dsub_rn((double)p, step);
}

// register forms of sgd_apply / adagrad_apply (the state is loaded and stored
// by the caller, so a thread's loads for several elements can all be in flight)
__device__ __forceinline__ float sgd_step(float p, float g, double v_in, double* v_out, bool has_v, double lr,
                                          double mu) {
  double step;
  if (has_v) {
    const double v = __dadd_rn(__dmul_rn(v_in, mu), (double)g);
    *v_out = v;
    step = __dmul_rn(lr, v);
  } else {
    step = __dmul_rn(lr, (double)g);
  }
  return (float)__dsub_rn((double)p, step);
}
__device__ __forceinline__ float adagrad_step(float p, float g, double s_in, double* s_out, double lr, double eps) {
  const double gd = (double)g;
  const double ss = __fma_rn(gd, gd, s_in);
  *s_out = ss;
  const double step = __ddiv_rn(__dmul_rn(-lr, gd), __dadd_rn(__dsqrt_rn(ss), eps));
  return (float)__dadd_rn((double)p, step);
}

// Adagrad (torch.optim.Adagrad semantics, no weight / lr decay): the
// squared-gradient sum s in fp64, s <- fma(g, g, s), p <- f32(p + (-lr g) / (sqrt(s) + eps)),
// one rounding into the parameter like sgd_apply. (The reference has no
// Adagrad — SPEC.md:282; BASELINE north_star asks for it next to SGD.)
__device__ __forceinline__ float adagrad_apply(float p, float g, double* s, double lr, double eps) {
  const double gd = (double)g;
  const double ss = __fma_rn(gd, gd, *s);  // torch's addcmul_: one rounding
  *s = ss;
  const double step = __ddiv_rn(__dmul_rn(-lr, gd), __dadd_rn(__dsqrt_rn(ss), eps));
  return (float)__dadd_rn((double)p, step);
}

}  // namespace ttb
