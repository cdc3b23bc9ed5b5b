// Host-side handle and workspace layout shared by the launchers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ttb.h"
#include "ttb_common.cuh"

namespace ttb {


struct Workspace {
  // error word + device counters: [0] err bits, [1] P, [2] S, [3] U
  int* err;
  int* counts;
  // prefix table over the m1*m2 prefix keys (first position, then slot)
  unsigned* pmap;
  int* pslot;
  unsigned* work_key;  // P: prefix key of each slot, first-occurrence order
  // per index (T)
  unsigned* keys32;    // row index as u32
  int* bag_of;
  int* occ_slot;
  int* seg_inv;
  int* occ_tmp;
  // segments
  int* seg_slot;  // S
  int* seg_bag;   // S
  int* bag_seg;   // B + 1
  int* bag_off;   // B + 1 (copied, clamped offsets)
  // reuse buffer
  float* slots;   // Pmax x slot
  // radix sort (T items)
  unsigned *skA, *svA, *skB, *svB;
  unsigned* sort_hist;    // 4 passes x 256
  unsigned* sort_status;  // 4 passes x tiles x 256
  unsigned* sort_ctr;     // 8 counters
  // rows (U <= T), sorted by row index
  unsigned* urow;
  int* urow_start;  // U + 1
  unsigned* urow_i3;
  int* prow_begin;  // by slot
  int* prow_end;
  float* gU;        // U x N aggregated row gradients
  float* dH;        // U x (r2 n3) per-row G3 gradient blocks
  float* E;         // Pmax x (n1 r1) per-prefix G1 gradient blocks
  float* zbuf;      // Pmax x slot: dL/dslot per prefix (split backward)
  float* dG2part;   // m2 x cmax x G2 slice
  int* i3_start;    // m3 + 1
  int* grp_cnt;     // m2: present prefixes per i2
  unsigned *rkA, *rvA, *rkB, *rvB;  // rows-by-i3 sort buffers
  int* uid_first;   // T: first-occurrence rank flags / scratch
  int* qrow;        // T: row ordinal of each sorted position
  float* agg_hp;    // (T / 64 + 1) x N: per-block head partial row sums
  float* agg_tp;    // (T / 64 + 1) x N: per-block tail partial row sums
  int* span_list;   // rows spanning aggregation blocks
  // look-back scan state. Zero block A (cleared by every plan) holds the
  // error word / counts and the plan-scope scans; zero block B (cleared by
  // the plan, and again if a second backward reuses the plan) holds the
  // backward-scope scan and radix-sort state. A and B are contiguous.
  char* zeroA;
  size_t zeroA_bytes;
  char* zeroB;
  size_t zeroB_bytes;
  unsigned long long* scan_status;  // kNumScans x scan_tiles (runs region lives in B)
  unsigned* scan_ctr;               // kNumScans counters
  unsigned long long* runs_status;  // scan_tiles
  unsigned* runs_ctr;
  int* grp_done;                    // m2: finished chunk CTAs per i2 group (self-resetting)
  float* scratch1;                  // 1-float sink for the unit core of d = 2 tables
  // tensor-core pipeline (ttb_fast.cu); fast_hdr sits just before zero block A:
  // [0] err bits, [1] multi-index bags, [2] work items, [3] prefixes P, [4] tiles
  uint4* f_tgeom;  // batched handles: per table (m2, m3, rows, 0) for the plan's digits
  int* fast_hdr;
  unsigned* f_key;        // T: i2-major prefix key
  unsigned* f_i3;         // T
  int2* f_sbi;            // T: (bag, i3) in prefix-sorted order
  int* f_item_start;      // T + 1
  unsigned* f_item_key;   // T
  int* f_rk;              // T: rank of each position inside its prefix key
  int* f_cnt;             // m1 m2: positions per prefix key (self-resetting)
  int* f_start;           // m1 m2: position of each key's first full item
  int* f_rstart;          // m1 m2: position of its remainder item, minus the full items' lookups
  int* f_split;           // m1 m2: lookups of the key in full items
  int* f_cta;             // kMaxCtas + 1: first tile of each step-kernel CTA
  int2* f_chunks;         // <= T / 32 + 2: runs of a multi-item prefix's full items (position, count) sorted by row before the backward
  int4* f_gtot;           // m2: (positions, items, prefixes) per i2 group
  int4* f_tile_info;      // tiles (<= T / 32 + m2): (i2, first item, items)
  float* f_g1img;         // m1 x 768: split G1 row images (pre-swizzled, both parities) / transposed images
  float* f_g3t;           // G3 slice-major (i3, c, n3): one slice = 512 contiguous bytes (bulk copies)
  float* f_img;           // m2 x 4 x 16 KB: G2 slice images (cb hi/lo, k hi/lo)
  float* f_grad;          // |G1| + |G2| + |G3|: gradients for the fused update
  unsigned* f_rowbits;    // rows / 32 + 1: row bitmap of the on-demand U count
};

enum ScanId { kScanSlots = 0, kScanSegs = 1, kScanFirst = 2, kScanFast = 3, kNumScans = 4 };

}  // namespace ttb

namespace ttb {
// Optional per-kernel CUDA-event timing (ttb_profile_*): each launch site
// records an event pair on its stream; ttb_profile_read accumulates them.
constexpr int kMaxProfEvents = 256;
constexpr int kMaxProfNames = 48;
struct Profiler {
  int on;
  int n;  // pending event pairs
  cudaEvent_t ev[kMaxProfEvents][2];
  const char* pend_name[kMaxProfEvents];
  const char* names[kMaxProfNames];
  double ms[kMaxProfNames];
  long long calls[kMaxProfNames];
  int nnames;
};
}  // namespace ttb

struct ttb_handle {
  ttb_geom geom;
  ttb::KGeom kg;
  ttb::DynDims dims;
  int64_t maxT, maxB, Pmax, scan_tiles, sort_tiles;
  int chf, chb;          // prefixes per chunk (forward / backward kernels)
  int nsplitf, nsplitb;  // CTAs per i2 group (forward / backward)
  int cmaxb;             // chunks per i2 group in the backward (dG2 partials)
  int dg2_slots;         // dG2 partial slots per i2 written by the last backward
  int bwd_split;         // use the split backward (rows kernel + tensor-core GEMM kernel)
  int allow_empty;       // TTB_OPT_ALLOW_EMPTY: empty bags pool to zero rows (nn.EmbeddingBag) instead of an error
  int fast_ok, fast;     // tensor-core pipeline supported / selected (ttb_fast.cu)
  int batched;           // ttb_create_batched: several tables in one handle (tensor-core pipeline only)
  ttb_geom tables[TTB_MAX_TABLES];  // their geometries (batched)
  uint4 tgeom_host[TTB_MAX_TABLES];  // (m2, m3, rows, 0) per table: the source of w.f_tgeom
  int num_sms;
  const void* plan_idx;  // inputs of the current plan (the legacy plan behind
  const int64_t* plan_off;  // ttb_export_plan is built from them on demand)
  int plan_idx64;
  int legacy_planned;
  int idx_bits, i3_bits;
  char* base;
  size_t bytes;
  ttb::Workspace w;
  // host-side state of the current plan
  int64_t T, B;
  int planned, forwarded, backwarded;
  int pmap_clean;   // prefix table already reset (by the last backward)
  int bwd_zeroed;   // zero block B is clear for the next backward
  int fgrad_zeroed;  // the tensor-core pipeline's flat gradient buffer was cleared by the last plan
  int tilectr_zeroed;  // the pooled backward's tile counter was cleared by the last plan
  int64_t gen;
  // the f_img / f_g1img core images describe the cores at img_c0 / img_c1
  // (written by the last forward or fused update; cleared by
  // ttb_cores_modified and by a backward that hands gradients to the caller)
  int64_t su_gen;       // plan generation whose S / U were counted (fast pipeline), -1 none
  int64_t su[2];
  int img_valid;
  const float* img_c0;
  const float* img_c1;
  const float* img_c2;
  ttb::Profiler prof;
};

namespace ttb {
// Kernel launch with programmatic stream serialization (PDL): the kernel may
// be scheduled while its predecessor drains and synchronises on it with
// griddepcontrol.wait (pdl_enter()). Graph capture keeps the programmatic edge.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Same, launched cooperatively: the launch fails (instead of a later
// deadlock) unless every CTA of the grid is co-resident — required by
// kernels that synchronise their CTAs with software grid barriers.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_coop(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                   Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

extern long long g_launches;
inline void count_launch(int n = 1) { __atomic_add_fetch(&g_launches, n, __ATOMIC_RELAXED); }

// RAII timing scope around one (or a few) launches; free when profiling is off.
struct ProfScope {
  Profiler* p;
  cudaStream_t s;
  int slot;
  ProfScope(ttb_handle* h, cudaStream_t st, const char* name);
  ~ProfScope();
};

// launchers (return cudaError_t of the last launch)
cudaError_t launch_plan(ttb_handle* h, const void* idx, int idx64, const int64_t* offsets, cudaStream_t s);
cudaError_t launch_forward(ttb_handle* h, const float* c0, const float* c1, const float* c2, float* out,
                           cudaStream_t s);
cudaError_t launch_aggregate(ttb_handle* h, const float* gout, cudaStream_t s);
// mode 0: write grads into g0..g2; mode 1: SGD update in place
cudaError_t launch_backward(ttb_handle* h, const float* c0, const float* c1, const float* c2,
                            const float* gout, float* g0, float* g1, float* g2, float* p0, float* p1,
                            float* p2, double* v0, double* v1, double* v2, double lr, double mu,
                            int update_mask, int mode, cudaStream_t s);
cudaError_t launch_sort(ttb_handle* h, const unsigned* keys_in, const unsigned* vals_in, unsigned* kA,
                        unsigned* vA, unsigned* kB, unsigned* vB, const int* d_count, int max_n,
                        int bits, int region, unsigned** keys_out, unsigned** vals_out, cudaStream_t s);
cudaError_t launch_sort_raw(const unsigned* keys_in, const unsigned* vals_in, unsigned* kA, unsigned* vA, unsigned* kB,
                            unsigned* vB, int n, int bits, unsigned* hist, unsigned* status, int tiles_cap,
                            unsigned* ctr, unsigned** keys_out, unsigned** vals_out, cudaStream_t s);
bool fast_supported(const ttb_handle* h);
// Raises a kernel's max dynamic shared memory to >= bytes on the CURRENT
// device (cudaFuncSetAttribute is per device context). Thread safe; the
// attribute is set once per (kernel, device, size increase).
cudaError_t ensure_kernel_smem(const void* kernel, size_t bytes);
cudaError_t fast_plan(ttb_handle* h, const void* idx, int idx64, const int64_t* offsets, cudaStream_t s);
cudaError_t fast_count_su(ttb_handle* h, const void* idx, int idx64, const int64_t* offsets, int64_t su[2],
                          cudaStream_t s);
cudaError_t fast_forward(ttb_handle* h, const float* c0, const float* c1, const float* c2, float* out,
                         cudaStream_t s);
cudaError_t fast_backward(ttb_handle* h, const float* c0, const float* c1, const float* c2, const float* gout,
                          float* g0, float* g1, float* g2, float* p0, float* p1, float* p2, double* v0, double* v1,
                          double* v2, double lr, double mu, int mask, int mode, cudaStream_t s, int adagrad = 0);
constexpr int kSgdMulti = 32;  // tensors per k_sgd_multi launch
cudaError_t launch_sgd_multi(const ttb_sgd_tensor* t, int count, double lr, double mu, cudaStream_t s);
cudaError_t launch_sgd(float* p, const float* g, double* v, int64_t n, double lr, double mu, cudaStream_t s,
                       const int* err = nullptr);
cudaError_t launch_adagrad(float* p, const float* g, double* st, int64_t n, double lr, double eps, cudaStream_t s,
                           const int* err = nullptr);
cudaError_t launch_dp_exchange(const ttb_dp_peers& P, int64_t n, double lr, double mu, int adagrad, double* state,
                               int* err, int grid, cudaStream_t s);
cudaError_t launch_gradcheck(const float* g, int64_t n, int* err, int num_sms, cudaStream_t s,
                             const int* suspect = nullptr);
cudaError_t launch_export_plan(ttb_handle* h, int64_t* work, int64_t* slot_occ, int64_t* seg_ids,
                               int64_t* seg_inv, int64_t* digits, cudaStream_t s);
cudaError_t launch_export_unique(ttb_handle* h, int64_t* rows, float* grads, cudaStream_t s);
}  // namespace ttb
