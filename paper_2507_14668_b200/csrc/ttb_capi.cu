#include <vector>
// extern "C" entry points (include/ttb.h): handle, workspace layout, checks.
#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "ttb_internal.h"

namespace ttb {
long long g_launches = 0;
bool choose_chunks(const DynDims& d, int* chf, int* chb);
}  // namespace ttb

using namespace ttb;

namespace ttb {
// (kernel, device) -> dynamic shared memory bytes already allowed
namespace {
struct SmemAttr {
  const void* kernel;
  int device;
  size_t bytes;
};
std::mutex g_attr_mu;
SmemAttr g_attr[256];
int g_nattr = 0;
}  // namespace

cudaError_t ensure_kernel_smem(const void* kernel, size_t bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(g_attr_mu);
  int slot = -1;
  for (int i = 0; i < g_nattr; ++i)
    if (g_attr[i].kernel == kernel && g_attr[i].device == dev) {
      if (g_attr[i].bytes >= bytes) return cudaSuccess;
      slot = i;
      break;
    }
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  if (slot < 0 && g_nattr < 256) {
    slot = g_nattr++;
    g_attr[slot].kernel = kernel;
    g_attr[slot].device = dev;
  }
  if (slot >= 0) g_attr[slot].bytes = bytes;
  return cudaSuccess;
}
}  // namespace ttb

namespace {

int bits_for(uint64_t maxval) {  // bits to represent values in [0, maxval]
  int b = 0;
  while (b < 63 && (maxval >> b) != 0) ++b;
  return b < 1 ? 1 : b;
}

bool geom_ok(const ttb_geom* g) {
  if (!g) return false;
  for (int k = 0; k < 3; ++k)
    if (g->m[k] < 1 || g->n[k] < 1) return false;
  if (g->r[0] != 1 || g->r[3] != 1 || g->r[1] < 1 || g->r[2] < 1) return false;
  const double rows = (double)g->m[0] * (double)g->m[1] * (double)g->m[2];
  if (rows >= 2147483647.0) return false;
  return true;
}

struct Carver {
  char* base;
  size_t off = 0;
  template <class T>
  T* take(size_t count) {
    off = (off + 255) & ~(size_t)255;
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += sizeof(T) * (count ? count : 1);
    return p;
  }
};

// Lays the workspace out (base == nullptr: sizing only). Fills h.
void layout(ttb_handle& h, char* base) {
  const ttb_geom& g = h.geom;
  const int64_t T = h.maxT, B = h.maxB;
  const int64_t m1m2 = g.m[0] * g.m[1];
  // the deterministic pipeline's buffers (a batched handle has none)
  const int64_t dT = h.batched ? 0 : T, dB = h.batched ? 0 : B, dK = h.batched ? 0 : m1m2;
  const DynDims& d = h.dims;
  const int64_t N = (int64_t)d.n1 * d.n2 * d.n3;
  const int64_t SL = (int64_t)d.n1 * d.n2 * d.r2, G1S = (int64_t)d.n1 * d.r1, G2S = (int64_t)d.r1 * d.n2 * d.r2,
                G3S = (int64_t)d.r2 * d.n3;
  h.Pmax = T < m1m2 ? T : m1m2;
  // one CTA per chunk: the prefix kernels are latency bound and gain from
  // many co-resident CTAs overlapping their gather / GEMM phases (measured:
  // fewer, longer CTAs that loop over chunks were 25% slower)
  h.nsplitf = (int)((g.m[0] + h.chf - 1) / h.chf);
  h.nsplitb = (int)((g.m[0] + h.chb - 1) / h.chb);
  h.cmaxb = h.nsplitb;
  h.sort_tiles = (T + kSortTile - 1) / kSortTile + 1;
  int64_t st = (T + kTile - 1) / kTile;
  const int64_t bt = (B + 31) / 32;
  h.scan_tiles = (st > bt ? st : bt) + 1;
  Carver c{base};
  Workspace& w = h.w;
  w.fast_hdr = c.take<int>(64);  // right before zero block A (fast_plan clears both in one memset)
  // zero block A
  size_t a0 = c.off;
  w.err = c.take<int>(16);
  w.counts = w.err;  // [0] err bits, [1] P, [2] S, [3] U
  w.scan_ctr = c.take<unsigned>(16);
  w.scan_status = c.take<unsigned long long>((size_t)kNumScans * h.scan_tiles);
  c.off = (c.off + 255) & ~(size_t)255;
  w.zeroA = base ? base + a0 : nullptr;
  w.zeroA_bytes = c.off - a0;
  // zero block B
  size_t b0 = c.off;
  w.runs_ctr = c.take<unsigned>(16);
  w.runs_status = c.take<unsigned long long>(h.scan_tiles);
  w.sort_ctr = c.take<unsigned>(8);
  w.sort_hist = c.take<unsigned>(2 * 4 * 256);
  w.sort_status = c.take<unsigned>((size_t)2 * 4 * h.sort_tiles * 256);
  c.off = (c.off + 255) & ~(size_t)255;
  w.zeroB = base ? base + b0 : nullptr;
  w.zeroB_bytes = c.off - b0;
  const int64_t dP = h.batched ? 0 : h.Pmax;
  w.grp_done = c.take<int>(h.batched ? 0 : g.m[1]);
  w.pmap = c.take<unsigned>(dK);
  w.pslot = c.take<int>(dK);
  w.work_key = c.take<unsigned>(dP);
  w.keys32 = c.take<unsigned>(dT);
  w.bag_of = c.take<int>(T);  // (the tensor-core plan's bag ids too)
  w.occ_slot = c.take<int>(dT);
  w.seg_inv = c.take<int>(dT);
  w.occ_tmp = c.take<int>(dT);
  w.seg_slot = c.take<int>(dT);
  w.seg_bag = c.take<int>(dT);
  w.bag_seg = c.take<int>(dB + 1);
  w.bag_off = c.take<int>(dB + 1);
  w.slots = c.take<float>((size_t)dP * SL);
  w.skA = c.take<unsigned>(dT);
  w.svA = c.take<unsigned>(dT);
  w.skB = c.take<unsigned>(dT);
  w.svB = c.take<unsigned>(dT);
  w.urow = c.take<unsigned>(dT + 1);
  w.urow_start = c.take<int>(dT + 1);
  w.urow_i3 = c.take<unsigned>(dT);
  w.prow_begin = c.take<int>(dP);
  w.prow_end = c.take<int>(dP);
  w.gU = c.take<float>((size_t)dT * N);
  w.dH = c.take<float>((size_t)dT * G3S);
  w.E = c.take<float>((size_t)dP * G1S);
  w.zbuf = c.take<float>((size_t)dP * SL);
  w.dG2part = c.take<float>(h.batched ? 0 : (size_t)g.m[1] * h.cmaxb * G2S);
  w.i3_start = c.take<int>(h.batched ? 0 : g.m[2] + 1);
  w.grp_cnt = c.take<int>(h.batched ? 0 : g.m[1]);
  w.rkA = c.take<unsigned>(dT);
  w.rvA = c.take<unsigned>(dT);
  w.rkB = c.take<unsigned>(dT);
  w.rvB = c.take<unsigned>(dT);
  w.uid_first = c.take<int>(dT);
  w.qrow = c.take<int>(dT);
  w.agg_hp = c.take<float>((size_t)(dT / 64 + 2) * N);
  w.agg_tp = c.take<float>((size_t)(dT / 64 + 2) * N);
  w.span_list = c.take<int>(dT / 64 + 2);
  w.scratch1 = c.take<float>(16);
  const bool fz = h.fast_ok;
  w.f_key = c.take<unsigned>(fz ? T : 0);
  w.f_i3 = c.take<unsigned>(fz ? T : 0);
  w.f_sbi = c.take<int2>(fz ? T : 0);
  w.f_item_start = c.take<int>(fz ? T + 1 : 0);
  w.f_item_key = c.take<unsigned>(fz ? T : 0);
  w.f_rk = c.take<int>(fz ? T : 0);
  // tensor-core pipeline: prefix keys (M1 per i2 group), i2 groups, G1 rows,
  // G3 slices of the (possibly stacked) geometry — KGeom, set before layout()
  const int64_t fk = h.kg.m1m2, fg = h.kg.m2, fg1 = h.kg.g1rows, fg3 = h.kg.m3;
  w.f_cnt = c.take<int>(fz ? (size_t)fk : 0);
  w.f_start = c.take<int>(fz ? (size_t)fk : 0);
  w.f_rstart = c.take<int>(fz ? (size_t)fk : 0);
  w.f_split = c.take<int>(fz ? (size_t)fk : 0);
  w.f_cta = c.take<int>(fz ? 1025 : 0);
  w.f_chunks = c.take<int2>(fz ? T / 32 + 2 : 0);
  w.f_gtot = c.take<int4>(fz ? fg : 0);
  w.f_tile_info = c.take<int4>(fz ? T / 32 + fg + 2 : 0);
  w.f_g1img = c.take<float>(fz ? (size_t)fg1 * 768 : 0);
  w.f_g3t = c.take<float>(fz ? (size_t)G3S * fg3 : 0);
  w.f_img = c.take<float>(fz ? (size_t)fg * 16384 : 0);
  w.f_grad = c.take<float>(fz ? (size_t)(G1S * fg1 + G2S * fg + G3S * fg3) : 0);
  w.f_rowbits = c.take<unsigned>(fz && !h.batched ? (size_t)(g.m[0] * g.m[1] * g.m[2] / 32 + 1) : 0);
  w.f_tgeom = c.take<uint4>(h.kg.nt);
  h.bytes = c.off + 256;
}

bool init_handle(ttb_handle& h, const ttb_geom* g, int64_t max_T, int64_t max_B) {
  if (!geom_ok(g) || max_T < 1 || max_B < 1 || max_T >= (1ll << 29) || max_B > max_T) return false;
  memset(&h, 0, sizeof(h));
  h.geom = *g;
  h.kg.m1 = (unsigned)g->m[0];
  h.kg.m2 = (unsigned)g->m[1];
  h.kg.m3 = (unsigned)g->m[2];
  h.kg.m1m2 = (unsigned)(g->m[0] * g->m[1]);
  h.kg.rows = (unsigned)(g->m[0] * g->m[1] * g->m[2]);
  h.kg.nt = 1;
  h.kg.tm2 = h.kg.m2;
  h.kg.tm3 = h.kg.m3;
  h.kg.g1rows = h.kg.m1;
  h.kg.bpt = 0;
  h.tables[0] = *g;
  h.dims = DynDims{g->n[0], g->n[1], g->n[2], g->r[1], g->r[2]};
  if (!choose_chunks(h.dims, &h.chf, &h.chb)) return false;
  h.maxT = max_T;
  h.maxB = max_B;
  h.idx_bits = bits_for((uint64_t)h.kg.rows - 1);
  h.fast_ok = fast_supported(&h) ? 1 : 0;
  h.fast = h.fast_ok;
  h.i3_bits = bits_for((uint64_t)h.kg.m3 - 1);
  layout(h, nullptr);
  return true;
}

// nt tables sharing n and ranks, stacked at the common (M1, M2, M3); the
// tensor-core pipeline must support the geometry (n = (4, 4, 4), ranks
// (1, 32, 32, 1), M3 <= 288). max_B = nt * bags_per_table.
bool init_handle_batched(ttb_handle& h, const ttb_geom* tables, int nt, int64_t max_T, int64_t bpt) {
  if (!tables || nt < 1 || nt > TTB_MAX_TABLES || bpt < 1) return false;
  int64_t M[3] = {1, 1, 1};
  for (int f = 0; f < nt; ++f) {
    if (!geom_ok(&tables[f])) return false;
    for (int k = 0; k < 3; ++k) {
      if (tables[f].n[k] != tables[0].n[k]) return false;
      if (tables[f].m[k] > M[k]) M[k] = tables[f].m[k];
    }
    for (int k = 0; k < 4; ++k)
      if (tables[f].r[k] != tables[0].r[k]) return false;
  }
  ttb_geom v = tables[0];
  v.m[0] = M[0];
  v.m[1] = M[1];
  v.m[2] = M[2];
  const int64_t max_B = (int64_t)nt * bpt;
  if ((double)M[0] * (double)M[1] * (double)nt >= 2147483647.0 || (double)nt * M[2] * 4 >= 2147483647.0) return false;
  if (!init_handle(h, &v, max_T, max_B)) return false;
  h.batched = 1;
  h.kg.nt = (unsigned)nt;
  h.kg.m2 = (unsigned)(nt * M[1]);
  h.kg.m3 = (unsigned)(nt * M[2]);
  h.kg.m1m2 = (unsigned)(M[0] * nt * M[1]);
  h.kg.tm2 = (unsigned)M[1];
  h.kg.tm3 = (unsigned)M[2];
  h.kg.g1rows = (unsigned)(nt * M[0]);
  h.kg.bpt = (unsigned)bpt;
  h.kg.rows = 0;  // per table (f_tgeom)
  for (int f = 0; f < nt; ++f) h.tables[f] = tables[f];
  h.fast_ok = fast_supported(&h) ? 1 : 0;
  if (!h.fast_ok) return false;
  h.fast = 1;
  layout(h, nullptr);
  return true;
}

thread_local cudaError_t t_last_cuda = cudaSuccess;  // the calling thread's last failing CUDA call
int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return TTB_OK;
  t_last_cuda = e;
  return TTB_ECUDA;
}

}  // namespace

extern "C" {

int ttb_abi_version(void) { return TTB_ABI_VERSION; }

const char* ttb_strerror(int code) {
  switch (code) {
    case TTB_OK: return "ok";
    case TTB_EINVAL: return "invalid argument or geometry";
    case TTB_ERANGE: return "index outside [0, rows)";
    case TTB_EEMPTY: return "empty batch or empty bag";
    case TTB_EOFFSETS: return "malformed bag offsets";
    case TTB_ENONFINITE: return "non-finite gradient";
    case TTB_ECUDA: return "CUDA error";
    case TTB_ESTATE: return "call order violated";
    default: return "unknown error";
  }
}

const char* ttb_last_cuda_error(void) { return cudaGetErrorString(t_last_cuda); }

int64_t ttb_launch_count(void) { return (int64_t)__atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

int ttb_workspace_bytes(const ttb_geom* g, int64_t max_T, int64_t max_B, size_t* bytes) {
  if (!bytes) return TTB_EINVAL;
  ttb_handle h;
  if (!init_handle(h, g, max_T, max_B)) return TTB_EINVAL;
  *bytes = h.bytes;
  return TTB_OK;
}

static ttb_handle* create_from(const ttb_handle& tmp, void* workspace, size_t bytes, ttb_stream stream);

ttb_handle* ttb_create(const ttb_geom* g, int64_t max_T, int64_t max_B, void* workspace, size_t bytes,
                       ttb_stream stream) {
  ttb_handle tmp;
  if (!init_handle(tmp, g, max_T, max_B)) return nullptr;
  return create_from(tmp, workspace, bytes, stream);
}

int ttb_batched_workspace_bytes(const ttb_geom* tables, int ntables, int64_t max_T, int64_t bags_per_table,
                                size_t* bytes) {
  if (!bytes) return TTB_EINVAL;
  ttb_handle h;
  if (!init_handle_batched(h, tables, ntables, max_T, bags_per_table)) return TTB_EINVAL;
  *bytes = h.bytes;
  return TTB_OK;
}

ttb_handle* ttb_create_batched(const ttb_geom* tables, int ntables, int64_t max_T, int64_t bags_per_table,
                               void* workspace, size_t bytes, ttb_stream stream) {
  ttb_handle tmp;
  if (!init_handle_batched(tmp, tables, ntables, max_T, bags_per_table)) return nullptr;
  return create_from(tmp, workspace, bytes, stream);
}

static ttb_handle* create_from(const ttb_handle& tmp, void* workspace, size_t bytes, ttb_stream stream) {
  if (!workspace || bytes < tmp.bytes) return nullptr;
  ttb_handle* h = (ttb_handle*)malloc(sizeof(ttb_handle));
  if (!h) return nullptr;
  *h = tmp;
  // align the base to 256 bytes inside the caller's buffer
  char* base = (char*)(((uintptr_t)workspace + 255) & ~(uintptr_t)255);
  layout(*h, base);
  h->base = base;
  h->pmap_clean = 1;
  h->su_gen = -1;
  {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
      h->num_sms = sms > 1024 ? 1024 : sms;
    else
      h->num_sms = 148;
  }
  cudaStream_t s = (cudaStream_t)stream;
  for (unsigned f = 0; f < h->kg.nt; ++f) {
    const ttb_geom& t = h->tables[f];
    h->tgeom_host[f] = make_uint4((unsigned)t.m[1], (unsigned)t.m[2], (unsigned)(t.m[0] * t.m[1] * t.m[2]), 0u);
  }
  if (cudaMemsetAsync(h->w.zeroA, 0, h->w.zeroA_bytes + h->w.zeroB_bytes, s) != cudaSuccess ||
      (!h->batched && cudaMemsetAsync(h->w.grp_done, 0, sizeof(int) * h->kg.m2, s) != cudaSuccess) ||
      (!h->batched && cudaMemsetAsync(h->w.pmap, 0xFF, sizeof(unsigned) * h->kg.m1m2, s) != cudaSuccess) ||
      (h->fast_ok && cudaMemsetAsync(h->w.f_cnt, 0, sizeof(int) * h->kg.m1m2, s) != cudaSuccess) ||
      cudaMemsetAsync(h->w.fast_hdr, 0, 64 * sizeof(int), s) != cudaSuccess ||  // the plan's grid barrier words
      cudaMemcpyAsync(h->w.f_tgeom, h->tgeom_host, sizeof(uint4) * h->kg.nt, cudaMemcpyHostToDevice, s) !=
          cudaSuccess) {
    free(h);
    return nullptr;
  }
  return h;
}

void ttb_destroy(ttb_handle* h) { free(h); }

int ttb_plan(ttb_handle* h, const void* indices, int idx_is_64, const int64_t* offsets, int64_t T, int64_t B,
             ttb_stream stream) {
  if (!h || !indices || !offsets) return TTB_EINVAL;
  if (T < 1 || B < 1) return TTB_EEMPTY;
  if (T > h->maxT || B > h->maxB) return TTB_EINVAL;
  if (h->batched && B != (int64_t)h->kg.nt * h->kg.bpt) return TTB_EINVAL;  // bags_per_table bags per table
  h->T = T;
  h->B = B;
  h->planned = 0;
  h->forwarded = 0;
  h->backwarded = 0;
  h->plan_idx = indices;
  h->plan_off = offsets;
  h->plan_idx64 = idx_is_64;
  h->legacy_planned = 0;
  cudaError_t e = h->fast ? fast_plan(h, indices, idx_is_64, offsets, (cudaStream_t)stream)
                          : launch_plan(h, indices, idx_is_64, offsets, (cudaStream_t)stream);
  if (!h->fast) h->legacy_planned = 1;
  if (e != cudaSuccess) return cuda_status(e);
  h->planned = 1;
  ++h->gen;
  return TTB_OK;
}

int ttb_forward(ttb_handle* h, const float* c0, const float* c1, const float* c2, float* out, ttb_stream stream) {
  if (!h || !c0 || !c1 || !c2 || !out) return TTB_EINVAL;
  if (!h->planned) return TTB_ESTATE;
  if (!h->fast && h->pmap_clean) return TTB_ESTATE;  // a backward consumed this plan's prefix table
  cudaError_t e = h->fast ? fast_forward(h, c0, c1, c2, out, (cudaStream_t)stream)
                          : launch_forward(h, c0, c1, c2, out, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_status(e);
  h->forwarded = 1;
  return TTB_OK;
}

int ttb_backward(ttb_handle* h, const float* c0, const float* c1, const float* c2, const float* grad_out, float* g0,
                 float* g1, float* g2, ttb_stream stream) {
  if (!h || !c0 || !c1 || !c2 || !grad_out || !g0 || !g1 || !g2) return TTB_EINVAL;
  if (!h->forwarded) return TTB_ESTATE;
  cudaError_t e = h->fast ? fast_backward(h, c0, c1, c2, grad_out, g0, g1, g2, nullptr, nullptr, nullptr, nullptr,
                                          nullptr, nullptr, 0.0, 0.0, 0, 0, (cudaStream_t)stream)
                          : launch_backward(h, c0, c1, c2, grad_out, g0, g1, g2, nullptr, nullptr, nullptr, nullptr,
                                            nullptr, nullptr, 0.0, 0.0, 0, 0, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_status(e);
  h->backwarded = 1;
  h->pmap_clean = 1;
  return TTB_OK;
}

int ttb_aggregate(ttb_handle* h, const float* grad_out, ttb_stream stream) {
  if (!h || !grad_out) return TTB_EINVAL;
  if (!h->planned || h->fast) return TTB_ESTATE;  // legacy pipeline only
  cudaError_t e = launch_aggregate(h, grad_out, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_status(e);
  h->backwarded = 1;
  return TTB_OK;
}

int ttb_backward_sgd(ttb_handle* h, float* c0, float* c1, float* c2, const float* grad_out, double* v0, double* v1,
                     double* v2, double lr, double momentum, int update_mask, ttb_stream stream) {
  if (!h || !c0 || !c1 || !c2 || !grad_out) return TTB_EINVAL;
  if (!(lr >= 0.0) || !(momentum >= 0.0 && momentum < 1.0)) return TTB_EINVAL;
  if (momentum > 0.0 && (((update_mask & 1) && !v0) || ((update_mask & 2) && !v1) || ((update_mask & 4) && !v2)))
    return TTB_EINVAL;
  if (!h->forwarded) return TTB_ESTATE;
  if (momentum == 0.0) v0 = v1 = v2 = nullptr;
  cudaError_t e = h->fast ? fast_backward(h, c0, c1, c2, grad_out, nullptr, nullptr, nullptr, c0, c1, c2, v0, v1, v2,
                                          lr, momentum, update_mask, 1, (cudaStream_t)stream)
                          : launch_backward(h, c0, c1, c2, grad_out, nullptr, nullptr, nullptr, c0, c1, c2, v0, v1, v2,
                                            lr, momentum, update_mask, 1, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_status(e);
  h->backwarded = 1;
  h->pmap_clean = 1;
  return TTB_OK;
}

int ttb_backward_adagrad(ttb_handle* h, float* c0, float* c1, float* c2, const float* grad_out, double* s0,
                         double* s1, double* s2, double lr, double eps, int update_mask, ttb_stream stream) {
  if (!h || !c0 || !c1 || !c2 || !grad_out) return TTB_EINVAL;
  if (!(lr >= 0.0) || !(eps >= 0.0)) return TTB_EINVAL;
  if (((update_mask & 1) && !s0) || ((update_mask & 2) && !s1) || ((update_mask & 4) && !s2)) return TTB_EINVAL;
  if (!h->forwarded) return TTB_ESTATE;
  if (!h->fast) return TTB_ESTATE;  // deterministic pipeline: ttb_backward, then ttb_adagrad_update
  cudaError_t e = fast_backward(h, c0, c1, c2, grad_out, nullptr, nullptr, nullptr, c0, c1, c2, s0, s1, s2, lr, eps,
                                update_mask, 1, (cudaStream_t)stream, 1);
  if (e != cudaSuccess) return cuda_status(e);
  h->backwarded = 1;
  h->pmap_clean = 1;
  return TTB_OK;
}

int ttb_adagrad_update(float* param, const float* grad, double* state_sum, int64_t n, double lr, double eps,
                       int* err, ttb_stream stream) {
  if (!param || !grad || !state_sum || n < 0) return TTB_EINVAL;
  if (!(lr >= 0.0) || !(eps >= 0.0)) return TTB_EINVAL;
  if (err) {
    int rc = ttb_check_finite(grad, n, err, stream);
    if (rc) return rc;
  }
  return cuda_status(launch_adagrad(param, grad, state_sum, n, lr, eps, (cudaStream_t)stream, err));
}

int ttb_cores_modified(ttb_handle* h) {
  if (!h) return TTB_EINVAL;
  h->img_valid = 0;
  return TTB_OK;
}

int ttb_sgd_update(float* param, const float* grad, double* velocity, int64_t n, double lr, double momentum,
                   ttb_stream stream) {
  if (!param || !grad || n < 0) return TTB_EINVAL;
  if (!(lr >= 0.0) || !(momentum >= 0.0 && momentum < 1.0)) return TTB_EINVAL;
  if (momentum > 0.0 && !velocity) return TTB_EINVAL;
  if (momentum == 0.0) velocity = nullptr;
  return cuda_status(launch_sgd(param, grad, velocity, n, lr, momentum, (cudaStream_t)stream));
}

int ttb_sgd_update_multi(const ttb_sgd_tensor* tensors, int count, double lr, double momentum, ttb_stream stream) {
  if (count < 0 || (count > 0 && !tensors) || !(lr >= 0.0) || !(momentum >= 0.0 && momentum < 1.0)) return TTB_EINVAL;
  std::vector<ttb_sgd_tensor> t(tensors, tensors + count);
  for (auto& x : t) {
    if (x.n < 0 || (x.n > 0 && (!x.param || !x.grad)) || (momentum > 0.0 && x.n > 0 && !x.velocity))
      return TTB_EINVAL;
    if (momentum == 0.0) x.velocity = nullptr;  // (as ttb_sgd_update)
  }
  return cuda_status(launch_sgd_multi(t.data(), count, lr, momentum, (cudaStream_t)stream));
}

int ttb_check_finite(const float* grad, int64_t n, int* err, ttb_stream stream) {
  if (!grad || !err || n < 0) return TTB_EINVAL;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return cuda_status(launch_gradcheck(grad, n, err, sms, (cudaStream_t)stream));
}

int ttb_sgd_update_checked(float* param, const float* grad, double* velocity, int64_t n, double lr, double momentum,
                           int* err, ttb_stream stream) {
  if (!param || !grad || !err || n < 0) return TTB_EINVAL;
  if (!(lr >= 0.0) || !(momentum >= 0.0 && momentum < 1.0)) return TTB_EINVAL;
  if (momentum > 0.0 && !velocity) return TTB_EINVAL;
  if (momentum == 0.0) velocity = nullptr;
  int rc = ttb_check_finite(grad, n, err, stream);
  if (rc) return rc;
  return cuda_status(launch_sgd(param, grad, velocity, n, lr, momentum, (cudaStream_t)stream, err));
}

int* ttb_status_word(ttb_handle* h) {
  if (!h) return nullptr;
  return h->fast ? h->w.fast_hdr : h->w.err;
}

int ttb_read_status(ttb_handle* h, int64_t status[8], ttb_stream stream) {
  if (!h || !status) return TTB_EINVAL;
  int hdr[16];
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemcpyAsync(hdr, h->w.err, sizeof(hdr), cudaMemcpyDeviceToHost, s) != cudaSuccess) return TTB_ECUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return TTB_ECUDA;
  status[1] = h->T;
  status[2] = h->B;
  status[6] = h->gen;
  if (h->fast) {
    int fh[8];
    if (cudaMemcpyAsync(fh, h->w.fast_hdr, sizeof(fh), cudaMemcpyDeviceToHost, s) != cudaSuccess) return TTB_ECUDA;
    if (cudaStreamSynchronize(s) != cudaSuccess) return TTB_ECUDA;
    status[0] = fh[0] | (h->legacy_planned ? hdr[0] : 0);
    status[3] = fh[3];
    const bool counted = h->su_gen == h->gen;  // ttb_plan_counts ran on this plan
    status[4] = counted ? h->su[0] : (h->legacy_planned ? hdr[2] : -1);
    status[5] = counted ? h->su[1] : -1;  // unique rows: not formed by this pipeline's step kernels
    status[7] = fh[2];                            // work items
    return TTB_OK;
  }
  status[0] = hdr[0];
  status[3] = hdr[1];
  status[4] = hdr[2];
  status[5] = h->backwarded ? hdr[3] : 0;
  status[7] = 0;
  return TTB_OK;
}

int ttb_plan_counts(ttb_handle* h, int64_t su[2], ttb_stream stream) {
  if (!h || !su) return TTB_EINVAL;
  if (!h->planned) return TTB_ESTATE;
  if (h->batched) return TTB_ESTATE;  // per-table counters / reference plans: not for batched handles
  if (!h->fast) {  // the deterministic pipeline forms both (U after a backward)
    int64_t st[8];
    int rc = ttb_read_status(h, st, stream);
    if (rc) return rc;
    su[0] = st[4];
    su[1] = h->backwarded ? st[5] : -1;
    return TTB_OK;
  }
  if (h->su_gen != h->gen) {
    if (fast_count_su(h, h->plan_idx, h->plan_idx64, h->plan_off, h->su, (cudaStream_t)stream) != cudaSuccess)
      return TTB_ECUDA;
    h->su_gen = h->gen;
  }
  su[0] = h->su[0];
  su[1] = h->su[1];
  return TTB_OK;
}

int ttb_export_plan(ttb_handle* h, int64_t* work, int64_t* slot_occ, int64_t* seg_ids, int64_t* seg_inv,
                    int64_t* digits, ttb_stream stream) {
  if (!h) return TTB_EINVAL;
  if (!h->planned) return TTB_ESTATE;
  if (h->batched) return TTB_ESTATE;  // per-table counters / reference plans: not for batched handles
  if (!h->legacy_planned) {
    // the reference-ordered plan (first-occurrence slots, segments) on demand
    cudaError_t e = launch_plan(h, h->plan_idx, h->plan_idx64, h->plan_off, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_status(e);
    h->legacy_planned = 1;
  }
  return cuda_status(launch_export_plan(h, work, slot_occ, seg_ids, seg_inv, digits, (cudaStream_t)stream));
}

int ttb_export_fast_plan(ttb_handle* h, int64_t counts[4], int32_t* item_start, uint32_t* item_key,
                         int32_t* tile_info, int32_t* sbi, int32_t* cta_tiles, ttb_stream stream) {
  if (!h || !counts) return TTB_EINVAL;
  if (!h->planned || !h->fast) return TTB_ESTATE;
  cudaStream_t s = (cudaStream_t)stream;
  int fh[8];
  if (cudaMemcpyAsync(fh, h->w.fast_hdr, sizeof(fh), cudaMemcpyDeviceToHost, s) != cudaSuccess) return TTB_ECUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return TTB_ECUDA;
  const int64_t items = fh[2], tiles = fh[4];
  counts[0] = items;
  counts[1] = tiles;
  counts[2] = h->num_sms;
  counts[3] = h->T;
  const cudaMemcpyKind dd = cudaMemcpyDeviceToDevice;
  if (item_start && cudaMemcpyAsync(item_start, h->w.f_item_start, sizeof(int) * (items + 1), dd, s)) return TTB_ECUDA;
  if (item_key && cudaMemcpyAsync(item_key, h->w.f_item_key, sizeof(unsigned) * items, dd, s)) return TTB_ECUDA;
  if (tile_info && cudaMemcpyAsync(tile_info, h->w.f_tile_info, sizeof(int4) * tiles, dd, s)) return TTB_ECUDA;
  if (sbi && cudaMemcpyAsync(sbi, h->w.f_sbi, sizeof(int2) * h->T, dd, s)) return TTB_ECUDA;
  if (cta_tiles && cudaMemcpyAsync(cta_tiles, h->w.f_cta, sizeof(int) * (h->num_sms + 1), dd, s)) return TTB_ECUDA;
  return cudaStreamSynchronize(s) == cudaSuccess ? TTB_OK : TTB_ECUDA;
}

int ttb_export_unique(ttb_handle* h, int64_t* rows, float* grads, ttb_stream stream) {
  if (!h) return TTB_EINVAL;
  if (!h->backwarded || h->fast) return TTB_ESTATE;
  return cuda_status(launch_export_unique(h, rows, grads, (cudaStream_t)stream));
}

int ttb_export_slots(ttb_handle* h, float* slots, ttb_stream stream) {
  if (!h || !slots) return TTB_EINVAL;
  if (!h->forwarded || h->fast) return TTB_ESTATE;
  int64_t st[8];
  int rc = ttb_read_status(h, st, stream);
  if (rc) return rc;
  const size_t n = (size_t)st[3] * h->dims.n1 * h->dims.n2 * h->dims.r2;
  return cuda_status(
      cudaMemcpyAsync(slots, h->w.slots, n * sizeof(float), cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
}

}  // extern "C"
