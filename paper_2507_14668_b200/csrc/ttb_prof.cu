// Per-kernel CUDA-event timing and the FP32 FMA peak calibration kernel.
#include <string.h>

#include "ttb_internal.h"

namespace ttb {

static void prof_flush(Profiler* p) {
  for (int i = 0; i < p->n; ++i) {
    float ms = 0.f;
    cudaEventSynchronize(p->ev[i][1]);
    cudaEventElapsedTime(&ms, p->ev[i][0], p->ev[i][1]);
    int k = 0;
    while (k < p->nnames && strcmp(p->names[k], p->pend_name[i]) != 0) ++k;
    if (k == p->nnames) {
      if (p->nnames == kMaxProfNames) continue;
      p->names[p->nnames++] = p->pend_name[i];
      p->ms[k] = 0.0;
      p->calls[k] = 0;
    }
    p->ms[k] += ms;
    p->calls[k] += 1;
  }
  p->n = 0;
}

ProfScope::ProfScope(ttb_handle* h, cudaStream_t st, const char* name) : p(&h->prof), s(st), slot(-1) {
  if (!p->on) return;
  if (p->n == kMaxProfEvents) prof_flush(p);
  slot = p->n++;
  p->pend_name[slot] = name;
  cudaEventRecord(p->ev[slot][0], s);
}

ProfScope::~ProfScope() {
  if (slot >= 0) cudaEventRecord(p->ev[slot][1], s);
}

// 8 independent FMA chains per thread; 2 * 8 * iters flops per thread
__global__ void __launch_bounds__(256) k_fma_peak(float* sink, int iters, float a, float b) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-7f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
  }
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += x[i];
  if (acc == 1234.5f) sink[threadIdx.x] = acc;
}

}  // namespace ttb

using namespace ttb;

extern "C" {

int ttb_profile_enable(ttb_handle* h, int on) {
  if (!h) return TTB_EINVAL;
  Profiler* p = &h->prof;
  if (on && !p->on) {
    for (int i = 0; i < kMaxProfEvents; ++i)
      for (int j = 0; j < 2; ++j)
        if (cudaEventCreate(&p->ev[i][j]) != cudaSuccess) return TTB_ECUDA;
    p->n = 0;
    p->nnames = 0;
    p->on = 1;
  } else if (!on && p->on) {
    prof_flush(p);
    for (int i = 0; i < kMaxProfEvents; ++i)
      for (int j = 0; j < 2; ++j) cudaEventDestroy(p->ev[i][j]);
    p->on = 0;
  }
  return TTB_OK;
}

int ttb_profile_read(ttb_handle* h, char* names, double* ms, int64_t* calls, int cap, int* count) {
  if (!h || !count) return TTB_EINVAL;
  Profiler* p = &h->prof;
  if (p->on) prof_flush(p);
  int n = p->nnames < cap ? p->nnames : cap;
  for (int i = 0; i < n; ++i) {
    if (names) {
      strncpy(names + 32 * i, p->names[i], 31);
      names[32 * i + 31] = 0;
    }
    if (ms) ms[i] = p->ms[i];
    if (calls) calls[i] = p->calls[i];
  }
  *count = n;
  p->nnames = 0;
  return TTB_OK;
}

int ttb_set_option(ttb_handle* h, int option, int value) {
  if (!h) return TTB_EINVAL;
  switch (option) {
    case 1: h->bwd_split = value ? 1 : 0; return TTB_OK;  // TTB_OPT_BWD_SPLIT
    case 3: h->allow_empty = value ? 1 : 0; return TTB_OK;  // TTB_OPT_ALLOW_EMPTY
    case 2:                                                // TTB_OPT_FAST
      if (value && !h->fast_ok) return TTB_EINVAL;
      if (!value && h->batched) return TTB_EINVAL;  // a batched handle has only the tensor-core pipeline
      h->fast = value ? 1 : 0;
      h->planned = h->forwarded = h->backwarded = 0;  // a plan belongs to one pipeline
      return TTB_OK;
    default: return TTB_EINVAL;
  }
}

int ttb_fma_peak(float* sink, int iters, int blocks, ttb_stream stream) {
  if (!sink || iters < 1 || blocks < 1) return TTB_EINVAL;
  k_fma_peak<<<blocks, 256, 0, (cudaStream_t)stream>>>(sink, iters, 0.999999f, 1e-7f);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? TTB_OK : TTB_ECUDA;
}

}  // extern "C"
