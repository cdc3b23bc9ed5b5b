// Fused data-parallel exchange step over peer memory (NVLink / NVSwitch P2P):
// reduce-scatter of the flat gradient buffers -> the optimizer update of this
// rank's shard -> all-gather of the updated parameters, in ONE kernel per
// rank. It replaces Rec-AD's data-parallel exchange (the
// TT-core and MLP gradients all-reduced, then every replica applies
// fused_update, backward.py:186-204 / model.py:353-364) — NCCL all-reduce +
// a separate update kernel on every rank — with:
//
//   1. announce: rank r stores (epoch, bad) into every peer's ready[r]
//      (release, system scope) and waits for all ready[p] of this epoch;
//      "bad" is the caller's device error word (its local finiteness check):
//      if any rank is bad, no rank updates anything (all-or-nothing, as
//      fused_update rejects a non-finite gradient before touching a core).
//   2. rank r owns elements [n r / W, n (r + 1) / W): it loads the W peers'
//      gradients (P2P loads, fixed peer order 0..W-1, fp64 sum rounded once),
//      applies SGD(+momentum) or Adagrad with its fp64 state (only the shard
//      is touched), and stores the new value into every peer's parameter
//      buffer (P2P stores) — each element is computed by exactly one rank,
//      so the replicas stay bitwise identical.
//   3. done: the last CTA of rank r publishes done[r] on every peer after a
//      system fence and waits for all done[p]; the kernel (hence the next
//      kernel on the rank's stream) ends only when every peer has written
//      its shard into this rank's parameters and finished reading this
//      rank's gradients (so they may be overwritten by the next backward).
//
// The epoch lives in device memory (flags[2W + 1]) and advances by one per
// call, so the step can be captured in a CUDA graph. A peer that never
// arrives (crashed rank) trips a bounded spin: TTB_ERRBIT_PEER is latched and
// the kernel exits instead of hanging.
#include <cuda.h>

#include <cstring>

#include "ttb_common.cuh"
#include "ttb_internal.h"

namespace ttb {
namespace {

constexpr int kDpThreads = 512;
constexpr long long kSpinCycles = 20LL * 2000 * 1000 * 1000;  // ~20 s at 2 GHz

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// spin until *p >= target; false on timeout
__device__ bool wait_at_least(const unsigned* p, unsigned target) {
  const long long t0 = clock64();
  while (ld_acquire_sys(p) < target) {
    __nanosleep(64);
    if (clock64() - t0 > kSpinCycles) return false;
  }
  return true;
}

// flags (per rank, u32): [0, W) ready[p] = 2 epoch + bad written by rank p;
// [W, 2W) done[p] = epoch written by rank p; [2W] CTA arrivals; [2W + 1] epoch
__global__ void __launch_bounds__(kDpThreads) k_dp_exchange(ttb_dp_peers P, int64_t n, double lr, double mu,
                                                            int adagrad, double* __restrict__ state,
                                                            int* __restrict__ err) {
  pdl_enter();
  const int W = P.world, r = P.rank;
  unsigned* my = P.flags[r];
  __shared__ unsigned s_epoch;
  __shared__ int s_skip;
  if (threadIdx.x == 0) {
    s_epoch = *(volatile unsigned*)(my + 2 * W + 1) + 1;
    s_skip = 0;
  }
  __syncthreads();
  const unsigned epoch = s_epoch;
  // 1. announce (block 0) and wait for every peer (every block)
  if (blockIdx.x == 0 && threadIdx.x < W) {
    const unsigned bad = (err != nullptr && *(volatile int*)err != 0) ? 1u : 0u;
    __threadfence_system();
    st_release_sys(P.flags[threadIdx.x] + r, 2u * epoch + bad);
  }
  if (threadIdx.x < W) {
    if (!wait_at_least(my + threadIdx.x, 2u * epoch)) {
      if (err) atomicOr(err, TTB_ERRBIT_PEER);
      s_skip = 1;
    } else if (ld_acquire_sys(my + threadIdx.x) & 1u) {
      s_skip = 1;  // some rank holds a non-finite gradient: nobody updates
      if (err) atomicOr(err, TTB_ERRBIT_NONFINITE);
    }
  }
  __syncthreads();
  // 2. this rank's shard
  if (!s_skip) {
    const int64_t lo = n * r / W, hi = n * (r + 1) / W;
    for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi;
         i += (int64_t)gridDim.x * blockDim.x) {
      double sum = 0.0;
      for (int p = 0; p < W; ++p) sum += (double)__ldcv(P.grad[p] + i);
      const float g = (float)sum;
      float p_new;
      const float p_old = P.param[r][i];
      if (!isfinite(g)) {  // finite shards, overflowing sum: keep the element, report
        if (err) atomicOr(err, TTB_ERRBIT_NONFINITE);
        p_new = p_old;
      } else if (adagrad) {
        p_new = adagrad_apply(p_old, g, state + i, lr, mu);
      } else {
        p_new = sgd_apply(p_old, g, state ? state + i : nullptr, lr, mu);
      }
      for (int p = 0; p < W; ++p) __stcg(P.param[p] + i, p_new);
    }
  }
  // 3. done: the last CTA of this rank publishes and waits for the peers
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned arrived = atomicAdd(my + 2 * W, 1u) + 1;
    if (arrived == gridDim.x) {
      my[2 * W] = 0;
      __threadfence_system();
      for (int p = 0; p < W; ++p) st_release_sys(P.flags[p] + W + r, epoch);
      bool ok = true;
      for (int p = 0; p < W; ++p) ok = wait_at_least(my + W + p, epoch) && ok;
      if (!ok && err) atomicOr(err, TTB_ERRBIT_PEER);
      *(volatile unsigned*)(my + 2 * W + 1) = epoch;
    }
  }
}

}  // namespace

cudaError_t launch_dp_exchange(const ttb_dp_peers& P, int64_t n, double lr, double mu, int adagrad, double* state,
                               int* err, int grid, cudaStream_t s) {
  if (grid <= 0) {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid = sms;
  }
  cudaError_t e = launch_pdl(k_dp_exchange, dim3(grid), dim3(kDpThreads), 0, s, P, n, lr, mu, adagrad, state, err);
  if (e == cudaSuccess) count_launch();
  return e == cudaSuccess ? cudaGetLastError() : e;
}

// base address of the allocation holding `p` (cudaIpcGetMemHandle needs the base)
cudaError_t alloc_base(const void* p, void** base, size_t* size) {
  typedef CUresult (*Fn)(CUdeviceptr*, size_t*, CUdeviceptr);
  static Fn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !f) return cudaErrorNotSupported;
    fn = (Fn)f;
  }
  CUdeviceptr b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, (CUdeviceptr)p) != CUDA_SUCCESS) return cudaErrorInvalidValue;
  *base = (void*)b;
  *size = sz;
  return cudaSuccess;
}

}  // namespace ttb

using namespace ttb;

extern "C" {

size_t ttb_dp_flag_words(int world) { return (size_t)(2 * world + 2); }

int ttb_dp_exchange_update(const ttb_dp_peers* peers, int64_t n, double lr, double momentum, int adagrad,
                           double* state, int* err, int grid, ttb_stream stream) {
  if (!peers || n < 0 || peers->world < 1 || peers->world > TTB_DP_MAX_PEERS) return TTB_EINVAL;
  if (peers->rank < 0 || peers->rank >= peers->world) return TTB_EINVAL;
  for (int p = 0; p < peers->world; ++p)
    if (!peers->grad[p] || !peers->param[p] || !peers->flags[p]) return TTB_EINVAL;
  if (!(lr >= 0.0)) return TTB_EINVAL;
  if (adagrad) {
    if (!state || !(momentum >= 0.0)) return TTB_EINVAL;  // momentum carries eps
  } else {
    if (!(momentum >= 0.0 && momentum < 1.0)) return TTB_EINVAL;
    if (momentum > 0.0 && !state) return TTB_EINVAL;
    if (momentum == 0.0) state = nullptr;
  }
  return launch_dp_exchange(*peers, n, lr, momentum, adagrad, state, err, grid, (cudaStream_t)stream) == cudaSuccess
             ? TTB_OK
             : TTB_ECUDA;
}

int ttb_ipc_handle(const void* dev_ptr, void* handle, int64_t* offset) {
  if (!dev_ptr || !handle || !offset) return TTB_EINVAL;
  void* base = nullptr;
  size_t size = 0;
  if (alloc_base(dev_ptr, &base, &size) != cudaSuccess) return TTB_ECUDA;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, base) != cudaSuccess) return TTB_ECUDA;
  memcpy(handle, &h, sizeof(h));
  *offset = (int64_t)((const char*)dev_ptr - (const char*)base);
  return TTB_OK;
}

int ttb_ipc_open(const void* handle, int64_t offset, void** dev_ptr) {
  if (!handle || !dev_ptr || offset < 0) return TTB_EINVAL;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  if (cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return TTB_ECUDA;
  *dev_ptr = (char*)base + offset;
  return TTB_OK;
}

int ttb_ipc_close(void* dev_ptr, int64_t offset) {
  if (!dev_ptr) return TTB_EINVAL;
  return cudaIpcCloseMemHandle((char*)dev_ptr - offset) == cudaSuccess ? TTB_OK : TTB_ECUDA;
}

}  // extern "C"
