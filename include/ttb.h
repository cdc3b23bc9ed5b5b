/*
 * ttb.h — C ABI of the B200 (sm_100a) TT-EmbeddingBag hot path.
 *
 * One handle per TT table. All array arguments are DEVICE pointers owned by
 * the caller (PyTorch tensors on the Python side); the library never
 * allocates device memory — the caller sizes and passes a workspace. Every
 * call is stream-ordered and asynchronous unless documented as syncing, and
 * the compute calls (plan / forward / backward / update) are CUDA-graph
 * capturable: batch-dependent counts (distinct prefixes P, segments S,
 * distinct rows U) stay on the device and kernels are launched over upper
 * bounds.
 *
 * Each entry point replaces one reference (numpy) operator of Rec-AD's TT
 * path; citations are file:line in the reference artifact (pkg/src/ttemb):
 *
 *   ttb_plan          lookup.py:97-124   prepare_reuse_plan (first-occurrence
 *                                        prefix slots, hits/misses)
 *                     lookup.py:254-260, 280-284  bag validation, bag ids,
 *                                        (bag, slot) segments via np.unique
 *                     tt_core.py:210-224 linear_index_to_tt_index (digits)
 *   ttb_forward       lookup.py:127-149  execute_prefix_products (reuse buffer)
 *                     lookup.py:286-296  forward_batch close + sum pooling
 *   ttb_backward      backward.py:72-87  unique_aggregate (row-gradient merge)
 *                     backward.py:101-183 tt_core_grads (core gradients)
 *   ttb_aggregate     backward.py:72-87  unique_aggregate alone
 *   ttb_backward_sgd  backward.py:207-227 backward_batch = aggregate + grads +
 *                                        fused_update, in one device pass
 *   ttb_sgd_update    backward.py:186-204 fused_update / model.py:353-364
 *                                        DlrmModel.train_step update loop
 *   ttb_export_*      read back plan / unique-row outputs for parity checks
 *                     (ReusePlan.work / slot_of, seg ids, unique_aggregate)
 *
 * Status codes: 0 ok, negative on failure (see TTB_E*). Data-dependent
 * errors (index out of range, empty bag, malformed offsets) are detected on
 * the device and latched in the workspace; ttb_read_status() returns them.
 * The Python wrapper maps them to ValueError exactly where the reference
 * raises ValueError (lookup.py:88-94, 254-255).
 */
#ifndef TTB_H
#define TTB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TTB_ABI_VERSION 1

#define TTB_OK 0
#define TTB_EINVAL (-1)     /* bad geometry / argument / capacity */
#define TTB_ERANGE (-2)     /* an index lies outside [0, rows_padded) */
#define TTB_EEMPTY (-3)     /* empty batch or an empty bag */
#define TTB_EOFFSETS (-4)   /* offsets not 0 .. T, or decreasing */
#define TTB_ENONFINITE (-5) /* non-finite gradient */
#define TTB_ECUDA (-6)      /* CUDA launch / runtime failure */
#define TTB_ESTATE (-7)     /* call order violated (forward before plan, ...) */

/* device error-word bits (ttb_read_status status[0]) */
#define TTB_ERRBIT_RANGE 1
#define TTB_ERRBIT_EMPTY_BAG 2
#define TTB_ERRBIT_OFFSETS 4
#define TTB_ERRBIT_NONFINITE 8
#define TTB_ERRBIT_PEER 16 /* data-parallel exchange: a peer never arrived */

/*
 * Table geometry, reference TtShape (tt_core.py:41-82) with d = 3.
 * A d = 2 table (m1, m2), (n1, n2), (1, R, 1) is passed as
 * m = (1, m1, m2), n = (1, n1, n2), r = (1, 1, R, 1) with a 1x1x1 core of
 * value 1 in front: the arithmetic is identical.
 * Core k has the reference layout (r[k], m[k] * n[k], r[k+1]), C order.
 */
typedef struct ttb_geom {
  int64_t m[3];
  int32_t n[3];
  int32_t r[4];
} ttb_geom;

typedef struct ttb_handle ttb_handle; /* opaque host-side handle */
#define TTB_MAX_TABLES 64
typedef void *ttb_stream;             /* a cudaStream_t */

int ttb_abi_version(void);
const char *ttb_strerror(int code);
/* cudaGetErrorString of the calling thread's last CUDA failure behind a
 * TTB_ECUDA status (diagnostics; no reference counterpart) */
const char *ttb_last_cuda_error(void);
/* number of kernels this library has launched in the process (a counter) */
int64_t ttb_launch_count(void);

/* device workspace bytes for tables of geometry g, batches up to max_T
 * indices in up to max_B bags */
int ttb_workspace_bytes(const ttb_geom *g, int64_t max_T, int64_t max_B,
                        size_t *bytes);
/* bind a caller-owned workspace (>= ttb_workspace_bytes) to a new handle and
 * initialise it on `stream`. Returns NULL on bad arguments. */
ttb_handle *ttb_create(const ttb_geom *g, int64_t max_T, int64_t max_B,
                       void *workspace, size_t bytes, ttb_stream stream);
void ttb_destroy(ttb_handle *h);

/* K1: plan one batch. indices: T int64 (idx_is_64 = 1) or int32 values;
 * offsets: B + 1 int64 bag boundaries (offsets[0] = 0, offsets[B] = T). */
int ttb_plan(ttb_handle *h, const void *indices, int idx_is_64,
             const int64_t *offsets, int64_t T, int64_t B, ttb_stream stream);

/* K2 + K3: pooled bag embeddings out (B, N) fp32, N = n1 n2 n3. Also fills
 * the prefix-product (reuse) buffer kept in the workspace for backward. */
int ttb_forward(ttb_handle *h, const float *core0, const float *core1,
                const float *core2, float *out, ttb_stream stream);

/* K4: core gradients (fp32, core layout) for upstream grad_out (B, N).
 * Requires ttb_forward on the same plan with the same cores. */
int ttb_backward(ttb_handle *h, const float *core0, const float *core1,
                 const float *core2, const float *grad_out, float *grad0,
                 float *grad1, float *grad2, ttb_stream stream);

/* K4 first stage alone: order the indices by row and sum each distinct
 * row's upstream gradients (unique_aggregate, backward.py:72-87); read the
 * result back with ttb_export_unique. Requires ttb_plan only. */
int ttb_aggregate(ttb_handle *h, const float *grad_out, ttb_stream stream);

/* K4 + K5: core gradients applied in place as SGD(+momentum):
 *   v <- momentum * v + g (fp64 velocity); core <- f32(f64(core) - lr * v)
 * (momentum == 0: velocity pointers may be NULL). update_mask bit k enables
 * the update of core k (a d = 2 table disables its leading unit core). */
int ttb_backward_sgd(ttb_handle *h, float *core0, float *core1, float *core2,
                     const float *grad_out, double *vel0, double *vel1,
                     double *vel2, double lr, double momentum,
                     int update_mask, ttb_stream stream);

/* K4 + Adagrad (torch.optim.Adagrad semantics, no lr / weight decay) fused
 * like ttb_backward_sgd: s <- s + g^2 (fp64 squared-gradient sums, one per
 * core element, zero-initialised by the caller); core <- f32(f64(core) -
 * lr g / (sqrt(s) + eps)). North-star item (3) names Adagrad next to SGD;
 * the reference implements only SGD(+momentum), so this rule
 * follows PyTorch's published algorithm. Tensor-core pipeline only
 * (TTB_ESTATE otherwise: use ttb_backward + ttb_adagrad_update). */
int ttb_backward_adagrad(ttb_handle *h, float *core0, float *core1, float *core2,
                         const float *grad_out, double *sum0, double *sum1,
                         double *sum2, double lr, double eps, int update_mask,
                         ttb_stream stream);

/* The same Adagrad step on a flat parameter. err (DEVICE int, may be NULL):
 * when given, the gradient is checked first and a non-finite value latches
 * TTB_ERRBIT_NONFINITE and cancels the update (as ttb_sgd_update_checked). */
int ttb_adagrad_update(float *param, const float *grad, double *state_sum,
                       int64_t n, double lr, double eps, int *err,
                       ttb_stream stream);

/* The tensor-core pipeline keeps split-tf32 images of cores 0 and 1 in the
 * workspace. They are rebuilt by ttb_forward whenever the core pointers
 * differ from the last forward / fused update, and written directly by
 * ttb_backward_sgd's update; ttb_backward (gradients returned) drops them.
 * A caller that changes core VALUES by any other means (an optimizer step,
 * loading a checkpoint) while keeping the same pointers must call this
 * before the next ttb_forward. The Python layer does so automatically
 * (tensor version counters). */
int ttb_cores_modified(ttb_handle *h);

/* K5 alone on a flat parameter: used after the data-parallel all-reduce
 * and for dense parameters. velocity may be NULL when momentum == 0. */
int ttb_sgd_update(float *param, const float *grad, double *velocity,
                   int64_t n, double lr, double momentum, ttb_stream stream);

/* ttb_sgd_update over several parameters in ONE launch (DlrmModel's
 * per-parameter update loop, model.py:353-364): the same arithmetic per
 * element (fp64 velocity, one rounding), so the result is bitwise that of
 * `count` ttb_sgd_update calls. velocity may be NULL per tensor when
 * momentum == 0. The array lives in host memory (copied at launch). */
typedef struct {
  float *param;
  const float *grad;
  double *velocity;
  int64_t n;
} ttb_sgd_tensor;
int ttb_sgd_update_multi(const ttb_sgd_tensor *tensors, int count, double lr, double momentum,
                         ttb_stream stream);

/* fused_update with the reference's validation (backward.py:186-204): the
 * gradient is checked for non-finite values first (TTB_ERRBIT_NONFINITE is
 * OR-ed into the caller's DEVICE int *err), and the update runs only if *err
 * is still 0 — otherwise param and velocity are left untouched. Calling
 * ttb_check_finite on several gradients before their updates gives the
 * reference's all-or-nothing semantics across arrays. Stream-ordered. */
int ttb_check_finite(const float *grad, int64_t n, int *err, ttb_stream stream);
int ttb_sgd_update_checked(float *param, const float *grad, double *velocity,
                           int64_t n, double lr, double momentum, int *err,
                           ttb_stream stream);

/* ---- data parallel: fused exchange over peer memory (NVLink / NVSwitch)
 * Replaces the DP exchange of Rec-AD (all-reduce of the
 * TT-core / MLP gradients, then fused_update on every replica,
 * backward.py:186-204) by ONE kernel per rank: reduce-scatter (P2P loads of
 * the peers' gradients, fixed peer order, fp64 sum) -> SGD(+momentum) or
 * Adagrad on this rank's shard -> all-gather (P2P stores of the new values
 * into every peer's parameters). grad[p] / param[p] / flags[p] are rank p's
 * buffers as mapped in THIS process (ttb_ipc_open, or plain pointers when all
 * ranks share one process); flags[p] holds ttb_dp_flag_words(world) u32,
 * zeroed once before the first call. state: fp64 velocity (momentum > 0) or
 * Adagrad squared-gradient sums (adagrad = 1, momentum then carries eps),
 * full length n, only this rank's shard is touched. err (device int, may be
 * NULL): non-zero on entry marks this rank's gradients bad — then NO rank
 * updates (TTB_ERRBIT_NONFINITE is latched everywhere); TTB_ERRBIT_PEER is
 * latched if a peer does not arrive within ~20 s. grid <= 0: one CTA per SM.
 * Every rank must call it once per step with the same n and world. */
#define TTB_DP_MAX_PEERS 8
typedef struct {
  int rank, world;
  float *grad[TTB_DP_MAX_PEERS];
  float *param[TTB_DP_MAX_PEERS];
  unsigned *flags[TTB_DP_MAX_PEERS];
} ttb_dp_peers;
size_t ttb_dp_flag_words(int world);
int ttb_dp_exchange_update(const ttb_dp_peers *peers, int64_t n, double lr,
                           double momentum, int adagrad, double *state,
                           int *err, int grid, ttb_stream stream);
/* CUDA IPC of a device pointer inside any allocation (e.g. a PyTorch caching
 * allocator block): handle = 64 bytes of cudaIpcMemHandle_t of the
 * allocation, offset = dev_ptr - allocation base. */
int ttb_ipc_handle(const void *dev_ptr, void *handle, int64_t *offset);
int ttb_ipc_open(const void *handle, int64_t offset, void **dev_ptr);
int ttb_ipc_close(void *dev_ptr, int64_t offset);

/* The DEVICE int holding the handle's latched error bits (the word
 * ttb_read_status reports in status[0]) for the current pipeline — e.g. the
 * `err` of ttb_dp_exchange_update, so a rank's plan / gradient errors cancel
 * the exchange everywhere and the exchange's own errors surface in
 * ttb_read_status. Valid until ttb_destroy or a pipeline switch. */
int *ttb_status_word(ttb_handle *h);

/* ---- table-batched handles (the reference loops over fields,
 * model.py:295-298 lookups and 334-338 gradients; here ONE plan / forward /
 * backward / update launch set covers every TT field of the model).
 * ntables <= TTB_MAX_TABLES tables with identical n and ranks (the
 * tensor-core geometry: n = (4, 4, 4), ranks (1, 32, 32, 1)) and their own
 * row factors m_f. Their cores are passed STACKED and zero-padded to the
 * common (M1, M2, M3) = max_f m_f (M3 <= 288): core0 (1, nt M1 4, 32),
 * core1 (32, nt M2 4, 32), core2 (32, nt M3 4, 1); table f's core k is the
 * block starting at f M_k along the middle axis (rows past m_f stay zero:
 * nothing references them, so gradients and updates leave them zero).
 * A batch: every table's indices (table-local row ids) concatenated table by
 * table; offsets over nt * bags_per_table bags (table f owns bags
 * [f bags_per_table, (f + 1) bags_per_table)); the output is
 * (nt * bags_per_table, N), table-major. Every other entry point takes the
 * handle as usual (plan, forward, backward[_sgd|_adagrad], read_status);
 * the reference-ordered exports and per-table counters do not apply. */
int ttb_batched_workspace_bytes(const ttb_geom *tables, int ntables,
                                int64_t max_T, int64_t bags_per_table,
                                size_t *bytes);
ttb_handle *ttb_create_batched(const ttb_geom *tables, int ntables,
                               int64_t max_T, int64_t bags_per_table,
                               void *workspace, size_t bytes,
                               ttb_stream stream);

/* SYNCS `stream`. status[0] = device error bits (TTB_ERRBIT_*), [1] = T,
 * [2] = B, [3] = P (distinct prefixes), [4] = S (bag-prefix segments),
 * [5] = U (distinct rows; valid after backward), [6] = plan generation. */
int ttb_read_status(ttb_handle *h, int64_t status[8], ttb_stream stream);

/* The reference's work counters for the current plan (SYNCS `stream`):
 * su[0] = S, the (bag, prefix) segments (lookup.py:280-284, 294-295);
 * su[1] = U, the distinct rows (backward.py:81-87, 218-222). The tensor-core
 * pipeline counts them on demand from the plan's inputs (which must still be
 * valid) — its step kernels never form them; afterwards ttb_read_status
 * reports them too. The deterministic pipeline reports U = -1 until a
 * backward ran. */
int ttb_plan_counts(ttb_handle *h, int64_t su[2], ttb_stream stream);

/* Plan read-back (after ttb_plan). Any pointer may be NULL. Sizes use the
 * counts of ttb_read_status.
 *   work      P x 4 int64: (prefix key, i1, i2, slot), first-occurrence order
 *   slot_occ  T int64: buffer slot of each index's prefix
 *   seg_ids   S int64: sorted bag * P + slot
 *   seg_inv   T int64: segment of each index
 *   digits    T x 3 int64: (i1, i2, i3) of each index                   */
int ttb_export_plan(ttb_handle *h, int64_t *work, int64_t *slot_occ,
                    int64_t *seg_ids, int64_t *seg_inv, int64_t *digits,
                    ttb_stream stream);

/* Tensor-core pipeline plan read-back (after ttb_plan with TTB_OPT_FAST;
 * SYNCS `stream`). counts (host) = {work items, tiles, step-kernel CTAs, T};
 * every pointer is a nullable DEVICE buffer:
 *   item_start  items + 1 int32: first position of each item (last = T)
 *   item_key    items u32: the item's prefix key i2 * m1 + i1
 *   tile_info   tiles x 4 int32: (i2, first item, items, first position)
 *   sbi         T x 2 int32: (bag, i3) of every position, item order
 *   cta_tiles   CTAs + 1 int32: first tile of each step-kernel CTA
 * A work item is a run of <= 32 lookups of one prefix (the reuse unit of
 * lookup.py:127-149); a tile is <= 32 items of one i2. */
int ttb_export_fast_plan(ttb_handle *h, int64_t counts[4], int32_t *item_start,
                         uint32_t *item_key, int32_t *tile_info, int32_t *sbi,
                         int32_t *cta_tiles, ttb_stream stream);

/* unique_aggregate read-back (after ttb_backward / ttb_backward_sgd):
 * rows U int64 in first-occurrence order, grads U x N fp32 (nullable) —
 * the per-row summed upstream gradients (backward.py:72-87). */
int ttb_export_unique(ttb_handle *h, int64_t *rows, float *grads,
                      ttb_stream stream);

/* prefix-product (reuse) buffer read-back: P x (n1 n2) x r2 fp32, slot
 * order (ReuseBuffer.slots, lookup.py:79-85). After ttb_forward. */
int ttb_export_slots(ttb_handle *h, float *slots, ttb_stream stream);

/* ---- offline index reordering (reference reorder.py) -------------------
 * ttb_count_frequencies  reorder.py:90-104   counts[table_len] (u64) of all
 *                        indices; *err != 0 if one lies outside [0, table_len)
 * ttb_rank_rows          reorder.py:100-104  rows by (count desc, id asc):
 *                        row_of_rank and rank_of (int64, either nullable);
 *                        workspace of ttb_rank_workspace_bytes(table_len)
 * ttb_apply_bijection    reorder.py:286-296  out[i] = forward[in[i]]; *err set
 *                        (and out = -1) for indices outside [0, table_len)
 * Community detection (reorder.py:176-236) stays on the host. */
int ttb_count_frequencies(const int64_t *indices, int64_t n, int64_t table_len,
                          uint64_t *counts, int *err, ttb_stream stream);
int ttb_rank_workspace_bytes(int64_t table_len, size_t *bytes);
int ttb_rank_rows(const uint64_t *counts, int64_t table_len, int64_t *row_of_rank,
                  int64_t *rank_of, void *workspace, size_t bytes, ttb_stream stream);
int ttb_apply_bijection(const int64_t *forward, int64_t table_len, const int64_t *in,
                        int64_t *out, int64_t n, int *err, ttb_stream stream);

/* ---- measurement hooks (not part of the reference interface) ----------
 * Per-kernel CUDA-event timing of one handle's launches: enable, run, then
 * read the accumulated milliseconds and launch counts per kernel name
 * (names: cap x 32 chars). Reading syncs and resets the accumulators. */
int ttb_profile_enable(ttb_handle *h, int on);
int ttb_profile_read(ttb_handle *h, char *names, double *ms, int64_t *calls,
                     int cap, int *count);
/* Kernel-path options (defaults are the fastest measured):
 *   TTB_OPT_BWD_SPLIT (1): 1 = backward as a warp-per-prefix rows kernel plus
 *   an i2-chunk GEMM kernel (tcgen05 3xTF32 where the shape allows) instead
 *   of the fused backward kernel (deterministic pipeline only).
 *   TTB_OPT_FAST (2): 1 (default where n = (4,4,4), ranks (1,32,32,1)) = the
 *   tensor-core pipeline: prefix-sorted work tiles, X = G1.G2 formed in TMEM
 *   by tcgen05 3xTF32 in the forward and recomputed in the backward, core
 *   gradients accumulated with fp32 reductions (summation order not fixed).
 *   0 = the deterministic pipeline (fixed summation order, reference-ordered
 *   plan resident, ttb_aggregate / ttb_export_unique / ttb_export_slots).
 *   Under 1, ttb_export_plan builds the reference-ordered plan on demand from
 *   the buffers given to ttb_plan (they must still be valid then) and
 *   ttb_read_status reports S = -1 until it has, U = -1, and status[7] = the
 *   number of work items. Changing the option drops the current plan. */
#define TTB_OPT_BWD_SPLIT 1
#define TTB_OPT_FAST 2
/* TTB_OPT_ALLOW_EMPTY (3): 1 = empty bags are allowed and pool to zero rows,
 * as torch.nn.EmbeddingBag does (the drop-in promise); 0 (the
 * default) = the reference's ValueError for an empty bag (lookup.py:90-91).
 * The batch itself must still hold at least one index (ttb_plan: EEMPTY). */
#define TTB_OPT_ALLOW_EMPTY 3
int ttb_set_option(ttb_handle *h, int option, int value);
/* FP32 FMA throughput probe: blocks x 256 threads x iters x 16 flops; the
 * caller times it with CUDA events to get the measured FP32 peak. */
int ttb_fma_peak(float *sink, int iters, int blocks, ttb_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* TTB_H */
