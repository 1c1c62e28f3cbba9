/*
 * skewgcn_b200 — C ABI of the B200-native skewed-sampling GCN hot path.
 *
 * The reference (arXiv 2101.07706 simulator, /root/reference/pkg/src/skewgcn) is pure
 * Python; its "plugin interface" for this path is the set of Python functions the
 * training loop calls.  Each entry point below replaces one of them; the Python mirror
 * in paper_2101_07706_b200/ binds them with ctypes (INTEGRATION.md shows the binding).
 *
 * Conventions: every function returns 0 on success or a negative skg status
 * (SKG_ERR_*); skg_last_error() returns a message whose wording follows the reference's
 * exceptions.  Pointers named *_dev / uint64 "ptr" arguments are CUDA device pointers;
 * everything else is host memory.  `stream` is a cudaStream_t (NULL = legacy default).
 * Calls are stream-ordered and asynchronous unless documented as synchronous.
 */
#ifndef SKEWGCN_B200_H
#define SKEWGCN_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SKG_OK 0
#define SKG_ERR_CUDA (-1)
#define SKG_ERR_ARG (-2)
#define SKG_ERR_NOT_ADJACENT (-3) /* graph.py:217-219  "candidates not adjacent to s_l" */
#define SKG_ERR_NO_LABELS (-4)    /* training.py:296-297 "batch contains no labeled nodes" */
#define SKG_ERR_CAPACITY (-5)
#define SKG_ERR_EMPTY (-6)        /* training.py:172-173 "empty batch" */

#define SKG_MODE_FULL 0
#define SKG_MODE_LOCAL 1
#define SKG_MODE_SKEWED 2
#define SKG_KIND_LADIES 0
#define SKG_KIND_SAINT 1
#define SKG_DT_F32 0
#define SKG_DT_F64 1

#define SKG_RNG_PCG64 0    /* numpy PCG64 (default_rng / spawn_rng, seeding.py:27) */
#define SKG_RNG_PHILOX 1   /* numpy Philox (Philox4x64-10) */
#define SKG_RNG_EXPLICIT 2 /* uniforms drawn by the caller's Generator (any bit generator) */

/* The uniform stream of one plan: the `rng` argument of ladies_plan / saint_plan
 * (training.py:162-164, 216-219), consumed by Generator.choice's random(B) at
 * sampling.py:184.  Plan draws number d = 1, 2, ... in consumption order.
 *   PCG64:    w[0..3] = state_hi, state_lo, inc_hi, inc_lo; draw d = output after d steps.
 *   PHILOX:   w[0..3] = counter, w[4..5] = key, w[6..9] = buffer, buffer_pos in 0..4
 *             (numpy's bit_generator.state); draw d = numpy's d-th next_uint64.
 *   EXPLICIT: uniforms[d-1] (host memory, n_uniforms >= n_layers * budget covers every
 *             draw a plan can make); the caller advances its Generator by the consumed
 *             count (skg_plan_stats info[1]) afterwards. */
typedef struct skg_rng {
  int32_t kind;
  int32_t buffer_pos;
  uint64_t w[10];
  const double* uniforms;
  int64_t n_uniforms;
} skg_rng;

typedef struct skg_ctx skg_ctx;
typedef struct skg_plans skg_plans;
typedef struct skg_gcn skg_gcn;

int skg_abi_version(void);
const char* skg_last_error(void);
unsigned long long skg_kernel_launches(void);
int skg_device_count(void);
/* Per-kernel timing: bracket every launch of `kernel_name` with CUDA events on its
 * stream until skg_profile_stop, which synchronises and returns the summed time. */
int skg_profile_start(const char* kernel_name);
int skg_profile_stop(double* total_ms, int64_t* launches);
/* With kernel_name "*": every launch is bracketed; skg_profile_table then writes one
 * "name launches total_ms" line per launch name (template-qualified for the GEMMs). */
int skg_profile_table(char* out, int64_t cap);
/* Capture-only mode: launch sequences replayed as CUDA graphs (the LADIES sampler and the
 * batched training step) are captured and instantiated but not replayed while it is on. */
int skg_set_capture_only(int on);

/* ---------------------------------------------------------------- host RNG runtime
 * spawn_rng (seeding.py:17-27): SHA-256 of each label's repr -> SeedSequence -> PCG64.
 * out_state = {state_hi, state_lo, inc_hi, inc_lo} (numpy's PCG64 state). */
int skg_spawn_pcg64(uint64_t master_seed, const char* const* label_reprs, int n_labels,
                    uint64_t out_state[4]);
/* Generator.choice(pop, size, replace=False) on a PCG64 state (indices, unsorted). */
int skg_choice_noreplace(const uint64_t state[4], int has_uint32, uint32_t uinteger,
                         int64_t pop, int64_t size, int64_t* out_idx);
/* One worker-iteration of train_distributed's host work (training.py:488-493):
 * batch = node_set(spawn_rng(seed,"batch",epoch,it,w).choice(train_w, min(bs,|train_w|),
 * replace=False)) and the PCG64 state of spawn_rng(seed,"plan",epoch,it,w). */
int skg_iteration_inputs(uint64_t master_seed, int64_t epoch, int64_t it, int64_t worker,
                         const int64_t* train_w, int64_t n_train_w, int64_t batch_size,
                         int64_t* out_batch, int64_t* out_len, uint64_t plan_state[4]);
/* skg_iteration_inputs for n worker-iterations (a look-ahead group of training.py:
 * 488-493 iterations) on up to n_threads host threads: item i = (epochs[i], its[i],
 * workers[i]) over train_ptrs[i] (int64 node ids, train_lens[i] of them); batch i packed
 * at out_batch[out_off[i] .. out_off[i+1]), plan state at plan_states[4i..4i+3]. */
int skg_group_inputs(uint64_t master_seed, int n, const int64_t* epochs, const int64_t* its,
                     const int32_t* workers, const uint64_t* train_ptrs, const int64_t* train_lens,
                     int64_t batch_size, int64_t* out_batch, int64_t* out_off,
                     uint64_t* plan_states, int n_threads);

/* ---------------------------------------------------------------- graph store
 * WeightedGraph (graph.py:20-79) + Partition.owner (partition.py:21) replicated on one
 * device: int64 offsets, int32 columns, fp64 weights, int32 owner. Synchronous. */
int skg_ctx_create(int device, int64_t n_nodes, int64_t nnz, const int64_t* offsets,
                   const int32_t* neighbors, const double* weights, int32_t n_workers,
                   const int32_t* owner, skg_ctx** out);
int skg_ctx_destroy(skg_ctx* ctx);
/* Feature rows of this rank's shard (all n rows when n_ranks == 1), row-major n_rows x dim,
 * dtype SKG_DT_F32 / SKG_DT_F64.  Stored padded to a multiple of 4 elements. */
int skg_ctx_set_features(skg_ctx* ctx, int dtype, int64_t dim, int64_t n_rows,
                         const void* host_rows);
/* Multi-hot (0/1) features bit-packed (the YouTube shape's 2048-d
 * multi-hot rows; the reference keeps a dense float matrix, graph.py:30 Graph.features):
 * n_rows x words_per_row uint32, feature c at bit (c & 31) of word (c >> 5).  The layer-0
 * SpMM expands the bits to exact 0 / 1 in the compute dtype (dtype), so results equal
 * skg_ctx_set_features on the unpacked rows.  Shards uploaded afterwards are packed rows. */
int skg_ctx_set_features_bits(skg_ctx* ctx, int dtype, int64_t dim, int64_t n_rows,
                              const uint32_t* host_words, int64_t words_per_row);
/* Multi-GPU: feature rows are owned by ranks; node_rank/node_row give each node's home
 * (rank, row) and shard_ptrs the device pointers (local or NVLink-mapped peer) of every
 * rank's shard.  With one rank this is implicit (rank 0, row = node). */
int skg_ctx_set_feature_map(skg_ctx* ctx, int n_ranks, const uint64_t* shard_ptrs,
                            const int32_t* node_rank, const int32_t* node_row);
int skg_ctx_feature_ptr(skg_ctx* ctx, uint64_t* out_ptr, int64_t* out_ld);
/* Upload a feature shard (n_rows x dim host rows, the ctx's dtype) into its own device
 * allocation (exportable with skg_ipc_handle); owned and freed by the ctx. */
int skg_ctx_shard_upload(skg_ctx* ctx, const void* host_rows, int64_t n_rows,
                         uint64_t* out_dev_ptr);
// Multi-label targets (extension; no reference implementation):
// n x ceil(C/64) uint64 multi-hot words, bit k%64 of word k/64 = class k.
int skg_ctx_set_multilabels(skg_ctx* ctx, const uint64_t* words, int32_t n_classes);
int skg_ctx_set_labels(skg_ctx* ctx, const int64_t* labels);
/* Replace the ownership map (Partition.owner) without re-uploading the CSR. */
int skg_ctx_set_owner(skg_ctx* ctx, int32_t n_workers, const int32_t* owner);
/* info: n, nnz, symmetric, feature_ld, feature_dim, feature_dtype, device,
 * n_ranks | normalized << 32 | bit-packed features << 33 */
int skg_ctx_info(skg_ctx* ctx, int64_t out[8]);

/* CUDA IPC for peer feature shards over NVLink (one process per GPU). */
int skg_ipc_handle(uint64_t dev_ptr, uint8_t out_handle[64]);
int skg_ipc_open(const uint8_t handle[64], uint64_t* out_dev_ptr);
int skg_ipc_close(uint64_t dev_ptr);

/* ---------------------------------------------------------------- sample plans
 * A plan set holds n_slots device-resident SamplePlans (training.py:97-114) sampled by
 * one launch sequence.  kind = SKG_KIND_LADIES (ladies_plan, training.py:162-208) or
 * SKG_KIND_SAINT (saint_plan, training.py:216-254). */
int skg_plans_create(skg_ctx* ctx, int kind, int n_slots, int n_layers, int64_t budget,
                     int64_t max_batch, skg_plans** out);
int skg_plans_destroy(skg_plans* ps);
/* ladies_plan for slots [0, n): worker w[i], batch ids[batch_off[i]:batch_off[i+1]]
 * (sorted, unique), PCG64 states rng[4*i..4*i+3]. */
int skg_ladies_sample(skg_plans* ps, int n, const int32_t* workers, const int64_t* batch_off,
                      const int64_t* batch_ids, int mode, double skew_constant,
                      double min_scale, const uint64_t* rng_states, void* stream);
/* Same with batches already resident in HBM: slot i reads batch_len[i] sorted int32 ids
 * at d_batch + i*batch_stride (elements). */
int skg_ladies_sample_device(skg_plans* ps, int n, const int32_t* workers,
                             const int32_t* batch_len, uint64_t d_batch, int64_t batch_stride,
                             int mode, double skew_constant, double min_scale,
                             const uint64_t* rng_states, void* stream);
/* skg_ladies_sample with one skg_rng per slot (PCG64, Philox or explicit uniforms). */
int skg_ladies_sample_rng(skg_plans* ps, int n, const int32_t* workers, const int64_t* batch_off,
                          const int64_t* batch_ids, int mode, double skew_constant,
                          double min_scale, const skg_rng* rngs, void* stream);
/* SAINT candidate set (sorted training nodes).  precompute != 0 caches
 * train_column_norms (training.py:211-213) used by full / skewed modes. */
// column_norms(g, rows, candidates) for large row sets: pull formulation (ordered fold over
// each candidate's column, i ascending).  Replaces graph.py:198-220 when |rows| is large
// (GraphSAINT's training-set norms, training.py:211-213).  out: host double[n_cand].
int skg_column_norms_pull(skg_ctx* ctx, const int64_t* rows, int64_t n_rows, const int64_t* cand,
                          int64_t n_cand, double* out);
int skg_saint_set_candidates(skg_plans* ps, const int64_t* train_ids, int64_t n_train,
                             int precompute, void* stream);
/* saint_plan for slots [0, n) with subgraph size = budget (<= |candidates| assumed). */
int skg_saint_sample(skg_plans* ps, int n, const int32_t* workers, int mode,
                     double skew_constant, double min_scale, const uint64_t* rng_states,
                     void* stream);
/* skg_saint_sample with one skg_rng per slot. */
int skg_saint_sample_rng(skg_plans* ps, int n, const int32_t* workers, int mode,
                         double skew_constant, double min_scale, const skg_rng* rngs,
                         void* stream);
/* CommLedger.add_plan (training.py:127-128) on device: ledger_dev is int64 [k x n_layers]
 * (one epoch); adds remote_per_layer of slots [slot0, slot0+n) to their workers' rows. */
int skg_plans_ledger_add(skg_plans* ps, int slot0, int n, uint64_t ledger_dev, void* stream);
/* Sticky error state of a plan set: the err bits of every plan passed to
 * skg_plans_ledger_add since the last clear (sampling errors, and "batch contains no
 * labeled nodes" from its training step), which later sampling calls cannot erase.
 * Synchronises; returns the matching status (SKG_OK when clean). */
int skg_plans_sticky_error(skg_plans* ps, int clear);
/* Synchronous readback.  stats: n_layers x 16 int64 (doubles bit-cast):
 * [n_upper, n_cand, n_nodes, nnz, remote, has_dist, n_remote_cand, starved, skew,
 *  n_pairs, kept_pairs, s, total, T, pw_depth, 0]; info: [err_bits, draws_consumed,
 * starvation_total, n_layers].  Returns the status for err_bits. */
int skg_plan_stats(skg_plans* ps, int slot, int64_t* stats, int64_t info[4]);
/* Top-down layer t (0 = adjacent to the batch).  Any output pointer may be NULL. */
int skg_plan_layer(skg_plans* ps, int slot, int t, int32_t* nodes, int32_t* indptr,
                   int32_t* indices, double* values, int32_t* cand, double* norm,
                   uint8_t* is_local);

/* ---------------------------------------------------------------- GCN over plans
 * forward / loss_and_backward (training.py:261-318) on slot `slot`.  dims has
 * n_layers+1 entries; weights are row-major d_l x d_{l+1} device arrays. */
int skg_gcn_create(skg_plans* ps, int n_layers, const int64_t* dims, int dtype, skg_gcn** out);
// Loss of the GCN head: 0 = softmax cross-entropy (training.py:293-308, default),
// 1 = multi-label BCE-with-logits, positive weight pos_weight, mean over rows x classes.
int skg_gcn_set_loss(skg_gcn* g, int kind, double pos_weight);
int skg_gcn_destroy(skg_gcn* g);
/* forward + loss + backward; grads (device) += or = dW_l; loss_dev: one double. */
int skg_gcn_step(skg_gcn* g, int slot, const uint64_t* weight_ptrs, const uint64_t* grad_ptrs,
                 int accumulate, uint64_t loss_dev, void* stream);
/* All slots [slot0, slot0+n) in one batched launch per stage; grads (+)= sum over the
 * slots in slot order; loss_dev receives n doubles. */
int skg_gcn_step_batch(skg_gcn* g, int slot0, int n, const uint64_t* weight_ptrs,
                       const uint64_t* grad_ptrs, int accumulate, uint64_t loss_dev, void* stream);
int skg_gcn_forward(skg_gcn* g, int slot, const uint64_t* weight_ptrs, void* stream);
/* Synchronous: copies logits of the last forward (rows x dims[L], unpadded, in the gcn
 * dtype) to host; rows_out receives the batch size. */
int skg_gcn_read_logits(skg_gcn* g, int slot, void* host_out, int64_t* rows_out);
/* predict_logits (training.py:325-334) over the whole graph into out_dev (n x dims[L]). */
int skg_predict_logits(skg_ctx* ctx, int n_layers, const int64_t* dims,
                       const uint64_t* weight_ptrs, int dtype, uint64_t out_dev, void* stream);

/* ---------------------------------------------------------------- optimizer
 * w -= lr * (g / contributors)  (training.py:402-404, 506) */
int skg_sgd_step(int dtype, uint64_t w_dev, uint64_t g_dev, int64_t n, double lr,
                 double contributors, void* stream);
/* Adam (training.py:407-427); t is the step count after increment. */
int skg_adam_step(int dtype, uint64_t w_dev, uint64_t g_dev, uint64_t m_dev, uint64_t v_dev,
                  int64_t n, double lr, double contributors, int64_t t, void* stream);
int skg_zero(int dtype, uint64_t p_dev, int64_t n, void* stream);

/* fp32 GEMM engine: 0 = SIMT FP32, 1 = tcgen05 1xTF32, 3 = tcgen05 3xTF32 (default). */
int skg_set_gemm_mode(int mode);

/* ---------------------------------------------------------------- test hooks
 * Synchronous: numpy pairwise sum (total) and the exact sequential cumsum (cdf, T =
 * cdf[-1]) of a positive host array a[n], through the sampler's own kernels. */
int skg_debug_reduce(const double* a, int64_t n, double* cdf, double* total, double* T);
/* Synchronous: C = op(A) op(B) (row-major host arrays) with the given GEMM mode. */
int skg_debug_gemm(int mode, int ta, int tb, int M, int N, int K, const float* A, const float* B,
                   float* C);

#ifdef __cplusplus
}
#endif
#endif
