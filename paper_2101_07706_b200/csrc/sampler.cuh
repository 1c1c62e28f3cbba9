// Device-side data layout of the sampler (shared by sampler.cu, gcn.cu and capi.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace skg {

enum Mode : int32_t { MODE_FULL = 0, MODE_LOCAL = 1, MODE_SKEWED = 2 };
enum Kind : int32_t { KIND_LADIES = 0, KIND_SAINT = 1 };
// uniform streams a plan's draws come from (the rng argument of training.py:162-164, 216-219)
enum RngKind : int32_t { RNG_PCG64 = 0, RNG_PHILOX = 1, RNG_EXPLICIT = 2 };

// Replicated topology (int32 columns, fp64 weights as stored by the reference's
// WeightedGraph, graph.py:28-31) plus the ownership map (partition.py:21).
struct GraphDev {
  int64_t n, nnz;
  const int64_t* off;    // [n+1]
  const int32_t* col;    // [nnz]
  const double* w;       // [nnz]
  const int32_t* owner;  // [n]
  // transpose (CSC) used by the SAINT pull-norm pass; aliases off/col/w when symmetric
  const int64_t* t_off;
  const int32_t* t_row;
  const double* t_w;
  int32_t n_words;       // ceil(n/32)
  int32_t normalized;    // every w_ij == 1/sqrt(d_i d_j) (graph.py:182), checked at load
  const double* degd;    // [n] row lengths as double (normalized graphs)
  // fused range expand: rstart[i * (n_fr + 1) + q] = offset in row i of its first column
  // >= q * fr_size (q = n_fr: the row length); graph-static per range size, built once
  const int32_t* rstart;
  int32_t n_fr;
  int32_t fr_size;
};

// Per-layer scalars of one plan.  Layers are indexed top-down while sampling
// (t = 0 is the layer adjacent to the batch); the Python mirror reverses them like
// training.py:207 does.
struct LayerStat {
  int32_t n_upper;        // |S_{t-1}| (rows of this layer's block)
  int32_t n_cand;         // |N(S)| (after the local restriction in local mode)
  int32_t n_nodes;        // |S_t| sampled (== n_cand when saturated)
  int32_t nnz;            // block nnz
  int32_t remote;         // remote sampled nodes (ledger, training.py:199)
  int32_t has_dist;       // 1 when a distribution was drawn from (not saturated)
  int32_t n_remote_cand;  // |R| among candidates
  int32_t starved;        // local-mode starvation events at this layer
  int32_t skew;           // 1 when skewed weights were used (else linear)
  int32_t pw_depth;       // depth of numpy's pairwise-sum tree for n_cand
  int64_t n_pairs;        // sum of upper-row degrees
  int64_t kept_pairs;     // pairs that landed on a candidate
  double s;               // scale factor baked into q (1.0 for linear)
  double total;           // numpy pairwise sum of the scaled weights
  double T;               // exact sequential cumsum total (cdf[-1])
};

// Per-plan workspace; an array of these lives in device memory, one per slot.
struct PlanDev {
  // ---- configuration, written by the host for each sampling launch
  int32_t kind, worker, mode, n_layers;
  int64_t budget;
  double D, min_scale;
  uint64_t rng[4];          // PCG64 state (hi, lo) and increment (hi, lo)
  int32_t rng_kind;         // RNG_PCG64 (rng), RNG_PHILOX (phx, rng_pos), RNG_EXPLICIT (uniforms)
  int32_t rng_pos;          // Philox: numpy's buffer_pos (4 = buffer exhausted)
  uint64_t phx[10];         // Philox4x64-10: counter[4], key[2], buffer[4] (numpy's state)
  const double* uniforms;   // explicit: uniforms[d - 1] is the plan's d-th uniform
  int64_t n_uniforms;
  int32_t batch_len;        // LADIES: |batch|; SAINT: |candidates|
  int32_t pad0;
  const int32_t* batch;     // LADIES batch ids; SAINT candidate ids (sorted)
  const double* cand_norm;  // SAINT precomputed norms aligned with batch, or null
  // ---- capacities
  int32_t cap_rows;         // max(|batch|, budget) (LADIES), budget (SAINT)
  int32_t cap_cand;         // N_max
  int64_t cap_pairs;        // E_max
  int32_t cap_chunks, cap_supers, cap_slots, cap_tiles;
  // ---- scratch
  uint32_t* bitmap;         // [n_words]
  uint32_t* sbitmap;        // [n_words] sampled set
  uint32_t* bitmap1;        // [ceil(n_words / 32)] global expand: nonzero words of bitmap (zero at rest)
  int32_t* dirty;           // [1] a call failed with state that is zero at rest left set (arena, persistent)
  uint32_t* cnt_pack;       // [n/2+1] 16-bit pair counters per node, zero at rest
  // LADIES contributions (upper-row rank r of every pair (r, j)), by node: the first
  // kSlots arrivals in slots[j], later ones in the overflow list; candidates with more
  // than kSlots get a contiguous, row-sorted range hbuf[hoff[h] .. + count)
  // normalised graphs: the contributions' row ranks by candidate rank k (4 x 16 bits):
  // row-sorted for candidates with <= kSlots contributions, the first kSlots arrivals
  // (any order) for heavier ones
  uint2* cslots;            // [cap_cand]
  // fused range expand (n_fr > 0, GraphDev.rstart): look-back words of the range CTAs per
  // layer (in the per-call zeroed scalars)
  int32_t n_fr;
  int32_t pad1;
  unsigned long long* look; // [L * kMaxFR]
  uint16_t* slots;          // [n*kSlots]
  double* slotw;            // [n*kSlots] stored w_ij (graphs that are not normalised)
  int2* ov;                 // [cap_pairs] overflow pairs (j, r)
  double* ovw;              // [cap_pairs] (not normalised)
  int32_t* hidx;            // [n] node -> heavy index
  int32_t* hoff;            // [cap_cand] heavy range starts
  int32_t* hfill;           // [cap_cand] heavy fill counters
  int32_t* hbuf;            // [cap_pairs] heavy entries (row-sorted after the heavy fold)
  double* hbufw;            // [cap_pairs] (not normalised)
  int32_t* heavy;           // [cap_cand] candidate ranks with count > kSlots
  int32_t* huge;            // [cap_cand] heavy candidates with count > 32
  double* updeg;            // [cap_rows] degree of each upper row (normalised graphs)
  int32_t* row_any;         // [cap_rows] local mode: the upper row kept a column (range expand)
  int32_t* cand_cnt;        // [cap_cand] contributions per candidate
  int64_t* pair_off;        // [cap_rows+1]
  int32_t* word_prefix;     // [n_words]
  int64_t* tile_a;          // [cap_tiles]
  int32_t* counters;        // [8]: 0 heavy, 1 overflow, 2 huge
  double* pw_val;           // [cap_slots]
  int32_t* pw_lvl;          // [cap_slots]
  double* chunk_sum;        // [cap_chunks]
  double* chunk_approx;     // [cap_chunks] approximate exclusive starts
  long long* chunk_map;     // [2*cap_chunks]
  int32_t* chunk_e;         // [cap_chunks] assumed binade (INT_MIN: not flat)
  int32_t* chunk_mode;      // [cap_chunks]
  double* chunk_start;      // [cap_chunks]
  long long* super_map;     // [2*cap_supers]
  int32_t* super_e;         // [cap_supers]
  int32_t* super_mode;      // [cap_supers]
  double* super_start;      // [cap_supers]
  double* cdf;              // [cap_cand]
  int32_t* draw_idx;        // [budget]
  int64_t* draws_consumed;  // [1] uniforms consumed by this plan so far
  int32_t* err;             // [1] ErrBits
  int32_t* starvation;      // [1]
  // ---- per top-down layer results, strided by the capacities
  int32_t* cand;            // [L*cap_cand]
  double* norm;             // [L*cap_cand]
  uint8_t* is_local;        // [L*cap_cand]
  int32_t* nodes;           // [L*cap_rows]
  int32_t* samp_rank;       // [L*cap_rows]
  double* p;                // [L*cap_rows]
  int32_t* indptr;          // [L*(cap_rows+1)]   CSR (rows = upper)
  int32_t* indices;         // [L*cap_pairs]
  double* val;              // [L*cap_pairs]
  int32_t* tindptr;         // [L*(cap_rows+1)]   CSR of the transpose (rows = sampled)
  int32_t* tindices;        // [L*cap_pairs]
  double* tval;             // [L*cap_pairs]
  LayerStat* stat;          // [L]
};

constexpr int kSlots = 4;         // contributions kept per node before overflowing
constexpr int kFrGrain = 2048;   // fused range expand: range sizes are multiples of this
constexpr int kMaxFR = 32;        // at most this many ranges (graphs up to 512K nodes)
constexpr int kFusedMaxRows = 8192;  // upper rows per plan on the fused path
constexpr int kRangeNodes = 65536;  // nodes per CTA of the shared-memory-counting expand
constexpr int kMaxRanges = 16;      // beyond this many ranges per plan: global-atomic expand
constexpr int kTileWords = 256;    // bitmap words per compaction tile (8 warps x 32 words)
constexpr int kTileCand = 4096;    // candidates per scan tile
constexpr int kSmallBucket = 16;   // buckets folded in registers
constexpr int kChunk = 32;         // exact-cumsum chunk (one warp)
constexpr int kSuper = 1024;       // exact-cumsum superchunk (32 chunks)
constexpr int kPwSub = 256;        // pairwise-tree slots combined per CTA

// Host-side launch of the full sampling pipeline for n_plans slots.
int launch_ladies(const GraphDev& g, PlanDev* d_plans, int n_plans, int n_layers, int max_upper,
                  int cap_cand, int64_t cap_pairs, int budget_max, int n_fr, cudaStream_t st);
int launch_saint(const GraphDev& g, PlanDev* d_plans, int n_plans, int cap_rows, int cap_cand,
                 int64_t cap_pairs, int budget_max, cudaStream_t st);
int launch_pull_norms(const GraphDev& g, const int32_t* cand, int32_t n_cand,
                      const uint32_t* row_bitmap, double* out, int32_t* err, cudaStream_t st);
// GraphDev.rstart for a graph of n_fr ranges (stream 0, synchronous use at load)
int launch_build_rstart(const GraphDev& g, int32_t* rstart, int n_fr);
// fused range expand: range size (nodes per CTA, returned) and count for np plans per launch
int choose_fr(int64_t n, int np, int max_upper, int* n_fr);
size_t fr_smem_bytes(int fr_size, int ud_cap);
void launch_set_bitmap(const int32_t* ids, int32_t n, uint32_t* bitmap, int32_t n_words,
                       cudaStream_t st);
extern unsigned long long g_kernel_launches;

}  // namespace skg
