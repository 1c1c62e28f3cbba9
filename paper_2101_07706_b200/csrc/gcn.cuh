// GCN forward/backward kernels over sampled plans (training.py:261-318), batched over
// the plans (slots) of an iteration: every stage is one launch with the slot on a grid axis.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace skg {

enum DType : int32_t { DT_F32 = 0, DT_F64 = 1 };

// Where layer-0 input rows live: a table of shard base pointers (one per rank; peer
// entries are NVLink-mapped IPC pointers) and per-node (rank, row) coordinates.
struct FeatStore {
  const void* const* shards;  // device array [n_ranks] of shard base pointers
  const int32_t* node_rank;   // [n] rank holding node's row (null: all local, row == node)
  const int32_t* node_row;    // [n] row inside that rank's shard
  int64_t ld;                 // elements per row (padded to a multiple of 4); bits: 32-bit words
  int64_t dim;                // true feature dimension
  int32_t bits;               // 1: multi-hot rows bit-packed (feature c = bit c & 31 of word c >> 5)
  int32_t pad_;
};

// Block of bottom-up layer l of one slot (device pointers into the plan arena).
struct LayerDesc {
  const int32_t* rows;  // |S_{l+1}| (device scalar)
  const int32_t* cols;  // |S_l|     (device scalar)
  const int32_t* indptr;
  const int32_t* indices;
  const double* val;
  const int32_t* tindptr;
  const int32_t* tindices;
  const double* tval;
};

struct SlotDesc {
  const int32_t* in_nodes;  // S_0 ids
  const int32_t* n_in;      // |S_0|
  const int32_t* batch;     // output rows' node ids (loss labels)
  const int32_t* n_batch;   // rows of the logits
  int32_t* err;
};

// Strided view of one activation buffer: slot z at base + z*stride, rows of ld elements.
template <typename T>
struct Act {
  T* base;
  int64_t stride, ld;
  __host__ __device__ T* at(int z) const { return base + (int64_t)z * stride; }
};

// A GEMM operand for the tensor-core path: TF32 hi / lo parts (lo null for 1xTF32) with
// identical geometry, rows of ld elements (ld % 4 == 0), slot z at + z*stride (stride 0:
// shared by all slots), rows_cap rows allocated per slot.
struct TcOp {
  const float* hi;
  const float* lo;
  int64_t ld, stride, rows_cap;
};

constexpr int kMaxLayers = 16;
// weights of every layer -> padded TF32 hi / lo copies (k_split_weights)
struct WSplitTable {
  int L;
  const float* w[kMaxLayers];
  float* hi[kMaxLayers];
  float* lo[kMaxLayers];
  int64_t rows[kMaxLayers], cols[kMaxLayers], ld_out[kMaxLayers];
};

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

extern int g_gemm_mode;        // fp32 GEMMs: 0 SIMT, 1 1xTF32 tcgen05, 3 3xTF32 tcgen05
extern int g_bn_override;      // debug / tuning overrides of the GEMM tile plan
extern int g_ksplit_override;
// C_z = op(A_z) op(B_z) (+ C_z) on tcgen05 (TMA-fed); M (or K) per slot from dM / dK.
// ks > 1 splits every slot's K into ks contiguous runs of 32-wide chunks: output block
// z * ks + j holds run j of slot z (partials for a fixed-order reduction).
constexpr int kMaxKSplit = 4;
extern thread_local int g_gemm_layer;
int gemm_tc(int mode, bool ta, bool tb, int n, int M, int N, int K, const int32_t* const* dM,
            const int32_t* const* dK, const TcOp& A, const TcOp& B, Act<float> C, bool acc,
            cudaStream_t st, int ks = 1);
// K split (1 .. kMaxKSplit) for an n-slot GEMM whose output is reduced afterwards: 1
// unless forced (SKG_GEMM_KSPLIT / skg_debug_gemm_ksplit); see plan_bn in gemm_tc.cu
int gemm_tc_ksplit(int n, int M, int N, int K);
void split_tf32(const float* in, int64_t ld_in, int64_t rows, int64_t cols, float* hi, float* lo,
                int64_t ld_out, cudaStream_t st);
void split_weights(const WSplitTable& t, cudaStream_t st);

// out = Block_l (relu?(A))  or, transposed, out = (Block_l^T A) * [H > 0].
// With out_lo (fp32 only) the result is written TF32-split (hi into out, lo into out_lo)
// for the tensor-core GEMMs, and rows [rows, max_rows) of every slot are zeroed.
// layer-0 SpMM fused with the feature gather: out = Block_0 . X[S_0], rows of X read
// through the feature store (local shard or NVLink-mapped peer shard; fp32 / fp64 rows or
// bit-packed multi-hot rows expanded to 0 / 1 on the fly)
template <typename T>
void spmm_in_b(const FeatStore& fs, const SlotDesc* sd, const LayerDesc* ld, int n, int max_rows,
               Act<T> out, T* out_lo, int64_t width, cudaStream_t st);
// full-graph SpMM over bit-packed rows (predict_logits layer 0)
template <typename T>
void spmm_full_bits(int64_t n, const int64_t* off, const int32_t* col, const double* w,
                    const uint32_t* X, int64_t ldw, T* out, int64_t ldo, int64_t width, cudaStream_t st);
template <typename T>
void spmm_b(const LayerDesc* ld, int n, int max_rows, bool transposed, bool relu_in, Act<T> A,
            Act<T> H, Act<T> out, T* out_lo, int64_t width, cudaStream_t st);
// SIMT GEMM (fp64, and the fp32 fallback mode 0): C_z = op(A_z) op(B_z) (+ C_z).
// M (or K) per slot from device scalars rows[z] when given.
template <typename T>
void gemm_simt(bool ta, bool tb, int n, int M, int N, int K, const int32_t* const* dM,
               const int32_t* const* dK, Act<T> A, Act<T> B, Act<T> C, bool accumulate,
               cudaStream_t st);
// C (+)= sum_z P_z in slot order (deterministic split-K reduction)
template <typename T>
void reduce_slots(const T* parts, int64_t part_stride, int n, int64_t rows, int64_t cols,
                  int64_t ldp, T* C, int64_t ldc, bool accumulate, cudaStream_t st);
// G (and G_lo when given: TF32-split output, rows [n_batch, max_rows) zeroed)
template <typename T>
void softmax_ce_b(const SlotDesc* sd, int n, int max_rows, const int32_t* labels, Act<T> Z, int C,
                  Act<T> G, T* G_lo, double* row_loss, double* loss_out, int32_t* nlab, cudaStream_t st);
// its three parts (labelled-row count per slot, per-row gradient + loss, fixed-order mean),
// for callers that run the count and the mean on a side branch
void count_labels_b(const SlotDesc* sd, int n, const int32_t* labels, int32_t* nlab, cudaStream_t st);
void loss_mean_b(const SlotDesc* sd, int n, int max_rows, const int32_t* labels, const double* row_loss,
                 const int32_t* nlab, double* loss_out, cudaStream_t st);
template <typename T>
void softmax_ce_rows_b(const SlotDesc* sd, int n, int max_rows, const int32_t* labels, Act<T> Z, int C,
                       Act<T> G, T* G_lo, double* row_loss, const int32_t* nlab, cudaStream_t st);
// multi-label BCE-with-logits (pos_weight on positives), mean over rows x C; multi-hot
// targets y (y_words 64-bit words per node); G (+ TF32 G_lo, tail rows zeroed)
template <typename T>
void bce_b(const SlotDesc* sd, int n, int max_rows, const uint64_t* y, int y_words, Act<T> Z, int C,
           double pos_weight, Act<T> G, T* G_lo, double* row_loss, double* loss_out, cudaStream_t st);
template <typename T>
void sgd_step(T* w, const T* g, int64_t n, double lr, double contrib, cudaStream_t st);
template <typename T>
void adam_step(T* w, const T* g, T* m, T* v, int64_t n, double lr, double contrib, double b1,
               double b2, double one_m_b1, double one_m_b2, double bc1, double bc2, double eps,
               cudaStream_t st);
template <typename T>
void spmm_full(int64_t n, const int64_t* off, const int32_t* col, const double* w, const T* A,
               int64_t lda, bool relu_in, T* out, int64_t ldo, int64_t width, cudaStream_t st);
template <typename T>
void gemm_plain(int M, int N, int K, const T* A, int64_t lda, const T* B, int64_t ldb, T* C,
                int64_t ldc, cudaStream_t st);
template <typename T>
void fill_zero(T* p, int64_t n, cudaStream_t st);

}  // namespace skg
