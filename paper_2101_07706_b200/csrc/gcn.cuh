// GCN forward/backward kernels over a sampled plan (training.py:261-318).
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
  int64_t ld;                 // elements per row (padded to a multiple of 4)
  int64_t dim;                // true feature dimension
};

template <typename T>
void gather_rows(const FeatStore& fs, const int32_t* ids, const int32_t* d_n, int max_n, T* out,
                 int64_t ldo, cudaStream_t st);
template <typename T>
void spmm(const int32_t* d_rows, int max_rows, const int32_t* indptr, const int32_t* indices,
          const double* val, const T* A, int64_t lda, bool relu_in, T* out, int64_t ldo,
          int64_t width, cudaStream_t st);
template <typename T>
void spmm_t_mask(const int32_t* d_rows, int max_rows, const int32_t* indptr,
                 const int32_t* indices, const double* val, const T* G, int64_t ldg,
                 const T* H, int64_t ldh, T* out, int64_t ldo, int64_t width, cudaStream_t st);
// C = op(A) op(B) (+ C if accumulate).  M or K may be read from device (dM / dK non-null).
template <typename T>
void gemm(bool ta, bool tb, int M, int N, int K, const int32_t* dM, const int32_t* dK,
          const T* A, int64_t lda, const T* B, int64_t ldb, T* C, int64_t ldc, bool accumulate,
          cudaStream_t st);
template <typename T>
void softmax_ce(const int32_t* d_rows, int max_rows, const int32_t* batch, const int32_t* labels,
                const T* logits, int64_t ldz, int C, T* grad, int64_t ldg, double* loss_out,
                int32_t* err, cudaStream_t st);
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
void fill_zero(T* p, int64_t n, cudaStream_t st);

}  // namespace skg
