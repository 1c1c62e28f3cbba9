// GCN compute over sampled plans: fused feature gather (local shard or NVLink peer),
// CSR SpMM (ReLU fused on the input), transposed SpMM fused with the ReLU mask, tiled
// GEMMs for H·W, softmax cross-entropy forward+backward and the optimizer steps.
// Every stage handles all plans (slots) of an iteration in one launch.
//
// Reference: training.py:261-318 (forward / loss_and_backward), 398-427 (SGD / Adam),
// 325-334 (predict_logits).  Activation rows are padded to a multiple of 4 elements so
// every row access is a 16-byte vector; padding columns stay zero.
#include <cub/block/block_reduce.cuh>
#include <algorithm>
#include <cstdio>

#include "gcn.cuh"
#include "prof.h"
#include "sampler.cuh"
#include "skg_internal.h"

namespace skg {



constexpr unsigned FULLM = 0xffffffffu;

template <typename T>
struct Vec4;
template <>
struct Vec4<float> {
  float4 v;
  __device__ static Vec4 load(const float* p) { Vec4 r; r.v = *reinterpret_cast<const float4*>(p); return r; }
  __device__ void store(float* p) const { *reinterpret_cast<float4*>(p) = v; }
  __device__ static Vec4 zero() { Vec4 r; r.v = make_float4(0.f, 0.f, 0.f, 0.f); return r; }
  __device__ static Vec4 from4(float4 f) { Vec4 r; r.v = f; return r; }
  __device__ void fma(float a, const Vec4& x) {
    v.x = fmaf(a, x.v.x, v.x); v.y = fmaf(a, x.v.y, v.y);
    v.z = fmaf(a, x.v.z, v.z); v.w = fmaf(a, x.v.w, v.w);
  }
  __device__ void relu() { v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f); }
  __device__ void mask(const Vec4& h) {
    v.x = h.v.x > 0.f ? v.x : 0.f; v.y = h.v.y > 0.f ? v.y : 0.f;
    v.z = h.v.z > 0.f ? v.z : 0.f; v.w = h.v.w > 0.f ? v.w : 0.f;
  }
};
template <>
struct Vec4<double> {
  double2 a, b;
  __device__ static Vec4 load(const double* p) {
    Vec4 r; r.a = reinterpret_cast<const double2*>(p)[0]; r.b = reinterpret_cast<const double2*>(p)[1]; return r;
  }
  __device__ void store(double* p) const { reinterpret_cast<double2*>(p)[0] = a; reinterpret_cast<double2*>(p)[1] = b; }
  __device__ static Vec4 zero() { Vec4 r; r.a = make_double2(0, 0); r.b = make_double2(0, 0); return r; }
  __device__ static Vec4 from4(float4 f) { Vec4 r; r.a = make_double2(f.x, f.y); r.b = make_double2(f.z, f.w); return r; }
  __device__ void fma(double s, const Vec4& x) {
    a.x = ::fma(s, x.a.x, a.x); a.y = ::fma(s, x.a.y, a.y); b.x = ::fma(s, x.b.x, b.x); b.y = ::fma(s, x.b.y, b.y);
  }
  __device__ void relu() { a.x = fmax(a.x, 0.); a.y = fmax(a.y, 0.); b.x = fmax(b.x, 0.); b.y = fmax(b.y, 0.); }
  __device__ void mask(const Vec4& h) {
    a.x = h.a.x > 0. ? a.x : 0.; a.y = h.a.y > 0. ? a.y : 0.;
    b.x = h.b.x > 0. ? b.x : 0.; b.y = h.b.y > 0. ? b.y : 0.;
  }
};

static int sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static int row_blocks(int max_rows, int n) {
  // warp per row, 8 warps per CTA; cover all rows but keep >= ~2 waves overall
  int b = (max_rows + 7) / 8;
  int cap = std::max(1, (4 * sms() + n - 1) / n);
  return std::max(1, std::min(b, std::max(cap, 1)));
}

// ------------------------------------------------------------------ SpMM (K8 / K10)
// TF32 split of a result vector for the tensor-core GEMMs: hi into o, lo into o_lo
__device__ __forceinline__ void store_split(const Vec4<float>& a, float* o, float* o_lo) {
  float4 h, l;
  h.x = tf32_rna(a.v.x); l.x = tf32_rna(a.v.x - h.x);
  h.y = tf32_rna(a.v.y); l.y = tf32_rna(a.v.y - h.y);
  h.z = tf32_rna(a.v.z); l.z = tf32_rna(a.v.z - h.z);
  h.w = tf32_rna(a.v.w); l.w = tf32_rna(a.v.w - h.w);
  *reinterpret_cast<float4*>(o) = h;
  *reinterpret_cast<float4*>(o_lo) = l;
}
__device__ __forceinline__ void store_split(const Vec4<double>&, double*, double*) {}

template <typename T, bool TRANS, bool RELU>
__global__ void k_spmm_b(const LayerDesc* lds, Act<T> A, Act<T> H, Act<T> out, T* out_lo,
                         int max_rows, int64_t width) {
  SKG_PDL_WAIT();  // dependents are triggered at the end (GEMM CTAs must not wait on SMs)
  const LayerDesc d = lds[blockIdx.y];
  const int rows = TRANS ? *d.cols : *d.rows;
  const int32_t* __restrict__ ip = TRANS ? d.tindptr : d.indptr;
  const int32_t* __restrict__ ix = TRANS ? d.tindices : d.indices;
  const double* __restrict__ vv = TRANS ? d.tval : d.val;
  const T* a = A.at(blockIdx.y);
  const T* h = TRANS ? H.at(blockIdx.y) : nullptr;
  T* o = out.at(blockIdx.y);
  T* ol = out_lo ? out_lo + (int64_t)blockIdx.y * out.stride : nullptr;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  // split outputs feed the GEMM's contraction over rows: rows past the plan's are zero
  const int rows_all = ol ? max_rows : rows;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows_all; r += nw) {
    if (r >= rows) {
      for (int64_t c = lane * 4; c < width; c += 128) {
        Vec4<T>::zero().store(o + (int64_t)r * out.ld + c);
        Vec4<T>::zero().store(ol + (int64_t)r * out.ld + c);
      }
      continue;
    }
    const int b = ip[r], e = ip[r + 1];
    // one pass over the row's nonzeros feeds up to NB 128-column blocks: NB gathers of
    // every source row in flight per lane (each column still accumulates in nonzero order)
    constexpr int NB = 2;
    for (int64_t c0 = lane * 4; c0 < width; c0 += 128 * NB) {
      Vec4<T> acc[NB];
#pragma unroll
      for (int q = 0; q < NB; ++q) acc[q] = Vec4<T>::zero();
#pragma unroll 2
      for (int p = b; p < e; ++p) {
        const T s = (T)vv[p];
        const T* src = a + (int64_t)ix[p] * A.ld;
#pragma unroll
        for (int q = 0; q < NB; ++q) {
          if (c0 + 128 * q < width) {
            Vec4<T> x = Vec4<T>::load(src + c0 + 128 * q);
            if (RELU) x.relu();
            acc[q].fma(s, x);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        const int64_t c = c0 + 128 * q;
        if (c >= width) continue;
        if (TRANS) acc[q].mask(Vec4<T>::load(h + (int64_t)r * H.ld + c));
        if (ol) store_split(acc[q], o + (int64_t)r * out.ld + c, ol + (int64_t)r * out.ld + c);
        else acc[q].store(o + (int64_t)r * out.ld + c);
      }
    }
  }
  SKG_PDL_TRIGGER();
}

template <typename T>
void spmm_b(const LayerDesc* ld, int n, int max_rows, bool transposed, bool relu_in, Act<T> A,
            Act<T> H, Act<T> out, T* out_lo, int64_t width, cudaStream_t st) {
  dim3 grid(row_blocks(max_rows, n), n);
  if (transposed) launch_k("k_spmm_b<T,1,0>", st, dim3(grid), dim3(256), 0, k_spmm_b<T, true, false>, ld, A, H, out, out_lo, max_rows, width);
  else if (relu_in) launch_k("k_spmm_b<F,1>", st, dim3(grid), dim3(256), 0, k_spmm_b<T, false, true>, ld, A, H, out, out_lo, max_rows, width);
  else launch_k("k_spmm_b<F,0>", st, dim3(grid), dim3(256), 0, k_spmm_b<T, false, false>, ld, A, H, out, out_lo, max_rows, width);
}

// ------------------------------------------------------------------ fused gather + SpMM
// four features c .. c + 3 (c a multiple of 4) of a bit-packed row as 0 / 1
template <typename T>
__device__ __forceinline__ Vec4<T> bits4(const uint32_t* row, int64_t c) {
  const uint32_t nib = (row[c >> 5] >> (c & 31)) & 0xFu;
  float4 f = make_float4((float)(nib & 1u), (float)((nib >> 1) & 1u), (float)((nib >> 2) & 1u),
                         (float)(nib >> 3));
  return Vec4<T>::from4(f);
}

// out[r] = sum_p val[p] X[S_0[ix[p]]] over the layer-0 block's rows, X rows addressed through
// the feature store; same per-column accumulation order as k_spmm_b over a gathered X_0
template <typename T, bool BITS>
__global__ void k_spmm_in_b(FeatStore fs, const SlotDesc* sd, const LayerDesc* lds, Act<T> out,
                            T* out_lo, int max_rows, int64_t width) {
  SKG_PDL_WAIT();  // dependents are triggered at the end (GEMM CTAs must not wait on SMs)
  const LayerDesc d = lds[blockIdx.y];
  const int32_t* __restrict__ in_nodes = sd[blockIdx.y].in_nodes;
  const int rows = *d.rows;
  const int32_t* __restrict__ ip = d.indptr;
  const int32_t* __restrict__ ix = d.indices;
  const double* __restrict__ vv = d.val;
  T* o = out.at(blockIdx.y);
  T* ol = out_lo ? out_lo + (int64_t)blockIdx.y * out.stride : nullptr;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int rows_all = ol ? max_rows : rows;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows_all; r += nw) {
    if (r >= rows) {
      for (int64_t c = lane * 4; c < width; c += 128) {
        Vec4<T>::zero().store(o + (int64_t)r * out.ld + c);
        Vec4<T>::zero().store(ol + (int64_t)r * out.ld + c);
      }
      continue;
    }
    const int b = ip[r], e = ip[r + 1];
    constexpr int NB = 2;
    for (int64_t c0 = lane * 4; c0 < width; c0 += 128 * NB) {
      Vec4<T> acc[NB];
#pragma unroll
      for (int q = 0; q < NB; ++q) acc[q] = Vec4<T>::zero();
#pragma unroll 2
      for (int p = b; p < e; ++p) {
        const T s = (T)vv[p];
        const int node = in_nodes[ix[p]];
        const int rank = fs.node_rank ? fs.node_rank[node] : 0;
        const int64_t row = fs.node_row ? fs.node_row[node] : node;
#pragma unroll
        for (int q = 0; q < NB; ++q) {
          if (c0 + 128 * q < width) {
            Vec4<T> x;
            if (BITS) x = bits4<T>(reinterpret_cast<const uint32_t*>(fs.shards[rank]) + row * fs.ld, c0 + 128 * q);
            else x = Vec4<T>::load(reinterpret_cast<const T*>(fs.shards[rank]) + row * fs.ld + c0 + 128 * q);
            acc[q].fma(s, x);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        const int64_t c = c0 + 128 * q;
        if (c >= width) continue;
        if (ol) store_split(acc[q], o + (int64_t)r * out.ld + c, ol + (int64_t)r * out.ld + c);
        else acc[q].store(o + (int64_t)r * out.ld + c);
      }
    }
  }
  SKG_PDL_TRIGGER();
}

template <typename T>
void spmm_in_b(const FeatStore& fs, const SlotDesc* sd, const LayerDesc* ld, int n, int max_rows,
               Act<T> out, T* out_lo, int64_t width, cudaStream_t st) {
  dim3 grid(row_blocks(max_rows, n), n);
  if (fs.bits)
    launch_k("k_spmm_in_b<bits>", st, dim3(grid), dim3(256), 0, k_spmm_in_b<T, true>, fs, sd, ld, out, out_lo,
             max_rows, width);
  else
    launch_k("k_spmm_in_b", st, dim3(grid), dim3(256), 0, k_spmm_in_b<T, false>, fs, sd, ld, out, out_lo,
             max_rows, width);
}

template <typename T>
__global__ void k_spmm_full_bits(int64_t n, const int64_t* __restrict__ off, const int32_t* __restrict__ col,
                                 const double* __restrict__ w, const uint32_t* __restrict__ X, int64_t ldw,
                                 T* __restrict__ out, int64_t ldo, int64_t width) {
  SKG_PDL_PROLOGUE();
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
    const int64_t b = off[r], e = off[r + 1];
    for (int64_t c = lane * 4; c < width; c += 128) {
      Vec4<T> acc = Vec4<T>::zero();
      for (int64_t p = b; p < e; ++p) acc.fma((T)w[p], bits4<T>(X + (int64_t)col[p] * ldw, c));
      acc.store(out + r * ldo + c);
    }
  }
}

template <typename T>
void spmm_full_bits(int64_t n, const int64_t* off, const int32_t* col, const double* w, const uint32_t* X,
                    int64_t ldw, T* out, int64_t ldo, int64_t width, cudaStream_t st) {
  launch_k("k_spmm_full_bits", st, dim3(16 * sms()), dim3(256), 0, k_spmm_full_bits<T>, n, off, col, w, X, ldw,
           out, ldo, width);
}

// full-graph SpMM for predict_logits (int64 offsets)
template <typename T, bool RELU>
__global__ void k_spmm_full(int64_t n, const int64_t* __restrict__ off, const int32_t* __restrict__ col,
                            const double* __restrict__ w, const T* __restrict__ A, int64_t lda,
                            T* __restrict__ out, int64_t ldo, int64_t width) {
  SKG_PDL_PROLOGUE();
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
    const int64_t b = off[r], e = off[r + 1];
    for (int64_t c = lane * 4; c < width; c += 128) {
      Vec4<T> acc = Vec4<T>::zero();
      for (int64_t p = b; p < e; ++p) {
        Vec4<T> x = Vec4<T>::load(A + (int64_t)col[p] * lda + c);
        if (RELU) x.relu();
        acc.fma((T)w[p], x);
      }
      acc.store(out + r * ldo + c);
    }
  }
}

template <typename T>
void spmm_full(int64_t n, const int64_t* off, const int32_t* col, const double* w, const T* A,
               int64_t lda, bool relu_in, T* out, int64_t ldo, int64_t width, cudaStream_t st) {
  int blocks = 16 * sms();
  if (relu_in)
    launch_k("k_spmm_full", st, dim3(blocks), dim3(256), 0, k_spmm_full<T, true>, n, off, col, w, A, lda, out, ldo, width);
  else
    launch_k("k_spmm_full", st, dim3(blocks), dim3(256), 0, k_spmm_full<T, false>, n, off, col, w, A, lda, out, ldo, width);
}

// ------------------------------------------------------------------ GEMM (K9)
// Register-tiled SIMT GEMM, BMxBN tile per CTA, TMxTN outputs per thread, slot on
// blockIdx.z.  op(A) is M x K, op(B) is K x N (TA/TB select transposed storage).
template <typename T, bool TA, bool TB, int BM, int BN, int BK, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
    k_gemm_b(int Mfix, int N, int Kfix, const int32_t* const* dM, const int32_t* const* dK,
             Act<T> A, Act<T> B, Act<T> C, int accumulate) {
  SKG_PDL_PROLOGUE();
  constexpr int NT = (BM / TM) * (BN / TN);
  const int z = blockIdx.z;
  const int M = dM ? *dM[z] : Mfix;
  const int K = dK ? *dK[z] : Kfix;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= M) return;
  const T* __restrict__ a = A.at(z);
  const T* __restrict__ b = B.at(z);
  T* __restrict__ c = C.at(z);
  __shared__ T As[BK][BM + 4];
  __shared__ T Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);
  for (int k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int q = 0; q < (BM * BK) / NT; ++q) {
      const int idx = tid + q * NT;
      int m, k;
      if (TA) { k = idx / BM; m = idx % BM; } else { m = idx / BK; k = idx % BK; }
      const int gm = m0 + m, gk = k0 + k;
      T v = T(0);
      if (gm < M && gk < K) v = TA ? a[(int64_t)gk * A.ld + gm] : a[(int64_t)gm * A.ld + gk];
      As[k][m] = v;
    }
#pragma unroll
    for (int q = 0; q < (BN * BK) / NT; ++q) {
      const int idx = tid + q * NT;
      int n, k;
      if (TB) { n = idx / BK; k = idx % BK; } else { k = idx / BN; n = idx % BN; }
      const int gn = n0 + n, gk = k0 + k;
      T v = T(0);
      if (gn < N && gk < K) v = TB ? b[(int64_t)gn * B.ld + gk] : b[(int64_t)gk * B.ld + gn];
      Bs[k][n] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) av[i] = As[kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) bv[j] = Bs[kk][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int gm = m0 + ty * TM + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int gn = n0 + tx * TN + j;
      if (gn >= N) continue;
      T* p = c + (int64_t)gm * C.ld + gn;
      *p = accumulate ? *p + acc[i][j] : acc[i][j];
    }
  }
}

template <typename T, int BM, int BN, int BK, int TM, int TN>
static void gemm_launch(bool ta, bool tb, int n, int M, int N, int K, const int32_t* const* dM,
                        const int32_t* const* dK, Act<T> A, Act<T> B, Act<T> C, bool acc,
                        cudaStream_t st) {
  constexpr int NT = (BM / TM) * (BN / TN);
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, n);
  if (!ta && !tb) launch_k("k_gemm_b", st, dim3(grid), dim3(NT), 0, k_gemm_b<T, false, false, BM, BN, BK, TM, TN>, M, N, K, dM, dK, A, B, C, acc);
  else if (ta && !tb) launch_k("k_gemm_b", st, dim3(grid), dim3(NT), 0, k_gemm_b<T, true, false, BM, BN, BK, TM, TN>, M, N, K, dM, dK, A, B, C, acc);
  else if (!ta && tb) launch_k("k_gemm_b", st, dim3(grid), dim3(NT), 0, k_gemm_b<T, false, true, BM, BN, BK, TM, TN>, M, N, K, dM, dK, A, B, C, acc);
  else launch_k("k_gemm_b", st, dim3(grid), dim3(NT), 0, k_gemm_b<T, true, true, BM, BN, BK, TM, TN>, M, N, K, dM, dK, A, B, C, acc);
}

int g_gemm_mode = 3;  // fp32 GEMMs: 0 SIMT, 1 1xTF32 tcgen05, 3 3xTF32 tcgen05

template <typename T>
void gemm_simt(bool ta, bool tb, int n, int M, int N, int K, const int32_t* const* dM,
               const int32_t* const* dK, Act<T> A, Act<T> B, Act<T> C, bool accumulate,
               cudaStream_t st) {
  if (M <= 0 || N <= 0 || n <= 0) return;
  if (sizeof(T) == 4 && N > 32)
    gemm_launch<T, 128, 64, 16, 8, 4>(ta, tb, n, M, N, K, dM, dK, A, B, C, accumulate, st);
  else
    gemm_launch<T, 64, 64, 16, 4, 4>(ta, tb, n, M, N, K, dM, dK, A, B, C, accumulate, st);
}

template <typename T>
void gemm_plain(int M, int N, int K, const T* A, int64_t lda, const T* B, int64_t ldb, T* C,
                int64_t ldc, cudaStream_t st) {
  Act<T> a{const_cast<T*>(A), 0, lda}, b{const_cast<T*>(B), 0, ldb}, c{C, 0, ldc};
  // full-graph inference: M = n rows, split into grid-y chunks the hardware accepts
  const int chunk = 65535 * 64;
  for (int m0 = 0; m0 < M; m0 += chunk) {
    Act<T> a2 = a, c2 = c;
    a2.base += (int64_t)m0 * lda;
    c2.base += (int64_t)m0 * ldc;
    gemm_simt<T>(false, false, 1, std::min(chunk, M - m0), N, K, nullptr, nullptr, a2, b, c2, false, st);
  }
}

// deterministic split-K reduction: C (+)= P_0 + P_1 + ... in slot order
template <typename T>
__global__ void k_reduce_slots(const T* parts, int64_t pstride, int n, int64_t rows, int64_t cols,
                               int64_t ldp, T* C, int64_t ldc, int accumulate) {
  SKG_PDL_PROLOGUE();
  // VW consecutive columns per thread (VW = 4 when every row and part is 16-byte aligned);
  // the parts' loads of a run of 8 slots are all issued before the in-order adds, so the
  // sum (C or 0, then slot 0, 1, ...) keeps its order and the loads overlap
  const bool vec = sizeof(T) == 4 && cols % 4 == 0 && ldp % 4 == 0 && ldc % 4 == 0 && pstride % 4 == 0 &&
                   (reinterpret_cast<uintptr_t>(parts) & 15) == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0;
  const int vw = vec ? 4 : 1;
  const int64_t cv = cols / vw;
  const int64_t total = rows * cv;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cv, c = (i - r * cv) * vw;
    if (vec) {
      float4 s = accumulate ? *reinterpret_cast<const float4*>(C + r * ldc + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      for (int z0 = 0; z0 < n; z0 += 8) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (z0 + u < n) v[u] = *reinterpret_cast<const float4*>(parts + (z0 + u) * pstride + r * ldp + c);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (z0 + u < n) {
            s.x += v[u].x; s.y += v[u].y; s.z += v[u].z; s.w += v[u].w;
          }
      }
      *reinterpret_cast<float4*>(C + r * ldc + c) = s;
    } else {
      T s = accumulate ? C[r * ldc + c] : T(0);
      for (int z0 = 0; z0 < n; z0 += 8) {
        T v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (z0 + u < n) v[u] = parts[(z0 + u) * pstride + r * ldp + c];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (z0 + u < n) s += v[u];
      }
      C[r * ldc + c] = s;
    }
  }
}

template <typename T>
void reduce_slots(const T* parts, int64_t part_stride, int n, int64_t rows, int64_t cols,
                  int64_t ldp, T* C, int64_t ldc, bool accumulate, cudaStream_t st) {
  int64_t total = rows * cols;
  int blocks = (int)std::min<int64_t>((total + 255) / 256, 8 * sms());
  launch_k("k_reduce_slots", st, dim3(std::max(blocks, 1)), dim3(256), 0, k_reduce_slots<T>, parts, part_stride, n, rows, cols,
                                                                 ldp, C, ldc, accumulate);
}

// ------------------------------------------------------------------ softmax CE (K11)
// labelled rows of every slot's batch, once per slot (the mean's divisor)
__global__ void __launch_bounds__(1024) k_count_labels(const SlotDesc* sd, const int32_t* labels,
                                                       int32_t* nlab) {
  SKG_PDL_PROLOGUE();
  const SlotDesc d = sd[blockIdx.x];
  const int n = *d.n_batch;
  typedef cub::BlockReduce<int, 1024> BR;
  __shared__ typename BR::TempStorage tmp;
  int cnt = 0;
#pragma unroll 4
  for (int r = threadIdx.x; r < n; r += blockDim.x) cnt += labels[d.batch[r]] >= 0;
  const int tot = BR(tmp).Sum(cnt);
  if (threadIdx.x == 0) nlab[blockIdx.x] = tot;
}

// training.py:293-308: per-row LSE loss and gradient (warp per row, all slots), then a
// fixed-order per-slot mean.
template <typename T>
__global__ void k_softmax_ce_b(const SlotDesc* sd, const int32_t* labels, Act<T> Z, int C,
                               Act<T> G, T* G_lo, int max_rows, double* row_loss, int64_t rl_stride,
                               const int32_t* nlab_slot) {
  SKG_PDL_PROLOGUE();
  const SlotDesc d = sd[blockIdx.y];
  const int n = *d.n_batch;
  const int nlab = nlab_slot[blockIdx.y];  // labelled batch rows (k_count_labels)
  const T* z0 = Z.at(blockIdx.y);
  T* g0 = G.at(blockIdx.y);
  T* gl0 = G_lo ? G_lo + (int64_t)blockIdx.y * G.stride : nullptr;
  double* rl = row_loss + blockIdx.y * rl_stride;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int rows_all = gl0 ? max_rows : n;  // split output: zero rows past the batch
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows_all; r += nw) {
    T* g = g0 + (int64_t)r * G.ld;
    T* gl = gl0 ? gl0 + (int64_t)r * G.ld : nullptr;
    if (r >= n) {
      for (int k = lane; k < C; k += 32) g[k] = gl[k] = T(0);
      continue;
    }
    const int y = labels[d.batch[r]];
    if (y < 0 || nlab == 0) {
      for (int k = lane; k < C; k += 32) {
        g[k] = T(0);
        if (gl) gl[k] = T(0);
      }
      if (lane == 0) rl[r] = 0.0;
      continue;
    }
    const T* z = z0 + (int64_t)r * Z.ld;
    double zmax = -INFINITY;
    for (int k = lane; k < C; k += 32) zmax = fmax(zmax, (double)z[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) zmax = fmax(zmax, __shfl_xor_sync(FULLM, zmax, o));
    double se = 0.0;
    for (int k = lane; k < C; k += 32) se += exp((double)z[k] - zmax);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(FULLM, se, o);
    const double lse = zmax + log(se);
    for (int k = lane; k < C; k += 32) {
      double gz = exp((double)z[k] - lse) - (k == y ? 1.0 : 0.0);
      const T v = (T)(gz / nlab);
      if (gl) {
        const float h = tf32_rna((float)v);
        g[k] = (T)h;
        gl[k] = (T)tf32_rna((float)v - h);
      } else {
        g[k] = v;
      }
    }
    if (lane == 0) rl[r] = lse - (double)z[y];
  }
}

__global__ void __launch_bounds__(1024) k_loss_mean(const SlotDesc* sd, const int32_t* labels,
                                                    const double* row_loss, int64_t rl_stride,
                                                    const int32_t* nlab, double* loss_out) {
  SKG_PDL_PROLOGUE();
  const SlotDesc d = sd[blockIdx.x];
  const int n = *d.n_batch;
  typedef cub::BlockReduce<double, 1024> BRD;
  __shared__ typename BRD::TempStorage td;
  double s = 0.0;
  const double* rl = row_loss + blockIdx.x * rl_stride;
#pragma unroll 4
  for (int r = threadIdx.x; r < n; r += blockDim.x)  // fixed assignment: deterministic
    if (labels[d.batch[r]] >= 0) s += rl[r];
  const double tot = BRD(td).Sum(s);
  if (threadIdx.x == 0) {
    const int cnt = nlab[blockIdx.x];
    loss_out[blockIdx.x] = cnt ? tot / cnt : __longlong_as_double(0x7ff8000000000000LL);
    if (!cnt) atomicOr(d.err, EB_NO_LABELS);
  }
}

void count_labels_b(const SlotDesc* sd, int n, const int32_t* labels, int32_t* nlab, cudaStream_t st) {
  launch_k("k_count_labels", st, dim3(n), dim3(1024), 0, k_count_labels, sd, labels, nlab);
}

void loss_mean_b(const SlotDesc* sd, int n, int max_rows, const int32_t* labels, const double* row_loss,
                 const int32_t* nlab, double* loss_out, cudaStream_t st) {
  launch_k("k_loss_mean", st, dim3(n), dim3(1024), 0, k_loss_mean, sd, labels, row_loss, (int64_t)max_rows,
           nlab, loss_out);
}

template <typename T>
void softmax_ce_rows_b(const SlotDesc* sd, int n, int max_rows, const int32_t* labels, Act<T> Z, int C,
                       Act<T> G, T* G_lo, double* row_loss, const int32_t* nlab, cudaStream_t st) {
  launch_k("k_softmax_ce_b", st, dim3(dim3(row_blocks(max_rows, n), n)), dim3(256), 0, k_softmax_ce_b<T>, sd, labels, Z, C, G, G_lo, max_rows, row_loss, max_rows, nlab);
}

template <typename T>
void softmax_ce_b(const SlotDesc* sd, int n, int max_rows, const int32_t* labels, Act<T> Z, int C,
                  Act<T> G, T* G_lo, double* row_loss, double* loss_out, int32_t* nlab, cudaStream_t st) {
  count_labels_b(sd, n, labels, nlab, st);
  softmax_ce_rows_b<T>(sd, n, max_rows, labels, Z, C, G, G_lo, row_loss, nlab, st);
  loss_mean_b(sd, n, max_rows, labels, row_loss, nlab, loss_out, st);
}

// ------------------------------------------------------------------ multi-label BCE
// torch.nn.BCEWithLogitsLoss(pos_weight=pw, reduction="mean") semantics over the batch rows:
// l = pw*y*softplus(-z) + (1-y)*softplus(z), dl/dz = sigmoid(z)*(pw*y + 1 - y) - pw*y, both
// divided by rows*C; warp per row, row sums in fp64, fixed-order mean per slot.
template <typename T>
__global__ void k_bce_b(const SlotDesc* sd, const uint64_t* y, int y_words, Act<T> Z, int C, double pw,
                        Act<T> G, T* G_lo, int max_rows, double* row_loss, int64_t rl_stride) {
  SKG_PDL_PROLOGUE();
  const SlotDesc d = sd[blockIdx.y];
  const int n = *d.n_batch;
  const T* z0 = Z.at(blockIdx.y);
  T* g0 = G.at(blockIdx.y);
  T* gl0 = G_lo ? G_lo + (int64_t)blockIdx.y * G.stride : nullptr;
  double* rl = row_loss + blockIdx.y * rl_stride;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const double scale = n > 0 ? 1.0 / ((double)n * C) : 0.0;
  const int rows_all = gl0 ? max_rows : n;  // split output: zero rows past the batch
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows_all; r += nw) {
    T* g = g0 + (int64_t)r * G.ld;
    T* gl = gl0 ? gl0 + (int64_t)r * G.ld : nullptr;
    if (r >= n) {
      for (int k = lane; k < C; k += 32) g[k] = gl[k] = T(0);
      continue;
    }
    const uint64_t* yr = y + (int64_t)d.batch[r] * y_words;
    const T* z = z0 + (int64_t)r * Z.ld;
    double ls = 0.0;
    for (int k = lane; k < C; k += 32) {
      const double yk = (double)((yr[k >> 6] >> (k & 63)) & 1ull);
      const double zk = (double)z[k];
      const double e = exp(-fabs(zk));
      const double sp_pos = log1p(e) + fmax(-zk, 0.0);  // softplus(-z) = -log sigmoid(z)
      const double sp_neg = log1p(e) + fmax(zk, 0.0);   // softplus(z)  = -log(1 - sigmoid(z))
      ls += pw * yk * sp_pos + (1.0 - yk) * sp_neg;
      const double sig = zk >= 0.0 ? 1.0 / (1.0 + e) : e / (1.0 + e);
      const T v = (T)((sig * (pw * yk + 1.0 - yk) - pw * yk) * scale);
      if (gl) {
        const float h = tf32_rna((float)v);
        g[k] = (T)h;
        gl[k] = (T)tf32_rna((float)v - h);
      } else {
        g[k] = v;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ls += __shfl_xor_sync(FULLM, ls, o);
    if (lane == 0) rl[r] = ls;
  }
}

__global__ void k_bce_mean(const SlotDesc* sd, const double* row_loss, int64_t rl_stride, int C,
                           double* loss_out) {
  SKG_PDL_PROLOGUE();
  const SlotDesc d = sd[blockIdx.x];
  const int n = *d.n_batch;
  typedef cub::BlockReduce<double, 256> BRD;
  __shared__ typename BRD::TempStorage td;
  double s = 0.0;
  const double* rl = row_loss + blockIdx.x * rl_stride;
  for (int r = threadIdx.x; r < n; r += blockDim.x) s += rl[r];  // fixed assignment
  const double tot = BRD(td).Sum(s);
  if (threadIdx.x == 0) loss_out[blockIdx.x] = n ? tot / ((double)n * C) : 0.0;
}

template <typename T>
void bce_b(const SlotDesc* sd, int n, int max_rows, const uint64_t* y, int y_words, Act<T> Z, int C,
           double pos_weight, Act<T> G, T* G_lo, double* row_loss, double* loss_out, cudaStream_t st) {
  launch_k("k_bce_b", st, dim3(row_blocks(max_rows, n), n), dim3(256), 0, k_bce_b<T>, sd, y, y_words, Z, C,
           pos_weight, G, G_lo, max_rows, row_loss, (int64_t)max_rows);
  launch_k("k_bce_mean", st, dim3(n), dim3(256), 0, k_bce_mean, sd, row_loss, (int64_t)max_rows, C, loss_out);
}

// ------------------------------------------------------------------ optimizers (K12 epilogue)
template <typename T>
__device__ __forceinline__ T dv(T a, T b);
template <> __device__ __forceinline__ float dv(float a, float b) { return __fdiv_rn(a, b); }
template <> __device__ __forceinline__ double dv(double a, double b) { return __ddiv_rn(a, b); }
template <typename T>
__device__ __forceinline__ T ml(T a, T b);
template <> __device__ __forceinline__ float ml(float a, float b) { return __fmul_rn(a, b); }
template <> __device__ __forceinline__ double ml(double a, double b) { return __dmul_rn(a, b); }
template <typename T>
__device__ __forceinline__ T ad(T a, T b);
template <> __device__ __forceinline__ float ad(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ double ad(double a, double b) { return __dadd_rn(a, b); }

// training.py:402-404 with the average of training.py:506: w -= lr * (g / contributors)
template <typename T>
__global__ void k_sgd(T* w, const T* g, int64_t n, T lr, T contrib) {
  SKG_PDL_PROLOGUE();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    w[i] = ad(w[i], -ml(lr, dv(g[i], contrib)));
}

// training.py:415-427
template <typename T>
__global__ void k_adam(T* w, const T* g, T* m, T* v, int64_t n, T lr, T contrib, T b1, T b2,
                       T omb1, T omb2, T bc1, T bc2, T eps) {
  SKG_PDL_PROLOGUE();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    T gr = dv(g[i], contrib);
    T mi = ad(ml(m[i], b1), ml(omb1, gr));
    T vi = ad(ml(v[i], b2), ml(ml(omb2, gr), gr));
    m[i] = mi;
    v[i] = vi;
    T mh = dv(mi, bc1), vh = dv(vi, bc2);
    w[i] = ad(w[i], -dv(ml(lr, mh), ad((T)sqrt(vh), eps)));
  }
}

template <typename T>
void sgd_step(T* w, const T* g, int64_t n, double lr, double contrib, cudaStream_t st) {
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 8 * sms());
  launch_k("k_sgd", st, dim3(std::max(blocks, 1)), dim3(256), 0, k_sgd<T>, w, g, n, (T)lr, (T)contrib);
}

template <typename T>
void adam_step(T* w, const T* g, T* m, T* v, int64_t n, double lr, double contrib, double b1,
               double b2, double omb1, double omb2, double bc1, double bc2, double eps,
               cudaStream_t st) {
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 8 * sms());
  launch_k("k_adam", st, dim3(std::max(blocks, 1)), dim3(256), 0, k_adam<T>, w, g, m, v, n, (T)lr, (T)contrib, (T)b1, (T)b2,
                                                         (T)omb1, (T)omb2, (T)bc1, (T)bc2, (T)eps);
}

template <typename T>
__global__ void k_zero(T* p, int64_t n) {
  SKG_PDL_PROLOGUE();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = T(0);
}
template <typename T>
void fill_zero(T* p, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 8 * sms());
  launch_k("k_zero", st, dim3(std::max(blocks, 1)), dim3(256), 0, k_zero<T>, p, n);
}

#define INST(T)                                                                                     \
  template void spmm_b<T>(const LayerDesc*, int, int, bool, bool, Act<T>, Act<T>, Act<T>, T*,       \
                          int64_t, cudaStream_t);                                                   \
  template void gemm_simt<T>(bool, bool, int, int, int, int, const int32_t* const*,                 \
                             const int32_t* const*, Act<T>, Act<T>, Act<T>, bool, cudaStream_t);    \
  template void reduce_slots<T>(const T*, int64_t, int, int64_t, int64_t, int64_t, T*, int64_t,     \
                                bool, cudaStream_t);                                                \
  template void spmm_in_b<T>(const FeatStore&, const SlotDesc*, const LayerDesc*, int, int, Act<T>, T*, \
                             int64_t, cudaStream_t);                                                \
  template void spmm_full_bits<T>(int64_t, const int64_t*, const int32_t*, const double*,           \
                                  const uint32_t*, int64_t, T*, int64_t, int64_t, cudaStream_t);   \
  template void softmax_ce_b<T>(const SlotDesc*, int, int, const int32_t*, Act<T>, int, Act<T>, T*, \
                                double*, double*, int32_t*, cudaStream_t);                          \
  template void softmax_ce_rows_b<T>(const SlotDesc*, int, int, const int32_t*, Act<T>, int, Act<T>, \
                                     T*, double*, const int32_t*, cudaStream_t);                    \
  template void bce_b<T>(const SlotDesc*, int, int, const uint64_t*, int, Act<T>, int, double, Act<T>, \
                         T*, double*, double*, cudaStream_t);                                       \
  template void sgd_step<T>(T*, const T*, int64_t, double, double, cudaStream_t);                   \
  template void adam_step<T>(T*, const T*, T*, T*, int64_t, double, double, double, double, double, \
                             double, double, double, double, cudaStream_t);                         \
  template void spmm_full<T>(int64_t, const int64_t*, const int32_t*, const double*, const T*,      \
                             int64_t, bool, T*, int64_t, int64_t, cudaStream_t);                    \
  template void gemm_plain<T>(int, int, int, const T*, int64_t, const T*, int64_t, T*, int64_t,     \
                              cudaStream_t);                                                        \
  template void fill_zero<T>(T*, int64_t, cudaStream_t);
INST(float)
INST(double)

}  // namespace skg
