// GCN compute over a sampled plan: fused feature gather (local shard or NVLink peer),
// CSR SpMM (ReLU fused on the input), transposed SpMM fused with the ReLU mask, a tiled
// GEMM for H·W, softmax cross-entropy forward+backward and the optimizer steps.
//
// Reference: training.py:261-318 (forward / loss_and_backward), 398-427 (SGD / Adam),
// 325-334 (predict_logits).  Activation rows are padded to a multiple of 4 elements so
// every row access is a 16-byte vector; padding columns stay zero.
#include <cub/block/block_reduce.cuh>
#include <cstdio>

#include "gcn.cuh"
#include "sampler.cuh"
#include "skg_internal.h"

namespace skg {

#define GLAUNCH(...)       \
  do {                     \
    __VA_ARGS__;           \
    ++g_kernel_launches;   \
  } while (0)

constexpr unsigned FULLM = 0xffffffffu;

template <typename T>
struct Vec4;
template <>
struct Vec4<float> {
  float4 v;
  __device__ static Vec4 load(const float* p) { Vec4 r; r.v = *reinterpret_cast<const float4*>(p); return r; }
  __device__ void store(float* p) const { *reinterpret_cast<float4*>(p) = v; }
  __device__ static Vec4 zero() { Vec4 r; r.v = make_float4(0.f, 0.f, 0.f, 0.f); return r; }
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

// ------------------------------------------------------------------ gather (K7)
template <typename T>
__global__ void k_gather(FeatStore fs, const int32_t* ids, const int32_t* d_n, T* out, int64_t ldo) {
  const int n = *d_n;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
    const int node = ids[r];
    const int rank = fs.node_rank ? fs.node_rank[node] : 0;
    const int64_t row = fs.node_row ? fs.node_row[node] : node;
    const T* src = reinterpret_cast<const T*>(fs.shards[rank]) + row * fs.ld;
    for (int64_t c = lane * 4; c < fs.ld; c += 128) Vec4<T>::load(src + c).store(out + r * ldo + c);
  }
}

template <typename T>
void gather_rows(const FeatStore& fs, const int32_t* ids, const int32_t* d_n, int max_n, T* out,
                 int64_t ldo, cudaStream_t st) {
  int blocks = std::max(1, std::min((max_n + 7) / 8, 4 * sms()));
  GLAUNCH(k_gather<T><<<blocks, 256, 0, st>>>(fs, ids, d_n, out, ldo));
}

// ------------------------------------------------------------------ SpMM (K8 / K10)
template <typename T, bool RELU, bool MASK>
__global__ void k_spmm(const int32_t* d_rows, const int32_t* __restrict__ indptr,
                       const int32_t* __restrict__ indices, const double* __restrict__ val,
                       const T* __restrict__ A, int64_t lda, const T* __restrict__ H, int64_t ldh,
                       T* __restrict__ out, int64_t ldo, int64_t width) {
  const int rows = *d_rows;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += nw) {
    const int b = indptr[r], e = indptr[r + 1];
    for (int64_t c = lane * 4; c < width; c += 128) {
      Vec4<T> acc = Vec4<T>::zero();
      for (int p = b; p < e; ++p) {
        Vec4<T> x = Vec4<T>::load(A + (int64_t)indices[p] * lda + c);
        if (RELU) x.relu();
        acc.fma((T)val[p], x);
      }
      if (MASK) acc.mask(Vec4<T>::load(H + (int64_t)r * ldh + c));
      acc.store(out + (int64_t)r * ldo + c);
    }
  }
}

template <typename T>
void spmm(const int32_t* d_rows, int max_rows, const int32_t* indptr, const int32_t* indices,
          const double* val, const T* A, int64_t lda, bool relu_in, T* out, int64_t ldo,
          int64_t width, cudaStream_t st) {
  int blocks = std::max(1, std::min((max_rows + 7) / 8, 4 * sms()));
  if (relu_in)
    GLAUNCH((k_spmm<T, true, false><<<blocks, 256, 0, st>>>(d_rows, indptr, indices, val, A, lda,
                                                            nullptr, 0, out, ldo, width)));
  else
    GLAUNCH((k_spmm<T, false, false><<<blocks, 256, 0, st>>>(d_rows, indptr, indices, val, A, lda,
                                                             nullptr, 0, out, ldo, width)));
}

template <typename T>
void spmm_t_mask(const int32_t* d_rows, int max_rows, const int32_t* indptr,
                 const int32_t* indices, const double* val, const T* G, int64_t ldg,
                 const T* H, int64_t ldh, T* out, int64_t ldo, int64_t width, cudaStream_t st) {
  int blocks = std::max(1, std::min((max_rows + 7) / 8, 4 * sms()));
  GLAUNCH((k_spmm<T, false, true><<<blocks, 256, 0, st>>>(d_rows, indptr, indices, val, G, ldg, H,
                                                          ldh, out, ldo, width)));
}

// full-graph SpMM for predict_logits (int64 offsets)
template <typename T, bool RELU>
__global__ void k_spmm_full(int64_t n, const int64_t* __restrict__ off, const int32_t* __restrict__ col,
                            const double* __restrict__ w, const T* __restrict__ A, int64_t lda,
                            T* __restrict__ out, int64_t ldo, int64_t width) {
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
    GLAUNCH((k_spmm_full<T, true><<<blocks, 256, 0, st>>>(n, off, col, w, A, lda, out, ldo, width)));
  else
    GLAUNCH((k_spmm_full<T, false><<<blocks, 256, 0, st>>>(n, off, col, w, A, lda, out, ldo, width)));
}

// ------------------------------------------------------------------ GEMM (K9)
// 64x64x16 tiles, 256 threads, 4x4 outputs per thread; op(A) is M x K, op(B) is K x N.
constexpr int GBM = 64, GBN = 64, GBK = 16;

template <typename T, bool TA, bool TB>
__global__ void __launch_bounds__(256) k_gemm(int M, int N, int K, const int32_t* dM, const int32_t* dK,
                                              const T* __restrict__ A, int64_t lda,
                                              const T* __restrict__ B, int64_t ldb,
                                              T* __restrict__ C, int64_t ldc, bool accumulate) {
  if (dM) M = *dM;
  if (dK) K = *dK;
  const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * GBN;
  if (m0 >= M) return;
  __shared__ T As[GBK][GBM + 4];
  __shared__ T Bs[GBK][GBN + 4];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  T acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
  for (int k0 = 0; k0 < K; k0 += GBK) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = tid + q * 256;
      int m, k;
      if (TA) { k = idx / GBM; m = idx % GBM; } else { m = idx / GBK; k = idx % GBK; }
      const int gm = m0 + m, gk = k0 + k;
      T v = T(0);
      if (gm < M && gk < K) v = TA ? A[(int64_t)gk * lda + gm] : A[(int64_t)gm * lda + gk];
      As[k][m] = v;
      int n, kb;
      if (TB) { n = idx / GBK; kb = idx % GBK; } else { kb = idx / GBN; n = idx % GBN; }
      const int gn = n0 + n, gkb = k0 + kb;
      T u = T(0);
      if (gn < N && gkb < K) u = TB ? B[(int64_t)gn * ldb + gkb] : B[(int64_t)gkb * ldb + gn];
      Bs[kb][n] = u;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GBK; ++kk) {
      T a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn >= N) continue;
      T* c = C + (int64_t)gm * ldc + gn;
      *c = accumulate ? *c + acc[i][j] : acc[i][j];
    }
  }
}

template <typename T>
void gemm(bool ta, bool tb, int M, int N, int K, const int32_t* dM, const int32_t* dK, const T* A,
          int64_t lda, const T* B, int64_t ldb, T* C, int64_t ldc, bool accumulate,
          cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  dim3 grid((N + GBN - 1) / GBN, (M + GBM - 1) / GBM);
  if (!ta && !tb) GLAUNCH((k_gemm<T, false, false><<<grid, 256, 0, st>>>(M, N, K, dM, dK, A, lda, B, ldb, C, ldc, accumulate)));
  else if (ta && !tb) GLAUNCH((k_gemm<T, true, false><<<grid, 256, 0, st>>>(M, N, K, dM, dK, A, lda, B, ldb, C, ldc, accumulate)));
  else if (!ta && tb) GLAUNCH((k_gemm<T, false, true><<<grid, 256, 0, st>>>(M, N, K, dM, dK, A, lda, B, ldb, C, ldc, accumulate)));
  else GLAUNCH((k_gemm<T, true, true><<<grid, 256, 0, st>>>(M, N, K, dM, dK, A, lda, B, ldb, C, ldc, accumulate)));
}

// ------------------------------------------------------------------ softmax CE (K11)
// training.py:293-308: LSE loss averaged over labelled batch rows and its gradient.
template <typename T>
__global__ void k_softmax_ce(const int32_t* d_rows, const int32_t* batch, const int32_t* labels,
                             const T* Z, int64_t ldz, int C, T* G, int64_t ldg, double* loss_out,
                             int32_t* err) {
  const int n = *d_rows;
  __shared__ int s_nlab;
  __shared__ double wsum[32];
  typedef cub::BlockReduce<int, 1024> BR;
  __shared__ typename BR::TempStorage tmp;
  int c = 0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) c += labels[batch[r]] >= 0;
  int tot = BR(tmp).Sum(c);
  if (threadIdx.x == 0) s_nlab = tot;
  __syncthreads();
  const int nlab = s_nlab;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double part = 0.0;
  for (int r = w; r < n; r += 32) {
    const int y = labels[batch[r]];
    T* g = G + (int64_t)r * ldg;
    if (y < 0 || nlab == 0) {
      for (int k = lane; k < C; k += 32) g[k] = T(0);
      continue;
    }
    const T* z = Z + (int64_t)r * ldz;
    double zmax = -INFINITY;
    for (int k = lane; k < C; k += 32) zmax = fmax(zmax, (double)z[k]);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) zmax = fmax(zmax, __shfl_xor_sync(FULLM, zmax, d));
    double se = 0.0;
    for (int k = lane; k < C; k += 32) se += exp((double)z[k] - zmax);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) se += __shfl_xor_sync(FULLM, se, d);
    const double lse = zmax + log(se);
    for (int k = lane; k < C; k += 32) {
      double gz = exp((double)z[k] - lse) - (k == y ? 1.0 : 0.0);
      g[k] = (T)(gz / nlab);
    }
    if (lane == 0) part += lse - (double)z[y];
  }
  if (lane == 0) wsum[w] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < 32; ++i) s += wsum[i];
    *loss_out = nlab ? s / nlab : __longlong_as_double(0x7ff8000000000000LL);
    if (!nlab) atomicOr(err, EB_NO_LABELS);
  }
}

template <typename T>
void softmax_ce(const int32_t* d_rows, int max_rows, const int32_t* batch, const int32_t* labels,
                const T* logits, int64_t ldz, int C, T* grad, int64_t ldg, double* loss_out,
                int32_t* err, cudaStream_t st) {
  GLAUNCH((k_softmax_ce<T><<<1, 1024, 0, st>>>(d_rows, batch, labels, logits, ldz, C, grad, ldg,
                                               loss_out, err)));
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
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    w[i] = ad(w[i], -ml(lr, dv(g[i], contrib)));
}

// training.py:415-427
template <typename T>
__global__ void k_adam(T* w, const T* g, T* m, T* v, int64_t n, T lr, T contrib, T b1, T b2,
                       T omb1, T omb2, T bc1, T bc2, T eps) {
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
  GLAUNCH(k_sgd<T><<<std::max(blocks, 1), 256, 0, st>>>(w, g, n, (T)lr, (T)contrib));
}

template <typename T>
void adam_step(T* w, const T* g, T* m, T* v, int64_t n, double lr, double contrib, double b1,
               double b2, double omb1, double omb2, double bc1, double bc2, double eps,
               cudaStream_t st) {
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 8 * sms());
  GLAUNCH(k_adam<T><<<std::max(blocks, 1), 256, 0, st>>>(w, g, m, v, n, (T)lr, (T)contrib, (T)b1, (T)b2,
                                                         (T)omb1, (T)omb2, (T)bc1, (T)bc2, (T)eps));
}

template <typename T>
__global__ void k_zero(T* p, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = T(0);
}
template <typename T>
void fill_zero(T* p, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 8 * sms());
  GLAUNCH(k_zero<T><<<std::max(blocks, 1), 256, 0, st>>>(p, n));
}

#define INST(T)                                                                                      \
  template void gather_rows<T>(const FeatStore&, const int32_t*, const int32_t*, int, T*, int64_t,   \
                               cudaStream_t);                                                        \
  template void spmm<T>(const int32_t*, int, const int32_t*, const int32_t*, const double*, const T*, \
                        int64_t, bool, T*, int64_t, int64_t, cudaStream_t);                          \
  template void spmm_t_mask<T>(const int32_t*, int, const int32_t*, const int32_t*, const double*,   \
                               const T*, int64_t, const T*, int64_t, T*, int64_t, int64_t,           \
                               cudaStream_t);                                                        \
  template void gemm<T>(bool, bool, int, int, int, const int32_t*, const int32_t*, const T*, int64_t, \
                        const T*, int64_t, T*, int64_t, bool, cudaStream_t);                         \
  template void softmax_ce<T>(const int32_t*, int, const int32_t*, const int32_t*, const T*, int64_t, \
                              int, T*, int64_t, double*, int32_t*, cudaStream_t);                    \
  template void sgd_step<T>(T*, const T*, int64_t, double, double, cudaStream_t);                    \
  template void adam_step<T>(T*, const T*, T*, T*, int64_t, double, double, double, double, double,  \
                             double, double, double, double, cudaStream_t);                          \
  template void spmm_full<T>(int64_t, const int64_t*, const int32_t*, const double*, const T*,       \
                             int64_t, bool, T*, int64_t, int64_t, cudaStream_t);                     \
  template void fill_zero<T>(T*, int64_t, cudaStream_t);
INST(float)
INST(double)

}  // namespace skg
