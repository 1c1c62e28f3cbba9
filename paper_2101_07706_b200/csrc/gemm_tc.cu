// tcgen05 (5th-gen tensor core) GEMM for the GCN's dense contractions H·W, G·Wᵀ, Uᵀ·G.
//
// Warp-specialised, one 128 x BN output tile per CTA, fp32 accumulator in TMEM:
//   warp 0      : TMEM allocation; lane 0 issues tcgen05.mma.kind::tf32 for every K step of
//                 a full stage and commits it to that stage's "empty" mbarrier
//   warps 1..8  : producers.  They read operands from global memory (any transposition),
//                 split them into TF32 hi/lo parts and write the canonical no-swizzle
//                 K-major UMMA layout (8-row x 16-byte core matrices; LBO = next core matrix
//                 along K, SBO = next along M/N) into a STAGES-deep shared-memory ring, then
//                 arrive on the stage's "full" mbarrier.  The next chunk's global loads are
//                 issued before the current chunk is converted (register double buffer).
//                 After the last commit they drain TMEM (tcgen05.ld) into global memory.
//   MODE 1: 1xTF32 (10-bit mantissa inputs)
//   MODE 3: 3xTF32  D += Ahi Bhi + Ahi Blo + Alo Bhi  (~fp32 accuracy; default, keeps the
//           rtol 1e-4 parity of fp32 activations/gradients against the fp64 reference)
#include <cstdint>
#include <cstdio>

#include "gcn.cuh"
#include "prof.h"
#include "sampler.cuh"
#include "skg_internal.h"

namespace skg {

namespace tc {

constexpr int BM = 128;
constexpr int BK = 32;                 // K elements per stage (4 MMAs of K = 8)
constexpr int KGROUPS = BK / 4;        // core matrices along K per stage
constexpr int NPROD = 256;             // producer threads (8 warps)
constexpr int NTHREADS = 32 + NPROD;
constexpr int STAGES = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// canonical K-major, no swizzle: element (row, k) of a tile
__device__ __forceinline__ int kmaj_off(int row, int k) {
  return (((row >> 3) * KGROUPS + (k >> 2)) << 5) + ((row & 7) << 2) + (k & 3);
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  const uint64_t lbo = 128, sbo = (uint64_t)KGROUPS * 128;
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
  return d;                // base offset 0, legacy LBO mode, SWIZZLE_NONE
}

__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  // c_format F32 (bit 4), a/b format TF32 (=2 at bits 7, 10), K-major A and B,
  // n_dim = N >> 3 at bit 17, m_dim = M >> 4 at bit 24
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm volatile("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)));
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
      smem_u32(bar)));
}

// Each quad is 4 consecutive k of one tile row, stored as one 16-byte smem write.  The 8
// lanes of a warp sharing a k group cover the 8 rows of one core matrix (a full 128-byte
// smem row: conflict-free) and global reads stay coalesced (TRANS: lanes walk the
// contiguous row axis).
template <bool TRANS, int ROWS>
struct StageIO {
  static constexpr int Q = ROWS * BK / 4 / NPROD;  // float4 quads per producer thread
  __device__ static void coords(int p, int q, int& r, int& k) {
    const int qd = p + q * NPROD;
    if (TRANS) {
      r = qd % ROWS;
      k = (qd / ROWS) * 4;
    } else {
      r = (qd & 7) + 8 * (qd >> 6);
      k = ((qd >> 3) & 7) * 4;
    }
  }
  // tile element (r, k) = TRANS ? src[(k0+k)*ld + row0 + r] : src[(row0+r)*ld + k0 + k]
  __device__ static void gload(int p, const float* __restrict__ src, int64_t ld, int row0,
                               int nrows, int k0, int K, bool vec, float4 (&v)[Q]) {
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      int r, k;
      coords(p, q, r, k);
      const int gr = row0 + r, gk = k0 + k;
      float t[4];
      if (TRANS) {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          t[e] = (gr < nrows && gk + e < K) ? __ldg(src + (int64_t)(gk + e) * ld + gr) : 0.f;
      } else {
        if (vec && gr < nrows && gk + 3 < K) {
          v[q] = __ldg(reinterpret_cast<const float4*>(src + (int64_t)gr * ld + gk));
          continue;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e)
          t[e] = (gr < nrows && gk + e < K) ? __ldg(src + (int64_t)gr * ld + gk + e) : 0.f;
      }
      v[q] = make_float4(t[0], t[1], t[2], t[3]);
    }
  }
  __device__ static void sstore(int p, const float4 (&v)[Q], float* s_hi, float* s_lo, bool split) {
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      int r, k;
      coords(p, q, r, k);
      const float x[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
      float hi[4], lo[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        hi[e] = to_tf32(x[e]);
        lo[e] = to_tf32(x[e] - hi[e]);
      }
      const int o = kmaj_off(r, k);
      *reinterpret_cast<float4*>(s_hi + o) = make_float4(hi[0], hi[1], hi[2], hi[3]);
      if (split) *reinterpret_cast<float4*>(s_lo + o) = make_float4(lo[0], lo[1], lo[2], lo[3]);
    }
  }
};

}  // namespace tc

// C_z = op(A_z) op(B_z) (+ C_z) on tensor cores; op(A) M x K, op(B) K x N.
template <bool TA, bool TB, int BN, int MODE>
__global__ void __launch_bounds__(tc::NTHREADS, 1)
    k_gemm_tc(int Mfix, int N, int Kfix, const int32_t* const* dM, const int32_t* const* dK,
              Act<float> A, Act<float> B, Act<float> C, int accumulate) {
  using namespace tc;
  constexpr bool SPLIT = MODE == 3;
  constexpr int A_ELEMS = BM * BK, B_ELEMS = BN * BK;
  constexpr int STAGE = (A_ELEMS + B_ELEMS) * (SPLIT ? 2 : 1);
  constexpr int TCOLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  extern __shared__ __align__(1024) float smem[];
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES], done_bar;
  __shared__ uint32_t tmem_base;

  const int z = blockIdx.z;
  const int M = dM ? *dM[z] : Mfix;
  const int K = dK ? *dK[z] : Kfix;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= M) return;
  const float* __restrict__ a = A.at(z);
  const float* __restrict__ b = B.at(z);
  float* __restrict__ c = C.at(z);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (K + BK - 1) / BK;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "n"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    if (lane == 0) {
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&full_bar[s], NPROD / 32);  // one arrive per producer warp
        mbar_init(&empty_bar[s], 1);          // tcgen05.commit
      }
      mbar_init(&done_bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc(BM, BN);
      for (int kc = 0; kc < nk; ++kc) {
        const int s = kc % STAGES;
        mbar_wait(&full_bar[s], (uint32_t)((kc / STAGES) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;");
        float* st = smem + s * STAGE;
        const uint32_t a_hi = smem_u32(st), b_hi = smem_u32(st + A_ELEMS);
        const uint32_t a_lo = smem_u32(st + A_ELEMS + B_ELEMS);
        const uint32_t b_lo = a_lo + A_ELEMS * 4;
#pragma unroll
        for (int ks = 0; ks < BK / 8; ++ks) {
          const uint32_t koff = ks * 2 * 128;  // two core matrices along K per MMA
          const uint64_t ah = make_desc(a_hi + koff), bh = make_desc(b_hi + koff);
          mma_tf32(tmem, ah, bh, idesc, (kc > 0 || ks > 0) ? 1u : 0u);
          if (SPLIT) {
            mma_tf32(tmem, ah, make_desc(b_lo + koff), idesc, 1u);
            mma_tf32(tmem, make_desc(a_lo + koff), bh, idesc, 1u);
          }
        }
        mma_commit(&empty_bar[s]);  // stage s may be refilled once these MMAs complete
      }
      mma_commit(&done_bar);  // accumulator complete
    }
    __syncwarp();
  } else {
    // ---------------- producers
    const int p = threadIdx.x - 32;
    const bool vecA = (A.ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(a) & 15) == 0);
    const bool vecB = (B.ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(b) & 15) == 0);
    using IOA = StageIO<TA, BM>;
    using IOB = StageIO<!TB, BN>;
    float4 ra[IOA::Q], rb[IOB::Q];
    if (nk > 0) {
      IOA::gload(p, a, A.ld, m0, M, 0, K, vecA, ra);
      IOB::gload(p, b, B.ld, n0, N, 0, K, vecB, rb);
    }
    for (int kc = 0; kc < nk; ++kc) {
      const int s = kc % STAGES;
      if (kc >= STAGES) mbar_wait(&empty_bar[s], (uint32_t)(((kc / STAGES) - 1) & 1));
      float* st = smem + s * STAGE;
      IOA::sstore(p, ra, st, st + A_ELEMS + B_ELEMS, SPLIT);
      IOB::sstore(p, rb, st + A_ELEMS, st + A_ELEMS + B_ELEMS + A_ELEMS, SPLIT);
      if (kc + 1 < nk) {  // next chunk's loads fly while the MMA consumes this stage
        IOA::gload(p, a, A.ld, m0, M, (kc + 1) * BK, K, vecA, ra);
        IOB::gload(p, b, B.ld, n0, N, (kc + 1) * BK, K, vecB, rb);
      }
      asm volatile("fence.proxy.async.shared::cta;");  // generic smem writes -> async proxy
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_bar[s]);
    }
    // ---------------- epilogue: TMEM lane group (warp % 4), column half (warp - 1) / 4
    mbar_wait(&done_bar, 0u);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int lg = warp & 3;
    const int row = m0 + lg * 32 + lane;
    const uint32_t taddr_row = tmem + ((uint32_t)(lg * 32) << 16);
    const int half = (warp - 1) >> 2;
    constexpr int CH = BN / 2;
#pragma unroll 1
    for (int cb = half * CH; cb < half * CH + CH; cb += 16) {
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
            "=r"(v[14]), "=r"(v[15])
          : "r"(taddr_row + cb));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      if (row < M) {
        float* crow = c + (int64_t)row * C.ld;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int col = n0 + cb + j;
          if (col < N) crow[col] = accumulate ? crow[col] + __uint_as_float(v[j]) : __uint_as_float(v[j]);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS));
}

template <bool TA, bool TB, int BN, int MODE>
static int launch_tc(int n, int M, int N, int K, const int32_t* const* dM, const int32_t* const* dK,
                     Act<float> A, Act<float> B, Act<float> C, bool acc, cudaStream_t st) {
  constexpr int STAGE = (tc::BM * tc::BK + BN * tc::BK) * (MODE == 3 ? 2 : 1);
  const size_t smem = (size_t)tc::STAGES * STAGE * sizeof(float);
  auto kern = k_gemm_tc<TA, TB, BN, MODE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((N + BN - 1) / BN, (M + tc::BM - 1) / tc::BM, n);
  LAUNCH_NAMED("k_gemm_tc", st, kern<<<grid, tc::NTHREADS, smem, st>>>(M, N, K, dM, dK, A, B, C, acc ? 1 : 0));
  return 0;
}

template <bool TA, bool TB, int MODE>
static int dispatch_bn(int n, int M, int N, int K, const int32_t* const* dM, const int32_t* const* dK,
                       Act<float> A, Act<float> B, Act<float> C, bool acc, cudaStream_t st) {
  // narrow N tiles: more CTAs for these skinny problems (M <= a few thousand rows)
  if (N <= 32) return launch_tc<TA, TB, 32, MODE>(n, M, N, K, dM, dK, A, B, C, acc, st);
  return launch_tc<TA, TB, 64, MODE>(n, M, N, K, dM, dK, A, B, C, acc, st);
}

int gemm_tc(int mode, bool ta, bool tb, int n, int M, int N, int K, const int32_t* const* dM,
            const int32_t* const* dK, Act<float> A, Act<float> B, Act<float> C, bool acc,
            cudaStream_t st) {
  if (M <= 0 || N <= 0 || n <= 0) return 0;
#define TC_CASE(TA_, TB_)                                                                        \
  if (ta == TA_ && tb == TB_)                                                                    \
    return mode == 3 ? dispatch_bn<TA_, TB_, 3>(n, M, N, K, dM, dK, A, B, C, acc, st)            \
                     : dispatch_bn<TA_, TB_, 1>(n, M, N, K, dM, dK, A, B, C, acc, st);
  TC_CASE(false, false)
  TC_CASE(true, false)
  TC_CASE(false, true)
  TC_CASE(true, true)
#undef TC_CASE
  return 0;
}

// test hook: C = op(A) op(B) for host arrays (row-major, ld = inner dim)
int debug_gemm(int mode, int ta, int tb, int M, int N, int K, const float* hA, const float* hB,
               float* hC) {
  const size_t na = (size_t)M * K, nb = (size_t)K * N, nc = (size_t)M * N;
  float *dA, *dB, *dC;
  cudaMalloc(&dA, na * 4);
  cudaMalloc(&dB, nb * 4);
  cudaMalloc(&dC, nc * 4);
  cudaMemcpy(dA, hA, na * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, nb * 4, cudaMemcpyHostToDevice);
  cudaMemset(dC, 0, nc * 4);
  Act<float> a{dA, 0, ta ? M : K}, b{dB, 0, tb ? K : N}, c{dC, 0, N};
  if (mode == 0) gemm_b<float>(ta, tb, 1, M, N, K, nullptr, nullptr, a, b, c, false, 0);
  else gemm_tc(mode, ta, tb, 1, M, N, K, nullptr, nullptr, a, b, c, false, 0);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hC, dC, nc * 4, cudaMemcpyDeviceToHost);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dC);
  if (e != cudaSuccess) {
    set_error(std::string("debug_gemm: ") + cudaGetErrorString(e));
    return SKG_ERR_CUDA;
  }
  return SKG_OK;
}

}  // namespace skg

extern "C" int skg_debug_gemm(int mode, int ta, int tb, int M, int N, int K, const float* A,
                              const float* B, float* C) {
  return skg::debug_gemm(mode, ta, tb, M, N, K, A, B, C);
}
