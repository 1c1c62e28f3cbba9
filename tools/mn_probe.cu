// Standalone probe: TMA (SWIZZLE_128B) -> tcgen05.mma kind::tf32 with K-major and MN-major
// operands.  C[128 x 64] = A[128 x 32] B[32 x 64]; prints the max error per variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mn_probe tools/mn_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int M = 128, N = 64, K = 32;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

struct Params {
  int a_mn, b_mn, a_layout, b_layout;
  uint32_t a_lbo, a_sbo, a_kstep, b_lbo, b_sbo, b_kstep;
  int a_boxes, b_boxes;      // TMA boxes per operand
  int a_box_bytes, b_box_bytes;
};

__global__ void probe(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                      Params P, float* C) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;
  uint8_t* sB = sm + 16384;
  __shared__ __align__(8) uint64_t bar, mbar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    const int bytes = P.a_boxes * P.a_box_bytes + P.b_boxes * P.b_box_bytes;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes));
    for (int i = 0; i < P.a_boxes; ++i) {
      int c0 = P.a_mn ? i * 32 : 0, c1 = 0;  // MN: box i covers rows 32i..; K: one box
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              su32(sA + i * P.a_box_bytes)),
          "l"(&ta), "r"(c0), "r"(c1), "r"(su32(&bar)));
    }
    for (int i = 0; i < P.b_boxes; ++i) {
      int c0 = P.b_mn ? i * 32 : 0, c1 = 0;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              su32(sB + i * P.b_box_bytes)),
          "l"(&tb), "r"(c0), "r"(c1), "r"(su32(&bar)));
    }
    asm volatile(
        "{\n.reg .pred p;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W1;\n}\n" ::"r"(su32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)P.a_mn << 15) | ((uint32_t)P.b_mn << 16) |
                           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int ks = 0; ks < K / 8; ++ks) {
      uint64_t ad = desc(su32(sA) + ks * P.a_kstep, P.a_lbo, P.a_sbo, P.a_layout);
      uint64_t bd = desc(su32(sB) + ks * P.b_kstep, P.b_lbo, P.b_sbo, P.b_layout);
      uint32_t acc = ks > 0;
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                       tmem),
                   "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar)));
  }
  __syncwarp();
  asm volatile(
      "{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W2;\n}\n" ::"r"(su32(&mbar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = warp * 32 + (threadIdx.x & 31);
  for (int cb = 0; cb < N; cb += 16) {
    uint32_t v[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(tmem + ((uint32_t)(warp * 32) << 16) + cb));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 16; ++j) C[row * N + cb + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;

// 2D fp32 tensor map: inner dim `inner` (contiguous), outer dim `outer`, box {32, box_outer}
static CUtensorMap make_map(float* base, int inner, int outer, int box_outer,
                            CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)inner * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
  return m;
}

int main() {
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  std::vector<float> a(M * K), b(K * N);
  for (int i = 0; i < M * K; ++i) a[i] = (float)((i * 7 + 3) % 11 - 5);
  for (int i = 0; i < K * N; ++i) b[i] = (float)((i * 5 + 1) % 9 - 4);
  std::vector<double> ref(M * N, 0.0);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < K; ++k) ref[m * N + n] += (double)a[m * K + k] * b[k * N + n];
  // device copies in both storage orders
  std::vector<float> at(K * M), bt(N * K);
  for (int m = 0; m < M; ++m)
    for (int k = 0; k < K; ++k) at[k * M + m] = a[m * K + k];
  for (int k = 0; k < K; ++k)
    for (int n = 0; n < N; ++n) bt[n * K + k] = b[k * N + n];
  float *dA, *dAt, *dB, *dBt, *dC;
  cudaMalloc(&dA, M * K * 4); cudaMalloc(&dAt, M * K * 4); cudaMalloc(&dB, K * N * 4);
  cudaMalloc(&dBt, K * N * 4); cudaMalloc(&dC, M * N * 4);
  cudaMemcpy(dA, a.data(), M * K * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dAt, at.data(), M * K * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, b.data(), K * N * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dBt, bt.data(), K * N * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  // K-major tile (rows x 32 k): one box {32 k, rows}; SW128 atom = 8 rows x 128 B;
  // SBO = 1024 (next 8-row group), LBO unused (16), k step of 8 tf32 = 32 B.
  // MN-major tile (32 k x rows): boxes {32 mn, 32 k} (4 KB each); atom = 8 k-rows x 128 B;
  // per CUTLASS: LBO = next 32-mn block, SBO = next 8-k group; k step = 8 k-rows = 1024 B.
  // MN-major tf32 needs the SW128_32B layout (descriptor layout 1, TMA 128B_ATOM_32B):
  // atom = 4 k-rows x 128 B (Swizzle<2,5,2>), SBO = next 4-k group, LBO = next 32-mn block.
  struct V { const char* name; int a_mn, b_mn; uint32_t a_lbo, a_sbo, b_lbo, b_sbo; };
  V vs[] = {
      {"A K, B K", 0, 0, 16, 1024, 16, 1024},
      {"A K, B MN32 lbo4096 sbo512", 0, 1, 16, 1024, 4096, 512},
      {"A K, B MN32 lbo512 sbo4096", 0, 1, 16, 1024, 512, 4096},
      {"A MN32, B K lbo4096 sbo512", 1, 0, 4096, 512, 16, 1024},
      {"A MN32, B MN32 lbo4096 sbo512", 1, 1, 4096, 512, 4096, 512},
  };
  for (const V& v : vs) {
    Params P;
    P.a_mn = v.a_mn; P.b_mn = v.b_mn;
    P.a_lbo = v.a_lbo; P.a_sbo = v.a_sbo; P.b_lbo = v.b_lbo; P.b_sbo = v.b_sbo;
    P.a_kstep = v.a_mn ? 1024 : 32;
    P.b_kstep = v.b_mn ? 1024 : 32;
    P.a_layout = v.a_mn ? 1 : 2;
    P.b_layout = v.b_mn ? 1 : 2;
    CUtensorMap ta = v.a_mn ? make_map(dAt, M, K, K, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) : make_map(dA, K, M, M);
    CUtensorMap tb = v.b_mn ? make_map(dB, N, K, K, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) : make_map(dBt, K, N, N);
    P.a_boxes = v.a_mn ? M / 32 : 1;
    P.a_box_bytes = v.a_mn ? 32 * K * 4 : M * K * 4;
    P.b_boxes = v.b_mn ? N / 32 : 1;
    P.b_box_bytes = v.b_mn ? 32 * K * 4 : N * K * 4;
    cudaMemset(dC, 0, M * N * 4);
    probe<<<1, 128, 40 * 1024>>>(ta, tb, P, dC);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> c(M * N);
    cudaMemcpy(c.data(), dC, M * N * 4, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < M * N; ++i) err = fmax(err, fabs(c[i] - ref[i]));
    printf("%-30s maxerr %g  (%s)\n", v.name, err, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
