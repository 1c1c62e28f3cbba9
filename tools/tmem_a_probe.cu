// Standalone probe: tcgen05.mma kind::tf32 with the A operand in tensor memory ("TS":
// A written by tcgen05.st from registers, lane = row, one tf32 per 32-bit column) against
// the SS form (A and B both read from shared memory).  Prints the max error of
// C[128 x N] = A[128 x 32] B[32 x N] and the cycles per MMA of a long MMA loop in each form.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tmem_a_probe tools/tmem_a_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int M = 128, K = 32;

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

// ts: A from TMEM; reps: MMA loop length for timing (1 = correctness pass)
__global__ void probe(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                      const float* A, int N, int ts, int reps, float* C, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;
  uint8_t* sB = sm + 16384;
  __shared__ __align__(8) uint64_t bar, mbar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
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
  constexpr uint32_t ACOL = 256;  // A columns [256, 288)
  {
    // every warp writes its 32-lane quarter: lane = row, column = k
    const int row = warp * 32 + lane;
    uint32_t r[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) r[k] = __float_as_uint(A[row * K + k]);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tmem + ((uint32_t)(warp * 32) << 16) + ACOL),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    const int bytes = M * K * 4 + N * K * 4;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(sA)),
        "l"(&ta), "r"(0), "r"(0), "r"(su32(&bar)));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(sB)),
        "l"(&tb), "r"(0), "r"(0), "r"(su32(&bar)));
    asm volatile(
        "{\n.reg .pred p;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W1;\n}\n" ::"r"(su32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
      for (int ks = 0; ks < K / 8; ++ks) {
        const uint64_t bd = desc(su32(sB) + ks * 32, 16, 1024, 2);
        const uint32_t acc = (rep > 0 || ks > 0) ? 1u : 0u;
        if (ts) {
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(
                           tmem),
                       "r"(tmem + ACOL + ks * 8), "l"(bd), "r"(idesc), "r"(acc));
        } else {
          const uint64_t ad = desc(su32(sA) + ks * 32, 16, 1024, 2);
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                           tmem),
                       "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar)));
    asm volatile(
        "{\n.reg .pred p;\nW3:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W3;\n}\n" ::"r"(su32(&mbar)));
    *cycles = clock64() - t0;
  }
  __syncwarp();
  asm volatile(
      "{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W2;\n}\n" ::"r"(su32(&mbar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = warp * 32 + lane;
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
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;

static CUtensorMap make_map(float* base, int inner, int outer, int box_outer) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)inner * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
  return m;
}

int main() {
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  for (int N : {64, 128, 256}) {
    std::vector<float> a(M * K), bt(N * K);
    for (int i = 0; i < M * K; ++i) a[i] = (float)((i * 7 + 3) % 11 - 5);
    for (int i = 0; i < N * K; ++i) bt[i] = (float)((i * 5 + 1) % 9 - 4);
    std::vector<double> ref(M * N, 0.0);
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n)
        for (int k = 0; k < K; ++k) ref[m * N + n] += (double)a[m * K + k] * bt[n * K + k];
    float *dA, *dBt, *dC;
    long long* dcy;
    cudaMalloc(&dA, M * K * 4);
    cudaMalloc(&dBt, N * K * 4);
    cudaMalloc(&dC, M * N * 4);
    cudaMalloc(&dcy, 8);
    cudaMemcpy(dA, a.data(), M * K * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dBt, bt.data(), N * K * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    CUtensorMap ta = make_map(dA, K, M, M), tb = make_map(dBt, K, N, N);
    for (int ts = 0; ts < 2; ++ts) {
      for (int reps : {1, 4096}) {
        cudaMemset(dC, 0, M * N * 4);
        probe<<<1, 128, 64 * 1024>>>(ta, tb, dA, N, ts, reps, dC, dcy);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> c(M * N);
        long long cy = 0;
        cudaMemcpy(c.data(), dC, M * N * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(&cy, dcy, 8, cudaMemcpyDeviceToHost);
        double err = 0;
        for (int i = 0; i < M * N; ++i) err = fmax(err, fabs(c[i] - reps * ref[i]) / fmax(1.0, fabs(reps * ref[i])));
        printf("N=%3d %s reps=%5d  max rel err %-10g  cycles/MMA %.1f  (%s)\n", N, ts ? "TS (A in TMEM)" : "SS          ",
               reps, err, (double)cy / (reps * (K / 8)), cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
      }
    }
    cudaFree(dA);
    cudaFree(dBt);
    cudaFree(dC);
    cudaFree(dcy);
  }
  return 0;
}
