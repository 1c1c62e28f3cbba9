// Standalone probe: the GEMM epilogue of a 128 x 128 fp32 TMEM accumulator.
//   (a) tcgen05.ld 32x32b (lane = row) -> float4 stores, one row per thread (the kernel's
//       current epilogue)
//   (b) tcgen05.ld -> st.shared into SWIZZLE_128B boxes of 128 rows x 32 columns -> TMA
//       tensor stores (cp.async.bulk.tensor ... bulk_group)
// One CTA per SM (148 x 128 threads), each writes its own 128 rows of C [148*128 x 128];
// prints the mean / max epilogue cycles per CTA and checks the output.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/epi_probe tools/epi_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int BM = 128, BN = 128, NCTA = 148;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128, 1) epi(const __grid_constant__ CUtensorMap tc, float* C, int mode,
                                                 long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tbase;
  const int row = warp * 32 + lane;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  // fill: value = grow * 1000 + col
  const int grow = blockIdx.x * BM + row;
  for (int cb = 0; cb < BN; cb += 16) {
    uint32_t v[16];
    for (int j = 0; j < 16; ++j) v[j] = __float_as_uint((float)(grow % 4096) * 1000.f + (float)(cb + j));
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            trow + cb),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const long long t0 = clock64();
  if (mode == 0) {
    float* crow = C + (size_t)grow * BN;
#pragma unroll 1
    for (int cb = 0; cb < BN; cb += 16) {
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(trow + cb));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int j4 = 0; j4 < 16; j4 += 4)
        *reinterpret_cast<float4*>(crow + cb + j4) = make_float4(__uint_as_float(v[j4]), __uint_as_float(v[j4 + 1]),
                                                                 __uint_as_float(v[j4 + 2]), __uint_as_float(v[j4 + 3]));
    }
  } else if (mode == 3) {
    // per row: stage the row's 32-column segment at a 144-byte row pitch (8 consecutive rows
    // cover all banks), then the thread itself bulk-copies its 128 bytes (no tensor map: a
    // row mask / column bound is the issuing thread's choice)
    float* crow = C + (size_t)grow * BN;
#pragma unroll 1
    for (int b = 0; b < BN / 32; ++b) {
      uint32_t v[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(trow + b * 32));
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
            "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(trow + b * 32 + 16));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      uint8_t* seg = sm + (b * BM + row) * 144;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<uint4*>(seg + c * 16) = make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
      asm volatile("fence.proxy.async.shared::cta;");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 128;" ::"l"(crow + b * 32), "r"(su32(seg))
                   : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  } else if (mode == 4) {
    // two boxes per step: four TMEM loads in flight per wait
#pragma unroll 1
    for (int b = 0; b < BN / 32; b += 2) {
      uint32_t v[64];
#pragma unroll
      for (int h = 0; h < 4; ++h)
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[16 * h + 0]), "=r"(v[16 * h + 1]), "=r"(v[16 * h + 2]), "=r"(v[16 * h + 3]), "=r"(v[16 * h + 4]),
              "=r"(v[16 * h + 5]), "=r"(v[16 * h + 6]), "=r"(v[16 * h + 7]), "=r"(v[16 * h + 8]), "=r"(v[16 * h + 9]),
              "=r"(v[16 * h + 10]), "=r"(v[16 * h + 11]), "=r"(v[16 * h + 12]), "=r"(v[16 * h + 13]),
              "=r"(v[16 * h + 14]), "=r"(v[16 * h + 15])
            : "r"(trow + b * 32 + 16 * h));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int bb = 0; bb < 2; ++bb) {
        uint8_t* box = sm + (b + bb) * (BM * 128) + row * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<uint4*>(box + ((c ^ (row & 7)) * 16)) =
              make_uint4(v[32 * bb + 4 * c], v[32 * bb + 4 * c + 1], v[32 * bb + 4 * c + 2], v[32 * bb + 4 * c + 3]);
      }
      asm volatile("fence.proxy.async.shared::cta;");
      asm volatile("bar.sync 1, 128;");
      if (threadIdx.x == 0) {
        for (int bb = 0; bb < 2; ++bb)
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&tc),
                       "r"((b + bb) * 32), "r"(blockIdx.x * BM), "r"(su32(sm + (b + bb) * BM * 128))
                       : "memory");
        asm volatile("cp.async.bulk.commit_group;");
      }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  } else if (mode == 2) {
    // per box: two TMEM loads in flight per wait, stage the box, then one thread issues its
    // TMA store while the next box is read from TMEM
#pragma unroll 1
    for (int b = 0; b < BN / 32; ++b) {
      uint32_t v[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(trow + b * 32));
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
            "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(trow + b * 32 + 16));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      uint8_t* box = sm + b * (BM * 128) + row * 128;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<uint4*>(box + ((c ^ (row & 7)) * 16)) = make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
      asm volatile("fence.proxy.async.shared::cta;");
      asm volatile("bar.sync 1, 128;");
      if (threadIdx.x == 0) {
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&tc),
                     "r"(b * 32), "r"(blockIdx.x * BM), "r"(su32(sm + b * BM * 128))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;");
      }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  } else {
    // box b = columns [32b, 32b + 32): 128 rows x 128 B, 16-byte chunk c of row r at
    // chunk position c ^ (r & 7) (SWIZZLE_128B)
#pragma unroll 1
    for (int cb = 0; cb < BN; cb += 16) {
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(trow + cb));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      uint8_t* box = sm + (cb / 32) * (BM * 128) + row * 128;
#pragma unroll
      for (int j4 = 0; j4 < 16; j4 += 4) {
        const int c = ((cb % 32) + j4) / 4;  // 16-byte chunk within the 128-byte row
        *reinterpret_cast<uint4*>(box + ((c ^ (row & 7)) * 16)) = make_uint4(v[j4], v[j4 + 1], v[j4 + 2], v[j4 + 3]);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int b = 0; b < BN / 32; ++b)
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&tc),
                     "r"(b * 32), "r"(blockIdx.x * BM), "r"(su32(sm + b * BM * 128))
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const size_t rows = (size_t)NCTA * BM;
  float* dC;
  long long* dcy;
  cudaMalloc(&dC, rows * BN * 4);
  cudaMalloc(&dcy, NCTA * 8);
  CUtensorMap tc;
  cuuint64_t dims[2] = {(cuuint64_t)BN, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)BN * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)BM};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&tc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dC, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
  cudaFuncSetAttribute(epi, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  std::vector<float> c(rows * BN);
  for (int mode = 0; mode < 5; ++mode) {
    for (int it = 0; it < 3; ++it) {
      cudaMemset(dC, 0, rows * BN * 4);
      epi<<<NCTA, 128, 80 * 1024>>>(tc, dC, mode, dcy);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<long long> cy(NCTA);
      cudaMemcpy(cy.data(), dcy, NCTA * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(c.data(), dC, rows * BN * 4, cudaMemcpyDeviceToHost);
      long long bad = 0;
      for (size_t i = 0; i < rows; ++i)
        for (int j = 0; j < BN; ++j) bad += c[i * BN + j] != (float)(i % 4096) * 1000.f + (float)j;
      double mean = 0;
      long long mx = 0;
      for (long long v : cy) {
        mean += v;
        mx = v > mx ? v : mx;
      }
      printf("%s  epilogue cycles mean %.0f max %lld  (%.2f us at 1.965 GHz)  bad %lld  (%s)\n",
             mode == 4 ? "TMA store 2 boxes  " : mode == 3 ? "bulk copy per row  " : mode == 2 ? "TMA store per box  " : mode ? "TMA store via smem " : "row float4 stores  ", mean / NCTA, mx, mean / NCTA / 1965.0, bad,
             cudaGetErrorString(e));
      if (e != cudaSuccess) return 1;
    }
  }
  return 0;
}
