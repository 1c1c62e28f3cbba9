// tcgen05 (5th-gen tensor core) GEMM for the GCN's dense contractions H·W, G·Wᵀ, Uᵀ·G.
//
// Operands arrive pre-split into TF32 hi / lo fp32 arrays (the producing kernels write
// them: SpMM -> U, softmax / transposed SpMM -> G, k_split_weights -> W), so this kernel is
// a pure TMA -> tcgen05 pipeline:
//   warp 0 (one lane) : TMA producer.  Per 32-wide K chunk it loads the hi (and lo) boxes of
//                       A and B into one stage of a STAGES-deep ring (SWIZZLE_128B) and
//                       arms the stage's "full" mbarrier with the byte count.
//   warp 1 (one lane) : TMEM allocation + MMA issuer: tcgen05.mma.kind::tf32, 128 x BN x 8,
//                       3 per K step for 3xTF32 (Ahi·Bhi + Ahi·Blo + Alo·Bhi, ~fp32
//                       accuracy) or 1 for 1xTF32; tcgen05.commit frees the stage.
//   warps 2..5        : epilogue: tcgen05.ld of their TMEM lane quarter -> global (float4).
// Operand layouts in shared memory (both supported by the MMA, checked by
// tools/mn_probe.cu):
//   K-major  (operand contiguous along K):  one TMA box {32 k, rows}; 8-row x 128-byte
//            swizzle atoms, SBO = 1024 B; a K = 8 step advances the start by 32 B.
//   MN-major (operand contiguous along M/N, i.e. a transposed operand): boxes {32 mn, 32 k}
//            of 4 KB side by side (LBO = 4096 B) in the SW128_32B layout, the only one tf32
//            allows for MN-major (TMA SWIZZLE_128B_ATOM_32B; 4 k-rows x 128 B atoms, SBO =
//            512 B); a K = 8 step is 8 rows = 1024 B.
// The slot (plan) index is the third tensor-map dimension; per-slot M or K comes from
// device scalars.  Rows of a slot beyond its K are zero in the producers' buffers, so the
// contraction over a slot's rows needs no masking; rows beyond M are masked at the store.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "gcn.cuh"
#include "prof.h"
#include "sampler.cuh"
#include "skg_internal.h"

namespace skg {

namespace tc {

constexpr int BM = 128;
constexpr int BK = 32;         // K elements per stage (4 MMAs of K = 8)
constexpr int NTHREADS = 192;  // TMA warp, MMA warp, 4 epilogue warps

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// layout: 2 = SWIZZLE_128B (K-major), 1 = SWIZZLE_128B_BASE32B (MN-major tf32)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
  d |= (uint64_t)layout << 61;
  return d;
}

__host__ __device__ constexpr uint32_t make_idesc(int M, int N, bool a_mn, bool b_mn) {
  // c_format F32 (bit 4), a/b format TF32 (=2 at bits 7, 10), a/b major (bits 15/16,
  // 1 = MN-major), n_dim = N >> 3 at bit 17, m_dim = M >> 4 at bit 24
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
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
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes));
}

__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma4(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                     uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
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

template <int BN, int MODE>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 4, B_BYTES = BN * BK * 4;
  static constexpr int PARTS = MODE == 3 ? 2 : 1;
  static constexpr int STAGE = (A_BYTES + B_BYTES) * PARTS;
  static constexpr int STAGES_FIT = (200 * 1024) / STAGE;
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE + 1024;  // + 1 KB alignment slack
};

}  // namespace tc

struct TcMaps {
  CUtensorMap a_hi, a_lo, b_hi, b_lo;
  CUtensorMap c;  // output boxes {32 columns, 128 rows, 1 block} for the TMA-store epilogue
  int c_tma;      // 1: the epilogue stages the tile in shared memory and stores it by TMA
  int early;      // chunks whose TMA loads are issued before the setup sync (k_gemm_tc; <= STAGES)
  int a_blk, b_blk;  // 1: the MN-major operand's 32-wide blocks come in one 4D box (k_gemm_tc)
};

// debug timeline of CTA (0, 0, 0) (globaltimer ns): [0] start, [1] after setup,
// [2 + kc] stage kc full at the MMA warp, [34 + kc] TMA kc issued, [66] accumulator done
// at the epilogue, [67] epilogue end (kc < 32); tools/gemm_trace.py
__device__ unsigned long long g_tc_trace[68];
__device__ int g_tc_trace_on;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// C_z = op(A_z) op(B_z) (+ C_z) on tensor cores; op(A) M x K, op(B) K x N.
// TA: A stored K x M (contiguous along M); TB: B stored N x K (contiguous along K).
template <bool TA, bool TB, int BN, int MODE>
__global__ void __launch_bounds__(tc::NTHREADS, 1)
    k_gemm_tc(const __grid_constant__ TcMaps maps, int Mfix, int N, int Kfix,
              const int32_t* const* dM, const int32_t* const* dK, int a_slots, int b_slots,
              Act<float> C, int accumulate, int ks) {
  using namespace tc;
  using CF = Cfg<BN, MODE>;
  constexpr bool SPLIT = MODE == 3;
  constexpr int STAGES = CF::STAGES;
  constexpr int TCOLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  constexpr bool A_MN = TA, B_MN = !TB;
  static_assert(STAGES * CF::STAGE >= (BN / 32) * BM * 128, "the TMA-store epilogue stages the tile in the ring");
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES], done_bar;
  __shared__ uint32_t tmem_base;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  const bool tr = g_tc_trace_on && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
  if (tr && threadIdx.x == 0) g_tc_trace[0] = gtimer();
  const int zc = blockIdx.z;  // output block
  const int z = zc / ks, kz = zc - z * ks;
  const int M = dM ? *dM[z] : Mfix;
  const int K = dK ? *dK[z] : Kfix;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= M) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk_all = K > 0 ? (K + BK - 1) / BK : 0;
  const int kc0 = (int)((long long)nk_all * kz / ks);  // this CTA's run of K chunks
  const int nk = (int)((long long)nk_all * (kz + 1) / ks) - kc0;

  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "n"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // under PDL the CTA may start while the previous grid of the stream drains: TMEM is
  // allocated above, every global access waits here
  SKG_PDL_WAIT();
  const int za = a_slots > 1 ? z : 0, zb = b_slots > 1 ? z : 0;
  // TMA loads of K chunk kc into its ring stage (the producer thread only)
  auto load_stage = [&](int kc) {
    const int s = kc % STAGES;
    uint8_t* st = smem + s * CF::STAGE;
    mbar_expect_tx(&full_bar[s], (uint32_t)CF::STAGE);
    if (tr && kc < 32) g_tc_trace[34 + kc] = gtimer();
    const int k0 = (kc0 + kc) * BK;
#pragma unroll
    for (int part = 0; part < CF::PARTS; ++part) {
      uint8_t* sa = st + part * (CF::A_BYTES + CF::B_BYTES);
      uint8_t* sb = sa + CF::A_BYTES;
      const CUtensorMap* ma = part ? &maps.a_lo : &maps.a_hi;
      const CUtensorMap* mb = part ? &maps.b_lo : &maps.b_hi;
      if (A_MN && maps.a_blk) {
        tma4(sa, ma, 0, k0, m0 / 32, za, &full_bar[s]);  // BM / 32 blocks of {32 mn, 32 k}, 4 KB apart
      } else if (A_MN) {
#pragma unroll
        for (int i = 0; i < BM / 32; ++i) tma3(sa + i * 4096, ma, m0 + 32 * i, k0, za, &full_bar[s]);
      } else {
        tma3(sa, ma, k0, m0, za, &full_bar[s]);
      }
      if (B_MN && maps.b_blk) {
        tma4(sb, mb, 0, k0, n0 / 32, zb, &full_bar[s]);
      } else if (B_MN) {
#pragma unroll
        for (int i = 0; i < BN / 32; ++i) tma3(sb + i * 4096, mb, n0 + 32 * i, k0, zb, &full_bar[s]);
      } else {
        tma3(sb, mb, k0, n0, zb, &full_bar[s]);
      }
    }
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);   // producer's expect_tx arrival (+ TMA bytes)
      mbar_init(&empty_bar[s], 1);  // tcgen05.commit
    }
    mbar_init(&done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
    // the first chunk's loads fly while TMEM is allocated and the CTA synchronises
    for (int kc = 0; kc < maps.early && kc < nk && kc < STAGES; ++kc) load_stage(kc);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (tr && threadIdx.x == 0) g_tc_trace[1] = gtimer();

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      for (int kc = min(maps.early, STAGES); kc < nk; ++kc) {
        const int s = kc % STAGES;
        if (kc >= STAGES) mbar_wait(&empty_bar[s], (uint32_t)(((kc / STAGES) - 1) & 1));
        load_stage(kc);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc(BM, BN, A_MN, B_MN);
      // K-major: SW128 atoms of 8 rows x 128 B (SBO 1024), K step = 32 B inside the atom.
      // MN-major (tf32 allows only SW128_32B): atoms of 4 k-rows x 128 B (SBO 512), 32-wide
      // MN blocks 4 KB apart (LBO), K step = 8 rows = 1024 B.
      constexpr uint32_t A_STEP = A_MN ? 1024 : 32, B_STEP = B_MN ? 1024 : 32;
      constexpr uint32_t A_LBO = A_MN ? 4096 : 16, B_LBO = B_MN ? 4096 : 16;
      constexpr uint32_t A_SBO = A_MN ? 512 : 1024, B_SBO = B_MN ? 512 : 1024;
      constexpr uint32_t A_LAY = A_MN ? 1 : 2, B_LAY = B_MN ? 1 : 2;
      for (int kc = 0; kc < nk; ++kc) {
        const int s = kc % STAGES;
        mbar_wait(&full_bar[s], (uint32_t)((kc / STAGES) & 1));
        if (tr && kc < 32) g_tc_trace[2 + kc] = gtimer();
        asm volatile("tcgen05.fence::after_thread_sync;");
        uint8_t* st = smem + s * CF::STAGE;
        const uint32_t a_hi = smem_u32(st), b_hi = a_hi + CF::A_BYTES;
        const uint32_t a_lo = b_hi + CF::B_BYTES, b_lo = a_lo + CF::A_BYTES;
#pragma unroll
        for (int ks = 0; ks < BK / 8; ++ks) {
          const uint64_t ah = make_desc(a_hi + ks * A_STEP, A_LBO, A_SBO, A_LAY);
          const uint64_t bh = make_desc(b_hi + ks * B_STEP, B_LBO, B_SBO, B_LAY);
          mma_tf32(tmem, ah, bh, idesc, (kc > 0 || ks > 0) ? 1u : 0u);
          if (SPLIT) {
            mma_tf32(tmem, ah, make_desc(b_lo + ks * B_STEP, B_LBO, B_SBO, B_LAY), idesc, 1u);
            mma_tf32(tmem, make_desc(a_lo + ks * A_STEP, A_LBO, A_SBO, A_LAY), bh, idesc, 1u);
          }
        }
        mma_commit(&empty_bar[s]);  // stage s may be refilled once these MMAs complete
      }
      mma_commit(&done_bar);  // accumulator complete (arrives at once when nk == 0)
    }
    __syncwarp();
  } else {
    // ---------------- epilogue: TMEM lane quarter (warp % 4), all BN columns
    mbar_wait(&done_bar, 0u);
    if (threadIdx.x == 64) SKG_PDL_TRIGGER();  // the next grid may launch during the epilogue
    if (tr && threadIdx.x == 64) g_tc_trace[66] = gtimer();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int lg = warp & 3;
    const int row = m0 + lg * 32 + lane;
    const uint32_t taddr_row = tmem + ((uint32_t)(lg * 32) << 16);
    float* __restrict__ c = C.at(zc);
    const bool vecC = (C.ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(c) & 15) == 0);
    const bool empty_k = nk == 0;  // no MMA ran: the product is zero
    if (maps.c_tma) {
      // The stage ring is idle (every MMA has completed), so each 32-column box of the tile
      // is staged in it in the SWIZZLE_128B layout of the output map (16-byte chunk q of tile
      // row r at chunk q ^ (r & 7)) and stored by one TMA tensor store while the next box is
      // read from TMEM: whole 128-byte row segments leave the SM instead of a 16-byte store
      // per row and instruction (probe: 1.35 vs 2.57 us for a 128 x 128 tile).  Rows past the
      // block's M are written as zero (their A rows are zero, and no later GEMM contracts
      // over an output's rows); the map clips rows past the launch's M and columns past N.
      const int rl = lg * 32 + lane;
      const bool live = row < M && !empty_k;
#pragma unroll 1
      for (int b = 0; b < BN / 32 && n0 + 32 * b < N; ++b) {
        uint32_t v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr_row + 32 * b));
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
              "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(taddr_row + 32 * b + 16));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        uint8_t* box = smem + b * (BM * 128);
        uint8_t* srow = box + rl * 128;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint4 o = live ? make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]) : make_uint4(0, 0, 0, 0);
          *reinterpret_cast<uint4*>(srow + ((q ^ (rl & 7)) * 16)) = o;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 64) {
          asm volatile(
              "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(&maps.c),
              "r"(n0 + 32 * b), "r"(m0), "r"(zc), "r"(smem_u32(box))
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      // the ring must outlive the TMA's reads of it
      if (threadIdx.x == 64) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    } else {
#pragma unroll 1
    for (int cb = 0; cb < BN && n0 + cb < N; cb += 16) {
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
        for (int j4 = 0; j4 < 16; j4 += 4) {
          const int col = n0 + cb + j4;
          float o[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) o[e] = empty_k ? 0.f : __uint_as_float(v[j4 + e]);
          if (vecC && col + 3 < N) {
            float4* p4 = reinterpret_cast<float4*>(crow + col);
            float4 r4 = make_float4(o[0], o[1], o[2], o[3]);
            if (accumulate) {
              const float4 cur = *p4;
              r4.x += cur.x; r4.y += cur.y; r4.z += cur.z; r4.w += cur.w;
            }
            *p4 = r4;
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (col + e < N) crow[col + e] = accumulate ? crow[col + e] + o[e] : o[e];
          }
        }
      }
    }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tr && threadIdx.x == 64) g_tc_trace[67] = gtimer();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS));
}

// Persistent variant for multi-wave grids (GraphSAINT's 36K-row GEMMs): one CTA per SM
// walks the tiles blockIdx.x, + gridDim.x, ... (N tile fastest, so consecutive tiles reuse
// the A tile in L2).  The stage ring runs continuously across tiles (global chunk
// counters carry the phases), and two TMEM accumulators alternate between the MMA warp
// and the epilogue warps (acc_full / acc_empty), so a tile's epilogue and the next tile's
// first loads overlap the main loop instead of idling the SM.
template <bool TA, bool TB, int BN, int MODE>
__global__ void __launch_bounds__(tc::NTHREADS, 1)
    k_gemm_tc_p(const __grid_constant__ TcMaps maps, int Mfix, int N, int Kfix,
                const int32_t* const* dM, const int32_t* const* dK, int a_slots, int b_slots,
                Act<float> C, int accumulate, int ks, int n_tiles_n, int n_tiles_m, int n_tiles) {
  SKG_PDL_PROLOGUE();
  using namespace tc;
  using CF = Cfg<BN, MODE>;
  constexpr bool SPLIT = MODE == 3;
  constexpr int STAGES = CF::STAGES;
  constexpr int TCOLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  constexpr bool A_MN = TA, B_MN = !TB;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "n"(2 * TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);     // tcgen05.commit after a tile's last MMA
      mbar_init(&acc_empty[b], 128);  // every epilogue thread, after its TMEM reads
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  // tile -> (n0, m0, output block zc, slot z, K run); false when the tile is past the slot's M
  auto tile_at = [&](int tile, int& n0, int& m0, int& zc, int& z, int& kc0, int& nk, int& M) {
    const int nt = tile % n_tiles_n;
    const int rest = tile / n_tiles_n;
    const int mt = rest % n_tiles_m;
    zc = rest / n_tiles_m;
    z = zc / ks;
    const int kz = zc - z * ks;
    M = dM ? *dM[z] : Mfix;
    const int K = dK ? *dK[z] : Kfix;
    n0 = nt * BN;
    m0 = mt * BM;
    const int nk_all = K > 0 ? (K + BK - 1) / BK : 0;
    kc0 = (int)((long long)nk_all * kz / ks);
    nk = (int)((long long)nk_all * (kz + 1) / ks) - kc0;
    return m0 < M;
  };

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      uint32_t it = 0;  // chunks issued by this CTA so far
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        int n0, m0, zc, z, kc0, nk, M;
        if (!tile_at(tile, n0, m0, zc, z, kc0, nk, M)) continue;
        const int za = a_slots > 1 ? z : 0, zb = b_slots > 1 ? z : 0;
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait(&empty_bar[s], (uint32_t)(((it / STAGES) - 1) & 1));
          uint8_t* st = smem + s * CF::STAGE;
          mbar_expect_tx(&full_bar[s], (uint32_t)CF::STAGE);
          const int k0 = (kc0 + kc) * BK;
#pragma unroll
          for (int part = 0; part < CF::PARTS; ++part) {
            uint8_t* sa = st + part * (CF::A_BYTES + CF::B_BYTES);
            uint8_t* sb = sa + CF::A_BYTES;
            const CUtensorMap* ma = part ? &maps.a_lo : &maps.a_hi;
            const CUtensorMap* mb = part ? &maps.b_lo : &maps.b_hi;
            if (A_MN && maps.a_blk) {
              tma4(sa, ma, 0, k0, m0 / 32, za, &full_bar[s]);
            } else if (A_MN) {
#pragma unroll
              for (int i = 0; i < BM / 32; ++i) tma3(sa + i * 4096, ma, m0 + 32 * i, k0, za, &full_bar[s]);
            } else {
              tma3(sa, ma, k0, m0, za, &full_bar[s]);
            }
            if (B_MN && maps.b_blk) {
              tma4(sb, mb, 0, k0, n0 / 32, zb, &full_bar[s]);
            } else if (B_MN) {
#pragma unroll
              for (int i = 0; i < BN / 32; ++i) tma3(sb + i * 4096, mb, n0 + 32 * i, k0, zb, &full_bar[s]);
            } else {
              tma3(sb, mb, k0, n0, zb, &full_bar[s]);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc(BM, BN, A_MN, B_MN);
      constexpr uint32_t A_STEP = A_MN ? 1024 : 32, B_STEP = B_MN ? 1024 : 32;
      constexpr uint32_t A_LBO = A_MN ? 4096 : 16, B_LBO = B_MN ? 4096 : 16;
      constexpr uint32_t A_SBO = A_MN ? 512 : 1024, B_SBO = B_MN ? 512 : 1024;
      constexpr uint32_t A_LAY = A_MN ? 1 : 2, B_LAY = B_MN ? 1 : 2;
      uint32_t it = 0, lt = 0;  // chunks consumed, tiles computed by this CTA
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        int n0, m0, zc, z, kc0, nk, M;
        if (!tile_at(tile, n0, m0, zc, z, kc0, nk, M)) continue;
        const uint32_t b = lt & 1u, u = lt >> 1;
        if (u >= 1) mbar_wait(&acc_empty[b], (u - 1) & 1u);  // the epilogue drained buffer b
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t acc = tmem + b * TCOLS;
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full_bar[s], (uint32_t)((it / STAGES) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;");
          uint8_t* st = smem + s * CF::STAGE;
          const uint32_t a_hi = smem_u32(st), b_hi = a_hi + CF::A_BYTES;
          const uint32_t a_lo = b_hi + CF::B_BYTES, b_lo = a_lo + CF::A_BYTES;
#pragma unroll
          for (int k8 = 0; k8 < BK / 8; ++k8) {
            const uint64_t ah = make_desc(a_hi + k8 * A_STEP, A_LBO, A_SBO, A_LAY);
            const uint64_t bh = make_desc(b_hi + k8 * B_STEP, B_LBO, B_SBO, B_LAY);
            mma_tf32(acc, ah, bh, idesc, (kc > 0 || k8 > 0) ? 1u : 0u);
            if (SPLIT) {
              mma_tf32(acc, ah, make_desc(b_lo + k8 * B_STEP, B_LBO, B_SBO, B_LAY), idesc, 1u);
              mma_tf32(acc, make_desc(a_lo + k8 * A_STEP, A_LBO, A_SBO, A_LAY), bh, idesc, 1u);
            }
          }
          mma_commit(&empty_bar[s]);
        }
        mma_commit(&acc_full[b]);  // arrives at once when nk == 0 (no MMA ran)
        ++lt;
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue: TMEM lane quarter (warp % 4) of the tile's accumulator
    const int lg = warp & 3;
    uint32_t lt = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      int n0, m0, zc, z, kc0, nk, M;
      if (!tile_at(tile, n0, m0, zc, z, kc0, nk, M)) continue;
      const uint32_t b = lt & 1u, u = lt >> 1;
      mbar_wait(&acc_full[b], u & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int row = m0 + lg * 32 + lane;
      const uint32_t taddr_row = tmem + b * TCOLS + ((uint32_t)(lg * 32) << 16);
      float* __restrict__ c = C.at(zc);
      const bool vecC = (C.ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(c) & 15) == 0);
      const bool empty_k = nk == 0;
#pragma unroll 1
      for (int cb = 0; cb < BN && n0 + cb < N; cb += 16) {
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
          for (int j4 = 0; j4 < 16; j4 += 4) {
            const int col = n0 + cb + j4;
            float o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) o[e] = empty_k ? 0.f : __uint_as_float(v[j4 + e]);
            if (vecC && col + 3 < N) {
              float4* p4 = reinterpret_cast<float4*>(crow + col);
              float4 r4 = make_float4(o[0], o[1], o[2], o[3]);
              if (accumulate) {
                const float4 cur = *p4;
                r4.x += cur.x; r4.y += cur.y; r4.z += cur.z; r4.w += cur.w;
              }
              *p4 = r4;
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e)
                if (col + e < N) crow[col + e] = accumulate ? crow[col + e] + o[e] : o[e];
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      mbar_arrive(&acc_empty[b]);  // buffer b may take the next tile's accumulation
      ++lt;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * TCOLS));
}

// ------------------------------------------------------------------ tensor maps (cached)
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

struct MapKey {
  const void* base;
  int64_t inner, outer, slots, ld, stride;
  int64_t box_outer, mn;
  bool operator==(const MapKey& o) const { return memcmp(this, &o, sizeof(MapKey)) == 0; }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    const uint64_t* w = reinterpret_cast<const uint64_t*>(&k);
    uint64_t h = 1469598103934665603ull;
    for (size_t i = 0; i < sizeof(MapKey) / 8; ++i) h = (h ^ w[i]) * 1099511628211ull;
    return (size_t)h;
  }
};

std::mutex g_map_mu;
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

// 3D fp32 map {inner (contiguous), outer (row stride ld), slots (slot stride)}, box
// {32, box_outer, 1}, SWIZZLE_128B (K-major) or SWIZZLE_128B_ATOM_32B (MN-major), zero fill
// out of bounds
int get_map(const float* base, int64_t inner, int64_t outer, int64_t slots, int64_t ld, int64_t stride,
            int box_outer, int mn, CUtensorMap* out) {
  MapKey key;
  memset(&key, 0, sizeof(key));
  key.base = base;
  key.inner = inner;
  key.outer = outer;
  key.slots = slots;
  key.ld = ld;
  key.stride = stride;
  key.box_outer = box_outer;
  key.mn = mn;
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) {
      *out = it->second;
      return SKG_OK;
    }
  }
  auto fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return SKG_ERR_CUDA;
  }
  if ((ld * 4) % 16 || (reinterpret_cast<uintptr_t>(base) & 15) || (slots > 1 && (stride * 4) % 16)) {
    set_error("gemm operand not TMA-compatible (ld / base alignment)");
    return SKG_ERR_ARG;
  }
  CUtensorMap m;
  CUresult r;
  if (mn == 2) {
    // MN-major operand as 4D {32 mn, k rows, inner / 32 blocks, slots}, box {32, 32 k,
    // blk_count, 1}: one TMA lands blk_count {32 mn, 32 k} blocks 4 KB apart, the layout the
    // per-block boxes produce (inner must be a multiple of 32: no partial block to zero-fill)
    const int blk_count = (int)(box_outer >> 8), k_box = (int)(box_outer & 255);
    cuuint64_t dims[4] = {32, (cuuint64_t)outer, (cuuint64_t)(inner / 32), (cuuint64_t)std::max<int64_t>(slots, 1)};
    cuuint64_t strides[3] = {(cuuint64_t)ld * 4, 128, (cuuint64_t)std::max<int64_t>(stride, ld * outer) * 4};
    cuuint32_t box[4] = {32, (cuuint32_t)k_box, (cuuint32_t)blk_count, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)std::max<int64_t>(slots, 1)};
    cuuint64_t strides[2] = {(cuuint64_t)ld * 4, (cuuint64_t)std::max<int64_t>(stride, ld * outer) * 4};
    cuuint32_t box[3] = {32, (cuuint32_t)box_outer, 1};
    cuuint32_t es[3] = {1, 1, 1};
    r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, mn ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return SKG_ERR_CUDA;
  }
  std::lock_guard<std::mutex> lk(g_map_mu);
  if (g_maps.size() > 4096) g_maps.clear();
  g_maps[key] = m;
  *out = m;
  return SKG_OK;
}

// operand maps: K-major operands are boxed {32 k, rows}; MN-major {32 mn, 32 k}
// (blk: an MN-major operand whose extent is a multiple of 32 gets the 4D block map, one TMA
// per stage instead of rows_box / 32; *blk_out says which was built)
int op_maps(const TcOp& op, bool mn, int64_t mn_extent, int64_t k_extent, int rows_box, int n,
            bool split, CUtensorMap* hi, CUtensorMap* lo, bool blk = false, int* blk_out = nullptr) {
  const int64_t slots = op.stride ? n : 1;
  const int64_t inner = mn ? mn_extent : k_extent;
  if (blk_out) *blk_out = 0;
  if (mn && blk && mn_extent % 32 == 0) {
    const int bo = ((rows_box / 32) << 8) | tc::BK;
    if (get_map(op.hi, inner, op.rows_cap, slots, op.ld, op.stride, bo, 2, hi) == SKG_OK &&
        (!split || (op.lo && get_map(op.lo, inner, op.rows_cap, slots, op.ld, op.stride, bo, 2, lo) == SKG_OK))) {
      if (!split) *lo = *hi;
      if (blk_out) *blk_out = 1;
      return SKG_OK;
    }
  }
  const int box_outer = mn ? tc::BK : rows_box;
  int rc = get_map(op.hi, inner, op.rows_cap, slots, op.ld, op.stride, box_outer, mn ? 1 : 0, hi);
  if (rc) return rc;
  if (split) {
    if (!op.lo) {
      set_error("3xTF32 GEMM needs the lo operand");
      return SKG_ERR_ARG;
    }
    rc = get_map(op.lo, inner, op.rows_cap, slots, op.ld, op.stride, box_outer, mn ? 1 : 0, lo);
    if (rc) return rc;
  } else {
    *lo = *hi;
  }
  return SKG_OK;
}

}  // namespace

// GCN layer of the GEMM being launched (set by the training step; -1 elsewhere): launch
// names carry it ("k_gemm_tc<...>@l2") so per-kernel profiles can attribute flops
thread_local int g_gemm_layer = -1;

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <bool TA, bool TB, int BN, int MODE>
static int launch_tc(int n, int M, int N, int K, const int32_t* const* dM, const int32_t* const* dK,
                     const TcOp& A, const TcOp& B, Act<float> C, bool acc, cudaStream_t st, int ks) {
  using CF = tc::Cfg<BN, MODE>;
  TcMaps maps;
  // A: M x K (TA: stored K x M); B: K x N (TB: stored N x K)
  const int tn = (N + BN - 1) / BN, tm = (M + tc::BM - 1) / tc::BM;
  const long long tiles = (long long)tn * tm * n * ks;
  static const int persist = getenv("SKG_GEMM_PERSIST") ? atoi(getenv("SKG_GEMM_PERSIST")) : 1;
  const bool use_p = persist && tiles >= 3LL * sm_count();
  // MN-major operands in one 4D box per stage (SKG_GEMM_TMA4=0: per block; =2: not in the
  // persistent kernel)
  static const int tma4_on = getenv("SKG_GEMM_TMA4") ? atoi(getenv("SKG_GEMM_TMA4")) : 1;
  const bool blk = tma4_on == 1 || (tma4_on == 2 && !use_p);
  int rc = op_maps(A, TA, M, K, tc::BM, n, MODE == 3, &maps.a_hi, &maps.a_lo, blk, &maps.a_blk);
  if (rc) return rc;
  rc = op_maps(B, !TB, N, K, BN, n, MODE == 3, &maps.b_hi, &maps.b_lo, blk, &maps.b_blk);
  if (rc) return rc;
  maps.c_tma = 0;
  static const int early = getenv("SKG_GEMM_EARLY") ? atoi(getenv("SKG_GEMM_EARLY")) : 1;
  maps.early = early;
  const int as = A.stride ? n : 1, bs = B.stride ? n : 1;
  if (use_p) {
    // >= 3 waves (GraphSAINT's 36K-row GEMMs): persistent CTAs with double-buffered TMEM
    // accumulators.  Not for shorter grids: persistent CTAs hold every SM until the GEMM
    // ends, which starves the concurrent sampler streams (YouTube step: 1720 vs 1808 it/s
    // when its 256-tile dW went persistent)
    auto pk = k_gemm_tc_p<TA, TB, BN, MODE>;
    static bool pattr = false;
    if (!pattr) {
      cudaFuncSetAttribute(pk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM);
      pattr = true;
    }
    const int grid_p = (int)std::min<long long>(tiles, sm_count());
    static const std::string pname = "k_gemm_tc_p<" + std::to_string((int)TA) + "," + std::to_string((int)TB) + "," +
                                     std::to_string(BN) + "," + std::to_string(MODE) + ">";
    const std::string pn = g_gemm_layer >= 0 ? pname + "@l" + std::to_string(g_gemm_layer) : pname;
    launch_k(pn.c_str(), st, dim3(grid_p), dim3(tc::NTHREADS), CF::SMEM, pk, maps, M, N, K, dM, dK, as, bs, C,
             acc ? 1 : 0, ks, tn, tm, (int)tiles);
    return SKG_OK;
  }
  // TMA-store epilogue: plain (non-accumulating) stores into TMA-compatible outputs whose
  // blocks do not overlap (SKG_GEMM_TMA_STORE=0 keeps the per-row stores)
  static const int tma_store = getenv("SKG_GEMM_TMA_STORE") ? atoi(getenv("SKG_GEMM_TMA_STORE")) : 1;
  const int64_t nz = (int64_t)n * ks;
  if (tma_store && !acc && C.ld % 4 == 0 && (reinterpret_cast<uintptr_t>(C.base) & 15) == 0 &&
      (nz == 1 || (C.stride % 4 == 0 && C.stride >= C.ld * (int64_t)M)) &&
      get_map(C.base, N, M, nz, C.ld, nz == 1 ? 0 : C.stride, tc::BM, 0, &maps.c) == SKG_OK)
    maps.c_tma = 1;
  auto kern = k_gemm_tc<TA, TB, BN, MODE>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM);
    attr = true;
  }
  dim3 grid(tn, tm, n * ks);
  static const std::string kname = "k_gemm_tc<" + std::to_string((int)TA) + "," + std::to_string((int)TB) + "," +
                                   std::to_string(BN) + "," + std::to_string(MODE) + ">";
  const std::string kn = g_gemm_layer >= 0 ? kname + "@l" + std::to_string(g_gemm_layer) : kname;
  launch_k(kn.c_str(), st, dim3(grid), dim3(tc::NTHREADS), CF::SMEM, kern, maps, M, N, K, dM, dK, as, bs, C,
           acc ? 1 : 0, ks);
  return SKG_OK;
}

int g_bn_override = 0;      // debug / tuning: force the N tile (32, 64, 128, 256)
int g_ksplit_override = 0;  // debug / tuning: force the K split of split-K callers

// N tile.  The 3xTF32 main loop is bound by shared-memory bandwidth (tools/gemm_trace.py:
// one 128 x 64 x 32 stage per ~0.5 us = TMA write 48 KB + MMA operand reads 72 KB at
// ~128 B/clk), and a CTA holds its SM (~200 KB of stages) for its whole life, with ~2 us of
// fixed setup / first-load / epilogue time.  Inside the training step the GEMMs share the
// GPU with the sampler streams, so total SM time counts, not one GEMM's latency: measured
// on the Reddit-shaped step, BN = 128 everywhere gives 1358 it/s vs 1323 (BN = 64) and 1234
// (BN = 256: a 2-stage ring, and mostly padding on the 41-class layer); splitting K inside
// a slot (more, shorter CTAs) costs 1.5 %.  BN = 256 is kept for the wide (N >= 512)
// multi-wave GraphSAINT GEMMs, where it halved their time.
static int plan_bn(int n, int M, int N) {
  if (N <= 32) return 32;
  if (N <= 64) return 64;
  const long long tiles256 = (long long)((M + tc::BM - 1) / tc::BM) * ((N + 255) / 256) * std::max(n, 1);
  if (N >= 512 && tiles256 >= sm_count()) return 256;
  return 128;
}

// Long contractions (>= 64 K chunks per slot, e.g. GraphSAINT's dW over 4500 subgraph
// rows) with a grid under one wave: choose (BN, K split) jointly by the shared-memory
// traffic model, waves x (chunks per tile + 2) x (128 + BN).  GraphSAINT dW (8 slots of
// 512 x 512 x 4500): BN 256 with a 2-way split, one wave of 128 CTAs, instead of 128 CTAs
// walking all 141 chunks.  Short contractions keep ks = 1 (measured faster in the LADIES step).
constexpr int kLongK = 64 * tc::BK;
struct LongKPlan {
  int bn, ks;
};
static LongKPlan plan_long_k(int n, int M, int N, int K, int ks_fixed) {
  const long long sms = sm_count();
  const long long mt = (M + tc::BM - 1) / tc::BM;
  const long long nk = (K + tc::BK - 1) / tc::BK;
  LongKPlan best{128, 1};
  double best_cost = 1e300;
  for (int bn : {128, 256}) {
    if (bn == 256 && N < 256) continue;
    const int ks_lo = ks_fixed > 0 ? ks_fixed : 1, ks_hi = ks_fixed > 0 ? ks_fixed : kMaxKSplit;
    for (int ks = ks_lo; ks <= ks_hi; ++ks) {
      const long long tiles = mt * ((N + bn - 1) / bn) * std::max(n, 1) * ks;
      const long long waves = (tiles + sms - 1) / sms;
      const double cost = (double)waves * ((nk + ks - 1) / ks + 2) * (128 + bn);
      if (cost < best_cost * 0.97) {  // a split must win clearly (it adds a reduction)
        best_cost = cost;
        best = LongKPlan{bn, ks};
      }
    }
  }
  return best;
}

int gemm_tc_ksplit(int n, int M, int N, int K) {
  static const int env = getenv("SKG_GEMM_KSPLIT") ? atoi(getenv("SKG_GEMM_KSPLIT")) : 0;
  const int force = g_ksplit_override ? g_ksplit_override : env;
  if (force) return std::max(1, std::min(force, kMaxKSplit));
  if (K >= kLongK && N > 64) return plan_long_k(n, M, N, K, 0).ks;
  return 1;
}

template <bool TA, bool TB, int MODE>
static int dispatch_bn(int n, int M, int N, int K, const int32_t* const* dM, const int32_t* const* dM2,
                       const TcOp& A, const TcOp& B, Act<float> C, bool acc, cudaStream_t st, int ks) {
  const int32_t* const* dK = dM2;
  static const int env_bn = getenv("SKG_GEMM_BN") ? atoi(getenv("SKG_GEMM_BN")) : 0;
  const int force = g_bn_override ? g_bn_override : env_bn;
  // long contractions: the N tile for the K split actually used (1 for callers without
  // partial outputs; a forward GEMM must not take the tile of a split plan)
  const int bn = force ? force : (K >= kLongK && N > 64) ? plan_long_k(n, M, N, K, ks).bn : plan_bn(n, M, N);
  if (bn == 32) return launch_tc<TA, TB, 32, MODE>(n, M, N, K, dM, dK, A, B, C, acc, st, ks);
  if (bn == 128) return launch_tc<TA, TB, 128, MODE>(n, M, N, K, dM, dK, A, B, C, acc, st, ks);
  if (bn == 256) return launch_tc<TA, TB, 256, MODE>(n, M, N, K, dM, dK, A, B, C, acc, st, ks);
  return launch_tc<TA, TB, 64, MODE>(n, M, N, K, dM, dK, A, B, C, acc, st, ks);
}

int gemm_tc(int mode, bool ta, bool tb, int n, int M, int N, int K, const int32_t* const* dM,
            const int32_t* const* dK, const TcOp& A, const TcOp& B, Act<float> C, bool acc,
            cudaStream_t st, int ks) {
  if (M <= 0 || N <= 0 || n <= 0) return SKG_OK;
  ks = std::max(1, std::min(ks, kMaxKSplit));
#define TC_CASE(TA_, TB_)                                                                        \
  if (ta == TA_ && tb == TB_)                                                                    \
    return mode == 3 ? dispatch_bn<TA_, TB_, 3>(n, M, N, K, dM, dK, A, B, C, acc, st, ks)        \
                     : dispatch_bn<TA_, TB_, 1>(n, M, N, K, dM, dK, A, B, C, acc, st, ks);
  TC_CASE(false, false)
  TC_CASE(true, false)
  TC_CASE(false, true)
  TC_CASE(true, true)
#undef TC_CASE
  return SKG_OK;
}

// ------------------------------------------------------------------ TF32 splits
// hi = tf32(x), lo = tf32(x - hi) of a rows x cols matrix (row stride ld_in) into padded
// outputs (row stride ld_out); padding columns are written as zero
__global__ void k_split_tf32(const float* __restrict__ in, int64_t ld_in, int64_t rows, int64_t cols,
                             float* __restrict__ hi, float* __restrict__ lo, int64_t ld_out) {
  SKG_PDL_PROLOGUE();
  const int64_t total = rows * ld_out;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / ld_out, c = i % ld_out;
    const float x = c < cols ? in[r * ld_in + c] : 0.f;
    const float h = tf32_rna(x);
    hi[i] = h;
    if (lo) lo[i] = tf32_rna(x - h);
  }
}

void split_tf32(const float* in, int64_t ld_in, int64_t rows, int64_t cols, float* hi, float* lo,
                int64_t ld_out, cudaStream_t st) {
  const int64_t total = rows * ld_out;
  if (total <= 0) return;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 1184);
  launch_k("k_split_tf32", st, dim3(blocks), dim3(256), 0, k_split_tf32, in, ld_in, rows, cols, hi, lo, ld_out);
}

// all layers' weights in one launch: W_l (d_l x d_{l+1}, dense rows) -> padded hi / lo
__global__ void k_split_weights(WSplitTable t) {
  SKG_PDL_PROLOGUE();
  for (int l = 0; l < t.L; ++l) {
    const int64_t rows = t.rows[l], cols = t.cols[l], ldo = t.ld_out[l];
    const float* in = t.w[l];
    float* hi = t.hi[l];
    float* lo = t.lo[l];
    const int64_t total = rows * ldo;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t r = i / ldo, c = i % ldo;
      const float x = c < cols ? in[r * cols + c] : 0.f;
      const float h = tf32_rna(x);
      hi[i] = h;
      if (lo) lo[i] = tf32_rna(x - h);
    }
  }
}

void split_weights(const WSplitTable& t, cudaStream_t st) {
  launch_k("k_split_weights", st, dim3(296), dim3(256), 0, k_split_weights, t);
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
  int rc = SKG_OK;
  if (mode == 0) {
    Act<float> a{dA, 0, ta ? M : K}, b{dB, 0, tb ? K : N}, c{dC, 0, N};
    gemm_simt<float>(ta, tb, 1, M, N, K, nullptr, nullptr, a, b, c, false, 0);
  } else {
    // stored shapes: A (TA ? K x M : M x K), B (TB ? N x K : K x N); split into padded buffers
    const int64_t ar = ta ? K : M, ac = ta ? M : K, br = tb ? N : K, bc = tb ? K : N;
    const int64_t lda = round4(ac), ldb = round4(bc);
    float *ah, *al, *bh, *bl;
    cudaMalloc(&ah, std::max<int64_t>(ar * lda, 1) * 4);
    cudaMalloc(&al, std::max<int64_t>(ar * lda, 1) * 4);
    cudaMalloc(&bh, std::max<int64_t>(br * ldb, 1) * 4);
    cudaMalloc(&bl, std::max<int64_t>(br * ldb, 1) * 4);
    split_tf32(dA, ac, ar, ac, ah, mode == 3 ? al : nullptr, lda, 0);
    split_tf32(dB, bc, br, bc, bh, mode == 3 ? bl : nullptr, ldb, 0);
    TcOp A{ah, mode == 3 ? al : nullptr, lda, 0, ar}, B{bh, mode == 3 ? bl : nullptr, ldb, 0, br};
    Act<float> c{dC, 0, N};
    rc = gemm_tc(mode, ta, tb, 1, M, N, K, nullptr, nullptr, A, B, c, false, 0);
    cudaDeviceSynchronize();
    cudaFree(ah);
    cudaFree(al);
    cudaFree(bh);
    cudaFree(bl);
  }
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hC, dC, nc * 4, cudaMemcpyDeviceToHost);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dC);
  if (rc) return rc;
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

// debug: time `iters` GEMMs on device-resident (zero) split operands, M x K by K x N
extern "C" int skg_debug_gemm_bn(int bn) {
  skg::g_bn_override = bn;
  return 0;
}

// debug / tuning: force the per-slot K split of the dW GEMMs (0 = planned)
extern "C" int skg_debug_gemm_ksplit(int ks) {
  skg::g_ksplit_override = ks;
  return 0;
}

// debug: timeline of the next GEMMs' CTA (0, 0, 0); on = 1 arms, out (68 entries) reads
extern "C" int skg_debug_tc_trace(int on, unsigned long long* out) {
  cudaMemcpyToSymbol(skg::g_tc_trace_on, &on, sizeof(int));
  if (out) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, skg::g_tc_trace, sizeof(unsigned long long) * 68);
  }
  return 0;
}

extern "C" int skg_debug_gemm_timed(int mode, int ta, int tb, int M, int N, int K, int iters,
                                    float* us_out) {
  using namespace skg;
  const int64_t ar = ta ? K : M, ac = ta ? M : K, br = tb ? N : K, bc = tb ? K : N;
  const int64_t lda = round4(ac), ldb = round4(bc);
  float *ah, *al, *bh, *bl, *dC;
  cudaMalloc(&ah, ar * lda * 4);
  cudaMalloc(&al, ar * lda * 4);
  cudaMalloc(&bh, br * ldb * 4);
  cudaMalloc(&bl, br * ldb * 4);
  cudaMalloc(&dC, (size_t)M * N * 4);
  cudaMemset(ah, 0, ar * lda * 4);
  cudaMemset(al, 0, ar * lda * 4);
  cudaMemset(bh, 0, br * ldb * 4);
  cudaMemset(bl, 0, br * ldb * 4);
  TcOp A{ah, al, lda, 0, ar}, B{bh, bl, ldb, 0, br};
  Act<float> c{dC, 0, N};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int rc = 0;
  for (int i = 0; i < 3; ++i) rc |= gemm_tc(mode, ta, tb, 1, M, N, K, nullptr, nullptr, A, B, c, false, 0);
  cudaEventRecord(e0, 0);
  for (int i = 0; i < iters; ++i) gemm_tc(mode, ta, tb, 1, M, N, K, nullptr, nullptr, A, B, c, false, 0);
  cudaEventRecord(e1, 0);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  *us_out = ms * 1000.f / iters;
  cudaError_t e = cudaDeviceSynchronize();
  cudaFree(ah);
  cudaFree(al);
  cudaFree(bh);
  cudaFree(bl);
  cudaFree(dC);
  return (rc || e != cudaSuccess) ? -1 : 0;
}
