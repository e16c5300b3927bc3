// tcgen05 (5th-gen tensor core) TF32 GEMM for sm_100a with fused epilogues:
// the dense gate projections of the GILR / GILR-LSTM layers (layers.hpp:78-375).
//
//   C[M][N] (row-major fp32)  =  sum_k A(m,k) * B(n,k)   (+ fused epilogue)
//
// A is given K-major ([M][K] storage) or MN-major ([K][M] storage); same for
// B.  That covers every product of the layer without transposes:
//   x * W^T        (forward projections)          A K-major, B K-major
//   dpre * W       (input gradients)              A K-major, B MN-major
//   dpre^T * x     (weight gradients, split-K)    A MN-major, B MN-major
// The K range may be the concatenation of two (A, B) operand pairs (the gate
// projection [x | htil_{t-1}] * [V | U]^T in one pass).
//
// Structure (one 128 x BN output tile per CTA, 8 warps):
//   warp 0      TMA producer: 128B-swizzled 2-D boxes into a STAGES ring
//               (mbarrier complete_tx);
//   warp 1      allocates TMEM (BN fp32 columns) and a single elected thread
//               issues tcgen05.mma.cta_group::1.kind::tf32 (M=128, N=BN,
//               K=8 per instruction), committing each stage back to the
//               producer and the finished accumulator to the epilogue;
//   warps 4-7   epilogue: tcgen05.ld 32 lanes x 32 columns at a time, apply
//               the fused epilogue, store.
#pragma once

#include <cstdint>

#include "tma_util.cuh"

namespace linrec_dev {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 elements per k-block = one 128-byte swizzle row

// ---- tcgen05 wrappers -------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on an mbarrier once all previously issued tcgen05.mma have completed.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// 32 lanes x 32 consecutive fp32 columns; thread i of the warp gets lane
// (base lane + i), columns [col, col+32).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor (cute::UMMA::SmemDescriptor layout):
// start[0,14) LBO[16,30) SBO[32,46) version[46,48)=1 base[49,52) layout[61,64)
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm_100)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

// UMMA instruction descriptor, kind::tf32, fp32 accumulate
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4)                      // c_format F32
         | (2u << 7)                    // a_format TF32
         | (2u << 10)                   // b_format TF32
         | ((a_mn ? 1u : 0u) << 15)     // a_major
         | ((b_mn ? 1u : 0u) << 16)     // b_major
         | ((uint32_t)(N >> 3) << 17)   // n_dim
         | ((uint32_t)(M >> 4) << 24);  // m_dim
}

// Operand tile geometry in shared memory for ROWS (M or N) x BK:
//   K-major:  TMA box {BK=32 elems (128 B), ROWS} -> [ROWS][128 B] 8-row
//             swizzle atoms; SBO = 1024 B; a k-step of 8 = +32 B
//   MN-major: ROWS/32 boxes {32 elems (128 B), BK rows} -> [BK][128 B] per
//             32-wide MN slab, slabs LBO = BK*128 B apart; SBO = 1024 B;
//             a k-step of 8 = +1024 B
template <bool MN, int ROWS>
struct TileGeom {
  static constexpr int BYTES = ROWS * BK * 4;
  static constexpr uint32_t LBO = MN ? BK * 128 : 16;
  static constexpr uint32_t SBO = 1024;
  static constexpr uint32_t KSTEP = MN ? 1024 : 32;  // bytes per 8-element k-step
  static constexpr int NBOX = MN ? ROWS / 32 : 1;
  static constexpr int BOX_BYTES = MN ? BK * 128 : BYTES;
};

struct GemmParams {
  int M, N;          // output rows / columns
  int kb1, kb;       // k-blocks from the first operand pair / in total (per split)
  int ldc;
  int k_splits;      // grid.z
  int kb_total;      // k-blocks over all splits
  float* C;          // output (split-K: partials at C + z * M * ldc)
  int mode;          // 0 store, 1 accumulate, 2 split-K partial
  // fused epilogue operands
  const float* bias;
  float* o0;
  float* o1;
  float* o2;
  float* o3;
  int ldo;           // leading dim of o0..o2 ([M][ldo])
};

enum Epi : int { kEpiPlain = 0, kEpiGilr = 1, kEpiGates = 2 };

template <bool A_MN, bool B_MN, int BN, int STAGES>
struct GemmCfg {
  using GA = TileGeom<A_MN, BM>;
  using GB = TileGeom<B_MN, BN>;
  static constexpr int STAGE_BYTES = GA::BYTES + GB::BYTES;
  static constexpr int OFF_BAR = STAGES * STAGE_BYTES;
  static constexpr int SMEM = OFF_BAR + (2 * STAGES + 1) * 8 + 16 + 1024;  // + alignment slack
  static constexpr uint32_t IDESC = idesc_tf32(BM, BN, A_MN, B_MN);
};

template <bool A_MN, bool B_MN, int BN, int STAGES, int EPI>
__global__ void __launch_bounds__(256, 1)
k_gemm_tf32(const __grid_constant__ CUtensorMap ta1, const __grid_constant__ CUtensorMap tb1,
            const __grid_constant__ CUtensorMap ta2, const __grid_constant__ CUtensorMap tb2, const GemmParams p) {
  using Cfg = GemmCfg<A_MN, B_MN, BN, STAGES>;
  using GA = typename Cfg::GA;
  using GB = typename Cfg::GB;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* empty = full + STAGES;
  uint64_t* accum = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int kb_begin = blockIdx.z * p.kb;
  const int kb_end = min(kb_begin + p.kb, p.kb_total);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accum, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {  // ---------------------------------- TMA producer
    prefetch_tmap(&ta1);
    prefetch_tmap(&tb1);
    const uint64_t pol = policy_evict_first();
    for (int kb = kb_begin, i = 0; kb < kb_end; ++kb, ++i) {
      const int s = i % STAGES;
      if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) + 1) & 1);
      const bool second = kb >= p.kb1;
      const CUtensorMap* ta = second ? &ta2 : &ta1;
      const CUtensorMap* tb = second ? &tb2 : &tb1;
      const int k0 = (second ? kb - p.kb1 : kb) * BK;
      unsigned char* sa = smem + s * Cfg::STAGE_BYTES;
      unsigned char* sb = sa + GA::BYTES;
      mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
      if (A_MN) {
#pragma unroll
        for (int j = 0; j < GA::NBOX; ++j) tma_load_2d(sa + j * GA::BOX_BYTES, ta, m0 + 32 * j, k0, &full[s], pol);
      } else {
        tma_load_2d(sa, ta, k0, m0, &full[s], pol);
      }
      if (B_MN) {
#pragma unroll
        for (int j = 0; j < GB::NBOX; ++j) tma_load_2d(sb + j * GB::BOX_BYTES, tb, n0 + 32 * j, k0, &full[s], pol);
      } else {
        tma_load_2d(sb, tb, k0, n0, &full[s], pol);
      }
    }
  } else if (warp == 1 && lane == 0) {  // ------------------------- MMA issuer
    for (int kb = kb_begin, i = 0; kb < kb_end; ++kb, ++i) {
      const int s = i % STAGES;
      mbar_wait(&full[s], (i / STAGES) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * Cfg::STAGE_BYTES);
      const uint32_t sb = sa + GA::BYTES;
#pragma unroll
      for (int kk = 0; kk < BK / 8; ++kk) {
        const uint64_t ad = smem_desc_sw128(sa + kk * GA::KSTEP, GA::LBO, GA::SBO);
        const uint64_t bd = smem_desc_sw128(sb + kk * GB::KSTEP, GB::LBO, GB::SBO);
        mma_tf32(tmem, ad, bd, Cfg::IDESC, (i > 0 || kk > 0) ? 1u : 0u);
      }
      mma_commit(&empty[s]);  // stage free once these MMAs have read it
    }
    mma_commit(accum);
  } else if (warp >= 4) {  // ---------------------------------------- epilogue
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int row = m0 + q * 32 + lane;
    mbar_wait(accum, 0);
    tc_fence_after();
    const bool empty_k = kb_end <= kb_begin;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      float v[32];
      if (!empty_k) tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, v);
      else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.f;
      }
      if (row >= p.M) continue;
      const int col = n0 + c0;
      if (EPI == kEpiPlain) {
        float* dst = p.C + (size_t)(p.mode == 2 ? blockIdx.z : 0) * p.M * p.ldc + (size_t)row * p.ldc + col;
        const bool full_cols = col + 32 <= p.N;
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          if (full_cols || col + i < p.N) {
            float4 w = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
            if (p.mode == 1) {
              const float4 o = *reinterpret_cast<const float4*>(dst + i);
              w.x += o.x; w.y += o.y; w.z += o.z; w.w += o.w;
            }
            if (full_cols || col + i + 3 < p.N) *reinterpret_cast<float4*>(dst + i) = w;
            else {
              const float* ww = &w.x;
              for (int e = 0; e < 4 && col + i + e < p.N; ++e) dst[i + e] = ww[e];
            }
          }
        }
      } else if (EPI == kEpiGilr) {
        // interleaved columns (2j, 2j+1) = (g_pre, i_pre) of hidden unit j:
        // g = sigmoid, i = tanh, impulse = (1 - g) * i  (layers.hpp:88-92)
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const int j = (col + i) >> 1;
          const float g = 1.f / (1.f + expf(-(v[i] + p.bias[col + i])));
          const float z = tanhf(v[i + 1] + p.bias[col + i + 1]);
          p.o0[(size_t)row * p.ldo + j] = g;
          p.o1[(size_t)row * p.ldo + j] = z;
          p.o2[(size_t)row * p.ldo + j] = (1.f - g) * z;
        }
      } else {  // kEpiGates
        // interleaved columns (4j .. 4j+3) = (f, i, o, z) pre-activations:
        // f, i, o = sigmoid, z = tanh (layers.hpp:263, activate_gates :226-236);
        // outputs f, i*z, o and the activated gates (cache, interleaved)
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const int j = (col + i) >> 2;
          const float f = 1.f / (1.f + expf(-(v[i] + p.bias[col + i])));
          const float ig = 1.f / (1.f + expf(-(v[i + 1] + p.bias[col + i + 1])));
          const float o = 1.f / (1.f + expf(-(v[i + 2] + p.bias[col + i + 2])));
          const float z = tanhf(v[i + 3] + p.bias[col + i + 3]);
          p.o0[(size_t)row * p.ldo + j] = f;
          p.o1[(size_t)row * p.ldo + j] = ig * z;
          p.o2[(size_t)row * p.ldo + j] = o;
          *reinterpret_cast<float4*>(p.o3 + (size_t)row * 4 * p.ldo + 4 * j) = make_float4(f, ig, o, z);
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, BN);
  }
}

}  // namespace tc
}  // namespace linrec_dev
