// tcgen05 (5th-gen tensor core) GEMM for sm_100a with fused layer epilogues:
// the dense gate projections of the GILR / GILR-LSTM layers
// (layers.hpp:78-133, :245-375) and their gradients.
//
//   C[M][N] (row-major fp32)  =  sum_k A(m,k) * B(n,k)   (+ fused epilogue)
//
// A is given K-major ([M][K] storage) or MN-major ([K][M] storage); same for
// B.  That covers every product of the layers without transposes:
//   x * W^T        (forward projections)          A K-major, B K-major
//   dpre * W       (input gradients)              A K-major, B MN-major
//   dpre^T * x     (weight gradients, split-K)    A MN-major, B MN-major
// The K range may be the concatenation of two (A, B) operand pairs (the gate
// projection [x | htil_{t-1}] * [V | U]^T in one pass).  A K-major B may be
// "blocked": the BN rows of a tile are NB sub-boxes taken from NB row blocks
// of the weight (rows q*bstride + j0 ..), so the f/i/o/z (or g/i) rows of the
// same hidden units land in one tile and the epilogue sees every gate of a
// unit without any host-side weight permutation.
//
// Precision: kind::tf32 reads 10 mantissa bits of each operand.  With SPLIT3
// the kernel runs 3xTF32: two split warps write lo = v - tf32(v) of every
// staged A and B tile next to it and the MMA warp issues
//   A_lo*B + A*B_lo + A*B   per k-step,
// which recovers ~fp32 accuracy (the default for the layers); without it the
// kernel is plain TF32.
//
// Structure: persistent (grid <= #SMs, one CTA per SM), 256 threads:
//   warp 0      TMA producer (STAGES-deep ring of 128B-swizzled boxes)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//               (M=128, N=BN, K=8), two TMEM accumulators (2*BN columns) so
//               the epilogue of tile t overlaps the mainloop of tile t+1
//   warps 2-3   3xTF32 split (SPLIT3 only)
//   warps 4-7   epilogue: tcgen05.ld, fused epilogue, stores
//
// Shared-memory operand layouts (canonical UMMA layouts):
//   K-major:  TMA box {32 elems = 128 B, rows}, SWIZZLE_128B
//             -> [rows][128 B], 8-row atoms, SBO 1024 B, k-step of 8 = +32 B
//   MN-major: TMA box {32 elems, BK rows}, SWIZZLE_128B_ATOM_32B
//             -> per 32-wide MN slab [BK][128 B], 4-row atoms (Swizzle<2,5,2>),
//             SBO 512 B, slabs LBO = BK*128 B apart, k-step of 8 = +1024 B.
//             tf32 MN-major operands require this 32-byte-atom swizzle
//             (UMMA layout type SWIZZLE_128B_BASE32B).
#pragma once

#include <cstdint>

#include "tma_util.cuh"

namespace linrec_dev {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 elements per k-block = one 128-byte swizzle row
constexpr int kThreads = 256;

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
// 32 lanes x 8 consecutive fp32 columns; thread i of the warp gets lane
// (base lane + i).  The caller waits with tmem_wait_ld().
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor (sm_100 SmemDescriptor):
// start[0,14) LBO[16,30) SBO[32,46) version[46,48)=1 base[49,52) layout[61,64)
// layout: 2 = SWIZZLE_128B (16-byte atoms), 1 = SWIZZLE_128B_BASE32B.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                              uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm_100)
  d |= (uint64_t)layout << 61;
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

template <bool MN, int ROWS>
struct TileGeom {
  static constexpr int BYTES = ROWS * BK * 4;
  static constexpr uint32_t LBO = MN ? BK * 128 : 16;
  static constexpr uint32_t SBO = MN ? 512 : 1024;
  static constexpr uint32_t KSTEP = MN ? 1024 : 32;  // bytes per 8-element k-step
  static constexpr uint32_t LAYOUT = MN ? 1 : 2;
  static constexpr int NBOX = MN ? ROWS / 32 : 1;
  static constexpr int BOX_BYTES = MN ? BK * 128 : BYTES;
};

enum Epi : int { kEpiPlain = 0, kEpiGilr = 1, kEpiGates = 2 };

struct GemmParams {
  int M;             // output rows
  int units;         // output columns per block (N for NB == 1)
  int ntm, ntn, nz;  // tiles along M, along units, K splits
  int kb1, kb, kb_total;
  int kchunk;        // k-blocks per TMEM accumulation unit (promotion to fp32 registers)
  int b_bstride;     // row offset between B blocks (blocked K-major B)
  // plain epilogue
  float* C;
  int ldc;
  int mode;          // 0 store, 1 accumulate, 2 split-K partial (C + z*M*ldc)
  // layer epilogues
  int act;           // candidate activation (common.hpp:49-71): 0 tanh, 1 identity, 2 relu
  int64_t ldo;       // pitch (elements) of the [M][units] output planes
  const float* bias[4];
  float* out[5];
};

template <bool A_MN, bool B_MN, int BN, int NB, int STAGES, bool SPLIT3>
struct GemmCfg {
  using GA = TileGeom<A_MN, BM>;
  using GB = TileGeom<B_MN, BN>;
  static constexpr int UNITS = BN / NB;  // output columns (hidden units) per tile
  static constexpr int STAGE_BYTES = GA::BYTES + GB::BYTES;
  static constexpr int LO_OFF = STAGES * STAGE_BYTES;  // 3xTF32 lo tiles, same layout
  static constexpr int OFF_BAR = LO_OFF + (SPLIT3 ? STAGES * STAGE_BYTES : 0);
  static constexpr int NBARS = 3 * STAGES + 4;
  static constexpr int SMEM = OFF_BAR + NBARS * 8 + 16 + 1024;  // + alignment slack
  static constexpr uint32_t IDESC = idesc_tf32(BM, BN, A_MN, B_MN);
  static constexpr uint32_t TMEM_COLS = 2 * BN;
  static_assert(!B_MN || NB == 1, "blocked B operands are K-major weights");
  static_assert(UNITS % 8 == 0 && (NB == 1 || UNITS >= 8), "epilogue works in 8-column chunks");
};

__device__ __forceinline__ float sigmoidf_(float z) { return 1.f / (1.f + expf(-z)); }
__device__ __forceinline__ float actf_(int a, float z) { return a == 0 ? tanhf(z) : a == 1 ? z : fmaxf(z, 0.f); }

__device__ __forceinline__ void store8(float* dst, const float (&v)[8], bool full, int left) {
  if (full) {
    reinterpret_cast<float4*>(dst)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(dst)[1] = make_float4(v[4], v[5], v[6], v[7]);
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < left) dst[i] = v[i];
  }
}

// tf32 part the tensor core uses (it ignores the low 13 mantissa bits).
__device__ __forceinline__ float tf32_hi(float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }

template <bool A_MN, bool B_MN, int BN, int NB, int STAGES, bool SPLIT3, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
k_gemm(const __grid_constant__ CUtensorMap ta1, const __grid_constant__ CUtensorMap tb1,
       const __grid_constant__ CUtensorMap ta2, const __grid_constant__ CUtensorMap tb2, const GemmParams p) {
  using Cfg = GemmCfg<A_MN, B_MN, BN, NB, STAGES, SPLIT3>;
  using GA = typename Cfg::GA;
  using GB = typename Cfg::GB;
  constexpr int UNITS = Cfg::UNITS;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* empty = full + STAGES;
  uint64_t* split = empty + STAGES;
  uint64_t* acc_full = split + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = p.ntm * p.ntn * p.nz;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&split[s], 64);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 128);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {  // ------------------------------------------ TMA producer
    if (lane == 0) {
      prefetch_tmap(&ta1);
      prefetch_tmap(&tb1);
      uint32_t it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int tn = t % p.ntn, tm = (t / p.ntn) % p.ntm, z = t / (p.ntn * p.ntm);
        const int m0 = tm * BM, u0 = tn * UNITS;
        const int kb_begin = z * p.kb, kb_end = min(kb_begin + p.kb, p.kb_total);
        for (int kb = kb_begin; kb < kb_end; ++kb, ++it) {
          const int s = it % STAGES;
          if (it >= (uint32_t)STAGES) mbar_wait(&empty[s], ((it / STAGES) + 1) & 1);
          const bool second = kb >= p.kb1;
          const CUtensorMap* ta = second ? &ta2 : &ta1;
          const CUtensorMap* tb = second ? &tb2 : &tb1;
          const int k0 = (second ? kb - p.kb1 : kb) * BK;
          unsigned char* sa = smem + s * Cfg::STAGE_BYTES;
          unsigned char* sb = sa + GA::BYTES;
          mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
          if (A_MN) {
#pragma unroll
            for (int j = 0; j < GA::NBOX; ++j) tma_load_2d_nohint(sa + j * GA::BOX_BYTES, ta, m0 + 32 * j, k0, &full[s]);
          } else {
            tma_load_2d_nohint(sa, ta, k0, m0, &full[s]);
          }
          if (B_MN) {
#pragma unroll
            for (int j = 0; j < GB::NBOX; ++j) tma_load_2d_nohint(sb + j * GB::BOX_BYTES, tb, u0 + 32 * j, k0, &full[s]);
          } else {
#pragma unroll
            for (int q = 0; q < NB; ++q)
              tma_load_2d_nohint(sb + q * UNITS * 128, tb, k0, q * p.b_bstride + u0, &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {  // ------------------------------------- MMA issuer
    if (lane == 0) {
      // One accumulation unit = KCHUNK k-blocks of one tile, accumulated from
      // zero in TMEM slot (unit & 1); the epilogue sums the units in fp32
      // registers (the tensor-core accumulator loses ~2^-23 per K=8 step).
      uint32_t it = 0, unit = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int z = t / (p.ntn * p.ntm);
        const int kb_begin = z * p.kb, kb_end = min(kb_begin + p.kb, p.kb_total);
        for (int c0 = kb_begin; c0 < kb_end; c0 += p.kchunk, ++unit) {
          const uint32_t as = unit & 1, use = unit >> 1;
          if (use > 0) mbar_wait(&acc_empty[as], (use - 1) & 1);
          tc_fence_after();
          const uint32_t acc = tmem + as * BN;
          const int c1 = min(c0 + p.kchunk, kb_end);
          for (int kb = c0; kb < c1; ++kb, ++it) {
            const int s = it % STAGES;
            mbar_wait(&full[s], (it / STAGES) & 1);
            if (SPLIT3) mbar_wait(&split[s], (it / STAGES) & 1);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + s * Cfg::STAGE_BYTES);
            const uint32_t sb = sa + GA::BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const uint64_t ad = smem_desc(sa + kk * GA::KSTEP, GA::LBO, GA::SBO, GA::LAYOUT);
              const uint64_t bd = smem_desc(sb + kk * GB::KSTEP, GB::LBO, GB::SBO, GB::LAYOUT);
              uint32_t accum = (kb > c0 || kk > 0) ? 1u : 0u;
              if (SPLIT3) {
                const uint64_t adl = smem_desc(sa + Cfg::LO_OFF + kk * GA::KSTEP, GA::LBO, GA::SBO, GA::LAYOUT);
                const uint64_t bdl = smem_desc(sb + Cfg::LO_OFF + kk * GB::KSTEP, GB::LBO, GB::SBO, GB::LAYOUT);
                mma_tf32(acc, adl, bd, Cfg::IDESC, accum);
                mma_tf32(acc, ad, bdl, Cfg::IDESC, 1u);
                accum = 1u;
              }
              mma_tf32(acc, ad, bd, Cfg::IDESC, accum);
            }
            mma_commit(&empty[s]);  // stage (and its lo tiles) free once these MMAs have read it
          }
          mma_commit(&acc_full[as]);
        }
      }
    }
  } else if (warp < 4) {  // --------------------------------------- 3xTF32 split
    if (SPLIT3) {
      const int st = threadIdx.x - 64;  // 0..63
      uint32_t it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int z = t / (p.ntn * p.ntm);
        const int kb_begin = z * p.kb, kb_end = min(kb_begin + p.kb, p.kb_total);
        for (int kb = kb_begin; kb < kb_end; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          const float4* src = reinterpret_cast<const float4*>(smem + s * Cfg::STAGE_BYTES);
          float4* dst = reinterpret_cast<float4*>(smem + Cfg::LO_OFF + s * Cfg::STAGE_BYTES);
#pragma unroll 8
          for (int e = st; e < Cfg::STAGE_BYTES / 16; e += 64) {
            const float4 v = src[e];
            dst[e] = make_float4(v.x - tf32_hi(v.x), v.y - tf32_hi(v.y), v.z - tf32_hi(v.z), v.w - tf32_hi(v.w));
          }
          fence_proxy_async();  // generic-proxy writes -> visible to the tensor core
          mbar_arrive(&split[s]);
        }
      }
    }
  } else {  // ------------------------------------------------------- epilogue
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    uint32_t unit = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int tn = t % p.ntn, tm = (t / p.ntn) % p.ntm, z = t / (p.ntn * p.ntm);
      const int kb_begin = z * p.kb, kb_end = min(kb_begin + p.kb, p.kb_total);
      float acc[BN];
#pragma unroll
      for (int i = 0; i < BN; ++i) acc[i] = 0.f;
      for (int c0 = kb_begin; c0 < kb_end; c0 += p.kchunk, ++unit) {
        const uint32_t as = unit & 1, use = unit >> 1;
        mbar_wait(&acc_full[as], use & 1);
        tc_fence_after();
        const uint32_t tbase = tmem + as * BN + ((uint32_t)(q * 32) << 16);
#pragma unroll
        for (int c = 0; c < BN; c += 32) {
          uint32_t r[4][8];
#pragma unroll
          for (int g = 0; g < 4; ++g) tmem_ld8(tbase + (uint32_t)(c + 8 * g), r[g]);
          tmem_wait_ld();
#pragma unroll
          for (int g = 0; g < 4; ++g)
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[c + 8 * g + i] += __uint_as_float(r[g][i]);
        }
        tc_fence_before();
        mbar_arrive(&acc_empty[as]);
      }
      const int row = tm * BM + q * 32 + lane;
      const int u0 = tn * UNITS;
      if (row >= p.M) continue;
#pragma unroll
      for (int c = 0; c < UNITS; c += 8) {
        const int j = u0 + c;  // first unit (column) of this chunk
        if (j >= p.units) break;
        const bool full8 = j + 8 <= p.units;
        if (EPI == kEpiPlain) {
          float* dst = p.C + (size_t)(p.mode == 2 ? z : 0) * p.M * p.ldc + (size_t)row * p.ldc + j;
          float w[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) w[i] = acc[c + i];
          if (p.mode == 1) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (full8 || j + i < p.units) w[i] += dst[i];
          }
          store8(dst, w, full8, p.units - j);
        } else if (EPI == kEpiGilr) {
          // blocks (g, i) of hidden units j..j+7: g = sigmoid, i = act,
          // impulse = (1 - g) * i  (layers.hpp:86-92)
          float g[8], ci[8], imp[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int jj = min(j + i, p.units - 1);
            g[i] = sigmoidf_(acc[c + i] + p.bias[0][jj]);
            ci[i] = actf_(p.act, acc[(NB - 1) * UNITS + c + i] + p.bias[1][jj]);
            imp[i] = (1.f - g[i]) * ci[i];
          }
          const size_t o = (size_t)row * p.ldo + j;
          store8(p.out[0] + o, g, full8, p.units - j);
          store8(p.out[1] + o, ci, full8, p.units - j);
          store8(p.out[2] + o, imp, full8, p.units - j);
        } else {  // kEpiGates
          // blocks (f, i, o, z) of units j..j+7: f, i, o = sigmoid, z = tanh
          // (layers.hpp:263, activate_gates :226-236); planes f, i, o, z and
          // the cell impulse i*z (:271-279)
          constexpr int B1 = NB > 1 ? 1 : 0, B2 = NB > 2 ? 2 : 0, B3 = NB > 3 ? 3 : 0;
          float f[8], ig[8], og[8], zg[8], iz[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int jj = min(j + i, p.units - 1);
            f[i] = sigmoidf_(acc[c + i] + p.bias[0][jj]);
            ig[i] = sigmoidf_(acc[B1 * UNITS + c + i] + p.bias[1][jj]);
            og[i] = sigmoidf_(acc[B2 * UNITS + c + i] + p.bias[2][jj]);
            zg[i] = tanhf(acc[B3 * UNITS + c + i] + p.bias[3][jj]);
            iz[i] = ig[i] * zg[i];
          }
          const size_t o = (size_t)row * p.ldo + j;
          store8(p.out[0] + o, f, full8, p.units - j);
          store8(p.out[1] + o, ig, full8, p.units - j);
          store8(p.out[2] + o, og, full8, p.units - j);
          store8(p.out[3] + o, zg, full8, p.units - j);
          store8(p.out[4] + o, iz, full8, p.units - j);
        }
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, Cfg::TMEM_COLS);
  }
}

}  // namespace tc
}  // namespace linrec_dev
