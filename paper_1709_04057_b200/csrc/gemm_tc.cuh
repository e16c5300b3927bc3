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
// "blocked": the B rows of a tile are NB sub-boxes taken from NB row blocks
// of the weight (rows q*bstride + j0 ..), so the f/i/o/z (or g/i) rows of the
// same hidden units land in one tile and the epilogue sees every gate of a
// unit without any host-side weight permutation.
//
// CTA pair (cluster of 2, tcgen05 cta_group::2): one MMA is M=256 x N=256 x
// K=8; CTA r holds A rows [128r, 128r+128) and B rows [128r, 128r+128) of the
// tile in its own shared memory (each SM streams half of each operand) and
// rows [128r, +128) x all 256 columns of the accumulator in its TMEM.  The
// leader CTA's single MMA thread issues for both.
//
// Precision: kind::tf32 reads 10 mantissa bits of each operand.  With SPLIT3
// the kernel runs 3xTF32: split warps write lo = v - tf32(v) of every staged
// A and B tile next to it and the MMA issues  A_lo*B + A*B_lo + A*B  per
// k-step (~fp32 accuracy, the layers' default).  The tensor-core accumulator
// itself drops bits at every K=8 step, so K is accumulated in chunks of KCHUNK
// k-blocks in TMEM and the chunks are summed in fp32 registers by the
// epilogue ("promotion"): the error no longer grows with K.
//
// Persistent, 384 threads per CTA:
//   warp 0      TMA producer (STAGES-deep ring)
//   warp 1      TMEM allocator (cta_group::2); leader: tcgen05.mma issuer,
//               two 256-column accumulators so the epilogue of tile t
//               overlaps the mainloop of tile t+1
//   warps 2-7   3xTF32 split (SPLIT3) and relay of "stage landed + split" to
//               the leader (six warps: with two, the split's smem round trip
//               and not the tensor core bounded 3xTF32)
//   warps 8-15  epilogue: 2 warps per TMEM lane quadrant, 128 fp32 register
//               accumulators each; fused epilogue -> 128B-swizzled smem box
//               -> TMA store (or TMA reduce-add for C += A*B)
//   setmaxnreg moves registers from warps 0-7 (64) to the epilogue (192).
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

constexpr int BM = 128;      // A rows per CTA (the MMA's M = 256 spans the pair)
constexpr int BN = 256;      // widest MMA N; each CTA stages BN/2 B rows (QRNN tiles use N = 192)
constexpr int BK = 32;       // fp32 elements per k-block = one 128-byte swizzle row
constexpr int kThreads = 512;
constexpr int kEpiWarps = 8;
constexpr int kSplitWarps = 6;   // warps 2..7
constexpr int kEpiWarp0 = 8;     // first epilogue warp

// ---- tcgen05 / cluster wrappers ----------------------------------------------
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Address of the same shared variable in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait_cluster(bar, parity)) return;
  SpinGuard g;
  while (!mbar_try_wait_cluster(bar, parity)) g.tick();
}

// 2-D TMA load into this CTA's smem whose completion is signalled on the
// leader CTA's mbarrier (cta_group::2 form).
__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                                 uint32_t leader_bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* smem_src, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, const void* smem_src, int32_t c0,
                                                  int32_t c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void tmem_alloc2(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on the mbarrier at this smem offset in both CTAs of the pair once
// all previously issued tcgen05.mma have completed.
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
// 32 lanes x 32 consecutive fp32 columns; thread i of the warp gets lane
// (base lane + i).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// 32 lanes x 16 consecutive fp32 columns.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
template <int N>
__device__ __forceinline__ void setmaxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void setmaxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
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

enum Epi : int { kEpiPlain = 0, kEpiGilr = 1, kEpiGates = 2, kEpiQrnn = 3 };

struct GemmParams {
  int M;             // output rows
  int units;         // output columns per block (N for NB == 1)
  int ntm, ntn, nz;  // tiles along M (256 rows), along units, K splits
  int kb1, kb, kb_total;
  int kchunk;        // k-blocks per TMEM accumulation unit (promotion to fp32 registers)
  int b_bstride;     // row offset between B blocks (blocked K-major B)
  // tap-shifted K (QRNN causal convolution, layers.hpp:376-388): k-block kb
  // belongs to tap s = kb / tap_kb and reads A rows shifted by s*a_tap and B
  // rows (K-major) / K (MN-major) offset by s*b_tap.  tap_kb = 0: off.
  int tap_kb, a_tap, b_tap;
  int b_lo;          // SPLIT3: B's lo part comes precomputed (tb1lo/tb2lo); split only A
  int mode;          // plain: 0 store, 1 accumulate (TMA reduce-add), 2 split-K partial (rows z*Mp + row)
  int Mp;            // partial rows per split (M rounded up to the 256-row tile)
  int act;           // candidate activation (common.hpp:49-71): 0 tanh, 1 identity, 2 relu
  const float* bias[4];
};

template <bool A_MN, bool B_MN, int NB, int BNT, int STAGES, bool SPLIT3>
struct GemmCfg {
  using GA = TileGeom<A_MN, BM>;
  using GB = TileGeom<B_MN, BNT / 2>;
  static constexpr int UNITS = BNT / NB;  // output columns (hidden units) per tile
  static constexpr int HALF = UNITS / 2;  // units per epilogue warp of a quadrant pair
  static constexpr int ACCN = BNT / 2;    // fp32 accumulators per epilogue thread
  // K-major B: each CTA loads its BNT/2 tile rows as NSB boxes of SB rows
  static constexpr int SB = NB == 1 ? BNT / 2 : (NB == 3 ? 32 : UNITS);
  static constexpr int NSB = (BNT / 2) / SB;
  static constexpr int STAGE_BYTES = GA::BYTES + GB::BYTES;  // this CTA's halves
  static constexpr int LO_OFF = STAGES * STAGE_BYTES;        // 3xTF32 lo tiles, same layout
  static constexpr int EPI_OFF = LO_OFF + (SPLIT3 ? STAGES * STAGE_BYTES : 0);
  static constexpr int EPI_BYTES = 32 * 128;                  // one 32x32 fp32 staging box per epilogue warp
  static constexpr int OFF_BAR = EPI_OFF + kEpiWarps * EPI_BYTES;
  static constexpr int NBARS = 3 * STAGES + 4;
  static constexpr int SMEM = OFF_BAR + NBARS * 8 + 16 + 1024;  // + alignment slack
  static constexpr uint32_t IDESC = idesc_tf32(2 * BM, BNT, A_MN, B_MN);
  static constexpr uint32_t TMEM_COLS = 2 * BNT <= 256 ? 256 : 512;  // two accumulators
  static_assert(!B_MN || NB == 1, "blocked B operands are K-major weights");
  static_assert(BNT % (NB * 64) == 0 && BNT <= BN, "NB / tile width");
  static_assert(HALF % 32 == 0 && ACCN % 32 == 0 && (BNT / 2) % SB == 0, "epilogue groups");
  static_assert(SMEM <= 232448, "shared memory");
};

// Activations on the SFU (ex2.approx / rcp.approx, ~2 ulp each): far inside
// the layers' 2e-5 normwise bar and branch-free.  tanh via 1 - 2/(e^{2z}+1)
// keeps an absolute error of a few 1e-8 near 0.
__device__ __forceinline__ float ex2_(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sigmoidf_(float z) { return rcp_(1.f + ex2_(-1.4426950408889634f * z)); }
__device__ __forceinline__ float tanhf_(float z) {
  const float e = ex2_(2.8853900817779268f * fminf(fmaxf(z, -15.f), 15.f));
  return fmaf(-2.f, rcp_(e + 1.f), 1.f);
}
__device__ __forceinline__ float actf_(int a, float z) { return a == 0 ? tanhf_(z) : a == 1 ? z : fmaxf(z, 0.f); }
// bias[u0 + lane] for this warp's 32 units (0 beyond `units`); element i is
// then __shfl_sync(.., i) -- one load per lane instead of 32 per thread.
__device__ __forceinline__ float bias_lane(const float* b, int u0, int lane, int units) {
  const int j = u0 + lane;
  return j < units ? __ldg(b + j) : 0.f;
}
#define LINREC_BCAST(v, i) __shfl_sync(0xffffffffu, (v), (i))

// tf32 part the tensor core uses (it ignores the low 13 mantissa bits).
__device__ __forceinline__ float tf32_hi(float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }

// One 32-row x 32-column fp32 box in the 128B-swizzled layout TMA expects:
// lane = row; 16-byte chunk j of the row lives at chunk (j ^ (row & 7)).
__device__ __forceinline__ void stage_row(unsigned char* box, int lane, const float (&v)[32]) {
  float4* row = reinterpret_cast<float4*>(box + lane * 128);
#pragma unroll
  for (int j = 0; j < 8; ++j) row[j ^ (lane & 7)] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
}

// Start writing the staged box to global memory (one lane).  `red` = TMA
// reduce-add instead of a store.  box_wait() must precede the next
// stage_row() into the same box: callers compute the next values first, so
// the TMA engine's read of the box overlaps that math.
__device__ __forceinline__ void flush_box(const CUtensorMap* map, unsigned char* box, int lane, int c0, int c1,
                                          bool red) {
  fence_proxy_async();
  __syncwarp();
  if (lane == 0) {
    if (red) tma_reduce_add_2d(map, box, c0, c1);
    else tma_store_2d(map, box, c0, c1);
    bulk_commit();
  }
}
__device__ __forceinline__ void box_wait(int lane) {
  if (lane == 0) bulk_wait_read0();
  __syncwarp();
}

struct OutMaps {
  CUtensorMap m[5];
};

template <bool A_MN, bool B_MN, int NB, int BNT, int STAGES, bool SPLIT3, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
k_gemm(const __grid_constant__ CUtensorMap ta1, const __grid_constant__ CUtensorMap tb1,
       const __grid_constant__ CUtensorMap ta2, const __grid_constant__ CUtensorMap tb2,
       const __grid_constant__ CUtensorMap tb1lo, const __grid_constant__ CUtensorMap tb2lo,
       const __grid_constant__ OutMaps om, const GemmParams p) {
  using Cfg = GemmCfg<A_MN, B_MN, NB, BNT, STAGES, SPLIT3>;
  using GA = typename Cfg::GA;
  using GB = typename Cfg::GB;
  constexpr int UNITS = Cfg::UNITS;
  constexpr int HALF = Cfg::HALF;
  constexpr int ACCN = Cfg::ACCN;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* empty = full + STAGES;
  uint64_t* ready = empty + STAGES;  // leader: stage landed and split in both CTAs (SPLIT3)
  uint64_t* acc_full = ready + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int ncl = gridDim.x >> 1, cid = blockIdx.x >> 1;
  const int ntiles = p.ntm * p.ntn * p.nz;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&ready[s], 2 * kSplitWarps * 32);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 2 * kEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc2(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {  // ------------------------------------------ TMA producer
    setmaxnreg_dec<64>();
    if (lane == 0) {
      prefetch_tmap(&ta1);
      prefetch_tmap(&tb1);
      const uint32_t full_leader = mapa(smem_u32(full), 0);
      uint32_t it = 0;
      for (int t = cid; t < ntiles; t += ncl) {
        const int tn = t % p.ntn, tm = (t / p.ntn) % p.ntm, z = t / (p.ntn * p.ntm);
        const int m0 = tm * 2 * BM + (int)rank * BM, u0 = tn * UNITS;
        const int kb_begin = z * p.kb, kb_end = min(kb_begin + p.kb, p.kb_total);
        for (int kb = kb_begin; kb < kb_end; ++kb, ++it) {
          const int s = it % STAGES;
          if (it >= (uint32_t)STAGES) mbar_wait(&empty[s], ((it / STAGES) + 1) & 1);
          const bool second = kb >= p.kb1;
          const CUtensorMap* ta = second ? &ta2 : &ta1;
          const CUtensorMap* tb = second ? &tb2 : &tb1;
          const CUtensorMap* tbl = second ? &tb2lo : &tb1lo;
          int kk = second ? kb - p.kb1 : kb, a_off = 0, b_off = 0;
          if (p.tap_kb) {
            const int tap = kb / p.tap_kb;
            kk = kb - tap * p.tap_kb;
            a_off = tap * p.a_tap;
            b_off = tap * p.b_tap;
          }
          const int k0 = kk * BK;
          unsigned char* sa = smem + s * Cfg::STAGE_BYTES;
          unsigned char* sb = sa + GA::BYTES;
          // SPLIT3: local completion (the split warps relay to the leader);
          // else both CTAs' loads complete on the leader's barrier, which
          // the leader armed with the bytes of both halves.
          const uint32_t bar = full_leader + 8u * (uint32_t)s;
          if (SPLIT3) mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES + (p.b_lo ? GB::BYTES : 0));
          else if (leader) mbar_arrive_expect_tx(&full[s], 2 * Cfg::STAGE_BYTES);
#define LINREC_LOAD(dst, map, c0, c1)                          \
  do {                                                         \
    if (SPLIT3) tma_load_2d_nohint(dst, map, c0, c1, &full[s]); \
    else tma_load_2d_pair(dst, map, c0, c1, bar);              \
  } while (0)
          if (A_MN) {
#pragma unroll
            for (int j = 0; j < GA::NBOX; ++j) LINREC_LOAD(sa + j * GA::BOX_BYTES, ta, m0 + 32 * j, k0);
          } else {
            LINREC_LOAD(sa, ta, k0, m0 + a_off);
          }
          // B hi into the stage; with b_lo also B lo into the stage's lo tile
          for (int pass = 0; pass < (SPLIT3 && p.b_lo ? 2 : 1); ++pass) {
            unsigned char* dstb = pass == 0 ? sb : smem + Cfg::LO_OFF + s * Cfg::STAGE_BYTES + GA::BYTES;
            const CUtensorMap* mb = pass == 0 ? tb : tbl;
            if (B_MN) {
#pragma unroll
              for (int j = 0; j < GB::NBOX; ++j)
                LINREC_LOAD(dstb + j * GB::BOX_BYTES, mb, u0 + (int)rank * (BNT / 2) + 32 * j, k0 + b_off);
            } else {
              // tile row rho -> gate block rho / UNITS, unit u0 + rho % UNITS
#pragma unroll
              for (int j = 0; j < Cfg::NSB; ++j) {
                const int rho = (int)rank * (BNT / 2) + j * Cfg::SB;
                LINREC_LOAD(dstb + j * Cfg::SB * 128, mb, k0, (rho / UNITS) * p.b_bstride + u0 + rho % UNITS + b_off);
              }
            }
          }
#undef LINREC_LOAD
        }
      }
    }
  } else if (warp == 1) {  // ------------------------------------- MMA issuer
    setmaxnreg_dec<64>();
    if (leader && lane == 0) {
      // One accumulation unit = KCHUNK k-blocks of one tile, accumulated from
      // zero in TMEM slot (unit & 1); the epilogue sums the units in fp32.
      uint32_t it = 0, unit = 0;
      for (int t = cid; t < ntiles; t += ncl) {
        const int z = t / (p.ntn * p.ntm);
        const int kb_begin = z * p.kb, kb_end = min(kb_begin + p.kb, p.kb_total);
        for (int c0 = kb_begin; c0 < kb_end; c0 += p.kchunk, ++unit) {
          const uint32_t as = unit & 1, use = unit >> 1;
          if (use > 0) mbar_wait_cluster(&acc_empty[as], (use - 1) & 1);
          tc_fence_after();
          const uint32_t acc = tmem + as * BNT;
          const int c1 = min(c0 + p.kchunk, kb_end);
          for (int kb = c0; kb < c1; ++kb, ++it) {
            const int s = it % STAGES;
            if (SPLIT3) mbar_wait_cluster(&ready[s], (it / STAGES) & 1);
            else mbar_wait_cluster(&full[s], (it / STAGES) & 1);
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
                mma_tf32_pair(acc, adl, bd, Cfg::IDESC, accum);
                mma_tf32_pair(acc, ad, bdl, Cfg::IDESC, 1u);
                accum = 1u;
              }
              mma_tf32_pair(acc, ad, bd, Cfg::IDESC, accum);
            }
            mma_commit_pair(&empty[s]);  // both CTAs' stage s (and lo tiles) free once read
          }
          mma_commit_pair(&acc_full[as]);
        }
      }
    }
  } else if (warp < kEpiWarp0) {  // ------------------------------- 3xTF32 split
    setmaxnreg_dec<64>();
    if (SPLIT3) {
      const int st = threadIdx.x - 64;  // 0 .. kSplitWarps*32-1
      const uint32_t ready_leader = mapa(smem_u32(ready), 0);
      uint32_t it = 0;
      for (int t = cid; t < ntiles; t += ncl) {
        const int z = t / (p.ntn * p.ntm);
        const int kb_begin = z * p.kb, kb_end = min(kb_begin + p.kb, p.kb_total);
        for (int kb = kb_begin; kb < kb_end; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          const float4* src = reinterpret_cast<const float4*>(smem + s * Cfg::STAGE_BYTES);
          float4* dst = reinterpret_cast<float4*>(smem + Cfg::LO_OFF + s * Cfg::STAGE_BYTES);
          const int nsplit = (p.b_lo ? GA::BYTES : Cfg::STAGE_BYTES) / 16;  // A only when B's lo is loaded
#pragma unroll 4
          for (int e = st; e < nsplit; e += kSplitWarps * 32) {
            const float4 v = src[e];
            dst[e] = make_float4(v.x - tf32_hi(v.x), v.y - tf32_hi(v.y), v.z - tf32_hi(v.z), v.w - tf32_hi(v.w));
          }
          fence_proxy_async();  // generic-proxy writes -> visible to the tensor core
          mbar_arrive_cluster(ready_leader + 8u * (uint32_t)s);
        }
      }
    }
  } else {  // ------------------------------------------------------- epilogue
    setmaxnreg_inc<192>();
    const int q = warp & 3;          // TMEM lane quadrant this warp may access
    const int hf = (warp - kEpiWarp0) >> 2;  // which half of the tile's units
    unsigned char* box = smem + Cfg::EPI_OFF + (warp - kEpiWarp0) * Cfg::EPI_BYTES;
    const uint32_t acc_empty_leader = mapa(smem_u32(acc_empty), 0);
    uint32_t unit = 0;
    for (int t = cid; t < ntiles; t += ncl) {
      const int tn = t % p.ntn, tm = (t / p.ntn) % p.ntm, z = t / (p.ntn * p.ntm);
      const int kb_begin = z * p.kb, kb_end = min(kb_begin + p.kb, p.kb_total);
      float acc[ACCN];
#pragma unroll
      for (int i = 0; i < ACCN; ++i) acc[i] = 0.f;
      for (int c0 = kb_begin; c0 < kb_end; c0 += p.kchunk, ++unit) {
        const uint32_t as = unit & 1, use = unit >> 1;
        mbar_wait(&acc_full[as], use & 1);
        tc_fence_after();
        const uint32_t tbase = tmem + as * BNT + ((uint32_t)(q * 32) << 16);
#pragma unroll
        for (int g = 0; g < ACCN / 32; ++g) {
          // accumulator group g (32 values) <- TMEM columns of gate block b
          const int b = (32 * g) / HALF;
          const int col = b * UNITS + hf * HALF + (32 * g) % HALF;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            uint32_t r[16];
            tmem_ld16(tbase + (uint32_t)(col + 16 * hh), r);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[32 * g + 16 * hh + i] += __uint_as_float(r[i]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(acc_empty_leader + 8u * as);
      }
      const int row0 = tm * 2 * BM + (int)rank * BM + q * 32;  // this warp's 32 output rows
      const int u0 = tn * UNITS + hf * HALF;                   // and its first unit
      if (EPI == kEpiPlain) {
        const int rowc = row0 + (p.mode == 2 ? z * p.Mp : 0);
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = acc[32 * g + i];
          box_wait(lane);
          stage_row(box, lane, v);
          flush_box(&om.m[0], box, lane, u0 + 32 * g, rowc, p.mode == 1);
        }
      } else if (EPI == kEpiGilr) {
        // blocks (g, i) of hidden units: g = sigmoid, i = act,
        // impulse = (1 - g) * i  (layers.hpp:86-92)
#pragma unroll
        for (int k = 0; k < HALF / 32; ++k) {
          const float bg = bias_lane(p.bias[0], u0 + 32 * k, lane, p.units);
          const float bz = bias_lane(p.bias[1], u0 + 32 * k, lane, p.units);
          float gv[32], cv[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) gv[i] = sigmoidf_(acc[32 * k + i] + LINREC_BCAST(bg, i));
          box_wait(lane);
          stage_row(box, lane, gv);
          flush_box(&om.m[0], box, lane, u0 + 32 * k, row0, false);
#pragma unroll
          for (int i = 0; i < 32; ++i) cv[i] = actf_(p.act, acc[HALF + 32 * k + i] + LINREC_BCAST(bz, i));
          box_wait(lane);
          stage_row(box, lane, cv);
          flush_box(&om.m[1], box, lane, u0 + 32 * k, row0, false);
#pragma unroll
          for (int i = 0; i < 32; ++i) gv[i] = (1.f - gv[i]) * cv[i];
          box_wait(lane);
          stage_row(box, lane, gv);
          flush_box(&om.m[2], box, lane, u0 + 32 * k, row0, false);
        }
      } else if (EPI == kEpiQrnn) {
        // blocks (f, o, z): f, o = sigmoid, z = tanh (layers.hpp:472);
        // planes f, o, z and the cell impulse (1 - f) * z (:475-482)
        const float b0 = bias_lane(p.bias[0], u0, lane, p.units), b1 = bias_lane(p.bias[1], u0, lane, p.units);
        const float b2 = bias_lane(p.bias[2], u0, lane, p.units);
        float v[32], fv[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) fv[i] = sigmoidf_(acc[i] + LINREC_BCAST(b0, i));
        box_wait(lane);
        stage_row(box, lane, fv);
        flush_box(&om.m[0], box, lane, u0, row0, false);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = sigmoidf_(acc[32 + i] + LINREC_BCAST(b1, i));
        box_wait(lane);
        stage_row(box, lane, v);
        flush_box(&om.m[1], box, lane, u0, row0, false);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = tanhf_(acc[64 + i] + LINREC_BCAST(b2, i));
        box_wait(lane);
        stage_row(box, lane, v);
        flush_box(&om.m[2], box, lane, u0, row0, false);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] *= 1.f - fv[i];
        box_wait(lane);
        stage_row(box, lane, v);
        flush_box(&om.m[3], box, lane, u0, row0, false);
      } else {  // kEpiGates
        // blocks (f, i, o, z): f, i, o = sigmoid, z = tanh (layers.hpp:263,
        // activate_gates :226-236); planes f, i, o, z and the impulse i*z
        const float b0 = bias_lane(p.bias[0], u0, lane, p.units), b1 = bias_lane(p.bias[1], u0, lane, p.units);
        const float b2 = bias_lane(p.bias[2], u0, lane, p.units), b3 = bias_lane(p.bias[3], u0, lane, p.units);
        float v[32], iv[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = sigmoidf_(acc[i] + LINREC_BCAST(b0, i));
        box_wait(lane);
        stage_row(box, lane, v);
        flush_box(&om.m[0], box, lane, u0, row0, false);
#pragma unroll
        for (int i = 0; i < 32; ++i) iv[i] = sigmoidf_(acc[32 + i] + LINREC_BCAST(b1, i));
        box_wait(lane);
        stage_row(box, lane, iv);
        flush_box(&om.m[1], box, lane, u0, row0, false);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = sigmoidf_(acc[64 + i] + LINREC_BCAST(b2, i));
        box_wait(lane);
        stage_row(box, lane, v);
        flush_box(&om.m[2], box, lane, u0, row0, false);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = tanhf_(acc[96 + i] + LINREC_BCAST(b3, i));
        box_wait(lane);
        stage_row(box, lane, v);
        flush_box(&om.m[3], box, lane, u0, row0, false);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] *= iv[i];
        box_wait(lane);
        stage_row(box, lane, v);
        flush_box(&om.m[4], box, lane, u0, row0, false);
      }
    }
    if (lane == 0) bulk_wait0();
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem, Cfg::TMEM_COLS);
  }
}

}  // namespace tc
}  // namespace linrec_dev
