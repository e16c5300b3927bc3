// Host side of the tcgen05 GEMM (gemm_tc.cuh): tensor maps, persistent
// launch, split-K planning and the deterministic split-K reduction.
#include <cstdio>

#include "gemm_tc.cuh"
#include "launch.h"

namespace linrec_impl {

namespace {

using linrec_dev::tc::BK;
using linrec_dev::tc::BM;
using linrec_dev::tc::BN;

// 2-D fp32 tensor map: `inner` contiguous elements, `outer` rows at `pitch`
// elements; box {32, box_outer}.  swizzle: 128B (K-major operands) or
// 128B with 32-byte atoms (MN-major tf32 operands).
cudaError_t make_tmap(CUtensorMap* map, const float* ptr, int64_t inner, int64_t outer, int64_t pitch, int box_outer,
                      CUtensorMapSwizzle swz) {
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Fn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<Fn>(f);
  }();
  if (!fn) return cudaErrorNotSupported;
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  const cuuint64_t strides[1] = {(cuuint64_t)(pitch * 4)};
  const cuuint32_t box[2] = {32u, (cuuint32_t)box_outer};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Operand map: K-major [rows][K] (pitch >= K), box {32 k, tile_rows}, or
// MN-major [K][rows], box {32 rows, BK k}.
cudaError_t operand_map(CUtensorMap* map, const float* p, bool mn, int64_t rows, int64_t K, int64_t pitch,
                        int tile_rows) {
  if (mn) return make_tmap(map, p, rows, K, pitch, BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  return make_tmap(map, p, K, rows, pitch, tile_rows, CU_TENSOR_MAP_SWIZZLE_128B);
}

// Partials [nz][Mp][ldp] (Mp = M rounded up to the 256-row tile, so tail
// rows of one split never land in the next) -> C, summed in split order.
__global__ void k_splitk_reduce(const float* __restrict__ part, int splits, int64_t M, int64_t Mp, int64_t N,
                                int64_t ldp, int64_t ldc, float* __restrict__ C, int accumulate) {
  const int64_t MN = M * N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < MN; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / N, c = i - r * N;
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += part[((int64_t)z * Mp + r) * ldp + c];  // fixed order: deterministic
    float* d = C + r * ldc + c;
    *d = accumulate ? *d + s : s;
  }
}

int sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// Output map over a [rows][cols] fp32 plane (pitch elements), 32x32 boxes,
// 128B swizzle (the epilogue's staging layout).
cudaError_t out_map(CUtensorMap* map, float* ptr, int64_t cols, int64_t rows, int64_t pitch) {
  return make_tmap(map, ptr, cols, rows, pitch, 32, CU_TENSOR_MAP_SWIZZLE_128B);
}

template <bool A_MN, bool B_MN, int NB, int BNT, bool SPLIT3, int EPI>
cudaError_t launch_cfg(const GemmOperands& op, const GemmEpilogue& ep, linrec_dev::tc::GemmParams p,
                       float* partial, int64_t Mp, int64_t ldp, cudaStream_t st) {
  constexpr int STAGES = SPLIT3 ? 3 : 5;
  using Cfg = linrec_dev::tc::GemmCfg<A_MN, B_MN, NB, BNT, STAGES, SPLIT3>;
  constexpr int UNITS = Cfg::UNITS;
  constexpr int BROWS = Cfg::SB;  // rows of one K-major B box
  // rows (K-major) / K extent (MN-major) the B map must cover, all taps included
  int64_t b_rows = NB == 1 ? op.units : (NB - 1) * op.b_bstride + op.units;
  if (op.ntaps > 1 && !B_MN) b_rows += (op.ntaps - 1) * op.b_tap;
  const int64_t b_k1 = op.ntaps > 1 && B_MN ? (op.ntaps - 1) * op.b_tap + op.K1 : op.K1;
  CUtensorMap a1, b1, a2, b2, b1l, b2l;
  linrec_dev::tc::OutMaps om;
  cudaError_t e;
  if ((e = operand_map(&a1, op.a1, A_MN, op.M, op.K1, op.lda1, BM)) != cudaSuccess) return e;
  if ((e = operand_map(&b1, op.b1, B_MN, b_rows, b_k1, op.ldb1, BROWS)) != cudaSuccess) return e;
  if (op.a2 != nullptr) {
    if ((e = operand_map(&a2, op.a2, A_MN, op.M, op.K2, op.lda2, BM)) != cudaSuccess) return e;
    if ((e = operand_map(&b2, op.b2, B_MN, b_rows, op.K2, op.ldb2, BROWS)) != cudaSuccess) return e;
  } else {
    a2 = a1;
    b2 = b1;
  }
  p.b_lo = SPLIT3 && op.b1_lo != nullptr && (op.a2 == nullptr || op.b2_lo != nullptr) ? 1 : 0;
  if (p.b_lo) {
    if ((e = operand_map(&b1l, op.b1_lo, B_MN, b_rows, b_k1, op.ldb1, BROWS)) != cudaSuccess) return e;
    if (op.a2 != nullptr) {
      if ((e = operand_map(&b2l, op.b2_lo, B_MN, b_rows, op.K2, op.ldb2, BROWS)) != cudaSuccess) return e;
    } else {
      b2l = b1l;
    }
  } else {
    b1l = b1;
    b2l = b2;
  }
  if (EPI == linrec_dev::tc::kEpiPlain) {
    if (partial) e = out_map(&om.m[0], partial, op.units, Mp * p.nz, ldp);
    else e = out_map(&om.m[0], ep.C, op.units, op.M, ep.ldc);
    if (e != cudaSuccess) return e;
  } else {
    const int nout = EPI == linrec_dev::tc::kEpiGilr ? 3 : EPI == linrec_dev::tc::kEpiQrnn ? 4 : 5;
    for (int i = 0; i < nout; ++i)
      if ((e = out_map(&om.m[i], ep.out[i], op.units, op.M, ep.ldo)) != cudaSuccess) return e;
  }
  p.ntm = (int)((op.M + 2 * BM - 1) / (2 * BM));
  p.ntn = (int)((op.units + UNITS - 1) / UNITS);
  p.b_bstride = (int)op.b_bstride;
  auto kern = linrec_dev::tc::k_gemm<A_MN, B_MN, NB, BNT, STAGES, SPLIT3, EPI>;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
  if (e != cudaSuccess) return e;
  const int64_t ntiles = (int64_t)p.ntm * p.ntn * p.nz;
  const int64_t clusters = sm_count() / 2;
  const int grid = 2 * (int)(ntiles < clusters ? ntiles : clusters);
  kern<<<grid, linrec_dev::tc::kThreads, Cfg::SMEM, st>>>(a1, b1, a2, b2, b1l, b2l, om, p);
  return cudaGetLastError();
}

template <bool SPLIT3>
cudaError_t dispatch(const GemmOperands& op, int epi, const GemmEpilogue& ep, const linrec_dev::tc::GemmParams& p,
                     float* partial, int64_t Mp, int64_t ldp, cudaStream_t st) {
  using namespace linrec_dev::tc;
  if (epi == kEpiPlain) {
    if (op.nb != 1) return cudaErrorInvalidValue;
    if (!op.a_mn && !op.b_mn) return launch_cfg<false, false, 1, BN, SPLIT3, kEpiPlain>(op, ep, p, partial, Mp, ldp, st);
    if (!op.a_mn && op.b_mn) return launch_cfg<false, true, 1, BN, SPLIT3, kEpiPlain>(op, ep, p, partial, Mp, ldp, st);
    if (op.a_mn && op.b_mn) return launch_cfg<true, true, 1, BN, SPLIT3, kEpiPlain>(op, ep, p, partial, Mp, ldp, st);
    return launch_cfg<true, false, 1, BN, SPLIT3, kEpiPlain>(op, ep, p, partial, Mp, ldp, st);
  }
  if (op.a_mn || op.b_mn) return cudaErrorInvalidValue;
  if (epi == kEpiGilr && op.nb == 2)
    return launch_cfg<false, false, 2, BN, SPLIT3, kEpiGilr>(op, ep, p, nullptr, 0, 0, st);
  if (epi == kEpiGates && op.nb == 4)
    return launch_cfg<false, false, 4, BN, SPLIT3, kEpiGates>(op, ep, p, nullptr, 0, 0, st);
  if (epi == kEpiQrnn && op.nb == 3)
    return launch_cfg<false, false, 3, 192, SPLIT3, kEpiQrnn>(op, ep, p, nullptr, 0, 0, st);
  return cudaErrorInvalidValue;
}

}  // namespace

// ---------------------------------------------------------------------------
// CUDA-core path for plain GEMMs with at most 8 output columns (the first
// layer's input width m, e.g. bench_model's m = 4): a 256-wide tensor-core
// tile would be >= 97 % padding there, while these are HBM-bound on A.
// Exact fp32 FMAs in a fixed order (deterministic, at least as accurate as
// 3xTF32).
struct SkinnyArgs {
  // two K-concatenated operand pairs (the second with K2 = 0 when absent);
  // fields are selected with ternaries, never indexed at run time, so the
  // kernel parameters stay in constant space
  const float *a0, *a1, *b0, *b1;
  int64_t K0, K1, lda0, lda1, ldb0, ldb1;
  int64_t M, units;
  bool b_mn;
  __device__ const float* a(int p) const { return p == 0 ? a0 : a1; }
  __device__ int64_t lda(int p) const { return p == 0 ? lda0 : lda1; }
  __device__ int64_t K(int p) const { return p == 0 ? K0 : K1; }
  __device__ float B(int p, int64_t n, int64_t k) const {
    const float* b = p == 0 ? b0 : b1;
    const int64_t ld = p == 0 ? ldb0 : ldb1;
    return b_mn ? __ldg(b + k * ld + n) : __ldg(b + n * ld + k);
  }
};

// A K-major (rows of A contiguous along k): one warp per output row, lanes
// along k (float4 loads when V4), B [K][N] staged in shared memory,
// fixed-order warp reduction.
template <int N, bool V4>
__global__ void __launch_bounds__(256) k_skinny_rows(SkinnyArgs g, float* __restrict__ C, int64_t ldc, int acc) {
  extern __shared__ float Bs[];  // [N][K1 + K2]: lanes read consecutive k (no bank conflicts)
  const int64_t Kt = g.K0 + g.K1;
  for (int64_t i = threadIdx.x; i < Kt * N; i += blockDim.x) {
    const int64_t n = i / Kt, k = i - n * Kt;
    const int p = k < g.K0 ? 0 : 1;
    Bs[i] = n < g.units ? g.B(p, n, p == 0 ? k : k - g.K0) : 0.f;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warps = blockDim.x >> 5;
  for (int64_t m = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5); m < g.M; m += (int64_t)gridDim.x * warps) {
    float s[N];
#pragma unroll
    for (int n = 0; n < N; ++n) s[n] = 0.f;
    int64_t koff = 0;
    for (int p = 0; p < 2; ++p) {
      const float* a = g.a(p) + m * g.lda(p);
      const int64_t Kp = g.K(p);
      if (V4) {  // lane owns k = 4*lane + 128*i .. +3
        constexpr int U = 4;
        for (int64_t k = 4 * lane; k < Kp; k += 128 * U) {
          float4 v[U];
#pragma unroll
          for (int u = 0; u < U; ++u)
            v[u] = k + 128 * u < Kp ? __ldcs(reinterpret_cast<const float4*>(a + k + 128 * u))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (k + 128 * u >= Kp) break;
#pragma unroll
            for (int n = 0; n < N; ++n) {
              const float4 b = *reinterpret_cast<const float4*>(Bs + n * Kt + koff + k + 128 * u);
              s[n] = __fmaf_rn(v[u].x, b.x, s[n]);
              s[n] = __fmaf_rn(v[u].y, b.y, s[n]);
              s[n] = __fmaf_rn(v[u].z, b.z, s[n]);
              s[n] = __fmaf_rn(v[u].w, b.w, s[n]);
            }
          }
        }
      } else {
        int64_t k = lane;
        for (; k + 96 < Kp; k += 128) {
          float v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) v[u] = __ldcs(a + k + 32 * u);
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int n = 0; n < N; ++n) s[n] = __fmaf_rn(v[u], Bs[n * Kt + koff + k + 32 * u], s[n]);
        }
        for (; k < Kp; k += 32) {
          const float v = __ldcs(a + k);
#pragma unroll
          for (int n = 0; n < N; ++n) s[n] = __fmaf_rn(v, Bs[n * Kt + koff + k], s[n]);
        }
      }
      koff += Kp;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
      for (int n = 0; n < N; ++n) s[n] += __shfl_xor_sync(0xffffffffu, s[n], off);
    if (lane == 0)
#pragma unroll
      for (int n = 0; n < N; ++n)
        if (n < g.units) {
          float* d = C + m * ldc + n;
          *d = acc ? *d + s[n] : s[n];
        }
  }
}

// A MN-major (A(m,k) = a[k*lda + m], the weight gradients' dpre^T with K =
// T*b rows): a CTA covers 64 rows m (16 threads x float4) x 16 k-groups,
// split-K over blockIdx.y into the tensor-core path's partial layout
// [splits][Mp][ldp] (then k_splitk_reduce); the k-groups are summed in
// shared memory in a fixed order.  Needs M, lda % 4 == 0 and 16-byte
// aligned A (the ABI's pitch rule).
template <int N>
__global__ void __launch_bounds__(256) k_skinny_outer(SkinnyArgs g, float* __restrict__ part, int64_t Mp,
                                                      int64_t ldp, int64_t kper) {
  constexpr int KC = 1024, MQ = 16, KG = 256 / MQ, U = 8;  // 64 rows m x 16 k-groups per CTA
  static_assert(KC * N >= KG * MQ * N * 4, "the k-group reduction reuses the B stage");
  __shared__ float4 smem[KC * N / 4];
  float(*Bs)[N] = reinterpret_cast<float(*)[N]>(smem);
  float4(*red)[MQ][N] = reinterpret_cast<float4(*)[MQ][N]>(smem);
  const int mq = threadIdx.x % MQ, kg = threadIdx.x / MQ;
  const int64_t m0 = (int64_t)blockIdx.x * (4 * MQ) + 4 * mq;
  const bool mok = m0 < g.M;
  const int64_t Kt = g.K0 + g.K1;
  const int64_t k0 = (int64_t)blockIdx.y * kper, k1 = k0 + kper < Kt ? k0 + kper : Kt;
  float4 s[N];
#pragma unroll
  for (int n = 0; n < N; ++n) s[n] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t kc = k0; kc < k1; kc += KC) {
    const int kn = (int)(k1 - kc < KC ? k1 - kc : KC);
    __syncthreads();
    for (int i = threadIdx.x; i < kn * N; i += blockDim.x) {
      const int kk = i / N, n = i - kk * N;
      const int64_t k = kc + kk;
      const int p = k < g.K0 ? 0 : 1;
      Bs[kk][n] = n < g.units ? g.B(p, n, p == 0 ? k : k - g.K0) : 0.f;
    }
    __syncthreads();
    if (!mok) continue;
    for (int kk = kg; kk < kn; kk += KG * U) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t k = kc + kk + KG * u;
        const int p = k < g.K0 ? 0 : 1;
        v[u] = kk + KG * u < kn
                   ? __ldcs(reinterpret_cast<const float4*>(g.a(p) + (p == 0 ? k : k - g.K0) * g.lda(p) + m0))
                   : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (kk + KG * u >= kn) break;
#pragma unroll
        for (int n = 0; n < N; ++n) {
          const float b = Bs[kk + KG * u][n];
          s[n].x = __fmaf_rn(v[u].x, b, s[n].x);
          s[n].y = __fmaf_rn(v[u].y, b, s[n].y);
          s[n].z = __fmaf_rn(v[u].z, b, s[n].z);
          s[n].w = __fmaf_rn(v[u].w, b, s[n].w);
        }
      }
    }
  }
  __syncthreads();  // the B stage is free: reuse it for the k-group sums
#pragma unroll
  for (int n = 0; n < N; ++n) red[kg][mq][n] = s[n];
  __syncthreads();
  if (kg == 0 && mok) {
#pragma unroll
    for (int q = 1; q < KG; ++q)  // fixed order: deterministic
#pragma unroll
      for (int n = 0; n < N; ++n) {
        const float4 r = red[q][mq][n];
        s[n].x += r.x;
        s[n].y += r.y;
        s[n].z += r.z;
        s[n].w += r.w;
      }
    float* dst = part + ((int64_t)blockIdx.y * Mp + m0) * ldp;  // M % 4 == 0: all four rows exist
#pragma unroll
    for (int n = 0; n < N; ++n)
      if (n < g.units) {
        dst[n] = s[n].x;
        dst[ldp + n] = s[n].y;
        dst[2 * ldp + n] = s[n].z;
        dst[3 * ldp + n] = s[n].w;
      }
  }
}

// K-major A with taps (the QRNN input gradient dx[r] = sum_s dpre[r + s*a_tap]
// W_s, N <= 8): a CTA owns 64 output rows (8 warps x 8 rows) and walks the
// taps, staging tap s's B [N][K] in shared memory (double-buffered) and
// accumulating per-lane partials of its rows; rows past M read as zero (the
// tensor-core path's TMA zero fill).  Fixed-order reduction: deterministic.
template <int N, bool V4>
__global__ void __launch_bounds__(256) k_skinny_taps(const float* __restrict__ A, int64_t lda, int64_t K,
                                                     const float* __restrict__ Bm, int64_t ldb, bool b_mn,
                                                     int64_t b_tap, int ntaps, int64_t a_tap, int64_t M,
                                                     int64_t units, float* __restrict__ C, int64_t ldc,
                                                     int acc) {
  constexpr int RW = 8;  // rows per warp
  extern __shared__ float Bs[];  // [2][N][K]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * (8 * RW) + warp * RW;
  float s[RW][N];
#pragma unroll
  for (int i = 0; i < RW; ++i)
#pragma unroll
    for (int n = 0; n < N; ++n) s[i][n] = 0.f;
  auto stage = [&](int tap, float* dst) {
    for (int64_t i = threadIdx.x; i < N * K; i += blockDim.x) {
      const int64_t n = i / K, k = i - n * K;
      dst[i] = n < units ? (b_mn ? __ldg(Bm + (tap * b_tap + k) * ldb + n) : __ldg(Bm + (tap * b_tap + n) * ldb + k))
                         : 0.f;
    }
  };
  stage(0, Bs);
  for (int tap = 0; tap < ntaps; ++tap) {
    float* cur = Bs + (tap & 1) * N * K;
    __syncthreads();  // tap's B staged; the other buffer is free
    if (tap + 1 < ntaps) stage(tap + 1, Bs + ((tap + 1) & 1) * N * K);
    if (V4) {  // lane owns k = 4*lane + 128*j .. +3; all RW rows' float4 in flight together
      for (int64_t k = 4 * lane; k < K; k += 128) {
        float4 bk[N];
#pragma unroll
        for (int n = 0; n < N; ++n) bk[n] = *reinterpret_cast<const float4*>(cur + n * K + k);
        float4 v[RW];
#pragma unroll
        for (int i = 0; i < RW; ++i) {
          const int64_t ar = r0 + i + tap * a_tap;  // this tap's A row
          v[i] = (r0 + i < M && ar < M) ? __ldg(reinterpret_cast<const float4*>(A + ar * lda + k))
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < RW; ++i)
#pragma unroll
          for (int n = 0; n < N; ++n) {
            s[i][n] = __fmaf_rn(v[i].x, bk[n].x, s[i][n]);
            s[i][n] = __fmaf_rn(v[i].y, bk[n].y, s[i][n]);
            s[i][n] = __fmaf_rn(v[i].z, bk[n].z, s[i][n]);
            s[i][n] = __fmaf_rn(v[i].w, bk[n].w, s[i][n]);
          }
      }
    } else {
      for (int64_t k = lane; k < K; k += 32) {  // all RW rows' loads of this k in flight together
        float bk[N];
#pragma unroll
        for (int n = 0; n < N; ++n) bk[n] = cur[n * K + k];
        float v[RW];
#pragma unroll
        for (int i = 0; i < RW; ++i) {
          const int64_t ar = r0 + i + tap * a_tap;
          v[i] = (r0 + i < M && ar < M) ? __ldg(A + ar * lda + k) : 0.f;
        }
#pragma unroll
        for (int i = 0; i < RW; ++i)
#pragma unroll
          for (int n = 0; n < N; ++n) s[i][n] = __fmaf_rn(v[i], bk[n], s[i][n]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < RW; ++i) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
      for (int n = 0; n < N; ++n) s[i][n] += __shfl_xor_sync(0xffffffffu, s[i][n], off);
    if (lane == 0 && r0 + i < M)
#pragma unroll
      for (int n = 0; n < N; ++n)
        if (n < units) {
          float* d = C + (r0 + i) * ldc + n;
          *d = acc ? *d + s[i][n] : s[i][n];
        }
  }
}

// The QRNN weight gradients of all k taps in one launch, <= 8 input columns:
// dW_s[M][N] += sum_{t < R - s*shift} A[t + s*shift][.]^T B[t][.] with A
// (dpre, MN-major, lda) and B (x, MN-major, ldb).  Tap s = blockIdx.x is the
// fastest grid dimension, so the k CTAs reading the same rows of A (shifted
// by s*shift) run together and share them through L2 -- one HBM pass over
// dpre instead of k.  Per tap the split-K partials use the tensor-core
// path's layout [splits][Mp][ldp] at part + s * splits*Mp*ldp.
template <int N>
__global__ void __launch_bounds__(256) k_skinny_outer_taps(const float* __restrict__ A, int64_t lda,
                                                           const float* __restrict__ Bm, int64_t ldb, int64_t R,
                                                           int64_t shift, int64_t M, int64_t units,
                                                           float* __restrict__ part, int64_t Mp, int64_t ldp,
                                                           int splits) {
  constexpr int KC = 1024, MQ = 16, KG = 256 / MQ, U = 8;
  __shared__ float4 smem[KC * N / 4];
  float(*Bs)[N] = reinterpret_cast<float(*)[N]>(smem);
  float4(*red)[MQ][N] = reinterpret_cast<float4(*)[MQ][N]>(smem);
  const int tap = blockIdx.x, split = blockIdx.z;
  const int mq = threadIdx.x % MQ, kg = threadIdx.x / MQ;
  const int64_t m0 = (int64_t)blockIdx.y * (4 * MQ) + 4 * mq;
  const bool mok = m0 < M;
  const int64_t Kt = R - tap * shift;  // rows of this tap
  const int64_t kper = (Kt + splits - 1) / splits;
  const int64_t k0 = split * kper, k1 = k0 + kper < Kt ? k0 + kper : Kt;
  const float* a = A + tap * shift * lda;
  float4 s[N];
#pragma unroll
  for (int n = 0; n < N; ++n) s[n] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t kc = k0; kc < k1; kc += KC) {
    const int kn = (int)(k1 - kc < KC ? k1 - kc : KC);
    __syncthreads();
    for (int i = threadIdx.x; i < kn * N; i += blockDim.x) {
      const int kk = i / N, n = i - kk * N;
      Bs[kk][n] = n < units ? __ldg(Bm + (kc + kk) * ldb + n) : 0.f;
    }
    __syncthreads();
    if (!mok) continue;
    for (int kk = kg; kk < kn; kk += KG * U) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        v[u] = kk + KG * u < kn ? __ldg(reinterpret_cast<const float4*>(a + (kc + kk + KG * u) * lda + m0))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (kk + KG * u >= kn) break;
#pragma unroll
        for (int n = 0; n < N; ++n) {
          const float b = Bs[kk + KG * u][n];
          s[n].x = __fmaf_rn(v[u].x, b, s[n].x);
          s[n].y = __fmaf_rn(v[u].y, b, s[n].y);
          s[n].z = __fmaf_rn(v[u].z, b, s[n].z);
          s[n].w = __fmaf_rn(v[u].w, b, s[n].w);
        }
      }
    }
  }
  __syncthreads();  // the B stage is free: reuse it for the k-group sums
#pragma unroll
  for (int n = 0; n < N; ++n) red[kg][mq][n] = s[n];
  __syncthreads();
  if (kg == 0 && mok) {
#pragma unroll
    for (int q = 1; q < KG; ++q)
#pragma unroll
      for (int n = 0; n < N; ++n) {
        const float4 r = red[q][mq][n];
        s[n].x += r.x;
        s[n].y += r.y;
        s[n].z += r.z;
        s[n].w += r.w;
      }
    float* dst = part + (((int64_t)tap * splits + split) * Mp + m0) * ldp;
#pragma unroll
    for (int n = 0; n < N; ++n)
      if (n < units) {
        dst[n] = s[n].x;
        dst[ldp + n] = s[n].y;
        dst[2 * ldp + n] = s[n].z;
        dst[3 * ldp + n] = s[n].w;
      }
  }
}

// Per-tap split reduction of k_skinny_outer_taps (blockIdx.y = tap), summed in
// split order into dW_s (accumulating).
__global__ void k_splitk_reduce_taps(const float* __restrict__ part, int splits, int64_t M, int64_t Mp, int64_t N,
                                     int64_t ldp, float* __restrict__ dW) {
  const int tap = blockIdx.y;
  const float* pt = part + (int64_t)tap * splits * Mp * ldp;
  float* C = dW + (int64_t)tap * M * N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * N; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / N, c = i - r * N;
    float v = 0.f;
    for (int z = 0; z < splits; ++z) v += pt[((int64_t)z * Mp + r) * ldp + c];
    C[i] += v;
  }
}

bool skinny_enabled() {  // LINREC_SKINNY_GEMM=0: always the tensor cores (comparison runs)
  static const bool on = env_int("LINREC_SKINNY_GEMM", 1) != 0;
  return on;
}

// Runs the plain GEMM on CUDA cores when it qualifies; cudaErrorNotSupported
// otherwise (the caller then uses the tensor cores).
cudaError_t gemm_skinny(const GemmOperands& op, const GemmEpilogue& ep, int splits, float* partial, int64_t Mp,
                        int64_t ldp, cudaStream_t st) {
  if (op.units > 8 || op.nb != 1 || op.M < 1) return cudaErrorNotSupported;
  if (op.ntaps > 1) {  // taps: K-major A, one operand pair
    if (op.a_mn || op.a2 != nullptr) return cudaErrorNotSupported;
    const int npad = op.units <= 1 ? 1 : op.units <= 2 ? 2 : op.units <= 4 ? 4 : 8;
    const size_t smem = (size_t)2 * npad * op.K1 * sizeof(float);
    if (smem > 96 * 1024) return cudaErrorNotSupported;
    const unsigned grid = (unsigned)((op.M + 63) / 64);
    const bool v4 = op.K1 % 4 == 0 && op.lda1 % 4 == 0 && (reinterpret_cast<uintptr_t>(op.a1) & 15) == 0;
#define TAPS1(NN, V)                                                                                               \
  do {                                                                                                             \
    cudaFuncSetAttribute(k_skinny_taps<NN, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);             \
    k_skinny_taps<NN, V><<<grid, 256, smem, st>>>(op.a1, op.lda1, op.K1, op.b1, op.ldb1, op.b_mn, op.b_tap,         \
                                                  op.ntaps, op.a_tap, op.M, op.units, ep.C, ep.ldc,                \
                                                  ep.accumulate ? 1 : 0);                                          \
  } while (0)
#define TAPS(NN)            \
  do {                      \
    if (v4) TAPS1(NN, true);  \
    else TAPS1(NN, false);  \
  } while (0)
    switch (npad) {
      case 1: TAPS(1); break;
      case 2: TAPS(2); break;
      case 4: TAPS(4); break;
      default: TAPS(8); break;
    }
#undef TAPS
#undef TAPS1
    return cudaGetLastError();
  }
  SkinnyArgs g{};
  g.a0 = op.a1;
  g.b0 = op.b1;
  g.K0 = op.K1;
  g.lda0 = op.lda1;
  g.ldb0 = op.ldb1;
  g.a1 = op.a2 != nullptr ? op.a2 : op.a1;
  g.b1 = op.a2 != nullptr ? op.b2 : op.b1;
  g.K1 = op.a2 != nullptr ? op.K2 : 0;
  g.lda1 = op.a2 != nullptr ? op.lda2 : op.lda1;
  g.ldb1 = op.a2 != nullptr ? op.ldb2 : op.ldb1;
  g.M = op.M;
  g.units = op.units;
  g.b_mn = op.b_mn;
  const int npad = op.units <= 1 ? 1 : op.units <= 2 ? 2 : op.units <= 4 ? 4 : 8;
  const int64_t Kt = op.K1 + g.K1;
  if (!op.a_mn) {
    const size_t smem = (size_t)Kt * npad * sizeof(float);
    if (smem > 48 * 1024) return cudaErrorNotSupported;
    const bool v4 = op.K1 % 4 == 0 && op.lda1 % 4 == 0 && (reinterpret_cast<uintptr_t>(op.a1) & 15) == 0 &&
                    (op.a2 == nullptr ||
                     (op.K2 % 4 == 0 && op.lda2 % 4 == 0 && (reinterpret_cast<uintptr_t>(op.a2) & 15) == 0));
    // one wave of resident CTAs, each warp walking rows (the B stage is per CTA)
    int occ = 1;
    if (v4) {
      void (*kf)(SkinnyArgs, float*, int64_t, int) = npad <= 1 ? k_skinny_rows<1, true>
                                                     : npad <= 2 ? k_skinny_rows<2, true>
                                                     : npad <= 4 ? k_skinny_rows<4, true> : k_skinny_rows<8, true>;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kf, 256, smem);
    } else {
      void (*kf)(SkinnyArgs, float*, int64_t, int) = npad <= 1 ? k_skinny_rows<1, false>
                                                     : npad <= 2 ? k_skinny_rows<2, false>
                                                     : npad <= 4 ? k_skinny_rows<4, false> : k_skinny_rows<8, false>;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kf, 256, smem);
    }
    const int64_t blocks = (op.M + 7) / 8, wave = (int64_t)sm_count() * (occ < 1 ? 1 : occ);
    const unsigned grid = (unsigned)(blocks < wave ? blocks : wave);
#define ROWS(NN)                                                                                             \
  (v4 ? k_skinny_rows<NN, true><<<grid, 256, smem, st>>>(g, ep.C, ep.ldc, ep.accumulate ? 1 : 0)            \
      : k_skinny_rows<NN, false><<<grid, 256, smem, st>>>(g, ep.C, ep.ldc, ep.accumulate ? 1 : 0))
    switch (npad) {
      case 1: ROWS(1); break;
      case 2: ROWS(2); break;
      case 4: ROWS(4); break;
      default: ROWS(8); break;
    }
#undef ROWS
    return cudaGetLastError();
  }
  // needs the split-K scratch and float4 rows of A
  if (splits < 2 || partial == nullptr || op.M % 4 != 0 || op.lda1 % 4 != 0 ||
      (reinterpret_cast<uintptr_t>(op.a1) & 15) != 0 ||
      (op.a2 != nullptr && (op.lda2 % 4 != 0 || (reinterpret_cast<uintptr_t>(op.a2) & 15) != 0)))
    return cudaErrorNotSupported;
  const int64_t kper = (Kt + splits - 1) / splits;
  const dim3 grid((unsigned)((op.M + 63) / 64), (unsigned)splits);
#define OUTER(NN) k_skinny_outer<NN><<<grid, 256, 0, st>>>(g, partial, Mp, ldp, kper)
  switch (npad) {
    case 1: OUTER(1); break;
    case 2: OUTER(2); break;
    case 4: OUTER(4); break;
    default: OUTER(8); break;
  }
#undef OUTER
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t MN = op.M * op.units;
  const int64_t blocks = (MN + 255) / 256;
  k_splitk_reduce<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, st>>>(
      partial, splits, op.M, Mp, op.units, ldp, ep.ldc, ep.C, ep.accumulate ? 1 : 0);
  return cudaGetLastError();
}

int gemm_splits_for(int64_t M, int64_t N, int64_t K) {
  const int64_t tiles = ((M + 2 * BM - 1) / (2 * BM)) * ((N + BN - 1) / BN);
  const int64_t kb = (K + BK - 1) / BK;
  const int64_t clusters = sm_count() / 2;
  if (tiles >= clusters || kb < 8) return 1;
  // fill the persistent grid of CTA pairs evenly: the split count whose last
  // wave is fullest, preferring fewer partials, with >= 4 k-blocks per split
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= 64 && s <= kb / 4; ++s) {
    const double waves = double(tiles * s) / double(clusters);
    const double eff = waves / double((tiles * s + clusters - 1) / clusters);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = s;
    }
  }
  return best;
}

__global__ void k_tf32_lo(const float* __restrict__ src, float* __restrict__ dst, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i] - linrec_dev::tc::tf32_hi(src[i]);
}

cudaError_t tf32_lo(const float* src, float* dst, int64_t count, cudaStream_t st) {
  const int64_t blocks = (count + 255) / 256;
  k_tf32_lo<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, st>>>(src, dst, count);
  return cudaGetLastError();
}

int64_t gemm_partial_floats(int64_t M, int64_t N, int splits) {
  return splits > 1 ? (int64_t)splits * round_up(M, 2 * BM) * round_up(N, 4) : 0;
}

int64_t wgrad_taps_partial_floats(int64_t M, int64_t N, int64_t R, int ntaps) {
  // partials are written even for one split (gemm_partial_floats is 0 there)
  return (int64_t)ntaps * gemm_splits_for(M, N, R) * round_up(M, 2 * BM) * round_up(N, 4);
}

cudaError_t wgrad_taps_skinny(const float* A, int64_t lda, const float* B, int64_t ldb, int64_t R, int64_t shift,
                              int ntaps, int64_t M, int64_t N, float* dW, float* scratch, cudaStream_t st) {
  static const bool on = env_int("LINREC_TAP_WGRAD", 1) != 0;
  if (!on || N > 8 || M % 4 || lda % 4 || (reinterpret_cast<uintptr_t>(A) & 15) || ntaps < 1 || !skinny_enabled())
    return cudaErrorNotSupported;
  const int splits = gemm_splits_for(M, N, R);
  const int64_t Mp = round_up(M, 2 * BM), ldp = round_up(N, 4);
  const dim3 grid((unsigned)ntaps, (unsigned)((M + 63) / 64), (unsigned)splits);
  const int npad = N <= 1 ? 1 : N <= 2 ? 2 : N <= 4 ? 4 : 8;
#define TAPW(NN) k_skinny_outer_taps<NN><<<grid, 256, 0, st>>>(A, lda, B, ldb, R, shift, M, N, scratch, Mp, ldp, splits)
  switch (npad) {
    case 1: TAPW(1); break;
    case 2: TAPW(2); break;
    case 4: TAPW(4); break;
    default: TAPW(8); break;
  }
#undef TAPW
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t blocks = (M * N + 255) / 256;
  k_splitk_reduce_taps<<<dim3((unsigned)(blocks < 1024 ? blocks : 1024), (unsigned)ntaps), 256, 0, st>>>(
      scratch, splits, M, Mp, N, ldp, dW);
  return cudaGetLastError();
}

cudaError_t gemm_tf32(const GemmOperands& op, int epi, const GemmEpilogue& ep, cudaStream_t st) {
  if (op.ntaps > 1 && (op.a2 != nullptr || op.a_mn)) return cudaErrorInvalidValue;
  const int kb1 = (int)((op.K1 + BK - 1) / BK) * (op.ntaps > 1 ? op.ntaps : 1);
  const int kb2 = op.a2 != nullptr ? (int)((op.K2 + BK - 1) / BK) : 0;
  const int kb_total = kb1 + kb2;
  int splits = ep.k_splits < 1 ? 1 : ep.k_splits;
  if (splits > kb_total) splits = kb_total > 0 ? kb_total : 1;
  const int kb_per = kb_total > 0 ? (kb_total + splits - 1) / splits : 0;
  splits = kb_per > 0 ? (kb_total + kb_per - 1) / kb_per : 1;

  linrec_dev::tc::GemmParams p{};
  p.M = (int)op.M;
  p.units = (int)op.units;
  p.nz = splits;
  p.kb1 = kb1;
  p.kb = kb_per;
  p.kb_total = kb_total;
  p.kchunk = ep.split3 ? 4 : 16;  // K = 128 (3xTF32) / 512 (TF32) per TMEM accumulation
  if (op.ntaps > 1) {
    p.tap_kb = (int)((op.K1 + BK - 1) / BK);
    p.a_tap = (int)op.a_tap;
    p.b_tap = (int)op.b_tap;
  }
  p.mode = ep.accumulate ? 1 : 0;
  p.act = ep.act;
  for (int i = 0; i < 4; ++i) p.bias[i] = ep.bias[i];
  float* partial = nullptr;
  const int64_t Mp = round_up(op.M, 2 * BM), ldp = round_up(op.units, 4);
  if (splits > 1) {
    if (epi != linrec_dev::tc::kEpiPlain || ep.scratch == nullptr) return cudaErrorInvalidValue;
    partial = ep.scratch;
    p.mode = 2;
    p.Mp = (int)Mp;
  }
  if (epi == linrec_dev::tc::kEpiPlain && skinny_enabled()) {
    const cudaError_t es = gemm_skinny(op, ep, splits, partial, Mp, ldp, st);
    if (es != cudaErrorNotSupported) return es;
  }
  cudaError_t e = ep.split3 ? dispatch<true>(op, epi, ep, p, partial, Mp, ldp, st)
                            : dispatch<false>(op, epi, ep, p, partial, Mp, ldp, st);
  if (e != cudaSuccess) return e;
  if (splits > 1) {
    const int64_t MN = op.M * op.units;
    const int64_t blocks = (MN + 255) / 256;
    k_splitk_reduce<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, st>>>(
        partial, splits, op.M, Mp, op.units, ldp, ep.ldc, ep.C, ep.accumulate ? 1 : 0);
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace linrec_impl
