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
