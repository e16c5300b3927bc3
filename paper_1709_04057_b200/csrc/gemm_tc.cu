// Host side of the tcgen05 TF32 GEMM (gemm_tc.cuh): tensor maps, launch,
// deterministic split-K reduction.
#include <cstdio>

#include "gemm_tc.cuh"
#include "launch.h"
#include "tma_impl.cuh"

namespace linrec_impl {

namespace {

// 2-D fp32 tensor map with a 128-byte swizzle: `inner` contiguous elements,
// `outer` rows at `pitch` elements; box {32, box_outer}.
cudaError_t make_tmap_sw128(CUtensorMap* map, const float* ptr, int64_t inner, int64_t outer, int64_t pitch,
                            int box_outer) {
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
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Operand map: K-major [rows][K] (pitch >= K) or MN-major [K][rows].
cudaError_t operand_map(CUtensorMap* map, const float* p, bool mn, int64_t rows, int64_t K, int64_t pitch,
                        int tile_rows) {
  if (mn) return make_tmap_sw128(map, p, rows, K, pitch, linrec_dev::tc::BK);
  return make_tmap_sw128(map, p, K, rows, pitch, tile_rows);
}

__global__ void k_splitk_reduce(const float* __restrict__ part, int splits, int64_t MN, int64_t N, int64_t ldc,
                                float* __restrict__ C, int accumulate) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < MN; i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += part[(size_t)z * MN + i];  // fixed order: deterministic
    const int64_t r = i / N, c = i - r * N;
    float* d = C + r * ldc + c;
    *d = accumulate ? *d + s : s;
  }
}

template <bool A_MN, bool B_MN, int BN, int STAGES, int EPI>
cudaError_t launch_cfg(const GemmOperands& op, const linrec_dev::tc::GemmParams& p, int k_splits,
                       cudaStream_t st) {
  using Cfg = linrec_dev::tc::GemmCfg<A_MN, B_MN, BN, STAGES>;
  CUtensorMap a1, b1, a2, b2;
  cudaError_t e;
  if ((e = operand_map(&a1, op.a1, A_MN, op.M, op.K1, op.lda1, linrec_dev::tc::BM)) != cudaSuccess) return e;
  if ((e = operand_map(&b1, op.b1, B_MN, op.N, op.K1, op.ldb1, BN)) != cudaSuccess) return e;
  if (op.a2 != nullptr) {
    if ((e = operand_map(&a2, op.a2, A_MN, op.M, op.K2, op.lda2, linrec_dev::tc::BM)) != cudaSuccess) return e;
    if ((e = operand_map(&b2, op.b2, B_MN, op.N, op.K2, op.ldb2, BN)) != cudaSuccess) return e;
  } else {
    a2 = a1;
    b2 = b1;
  }
  auto kern = linrec_dev::tc::k_gemm_tf32<A_MN, B_MN, BN, STAGES, EPI>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
  const dim3 grid((unsigned)((op.N + BN - 1) / BN), (unsigned)((op.M + 127) / 128), (unsigned)k_splits);
  kern<<<grid, 256, Cfg::SMEM, st>>>(a1, b1, a2, b2, p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t gemm_tf32(const GemmOperands& op, int epi, const GemmEpilogue& ep, cudaStream_t st) {
  using linrec_dev::tc::BK;
  const int kb1 = (int)((op.K1 + BK - 1) / BK);
  const int kb2 = op.a2 != nullptr ? (int)((op.K2 + BK - 1) / BK) : 0;
  const int kb_total = kb1 + kb2;
  int splits = ep.k_splits < 1 ? 1 : ep.k_splits;
  if (splits > kb_total) splits = kb_total > 0 ? kb_total : 1;
  const int kb_per = (kb_total + splits - 1) / splits;
  splits = kb_total > 0 ? (kb_total + kb_per - 1) / kb_per : 1;

  linrec_dev::tc::GemmParams p{};
  p.M = (int)op.M;
  p.N = (int)op.N;
  p.kb1 = kb1;
  p.kb = kb_per;
  p.kb_total = kb_total;
  p.k_splits = splits;
  p.ldc = (int)ep.ldc;
  p.C = ep.C;
  p.mode = ep.accumulate ? 1 : 0;
  p.bias = ep.bias;
  p.o0 = ep.o0;
  p.o1 = ep.o1;
  p.o2 = ep.o2;
  p.o3 = ep.o3;
  p.ldo = (int)ep.ldo;
  float* partial = nullptr;
  if (splits > 1) {
    if (epi != linrec_dev::tc::kEpiPlain || ep.scratch == nullptr) return cudaErrorInvalidValue;
    partial = ep.scratch;
    p.C = partial;
    p.ldc = (int)op.N;
    p.mode = 2;
  }
  cudaError_t e;
#define GEMM_CASE(AM, BMN, EP)                                                          \
  if (op.a_mn == AM && op.b_mn == BMN && epi == EP) {                                   \
    e = launch_cfg<AM, BMN, 128, 4, EP>(op, p, splits, st);                            \
    goto launched;                                                                      \
  }
  GEMM_CASE(false, false, linrec_dev::tc::kEpiPlain)
  GEMM_CASE(false, false, linrec_dev::tc::kEpiGilr)
  GEMM_CASE(false, false, linrec_dev::tc::kEpiGates)
  GEMM_CASE(false, true, linrec_dev::tc::kEpiPlain)
  GEMM_CASE(true, true, linrec_dev::tc::kEpiPlain)
  GEMM_CASE(true, false, linrec_dev::tc::kEpiPlain)
#undef GEMM_CASE
  return cudaErrorInvalidConfiguration;
launched:
  if (e != cudaSuccess) return e;
  if (splits > 1) {
    const int64_t MN = op.M * op.N;
    const int64_t blocks = (MN + 255) / 256;
    k_splitk_reduce<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, st>>>(partial, splits, MN, op.N, ep.ldc,
                                                                               ep.C, ep.accumulate ? 1 : 0);
    e = cudaGetLastError();
  }
  return e;
}

int gemm_splits_for(int64_t M, int64_t N, int64_t K) {
  const int64_t tiles = ((M + 127) / 128) * ((N + 127) / 128);
  const int64_t kb = (K + 31) / 32;
  int64_t s = (2 * 148 + tiles - 1) / tiles;  // ~2 waves of CTAs
  if (s > kb / 4) s = kb / 4;                  // >= 4 k-blocks per split
  if (s < 1) s = 1;
  if (s > 64) s = 64;
  return (int)s;
}

}  // namespace linrec_impl
