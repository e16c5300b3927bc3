// GILR and GILR-LSTM layers on the B200 (layers.hpp:23-375): host
// orchestration in C++ over the library's own building blocks, plus the
// pointwise kernels that sit between them.
//
// Forward (gilr_lstm_forward, layers.hpp:245-293), R = T*b rows:
//   1. gemm  x * [U_s; V_s]^T  -> epilogue sigmoid / act / (1-g)*i   (g, i, imp)
//   2. scan  htil = scan(g, imp, htil0)            written after a copy of htil0,
//            so htil_prev (shift_right, :213-220) is a pointer, not a copy
//   3. gemm  [x | htil_prev] * [V | U]^T + bias -> epilogue f,i,o,z planes and i*z
//   4. scan  c = scan(f, i*z, c0)
//   5. h = o * c
// Backward (gilr_lstm_backward, :295-375):
//   dc = dh*o; cell scan backward -> df, diz, dc0; pointwise dpre (+ bias
//   column sums); dU += dpre^T htil_prev, dV += dpre^T x (split-K);
//   dhp = dpre U; surrogate scan backward on dhp shifted one step (again a
//   pointer offset: the row after the last is zeroed); pointwise dg, di
//   (+ bias sums); dU_s, dV_s (split-K); dx = [dpre | dg di] [V; U_s; V_s]
//   in ONE K-concatenated GEMM; dhtil0 = scan dh0 + dhp[0].
// Every GEMM runs on the tcgen05 kernel (gemm_tc.cuh), every recurrence on
// the chained scans (linrec_scan_f32 / linrec_scan_backward_f32).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "launch.h"
#include "linrec_cuda.h"

namespace linrec_dev {
namespace layers {

__device__ __forceinline__ float4 ld4(const float* p) { return __ldcs(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

// out = a * b over n4 float4s
__global__ void k_mul(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ out, int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 x = ld4(a + 4 * i), y = ld4(b + 4 * i);
    st4(out + 4 * i, make_float4(x.x * y.x, x.y * y.y, x.z * y.z, x.w * y.w));
  }
}

__global__ void k_add(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[i] + b[i];
}

// dst[c] += sum_k part[k * pitch + c], deterministic: block = 32 columns x
// 32 part-groups; group g sums parts g, g+32, ... in order, then the 32 group
// sums are added in group order.
__global__ void __launch_bounds__(1024) k_colsum(const float* __restrict__ part, int64_t nparts, int64_t pitch,
                                                 int64_t ncols, float* __restrict__ dst) {
  __shared__ float red[32][33];
  const int cx = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * 32 + cx;
  float s = 0.f;
  if (c < ncols)
    for (int64_t k = g; k < nparts; k += 32) s += __ldg(part + k * pitch + c);
  red[g][cx] = s;
  __syncthreads();
  if (g == 0 && c < ncols) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i) t += red[i][cx];
    dst[c] += t;
  }
}

__device__ __forceinline__ float dact(int a, float v) {  // activation_deriv_from_value (common.hpp:62-71)
  return a == 0 ? 1.f - v * v : a == 1 ? 1.f : (v > 0.f ? 1.f : 0.f);
}

// GILR-LSTM fused pre-activation gradients (layers.hpp:327-342), written
// blocked [R][4n] (f, i, o, z) like the reference's dpre, plus per-block
// partial column sums for the bias gradient.  Thread = 4 units of one row
// range; rows [blockIdx.x * rpb, ...).
// The decay gradient df = c_{t-1} * diz (recurrence.hpp:338-343) is formed
// here from the cell state instead of being stored by the scan: row r - b of
// c (c0 for t = 0), read b rows after this thread last touched it.
__global__ void k_lstm_dpre(const float* __restrict__ gf, const float* __restrict__ gi, const float* __restrict__ go,
                            const float* __restrict__ gz, const float* __restrict__ c0, const float* __restrict__ diz,
                            const float* __restrict__ dh, const float* __restrict__ c, float* __restrict__ dpre,
                            float* __restrict__ part, int64_t R, int64_t n, int64_t b, int64_t rpb) {
  const int64_t u = 4 * ((int64_t)blockIdx.y * blockDim.x + threadIdx.x);
  if (u >= n) return;
  const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = min(r0 + rpb, R);
  float4 sf = make_float4(0, 0, 0, 0), si = sf, so = sf, sz = sf;
#pragma unroll 2
  for (int64_t r = r0; r < r1; ++r) {
    const int64_t o = r * n + u;
    const float4 f = ld4(gf + o), i = ld4(gi + o), og = ld4(go + o), z = ld4(gz + o);
    const float4 d_iz = ld4(diz + o), d_h = ld4(dh + o), cc = ld4(c + o);
    const float4 cp = r >= b ? *reinterpret_cast<const float4*>(c + o - b * n)
                             : (c0 != nullptr ? *reinterpret_cast<const float4*>(c0 + r * n + u) : make_float4(0, 0, 0, 0));
    float4 pf, pi, po, pz;
#define LINREC_DPRE(X)                                                 \
  pf.X = (cp.X * d_iz.X) * f.X * (1.f - f.X);                          \
  pi.X = d_iz.X * z.X * i.X * (1.f - i.X);                             \
  po.X = (d_h.X * cc.X) * og.X * (1.f - og.X);                         \
  pz.X = d_iz.X * i.X * (1.f - z.X * z.X);                             \
  sf.X += pf.X; si.X += pi.X; so.X += po.X; sz.X += pz.X;
    LINREC_DPRE(x) LINREC_DPRE(y) LINREC_DPRE(z) LINREC_DPRE(w)
#undef LINREC_DPRE
    float* d = dpre + r * 4 * n + u;
    st4(d, pf);
    st4(d + n, pi);
    st4(d + 2 * n, po);
    st4(d + 3 * n, pz);
  }
  float* pp = part + (int64_t)blockIdx.x * 4 * n + u;
  st4(pp, sf);
  st4(pp + n, si);
  st4(pp + 2 * n, so);
  st4(pp + 3 * n, sz);
}

// GILR pre-activation gradients (layers.hpp:112-121): dg, di written blocked
// [R][2n], plus partial column sums for b_g, b_z.
// dl = h_{t-1} * G formed here (h0 for t = 0), see k_lstm_dpre.
__global__ void k_gilr_dpre(const float* __restrict__ g, const float* __restrict__ ci, const float* __restrict__ h,
                            const float* __restrict__ h0, const float* __restrict__ G, int act,
                            float* __restrict__ dpre, float* __restrict__ part, int64_t R, int64_t n, int64_t b,
                            int64_t rpb) {
  const int64_t u = 4 * ((int64_t)blockIdx.y * blockDim.x + threadIdx.x);
  if (u >= n) return;
  const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = min(r0 + rpb, R);
  float4 sg = make_float4(0, 0, 0, 0), si = sg;
#pragma unroll 2
  for (int64_t r = r0; r < r1; ++r) {
    const int64_t o = r * n + u;
    const float4 gv = ld4(g + o), iv = ld4(ci + o), Gv = ld4(G + o);
    const float4 hp = r >= b ? *reinterpret_cast<const float4*>(h + o - b * n)
                             : (h0 != nullptr ? *reinterpret_cast<const float4*>(h0 + r * n + u) : make_float4(0, 0, 0, 0));
    float4 pg, pi;
#define LINREC_GDPRE(X)                                              \
  pg.X = (hp.X * Gv.X - Gv.X * iv.X) * gv.X * (1.f - gv.X);          \
  pi.X = Gv.X * (1.f - gv.X) * dact(act, iv.X);                      \
  sg.X += pg.X; si.X += pi.X;
    LINREC_GDPRE(x) LINREC_GDPRE(y) LINREC_GDPRE(z) LINREC_GDPRE(w)
#undef LINREC_GDPRE
    float* d = dpre + r * 2 * n + u;
    st4(d, pg);
    st4(d + n, pi);
  }
  float* pp = part + (int64_t)blockIdx.x * 2 * n + u;
  st4(pp, sg);
  st4(pp + n, si);
}

// QRNN fused pre-activation gradients (layers.hpp:519-531), blocked [R][3n]
// (f, o, z), plus per-block partial column sums for the bias gradient.
// df = c_{t-1} * dimp formed here (c0 for t = 0), see k_lstm_dpre.
__global__ void k_qrnn_dpre(const float* __restrict__ gf, const float* __restrict__ go, const float* __restrict__ gz,
                            const float* __restrict__ c0, const float* __restrict__ dimp,
                            const float* __restrict__ dh, const float* __restrict__ c, float* __restrict__ dpre,
                            float* __restrict__ part, int64_t R, int64_t n, int64_t b, int64_t rpb) {
  const int64_t u = 4 * ((int64_t)blockIdx.y * blockDim.x + threadIdx.x);
  if (u >= n) return;
  const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = min(r0 + rpb, R);
  float4 sf = make_float4(0, 0, 0, 0), so = sf, sz = sf;
#pragma unroll 2
  for (int64_t r = r0; r < r1; ++r) {
    const int64_t o = r * n + u;
    const float4 f = ld4(gf + o), og = ld4(go + o), z = ld4(gz + o);
    const float4 d_i = ld4(dimp + o), d_h = ld4(dh + o), cc = ld4(c + o);
    const float4 cp = r >= b ? *reinterpret_cast<const float4*>(c + o - b * n)
                             : (c0 != nullptr ? *reinterpret_cast<const float4*>(c0 + r * n + u) : make_float4(0, 0, 0, 0));
    float4 pf, po, pz;
#define LINREC_QDPRE(X)                                              \
  pf.X = (cp.X * d_i.X - d_i.X * z.X) * f.X * (1.f - f.X);           \
  po.X = (d_h.X * cc.X) * og.X * (1.f - og.X);                       \
  pz.X = d_i.X * (1.f - f.X) * (1.f - z.X * z.X);                    \
  sf.X += pf.X; so.X += po.X; sz.X += pz.X;
    LINREC_QDPRE(x) LINREC_QDPRE(y) LINREC_QDPRE(z) LINREC_QDPRE(w)
#undef LINREC_QDPRE
    float* d = dpre + r * 3 * n + u;
    st4(d, pf);
    st4(d + n, po);
    st4(d + 2 * n, pz);
  }
  float* pp = part + (int64_t)blockIdx.x * 3 * n + u;
  st4(pp, sf);
  st4(pp + n, so);
  st4(pp + 2 * n, sz);
}

}  // namespace layers
}  // namespace linrec_dev

// ---- optional per-stage timing (linrec_profile_begin / _end) ------------------
namespace {
struct Prof {
  bool on = false;
  std::vector<std::pair<std::string, cudaEvent_t>> marks;  // (stage that ENDS here, event)
};
Prof& prof() {
  static thread_local Prof p;
  return p;
}
// Records an event on `st` closing stage `name` (the previous mark opens it).
void mark(cudaStream_t st, const char* name) {
  Prof& p = prof();
  if (!p.on) return;
  cudaEvent_t e;
  if (cudaEventCreate(&e) != cudaSuccess) return;
  cudaEventRecord(e, st);
  p.marks.emplace_back(name, e);
}
}  // namespace

namespace {

using namespace linrec_dev::layers;
using linrec_impl::GemmEpilogue;
using linrec_impl::GemmOperands;

constexpr int kEpiPlain = 0, kEpiGilr = 1, kEpiGates = 2, kEpiQrnn = 3;

int sms() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

// Row partition of the pointwise gradient kernels: blocks of `thr` threads
// over n/4 unit quads, row chunks so the grid holds ~sms*1024 threads.
struct RowPlan {
  int thr;
  int64_t gy, nbx, rpb;
};
RowPlan row_plan(int64_t R, int64_t n) {
  RowPlan p;
  const int64_t quads = n / 4;
  p.thr = (int)(quads < 128 ? quads : 128);
  p.gy = (quads + p.thr - 1) / p.thr;
  const int64_t want = ((int64_t)sms() * 1024) / (p.thr * p.gy);
  p.nbx = want < 1 ? 1 : (want > R ? R : want);
  p.rpb = (R + p.nbx - 1) / p.nbx;
  p.nbx = (R + p.rpb - 1) / p.rpb;
  return p;
}

int64_t al(int64_t floats) { return (floats + 63) / 64 * 64; }  // 256-byte aligned carve-outs

struct Carve {
  float* base;
  int64_t off = 0;
  float* take(int64_t floats) {
    float* p = base ? base + off : nullptr;
    off += al(floats);
    return p;
  }
};

int64_t wsplit_floats(int64_t R, int64_t M, int64_t N) {
  return linrec_impl::gemm_partial_floats(M, N, linrec_impl::gemm_splits_for(M, N, R));
}

// ---- scratch layouts (one function drives sizing and carving) -------------
struct GilrScratch {
  float *imp, *uv, *uv_lo, *dl, *G, *dpre, *part, *split, *dh0;
};
int64_t gilr_scratch(float* base, int64_t T, int64_t b, int64_t m, int64_t n, GilrScratch* s) {
  const int64_t R = T * b;
  Carve c{base};
  GilrScratch t;
  t.uv = c.take(2 * n * m);
  t.uv_lo = c.take(2 * n * m);
  t.dh0 = c.take(b * n);
  const RowPlan rp = row_plan(R, n);
  t.part = c.take(rp.nbx * 2 * n);
  t.split = c.take(wsplit_floats(R, n, m));
  const int64_t common = c.off;
  // forward: imp; backward: dl, G, dpre (2n)
  Carve f{base, common};
  t.imp = f.take(R * n);
  Carve bw{base, common};
  t.dl = bw.take(R * n);
  t.G = bw.take(R * n);
  t.dpre = bw.take(2 * R * n);
  if (s) *s = t;
  return f.off > bw.off ? f.off : bw.off;
}

struct LstmScratch {
  float *uv, *uv_lo, *v_lo, *u_lo, *part, *split, *tmp0, *tmp1;
  float *iz;                                  // forward (also the surrogate impulses)
  float *dc, *df, *diz, *dpre, *dhp, *G;      // backward; dpre_s aliases df|diz, dls aliases dc
};
int64_t lstm_scratch(float* base, int64_t T, int64_t b, int64_t m, int64_t n, LstmScratch* s) {
  const int64_t R = T * b;
  Carve c{base};
  LstmScratch t;
  t.uv = c.take(2 * n * m);
  t.uv_lo = c.take(2 * n * m);
  t.v_lo = c.take(4 * n * m);
  t.u_lo = c.take(4 * n * n);
  t.tmp0 = c.take(b * n);
  t.tmp1 = c.take(b * n);
  const RowPlan rp = row_plan(R, n);
  t.part = c.take(rp.nbx * 4 * n);
  int64_t sp = wsplit_floats(R, 4 * n, n);
  const int64_t s2 = wsplit_floats(R, 4 * n, m), s3 = wsplit_floats(R, n, m);
  sp = sp > s2 ? sp : s2;
  sp = sp > s3 ? sp : s3;
  t.split = c.take(sp);
  const int64_t common = c.off;
  Carve f{base, common};
  t.iz = f.take(R * n);
  Carve bw{base, common};
  t.dc = bw.take(R * n);
  t.df = bw.take(2 * R * n);  // df | diz contiguous: reused as dpre_s [R][2n]
  t.diz = t.df ? t.df + R * n : nullptr;
  t.dpre = bw.take(4 * R * n);
  t.dhp = bw.take((R + b) * n);
  t.G = bw.take(R * n);
  if (s) *s = t;
  return f.off > bw.off ? f.off : bw.off;
}

struct QrnnScratch {
  float *part, *split, *tmp0, *w_lo;
  float *imp;                // forward
  float *dc, *df, *dimp, *dpre;  // backward
};
int64_t qrnn_scratch(float* base, int64_t T, int64_t b, int64_t m, int64_t n, int64_t k, QrnnScratch* s) {
  const int64_t R = T * b;
  Carve c{base};
  QrnnScratch t;
  t.tmp0 = c.take(b * n);
  t.w_lo = c.take(k * 3 * n * m);
  const RowPlan rp = row_plan(R, n);
  t.part = c.take(rp.nbx * 3 * n);
  const int64_t sp1 = wsplit_floats(R, 3 * n, m);
  const int64_t spk = m <= 8 ? linrec_impl::wgrad_taps_partial_floats(3 * n, m, R, (int)k) : 0;
  t.split = c.take(sp1 > spk ? sp1 : spk);  // one tap's partials, or all taps' (CUDA-core tap batch)
  const int64_t common = c.off;
  Carve f{base, common};
  t.imp = f.take(R * n);
  Carve bw{base, common};
  t.dc = bw.take(R * n);
  t.df = bw.take(R * n);
  t.dimp = bw.take(R * n);
  t.dpre = bw.take(3 * R * n);
  if (s) *s = t;
  return f.off > bw.off ? f.off : bw.off;
}

int err(int code, const std::string& m) { return linrec_impl::set_error(code, m.c_str()); }

#define LTRY(expr)                                                                      \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return err(LINREC_ERR_CUDA, std::string("linrec: CUDA error in ") + #expr + ": " + \
                                      cudaGetErrorString(e_));                          \
  } while (0)
#define LRC(expr)              \
  do {                         \
    int rc_ = (expr);          \
    if (rc_ != LINREC_OK) return rc_; \
  } while (0)

unsigned grid_for(int64_t n, int thr) {
  int64_t g = (n + thr - 1) / thr;
  const int64_t cap = (int64_t)sms() * 16;
  return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
}

int check_common(int64_t T, int64_t b, int64_t m, int64_t n, int mode, int precision, const void* x) {
  if (T < 1 || b < 1 || m < 1 || n < 1) return err(LINREC_ERR_SHAPE, "Tensor3 dimensions must be >= 1");
  if (m % 4 || n % 4)
    return err(LINREC_ERR_SHAPE, "layers: input and hidden sizes must be multiples of 4 (16-byte TMA rows)");
  if (T * b >= (int64_t(1) << 31)) return err(LINREC_ERR_SHAPE, "layers: T*b must be < 2^31");
  if (mode != LINREC_SERIAL && mode != LINREC_PARALLEL)
    return err(LINREC_ERR_VALUE, "mode must be \"parallel\" or \"serial\"");
  if (precision != LINREC_PREC_FP32 && precision != LINREC_PREC_TF32)
    return err(LINREC_ERR_VALUE, "precision must be LINREC_PREC_FP32 or LINREC_PREC_TF32");
  if (!x) return err(LINREC_ERR_VALUE, "x must not be NULL");
  return LINREC_OK;
}

int check_scratch(void* scratch, size_t have, int64_t need_floats) {
  if (!scratch || have < (size_t)need_floats * 4)
    return err(LINREC_ERR_VALUE, "layers: scratch is NULL or smaller than linrec_*_scratch_bytes()");
  if (reinterpret_cast<uintptr_t>(scratch) & 255) return err(LINREC_ERR_VALUE, "layers: scratch must be 256-byte aligned");
  return LINREC_OK;
}

// C (+)= A * B with the planner's split count
cudaError_t gemm(const GemmOperands& op, int epi, GemmEpilogue ep, bool split3, float* split_scratch,
                 cudaStream_t st) {
  ep.split3 = split3;
  if (epi == kEpiPlain && op.a_mn) {  // weight gradient: K = R rows, split across the grid
    ep.k_splits = linrec_impl::gemm_splits_for(op.M, op.units, op.K1);
    ep.scratch = split_scratch;
  }
  return linrec_impl::gemm_tf32(op, epi, ep, st);
}

// dW[M][N] += dpre_block^T * act, dpre_block = columns [0, M) of a [R][lda] matrix
cudaError_t wgrad(const float* dpre, int64_t lda, int64_t M, const float* act, int64_t N, int64_t R, float* dW,
                  bool split3, float* split_scratch, cudaStream_t st) {
  GemmOperands op;
  op.a1 = dpre;
  op.lda1 = lda;
  op.b1 = act;
  op.ldb1 = N;
  op.K1 = R;
  op.M = M;
  op.units = N;
  op.a_mn = op.b_mn = true;
  GemmEpilogue ep;
  ep.C = dW;
  ep.ldc = N;
  ep.accumulate = true;
  return gemm(op, kEpiPlain, ep, split3, split_scratch, st);
}

// gilr_forward core: g, i (cache), imp; then h = scan(g, imp, h0)
int gilr_forward_core(const linrec_gilr_params_f32* p, const float* x, const float* h0, float* h, float* g, float* ci,
                      float* imp, float* uv, float* uv_lo, int64_t T, int64_t b, int64_t m, int64_t n, int mode,
                      bool split3, cudaStream_t st) {
  const int64_t R = T * b;
  LTRY(cudaMemcpyAsync(uv, p->U, sizeof(float) * n * m, cudaMemcpyDeviceToDevice, st));
  LTRY(cudaMemcpyAsync(uv + n * m, p->V, sizeof(float) * n * m, cudaMemcpyDeviceToDevice, st));
  if (split3) LTRY(linrec_impl::tf32_lo(uv, uv_lo, 2 * n * m, st));
  mark(st, "prep");
  GemmOperands op;
  op.a1 = x;
  op.lda1 = m;
  op.b1 = uv;
  op.ldb1 = m;
  op.K1 = m;
  op.M = R;
  op.units = n;
  op.nb = 2;
  op.b_bstride = n;
  if (split3) op.b1_lo = uv_lo;
  GemmEpilogue ep;
  ep.act = p->act;
  ep.bias[0] = p->b_g;
  ep.bias[1] = p->b_z;
  ep.out[0] = g;
  ep.out[1] = ci;
  ep.out[2] = imp;
  ep.ldo = n;
  LTRY(gemm(op, kEpiGilr, ep, split3, nullptr, st));
  mark(st, "gemm_surrogate");
  LRC(linrec_scan_f32(g, imp, h0, h, T, b * n, mode, nullptr, st));
  mark(st, "scan_surrogate");
  return LINREC_OK;
}

// gilr_backward core.  dpre_s [R][2n] (dg | di), dl / G scratch; dx written
// (or, for the LSTM, produced by the caller's concatenated GEMM when
// dx == nullptr).
int gilr_backward_core(const linrec_gilr_params_f32* p, const float* x, const float* h0, const float* g,
                       const float* ci, const float* h, const float* dh, linrec_gilr_grads_f32* gr, float* dx,
                       float* dh0, float* dl, float* G, float* dpre_s, float* part, float* split, float* uv,
                       float* uv_lo, float* dh0_tmp, int64_t T, int64_t b, int64_t m, int64_t n, int mode,
                       bool split3, cudaStream_t st) {
  const int64_t R = T * b;
  mark(st, "prep");
  LRC(linrec_scan_backward_f32(g, h0, h, dh, nullptr, G, dh0 ? dh0 : dh0_tmp, T, b * n, mode, nullptr, st));
  mark(st, "scan_bwd_surrogate");
  const RowPlan rp = row_plan(R, n);
  (void)dl;
  k_gilr_dpre<<<dim3((unsigned)rp.nbx, (unsigned)rp.gy), rp.thr, 0, st>>>(g, ci, h, h0, G, p->act, dpre_s, part, R, n,
                                                                          b, rp.rpb);
  LTRY(cudaGetLastError());
  if (gr->b_g) {
    k_colsum<<<(unsigned)((n + 31) / 32), 1024, 0, st>>>(part, rp.nbx, 2 * n, n, gr->b_g);
    LTRY(cudaGetLastError());
  }
  if (gr->b_z) {  // partial sums of di are columns [n, 2n)
    k_colsum<<<(unsigned)((n + 31) / 32), 1024, 0, st>>>(part + n, rp.nbx, 2 * n, n, gr->b_z);
    LTRY(cudaGetLastError());
  }
  mark(st, "dpre_surrogate");
  if (gr->U) LTRY(wgrad(dpre_s, 2 * n, n, x, m, R, gr->U, split3, split, st));
  mark(st, "wgrad_surrogate_U");
  if (gr->V) LTRY(wgrad(dpre_s + n, 2 * n, n, x, m, R, gr->V, split3, split, st));
  mark(st, "wgrad_surrogate_V");
  if (dx) {
    LTRY(cudaMemcpyAsync(uv, p->U, sizeof(float) * n * m, cudaMemcpyDeviceToDevice, st));
    LTRY(cudaMemcpyAsync(uv + n * m, p->V, sizeof(float) * n * m, cudaMemcpyDeviceToDevice, st));
    if (split3) LTRY(linrec_impl::tf32_lo(uv, uv_lo, 2 * n * m, st));
    mark(st, "prep");
    GemmOperands op;  // dx = [dg | di] * [U; V]
    op.a1 = dpre_s;
    op.lda1 = 2 * n;
    op.b1 = uv;
    op.ldb1 = m;
    op.K1 = 2 * n;
    op.M = R;
    op.units = m;
    op.b_mn = true;
    if (split3) op.b1_lo = uv_lo;
    GemmEpilogue ep;
    ep.C = dx;
    ep.ldc = m;
    LTRY(gemm(op, kEpiPlain, ep, split3, nullptr, st));
    mark(st, "dx");
  }
  return LINREC_OK;
}

}  // namespace

extern "C" {

size_t linrec_qrnn_scratch_bytes(int64_t T, int64_t b, int64_t m, int64_t n, int64_t k) {
  if (T < 1 || b < 1 || m < 1 || n < 1 || k < 1) return 0;
  return (size_t)qrnn_scratch(nullptr, T, b, m, n, k, nullptr) * 4;
}

int linrec_qrnn_forward_f32(const float* W, const float* bias, const float* x, const float* c0, float* h,
                            float* gates, float* c, int64_t T, int64_t b, int64_t m, int64_t n, int64_t k, int mode,
                            int precision, void* scratch, size_t scratch_bytes, void* stream) {
  LRC(check_common(T, b, m, n, mode, precision, x));
  if (k < 1) return err(LINREC_ERR_SHAPE, "qrnn_init: window must be >= 1");
  if (k > T) return err(LINREC_ERR_SHAPE, "qrnn_forward: filter window exceeds sequence length");
  if (!W || !bias || !h || !gates || !c)
    return err(LINREC_ERR_VALUE, "qrnn_forward: W, bias, h, gates and c must not be NULL");
  LRC(check_scratch(scratch, scratch_bytes, qrnn_scratch(nullptr, T, b, m, n, k, nullptr)));
  QrnnScratch s;
  qrnn_scratch(static_cast<float*>(scratch), T, b, m, n, k, &s);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t R = T * b, N = R * n;
  float* gf = gates;
  float* go = gf + N;
  float* gz = go + N;
  mark(st, "begin");
  if (precision == LINREC_PREC_FP32) LTRY(linrec_impl::tf32_lo(W, s.w_lo, k * 3 * n * m, st));
  // pre[r] = bias + sum_s x[r - s*b] W_s^T: one GEMM whose K runs over the k
  // taps, tap s reading x shifted s*b rows down (zero-filled above row 0)
  GemmOperands op;
  op.a1 = x;
  op.lda1 = m;
  op.b1 = W;
  op.ldb1 = m;
  op.K1 = m;
  op.ntaps = (int)k;
  op.a_tap = -b;
  op.b_tap = 3 * n;
  op.M = R;
  op.units = n;
  op.nb = 3;
  op.b_bstride = n;
  if (precision == LINREC_PREC_FP32) op.b1_lo = s.w_lo;
  GemmEpilogue ep;
  for (int q = 0; q < 3; ++q) ep.bias[q] = bias + q * n;
  ep.out[0] = gf;
  ep.out[1] = go;
  ep.out[2] = gz;
  ep.out[3] = s.imp;
  ep.ldo = n;
  LTRY(gemm(op, kEpiQrnn, ep, precision == LINREC_PREC_FP32, nullptr, st));
  mark(st, "gemm_gates");
  LRC(linrec_scan_f32(gf, s.imp, c0, c, T, b * n, mode, nullptr, st));
  mark(st, "scan_cell");
  k_mul<<<grid_for(N / 4, 256), 256, 0, st>>>(go, c, h, N / 4);
  LTRY(cudaGetLastError());
  mark(st, "h_out");
  return LINREC_OK;
}

int linrec_qrnn_backward_f32(const float* W, const float* x, const float* c0, const float* gates, const float* c,
                             const float* dh, float* dW, float* dbias, float* dx, float* dc0, int64_t T, int64_t b,
                             int64_t m, int64_t n, int64_t k, int mode, int precision, void* scratch,
                             size_t scratch_bytes, void* stream) {
  LRC(check_common(T, b, m, n, mode, precision, x));
  if (k < 1 || k > T) return err(LINREC_ERR_SHAPE, "qrnn_backward: window must be in [1, T]");
  if (!W || !gates || !c || !dh || !dx)
    return err(LINREC_ERR_VALUE, "qrnn_backward: W, gates, c, d_h and dx must not be NULL");
  LRC(check_scratch(scratch, scratch_bytes, qrnn_scratch(nullptr, T, b, m, n, k, nullptr)));
  QrnnScratch s;
  qrnn_scratch(static_cast<float*>(scratch), T, b, m, n, k, &s);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool split3 = precision == LINREC_PREC_FP32;
  const int64_t R = T * b, N = R * n;
  const float* gf = gates;
  const float* go = gf + N;
  const float* gz = go + N;
  mark(st, "begin");
  // dc = dh * o fused into the cell scan's backward (layers.hpp:510-521)
  LRC(linrec_scan_backward_gated_f32(gf, c0, c, dh, go, nullptr, s.dimp, dc0 ? dc0 : s.tmp0, T, b * n, mode, nullptr,
                                     st));
  mark(st, "scan_bwd_cell");
  const RowPlan rp = row_plan(R, n);
  k_qrnn_dpre<<<dim3((unsigned)rp.nbx, (unsigned)rp.gy), rp.thr, 0, st>>>(gf, go, gz, c0, s.dimp, dh, c, s.dpre,
                                                                          s.part, R, n, b, rp.rpb);
  LTRY(cudaGetLastError());
  if (dbias) {
    k_colsum<<<(unsigned)((3 * n + 31) / 32), 1024, 0, st>>>(s.part, rp.nbx, 3 * n, 3 * n, dbias);
    LTRY(cudaGetLastError());
  }
  mark(st, "dpre_gates");
  // dW_s += dpre[s*b ..]^T x[.. R - s*b]  (layers.hpp:536-539): all taps in one
  // CUDA-core launch when x is narrow (one HBM pass over dpre), else per tap
  if (dW) {
    const cudaError_t et =
        linrec_impl::wgrad_taps_skinny(s.dpre, 3 * n, x, m, R, b, (int)k, 3 * n, m, dW, s.split, st);
    if (et == cudaErrorNotSupported) {
      for (int64_t tap = 0; tap < k; ++tap)
        LTRY(wgrad(s.dpre + tap * b * 3 * n, 3 * n, 3 * n, x, m, R - tap * b, dW + tap * 3 * n * m, split3,
                   s.split, st));
    } else {
      LTRY(et);
    }
  }
  mark(st, "wgrad_W");
  // dx[r] = sum_s dpre[r + s*b] W_s  (:540-543): one GEMM over the taps,
  // tap s reading dpre shifted s*b rows up (zero-filled past row R)
  {
    GemmOperands op;
    op.a1 = s.dpre;
    op.lda1 = 3 * n;
    op.b1 = W;
    op.ldb1 = m;
    op.K1 = 3 * n;
    op.ntaps = (int)k;
    op.a_tap = b;
    op.b_tap = 3 * n;
    op.M = R;
    op.units = m;
    op.b_mn = true;
    if (split3) {
      LTRY(linrec_impl::tf32_lo(W, s.w_lo, k * 3 * n * m, st));
      op.b1_lo = s.w_lo;
    }
    GemmEpilogue ep;
    ep.C = dx;
    ep.ldc = m;
    LTRY(gemm(op, kEpiPlain, ep, split3, nullptr, st));
  }
  mark(st, "dx");
  return LINREC_OK;
}

int linrec_profile_begin(void) {
  Prof& p = prof();
  for (auto& m : p.marks) cudaEventDestroy(m.second);
  p.marks.clear();
  p.on = true;
  return LINREC_OK;
}

int linrec_profile_end(char* out, size_t cap) {
  Prof& p = prof();
  p.on = false;
  std::map<std::string, std::pair<double, int>> acc;  // name -> (ms, count)
  std::vector<std::string> order;
  int rc = LINREC_OK;
  for (size_t k = 1; k < p.marks.size(); ++k) {
    if (p.marks[k].first == "begin") continue;
    float ms = 0.f;
    if (cudaEventSynchronize(p.marks[k].second) != cudaSuccess ||
        cudaEventElapsedTime(&ms, p.marks[k - 1].second, p.marks[k].second) != cudaSuccess) {
      rc = err(LINREC_ERR_CUDA, "linrec_profile_end: event timing failed");
      break;
    }
    auto it = acc.find(p.marks[k].first);
    if (it == acc.end()) {
      order.push_back(p.marks[k].first);
      acc[p.marks[k].first] = {ms, 1};
    } else {
      it->second.first += ms;
      it->second.second += 1;
    }
  }
  for (auto& m : p.marks) cudaEventDestroy(m.second);
  p.marks.clear();
  std::string s;
  for (auto& n : order) {
    char buf[160];
    snprintf(buf, sizeof buf, "%s %.6f %d\n", n.c_str(), acc[n].first, acc[n].second);
    s += buf;
  }
  if (out && cap) {
    const size_t k = s.size() < cap - 1 ? s.size() : cap - 1;
    memcpy(out, s.data(), k);
    out[k] = 0;
    if (s.size() >= cap) return err(LINREC_ERR_VALUE, "linrec_profile_end: buffer too small");
  }
  return rc;
}

size_t linrec_gilr_scratch_bytes(int64_t T, int64_t b, int64_t m, int64_t n) {
  if (T < 1 || b < 1 || m < 1 || n < 1) return 0;
  return (size_t)gilr_scratch(nullptr, T, b, m, n, nullptr) * 4;
}

size_t linrec_gilr_lstm_scratch_bytes(int64_t T, int64_t b, int64_t m, int64_t n) {
  if (T < 1 || b < 1 || m < 1 || n < 1) return 0;
  return (size_t)lstm_scratch(nullptr, T, b, m, n, nullptr) * 4;
}

int linrec_gilr_forward_f32(const linrec_gilr_params_f32* p, const float* x, const float* h0, float* h, float* g,
                            float* i, int64_t T, int64_t b, int64_t m, int64_t n, int mode, int precision,
                            void* scratch, size_t scratch_bytes, void* stream) {
  LRC(check_common(T, b, m, n, mode, precision, x));
  if (!p || !p->U || !p->V || !p->b_g || !p->b_z || !h || !g || !i)
    return err(LINREC_ERR_VALUE, "gilr_forward: parameters, h and the cache (g, i) must not be NULL");
  GilrScratch s;
  LRC(check_scratch(scratch, scratch_bytes, gilr_scratch(nullptr, T, b, m, n, nullptr)));
  gilr_scratch(static_cast<float*>(scratch), T, b, m, n, &s);
  mark(static_cast<cudaStream_t>(stream), "begin");
  return gilr_forward_core(p, x, h0, h, g, i, s.imp, s.uv, s.uv_lo, T, b, m, n, mode,
                           precision == LINREC_PREC_FP32, static_cast<cudaStream_t>(stream));
}

int linrec_gilr_backward_f32(const linrec_gilr_params_f32* p, const float* x, const float* h0, const float* g,
                             const float* i, const float* h, const float* dh, linrec_gilr_grads_f32* grads,
                             float* dx, float* dh0, int64_t T, int64_t b, int64_t m, int64_t n, int mode,
                             int precision, void* scratch, size_t scratch_bytes, void* stream) {
  LRC(check_common(T, b, m, n, mode, precision, x));
  if (!p || !p->U || !p->V || !g || !i || !h || !dh || !grads || !dx)
    return err(LINREC_ERR_VALUE, "gilr_backward: parameters, cache, d_h, grads and dx must not be NULL");
  GilrScratch s;
  LRC(check_scratch(scratch, scratch_bytes, gilr_scratch(nullptr, T, b, m, n, nullptr)));
  gilr_scratch(static_cast<float*>(scratch), T, b, m, n, &s);
  mark(static_cast<cudaStream_t>(stream), "begin");
  return gilr_backward_core(p, x, h0, g, i, h, dh, grads, dx, dh0, s.dl, s.G, s.dpre, s.part, s.split, s.uv,
                            s.uv_lo, s.dh0, T, b, m, n, mode, precision == LINREC_PREC_FP32,
                            static_cast<cudaStream_t>(stream));
}

int linrec_gilr_lstm_forward_f32(const linrec_gilr_lstm_params_f32* p, const float* x, const float* htil0,
                                 const float* c0, float* h, const linrec_gilr_lstm_cache_f32* cache, int64_t T,
                                 int64_t b, int64_t m, int64_t n, int mode, int precision, void* scratch,
                                 size_t scratch_bytes, void* stream) {
  LRC(check_common(T, b, m, n, mode, precision, x));
  if (!p || !p->U || !p->V || !p->bias || !p->surrogate.U || !p->surrogate.V || !p->surrogate.b_g ||
      !p->surrogate.b_z || !h || !cache || !cache->sg || !cache->si || !cache->htil || !cache->gates || !cache->c)
    return err(LINREC_ERR_VALUE, "gilr_lstm_forward: parameters, h and every cache buffer must not be NULL");
  LRC(check_scratch(scratch, scratch_bytes, lstm_scratch(nullptr, T, b, m, n, nullptr)));
  LstmScratch s;
  lstm_scratch(static_cast<float*>(scratch), T, b, m, n, &s);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool split3 = precision == LINREC_PREC_FP32;
  const int64_t R = T * b, BN = b * n, N = R * n;
  mark(st, "begin");
  // 1-2. surrogate; its output lands one row block after htil0
  if (htil0) LTRY(cudaMemcpyAsync(cache->htil, htil0, sizeof(float) * BN, cudaMemcpyDeviceToDevice, st));
  else LTRY(cudaMemsetAsync(cache->htil, 0, sizeof(float) * BN, st));
  LRC(gilr_forward_core(&p->surrogate, x, htil0, cache->htil + BN, cache->sg, cache->si, s.iz, s.uv, s.uv_lo, T, b,
                        m, n, mode, split3, st));
  if (split3) {
    LTRY(linrec_impl::tf32_lo(p->V, s.v_lo, 4 * n * m, st));
    LTRY(linrec_impl::tf32_lo(p->U, s.u_lo, 4 * n * n, st));
  }
  // 3. gates = act([x | htil_prev] [V | U]^T + bias)
  float* gf = cache->gates;
  float* gi = gf + N;
  float* go = gi + N;
  float* gz = go + N;
  GemmOperands op;
  op.a1 = x;
  op.lda1 = m;
  op.b1 = p->V;
  op.ldb1 = m;
  op.K1 = m;
  op.a2 = cache->htil;  // rows 0..R-1 = htil_prev
  op.lda2 = n;
  op.b2 = p->U;
  op.ldb2 = n;
  op.K2 = n;
  op.M = R;
  op.units = n;
  op.nb = 4;
  op.b_bstride = n;
  if (split3) {
    op.b1_lo = s.v_lo;
    op.b2_lo = s.u_lo;
  }
  GemmEpilogue ep;
  for (int q = 0; q < 4; ++q) ep.bias[q] = p->bias + q * n;
  ep.out[0] = gf;
  ep.out[1] = gi;
  ep.out[2] = go;
  ep.out[3] = gz;
  ep.out[4] = s.iz;
  ep.ldo = n;
  LTRY(gemm(op, kEpiGates, ep, split3, nullptr, st));
  mark(st, "gemm_gates");
  // 4-5. c = scan(f, i*z, c0); h = o * c
  LRC(linrec_scan_f32(gf, s.iz, c0, cache->c, T, BN, mode, nullptr, st));
  mark(st, "scan_cell");
  k_mul<<<grid_for(N / 4, 256), 256, 0, st>>>(go, cache->c, h, N / 4);
  LTRY(cudaGetLastError());
  mark(st, "h_out");
  return LINREC_OK;
}

int linrec_gilr_lstm_backward_f32(const linrec_gilr_lstm_params_f32* p, const float* x, const float* htil0,
                                  const float* c0, const linrec_gilr_lstm_cache_f32* cache, const float* dh,
                                  linrec_gilr_lstm_grads_f32* grads, float* dx, float* dhtil0, float* dc0,
                                  int64_t T, int64_t b, int64_t m, int64_t n, int mode, int precision,
                                  void* scratch, size_t scratch_bytes, void* stream) {
  LRC(check_common(T, b, m, n, mode, precision, x));
  if (!p || !p->U || !p->V || !p->surrogate.U || !p->surrogate.V || !cache || !cache->sg || !cache->si ||
      !cache->htil || !cache->gates || !cache->c || !dh || !grads || !dx)
    return err(LINREC_ERR_VALUE, "gilr_lstm_backward: parameters, cache, d_h, grads and dx must not be NULL");
  LRC(check_scratch(scratch, scratch_bytes, lstm_scratch(nullptr, T, b, m, n, nullptr)));
  LstmScratch s;
  lstm_scratch(static_cast<float*>(scratch), T, b, m, n, &s);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool split3 = precision == LINREC_PREC_FP32;
  const int64_t R = T * b, BN = b * n, N = R * n;
  const float* gf = cache->gates;
  const float* gi = gf + N;
  const float* go = gi + N;
  const float* gz = go + N;
  mark(st, "begin");
  if (split3) {
    LTRY(linrec_impl::tf32_lo(p->V, s.v_lo, 4 * n * m, st));
    LTRY(linrec_impl::tf32_lo(p->U, s.u_lo, 4 * n * n, st));
  }
  // h = o * c  ->  dc = dh * o, fused into the cell scan's backward (the scan
  // stages dh and o and multiplies them as it reads; layers.hpp:312-324);
  // d_o is formed inside k_lstm_dpre
  LRC(linrec_scan_backward_gated_f32(gf, c0, cache->c, dh, go, nullptr, s.diz, dc0 ? dc0 : s.tmp0, T, BN, mode,
                                     nullptr, st));
  mark(st, "scan_bwd_cell");
  const RowPlan rp = row_plan(R, n);
  k_lstm_dpre<<<dim3((unsigned)rp.nbx, (unsigned)rp.gy), rp.thr, 0, st>>>(gf, gi, go, gz, c0, s.diz, dh, cache->c,
                                                                          s.dpre, s.part, R, n, b, rp.rpb);
  LTRY(cudaGetLastError());
  if (grads->bias) {
    k_colsum<<<(unsigned)((4 * n + 31) / 32), 1024, 0, st>>>(s.part, rp.nbx, 4 * n, 4 * n, grads->bias);
    LTRY(cudaGetLastError());
  }
  mark(st, "dpre_gates");
  // dU += dpre^T htil_prev ; dV += dpre^T x
  if (grads->U) LTRY(wgrad(s.dpre, 4 * n, 4 * n, cache->htil, n, R, grads->U, split3, s.split, st));
  mark(st, "wgrad_U");
  if (grads->V) LTRY(wgrad(s.dpre, 4 * n, 4 * n, x, m, R, grads->V, split3, s.split, st));
  mark(st, "wgrad_V");
  // dhp = dpre U  (gradient w.r.t. htil_prev); the row block after the last is 0
  {
    GemmOperands op;
    op.a1 = s.dpre;
    op.lda1 = 4 * n;
    op.b1 = p->U;
    op.ldb1 = n;
    op.K1 = 4 * n;
    op.M = R;
    op.units = n;
    op.b_mn = true;
    if (split3) op.b1_lo = s.u_lo;
    GemmEpilogue ep;
    ep.C = s.dhp;
    ep.ldc = n;
    LTRY(gemm(op, kEpiPlain, ep, split3, nullptr, st));
    LTRY(cudaMemsetAsync(s.dhp + N, 0, sizeof(float) * BN, st));
    mark(st, "dhtil_prev");
  }
  // surrogate backward on d_htil[t] = dhp[t+1] (pointer shift); dpre_s in df|diz
  float* dpre_s = s.df;
  LRC(gilr_backward_core(&p->surrogate, x, htil0, cache->sg, cache->si, cache->htil + BN, s.dhp + BN,
                         &grads->surrogate, nullptr, nullptr, s.dc, s.G, dpre_s, s.part, s.split, s.uv, s.uv_lo, s.tmp1,
                         T, b, m, n, mode, split3, st));
  // dx = dpre V + [dg | di] [U_s; V_s]   (one K-concatenated GEMM)
  LTRY(cudaMemcpyAsync(s.uv, p->surrogate.U, sizeof(float) * n * m, cudaMemcpyDeviceToDevice, st));
  LTRY(cudaMemcpyAsync(s.uv + n * m, p->surrogate.V, sizeof(float) * n * m, cudaMemcpyDeviceToDevice, st));
  if (split3) LTRY(linrec_impl::tf32_lo(s.uv, s.uv_lo, 2 * n * m, st));
  mark(st, "prep");
  {
    GemmOperands op;
    op.a1 = s.dpre;
    op.lda1 = 4 * n;
    op.b1 = p->V;
    op.ldb1 = m;
    op.K1 = 4 * n;
    op.a2 = dpre_s;
    op.lda2 = 2 * n;
    op.b2 = s.uv;
    op.ldb2 = m;
    op.K2 = 2 * n;
    op.M = R;
    op.units = m;
    op.b_mn = true;
    if (split3) {
      op.b1_lo = s.v_lo;
      op.b2_lo = s.uv_lo;
    }
    GemmEpilogue ep;
    ep.C = dx;
    ep.ldc = m;
    LTRY(gemm(op, kEpiPlain, ep, split3, nullptr, st));
    mark(st, "dx");
  }
  // htil0 feeds the surrogate scan and the t=1 gate input (:364-370)
  if (dhtil0) {
    k_add<<<grid_for(BN, 256), 256, 0, st>>>(s.tmp1, s.dhp, dhtil0, BN);
    LTRY(cudaGetLastError());
    mark(st, "dhtil0");
  }
  return LINREC_OK;
}

}  // extern "C"
