// GILR, GILR-LSTM and QRNN in double precision (layers.hpp:23-548 are
// templated on S; proj/tests/test_layers.cpp runs them in double).  Same
// orchestration as the fp32 layers (layers.cu), with the projections on a
// CUDA-core fp64 GEMM (the tcgen05 kind::tf32 path has no fp64 operand
// type) and the activations as separate pointwise passes:
//
//   forward   pre = x W^T (+ htil_prev U^T, + the QRNN taps)   k_dgemm
//             gates / impulses from pre + bias                 k_*_gates64
//             state = scan(decay, impulse, initial)            linrec_scan_f64
//             h = o * c                                        k_mul64
//   backward  dc = dh * o; scan_backward (dlam folded below)   linrec_scan_backward_f64
//             dpre (+ per-block bias partials)                  k_*_dpre64, k_colpart64
//             dW += dpre^T act (split-K, fixed-order reduce)    k_dgemm + k_dsplit_reduce
//             dx  = dpre W (+ the second operand / taps)       k_dgemm
//
// Every sum has a fixed association (run-to-run bit-identical).  Widths need
// not be multiples of 4 (no TMA rows here).
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "launch.h"
#include "linrec_cuda.h"

namespace linrec_dev {
namespace layers64 {

// ---- C[M][N] (+)= sum_k A(m,k) B(k,n), A(m,k) = A[m*sam + k*sak], B(k,n) = B[k*sbk + n*sbn]
constexpr int BM = 64, BN = 64, BK = 16;

struct Gm {
  const double* A;
  int64_t sam, sak;
  const double* B;
  int64_t sbk, sbn;
  double* C;
  int64_t ldc, M, N, K, kchunk;
  int accumulate;
  double* part;  // split-K partials [splits][M][N] (nullptr: write C)
};

// 64 x 64 tile per CTA of 256 threads, 4 x 4 outputs per thread (rows
// ty + 16 i, columns tx + 16 j), K in steps of 16 through shared memory;
// blockIdx.z = the K split.  Loads run along whichever index is unit-stride.
__global__ void __launch_bounds__(256) k_dgemm(Gm g) {
  __shared__ double As[BK][BM + 1], Bs[BK][BN + 1];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;  // rows on x: R may exceed 65535 tiles
  const int64_t kb = (int64_t)blockIdx.z * g.kchunk;
  const int64_t ke = kb + g.kchunk < g.K ? kb + g.kchunk : g.K;
  const bool a_m1 = g.sam == 1, b_n1 = g.sbn == 1;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int64_t k0 = kb; k0 < ke; k0 += BK) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int mm, kk;
      if (a_m1) {
        mm = tid & 63;
        kk = (tid >> 6) + 4 * e;
      } else {
        kk = tid & 15;
        mm = (tid >> 4) + 16 * e;
      }
      const int64_t m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < g.M && k < ke) ? g.A[m * g.sam + k * g.sak] : 0.0;
      int nn, kq;
      if (b_n1) {
        nn = tid & 63;
        kq = (tid >> 6) + 4 * e;
      } else {
        kq = tid & 15;
        nn = (tid >> 4) + 16 * e;
      }
      const int64_t n = n0 + nn, k2 = k0 + kq;
      Bs[kq][nn] = (n < g.N && k2 < ke) ? g.B[k2 * g.sbk + n * g.sbn] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty + 16 * i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + tx + 16 * j;
      if (n >= g.N) continue;
      if (g.part != nullptr) {
        g.part[((int64_t)blockIdx.z * g.M + m) * g.N + n] = acc[i][j];
      } else {
        double* c = g.C + m * g.ldc + n;
        *c = g.accumulate ? *c + acc[i][j] : acc[i][j];
      }
    }
  }
}

// C (+)= sum over splits z = 0, 1, ... of part[z] (fixed order)
__global__ void k_dsplit_reduce(const double* __restrict__ part, int splits, int64_t M, int64_t N,
                                double* __restrict__ C, int64_t ldc, int accumulate) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < M * N; e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += part[(int64_t)z * M * N + e];
    double* c = C + (e / N) * ldc + e % N;
    *c = accumulate ? *c + s : s;
  }
}

// ---- pointwise (activation_fn / activation_deriv_from_value, common.hpp:49-71)
__device__ __forceinline__ double sigm(double z) { return 1.0 / (1.0 + exp(-z)); }
__device__ __forceinline__ double actf(int a, double z) { return a == 0 ? tanh(z) : a == 1 ? z : (z > 0.0 ? z : 0.0); }
__device__ __forceinline__ double dactv(int a, double v) {
  return a == 0 ? 1.0 - v * v : a == 1 ? 1.0 : (v > 0.0 ? 1.0 : 0.0);
}

#define LINREC_GRID_LOOP(i, n) \
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// GILR gates (layers.hpp:84-95): pre [R][2n] = (x U^T | x V^T)
__global__ void k_gilr_gates64(const double* __restrict__ pre, const double* __restrict__ bg,
                               const double* __restrict__ bz, int act, double* __restrict__ g,
                               double* __restrict__ ci, double* __restrict__ imp, int64_t R, int64_t n) {
  LINREC_GRID_LOOP(e, R * n) {
    const int64_t r = e / n, j = e % n;
    const double gv = sigm(pre[r * 2 * n + j] + bg[j]);
    const double iv = actf(act, pre[r * 2 * n + n + j] + bz[j]);
    g[e] = gv;
    ci[e] = iv;
    imp[e] = (1.0 - gv) * iv;
  }
}

// GILR-LSTM gates (layers.hpp:262-285): pre [R][4n] blocks f, i, o, z ->
// activated planes and the cell impulses i * z
__global__ void k_lstm_gates64(const double* __restrict__ pre, const double* __restrict__ bias,
                               double* __restrict__ gates, double* __restrict__ iz, int64_t R, int64_t n) {
  const int64_t N = R * n;
  LINREC_GRID_LOOP(e, N) {
    const int64_t r = e / n, j = e % n;
    const double* p = pre + r * 4 * n;
    const double f = sigm(p[j] + bias[j]), i = sigm(p[n + j] + bias[n + j]);
    const double o = sigm(p[2 * n + j] + bias[2 * n + j]), z = tanh(p[3 * n + j] + bias[3 * n + j]);
    gates[e] = f;
    gates[N + e] = i;
    gates[2 * N + e] = o;
    gates[3 * N + e] = z;
    iz[e] = i * z;
  }
}

// QRNN gates (layers.hpp:471-484): pre [R][3n] blocks f, o, z -> planes and
// the impulses (1 - f) * z
__global__ void k_qrnn_gates64(const double* __restrict__ pre, const double* __restrict__ bias,
                               double* __restrict__ gates, double* __restrict__ imp, int64_t R, int64_t n) {
  const int64_t N = R * n;
  LINREC_GRID_LOOP(e, N) {
    const int64_t r = e / n, j = e % n;
    const double* p = pre + r * 3 * n;
    const double f = sigm(p[j] + bias[j]), o = sigm(p[n + j] + bias[n + j]), z = tanh(p[2 * n + j] + bias[2 * n + j]);
    gates[e] = f;
    gates[N + e] = o;
    gates[2 * N + e] = z;
    imp[e] = (1.0 - f) * z;
  }
}

__global__ void k_mul64(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out,
                        int64_t n) {
  LINREC_GRID_LOOP(e, n) out[e] = a[e] * b[e];
}

__global__ void k_add64(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out,
                        int64_t n) {
  LINREC_GRID_LOOP(e, n) out[e] = a[e] + b[e];
}

// The state row before row r: row r - b of s, or the initial state (zeros if
// NULL) for the first time step.
__device__ __forceinline__ double prev_row(const double* s, const double* s0, int64_t r, int64_t j, int64_t n,
                                           int64_t b) {
  return r >= b ? s[(r - b) * n + j] : (s0 != nullptr ? s0[r * n + j] : 0.0);
}

// GILR pre-activation gradients (layers.hpp:112-121), dl = h_{t-1} G formed
// here: dpre [R][2n] = (dg | di)
__global__ void k_gilr_dpre64(const double* __restrict__ g, const double* __restrict__ ci,
                              const double* __restrict__ h, const double* __restrict__ h0,
                              const double* __restrict__ G, int act, double* __restrict__ dpre, int64_t R, int64_t n,
                              int64_t b) {
  LINREC_GRID_LOOP(e, R * n) {
    const int64_t r = e / n, j = e % n;
    const double gv = g[e], iv = ci[e], Gv = G[e];
    const double dl = prev_row(h, h0, r, j, n, b) * Gv;
    dpre[r * 2 * n + j] = (dl - Gv * iv) * gv * (1.0 - gv);
    dpre[r * 2 * n + n + j] = Gv * (1.0 - gv) * dactv(act, iv);
  }
}

// GILR-LSTM pre-activation gradients (layers.hpp:327-342): dpre [R][4n]
__global__ void k_lstm_dpre64(const double* __restrict__ gates, const double* __restrict__ c0,
                              const double* __restrict__ diz, const double* __restrict__ dh,
                              const double* __restrict__ c, double* __restrict__ dpre, int64_t R, int64_t n,
                              int64_t b) {
  const int64_t N = R * n;
  LINREC_GRID_LOOP(e, N) {
    const int64_t r = e / n, j = e % n;
    const double f = gates[e], i = gates[N + e], o = gates[2 * N + e], z = gates[3 * N + e];
    const double d_iz = diz[e], df = prev_row(c, c0, r, j, n, b) * d_iz;
    double* d = dpre + r * 4 * n;
    d[j] = df * f * (1.0 - f);
    d[n + j] = d_iz * z * i * (1.0 - i);
    d[2 * n + j] = (dh[e] * c[e]) * o * (1.0 - o);
    d[3 * n + j] = d_iz * i * (1.0 - z * z);
  }
}

// QRNN pre-activation gradients (layers.hpp:519-531): dpre [R][3n]
__global__ void k_qrnn_dpre64(const double* __restrict__ gates, const double* __restrict__ c0,
                              const double* __restrict__ dimp, const double* __restrict__ dh,
                              const double* __restrict__ c, double* __restrict__ dpre, int64_t R, int64_t n,
                              int64_t b) {
  const int64_t N = R * n;
  LINREC_GRID_LOOP(e, N) {
    const int64_t r = e / n, j = e % n;
    const double f = gates[e], o = gates[N + e], z = gates[2 * N + e];
    const double di = dimp[e], df = prev_row(c, c0, r, j, n, b) * di;
    double* d = dpre + r * 3 * n;
    d[j] = (df - di * z) * f * (1.0 - f);
    d[n + j] = (dh[e] * c[e]) * o * (1.0 - o);
    d[2 * n + j] = di * (1.0 - f) * (1.0 - z * z);
  }
}

// Column sums of d [R][ld] columns [0, C): block (x, y) sums rows
// [y*rpb, (y+1)*rpb) of its 256 columns in row order into part[y][C]; then
// dst[c] += the partials in block order (accumulate_bias_grad, tensor.hpp:286-296).
__global__ void k_colpart64(const double* __restrict__ d, int64_t R, int64_t C, int64_t ld, int64_t rpb,
                            double* __restrict__ part) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const int64_t r0 = (int64_t)blockIdx.y * rpb, r1 = r0 + rpb < R ? r0 + rpb : R;
  double s = 0.0;
  for (int64_t r = r0; r < r1; ++r) s += d[r * ld + c];
  part[(int64_t)blockIdx.y * C + c] = s;
}

__global__ void k_colsum64(const double* __restrict__ part, int64_t nb, int64_t C, double* __restrict__ dst) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double s = 0.0;
  for (int64_t y = 0; y < nb; ++y) s += part[y * C + c];
  dst[c] += s;
}

}  // namespace layers64
}  // namespace linrec_dev

namespace {

using namespace linrec_dev::layers64;

constexpr int kMaxSplits = 16;

int sms64() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

int err64(int code, const std::string& m) { return linrec_impl::set_error(code, m.c_str()); }

#define DTRY(expr)                                                                        \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return err64(LINREC_ERR_CUDA, std::string("linrec: CUDA error in ") + #expr + ": " + \
                                        cudaGetErrorString(e_));                          \
  } while (0)
#define DRC(expr)                     \
  do {                                \
    int rc_ = (expr);                 \
    if (rc_ != LINREC_OK) return rc_; \
  } while (0)

unsigned grid64(int64_t n) {
  const int64_t g = (n + 255) / 256, cap = (int64_t)sms64() * 8;
  return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
}

// split count for an M x N x K product: fill ~2 waves of CTAs when the tile
// grid alone does not, keep >= 256 K per split
int splits_for(int64_t M, int64_t N, int64_t K) {
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  int64_t s = (2 * sms64() + tiles - 1) / tiles;
  if (s > K / 256) s = K / 256;
  if (s > kMaxSplits) s = kMaxSplits;
  return (int)(s < 1 ? 1 : s);
}

// C[M][N] (+)= A B with the strides of Gm; split-K through `part` (room for
// kMaxSplits * M * N doubles) when it is given and the product is tall in K.
int dgemm(const double* A, int64_t sam, int64_t sak, const double* B, int64_t sbk, int64_t sbn, double* C,
          int64_t ldc, int64_t M, int64_t N, int64_t K, bool accumulate, double* part, cudaStream_t st) {
  if (M <= 0 || N <= 0) return LINREC_OK;
  if (K <= 0) {  // empty sum: C = 0 or unchanged
    if (!accumulate)
      for (int64_t m = 0; m < M; ++m) DTRY(cudaMemsetAsync(C + m * ldc, 0, sizeof(double) * N, st));
    return LINREC_OK;
  }
  const int splits = part != nullptr ? splits_for(M, N, K) : 1;
  int64_t kchunk = (K + splits - 1) / splits;
  kchunk = (kchunk + BK - 1) / BK * BK;
  const int used = (int)((K + kchunk - 1) / kchunk);
  Gm g{A, sam, sak, B, sbk, sbn, C, ldc, M, N, K, kchunk, accumulate ? 1 : 0, used > 1 ? part : nullptr};
  if ((N + BN - 1) / BN > 65535) return err64(LINREC_ERR_SHAPE, "gemm_f64: N too large");
  const dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((N + BN - 1) / BN), (unsigned)used);
  k_dgemm<<<grid, 256, 0, st>>>(g);
  DTRY(cudaGetLastError());
  if (used > 1) {
    k_dsplit_reduce<<<grid64(M * N), 256, 0, st>>>(part, used, M, N, C, ldc, accumulate ? 1 : 0);
    DTRY(cudaGetLastError());
  }
  return LINREC_OK;
}

// out[R][N] (+)= act[R][K] W^T, W [N][K] row-major (affine, tensor.hpp:249-270)
int affine64(const double* act, int64_t lda, const double* W, int64_t ldw, double* out, int64_t ldo, int64_t R,
             int64_t N, int64_t K, bool accumulate, cudaStream_t st) {
  return dgemm(act, lda, 1, W, 1, ldw, out, ldo, R, N, K, accumulate, nullptr, st);
}

// dW[N][K] += d[R][N]^T act[R][K] (accumulate_weight_grad, tensor.hpp:272-284)
int wgrad64(const double* d, int64_t ldd, const double* act, int64_t lda, double* dW, int64_t ldw, int64_t R,
            int64_t N, int64_t K, double* part, cudaStream_t st) {
  return dgemm(d, 1, ldd, act, lda, 1, dW, ldw, N, K, R, true, part, st);
}

// dx[R][K] (+)= d[R][N] W, W [N][K] (accumulate_input_grad, tensor.hpp:298-308)
int igrad64(const double* d, int64_t ldd, const double* W, int64_t ldw, double* dx, int64_t ldx, int64_t R,
            int64_t N, int64_t K, bool accumulate, cudaStream_t st) {
  return dgemm(d, ldd, 1, W, ldw, 1, dx, ldx, R, K, N, accumulate, nullptr, st);
}

// dst[C] += column sums of d [R][ld] columns [0, C)
int bgrad64(const double* d, int64_t ld, int64_t R, int64_t C, double* part, double* dst, cudaStream_t st) {
  if (dst == nullptr) return LINREC_OK;
  const int64_t rpb = R > 512 ? (R + 511) / 512 : 1, nb = (R + rpb - 1) / rpb;
  k_colpart64<<<dim3((unsigned)((C + 255) / 256), (unsigned)nb), 256, 0, st>>>(d, R, C, ld, rpb, part);
  DTRY(cudaGetLastError());
  k_colsum64<<<(unsigned)((C + 255) / 256), 256, 0, st>>>(part, nb, C, dst);
  DTRY(cudaGetLastError());
  return LINREC_OK;
}

int64_t part_rows(int64_t R) { return R > 512 ? 512 : R; }

struct Carve64 {
  double* base;
  int64_t off = 0;
  double* take(int64_t n) {
    double* p = base ? base + off : nullptr;
    off += (n + 31) / 32 * 32;  // 256-byte aligned carve-outs
    return p;
  }
};

// ---- scratch layouts (doubles; one function sizes and carves) --------------
struct Gilr64 {
  double *pre, *imp, *G, *dpre, *dh0, *part, *split;
};
int64_t gilr64_scratch(double* base, int64_t T, int64_t b, int64_t m, int64_t n, Gilr64* s) {
  const int64_t R = T * b, N = R * n;
  Carve64 c{base};
  Gilr64 t;
  t.dh0 = c.take(b * n);
  t.part = c.take(part_rows(R) * 2 * n);
  t.split = c.take((int64_t)kMaxSplits * n * m);
  const int64_t common = c.off;
  Carve64 f{base, common};
  t.pre = f.take(2 * N);
  t.imp = f.take(N);
  Carve64 bw{base, common};
  t.G = bw.take(N);
  t.dpre = bw.take(2 * N);
  if (s) *s = t;
  return f.off > bw.off ? f.off : bw.off;
}

struct Lstm64 {
  double *pre, *iz, *pre_s, *imp_s;                       // forward
  double *dc, *diz, *dpre, *dhp, *G, *dpre_s, *tmp0, *tmp1;  // backward
  double *part, *split;
};
int64_t lstm64_scratch(double* base, int64_t T, int64_t b, int64_t m, int64_t n, Lstm64* s) {
  const int64_t R = T * b, N = R * n, mx = m > n ? m : n;
  Carve64 c{base};
  Lstm64 t;
  t.tmp0 = c.take(b * n);
  t.tmp1 = c.take(b * n);
  t.part = c.take(part_rows(R) * 4 * n);
  t.split = c.take((int64_t)kMaxSplits * 4 * n * mx);
  const int64_t common = c.off;
  Carve64 f{base, common};
  t.pre = f.take(4 * N);
  t.iz = f.take(N);
  t.pre_s = f.take(2 * N);
  t.imp_s = f.take(N);
  Carve64 bw{base, common};
  t.dc = bw.take(N);
  t.diz = bw.take(N);
  t.dpre = bw.take(4 * N);
  t.dhp = bw.take(N + b * n);
  t.G = bw.take(N);
  t.dpre_s = bw.take(2 * N);
  if (s) *s = t;
  return f.off > bw.off ? f.off : bw.off;
}

struct Qrnn64 {
  double *pre, *imp, *dc, *dimp, *dpre, *tmp0, *part, *split;
};
int64_t qrnn64_scratch(double* base, int64_t T, int64_t b, int64_t m, int64_t n, Qrnn64* s) {
  const int64_t R = T * b, N = R * n;
  Carve64 c{base};
  Qrnn64 t;
  t.tmp0 = c.take(b * n);
  t.part = c.take(part_rows(R) * 3 * n);
  t.split = c.take((int64_t)kMaxSplits * 3 * n * m);
  const int64_t common = c.off;
  Carve64 f{base, common};
  t.pre = f.take(3 * N);
  t.imp = f.take(N);
  Carve64 bw{base, common};
  t.dc = bw.take(N);
  t.dimp = bw.take(N);
  t.dpre = bw.take(3 * N);
  if (s) *s = t;
  return f.off > bw.off ? f.off : bw.off;
}

int check64(int64_t T, int64_t b, int64_t m, int64_t n, int mode, const void* x) {
  if (T < 1 || b < 1 || m < 1 || n < 1) return err64(LINREC_ERR_SHAPE, "Tensor3 dimensions must be >= 1");
  if (T * b >= (int64_t(1) << 31)) return err64(LINREC_ERR_SHAPE, "layers: T*b must be < 2^31");
  if (mode != LINREC_SERIAL && mode != LINREC_PARALLEL)
    return err64(LINREC_ERR_VALUE, "mode must be \"parallel\" or \"serial\"");
  if (!x) return err64(LINREC_ERR_VALUE, "x must not be NULL");
  return LINREC_OK;
}

int check_scratch64(void* scratch, size_t have, int64_t need_doubles) {
  if (!scratch || have < (size_t)need_doubles * 8)
    return err64(LINREC_ERR_VALUE, "layers: scratch is NULL or smaller than linrec_*_scratch_bytes_f64()");
  if (reinterpret_cast<uintptr_t>(scratch) & 255)
    return err64(LINREC_ERR_VALUE, "layers: scratch must be 256-byte aligned");
  return LINREC_OK;
}

// gilr_forward core (layers.hpp:78-100): pre = x [U; V]^T, gates, h = scan
int gilr64_forward(const linrec_gilr_params_f64* p, const double* x, const double* h0, double* h, double* g,
                   double* ci, double* pre, double* imp, int64_t T, int64_t b, int64_t m, int64_t n, int mode,
                   cudaStream_t st) {
  const int64_t R = T * b;
  DRC(affine64(x, m, p->U, m, pre, 2 * n, R, n, m, false, st));
  DRC(affine64(x, m, p->V, m, pre + n, 2 * n, R, n, m, false, st));
  k_gilr_gates64<<<grid64(R * n), 256, 0, st>>>(pre, p->b_g, p->b_z, p->act, g, ci, imp, R, n);
  DTRY(cudaGetLastError());
  return linrec_scan_f64(g, imp, h0, h, T, b * n, mode, nullptr, st);
}

// gilr_backward core (layers.hpp:102-133); dx == nullptr: dpre is left for
// the caller's own input-gradient GEMM (the LSTM)
int gilr64_backward(const linrec_gilr_params_f64* p, const double* x, const double* h0, const double* g,
                    const double* ci, const double* h, const double* dh, linrec_gilr_grads_f64* gr, double* dx,
                    double* dh0, double* G, double* dpre, double* part, double* split, int64_t T, int64_t b,
                    int64_t m, int64_t n, int mode, cudaStream_t st) {
  const int64_t R = T * b;
  DRC(linrec_scan_backward_f64(g, h0, h, dh, nullptr, G, dh0, T, b * n, mode, nullptr, st));
  k_gilr_dpre64<<<grid64(R * n), 256, 0, st>>>(g, ci, h, h0, G, p->act, dpre, R, n, b);
  DTRY(cudaGetLastError());
  DRC(bgrad64(dpre, 2 * n, R, n, part, gr->b_g, st));
  DRC(bgrad64(dpre + n, 2 * n, R, n, part, gr->b_z, st));
  if (gr->U) DRC(wgrad64(dpre, 2 * n, x, m, gr->U, m, R, n, m, split, st));
  if (gr->V) DRC(wgrad64(dpre + n, 2 * n, x, m, gr->V, m, R, n, m, split, st));
  if (dx) {
    DRC(igrad64(dpre, 2 * n, p->U, m, dx, m, R, n, m, false, st));
    DRC(igrad64(dpre + n, 2 * n, p->V, m, dx, m, R, n, m, true, st));
  }
  return LINREC_OK;
}

}  // namespace

extern "C" {

int linrec_gemm_f64(const double* A, int a_mn, int64_t lda, const double* B, int b_mn, int64_t ldb, double* C,
                    int64_t ldc, int64_t M, int64_t N, int64_t K, int accumulate, void* stream) {
  if (M < 0 || N < 0 || K < 0) return err64(LINREC_ERR_SHAPE, "gemm: negative dimension");
  if ((M > 0 && N > 0) && (!C || (K > 0 && (!A || !B)))) return err64(LINREC_ERR_VALUE, "gemm: NULL operand");
  // A(m, k): K-major [M][K] or MN-major [K][M]; B(n, k) likewise
  const int64_t sam = a_mn ? 1 : lda, sak = a_mn ? lda : 1;
  const int64_t sbn = b_mn ? 1 : ldb, sbk = b_mn ? ldb : 1;
  return dgemm(A, sam, sak, B, sbk, sbn, C, ldc, M, N, K, accumulate != 0, nullptr,
               static_cast<cudaStream_t>(stream));
}

size_t linrec_gilr_scratch_bytes_f64(int64_t T, int64_t b, int64_t m, int64_t n) {
  if (T < 1 || b < 1 || m < 1 || n < 1) return 0;
  return (size_t)gilr64_scratch(nullptr, T, b, m, n, nullptr) * 8;
}
size_t linrec_gilr_lstm_scratch_bytes_f64(int64_t T, int64_t b, int64_t m, int64_t n) {
  if (T < 1 || b < 1 || m < 1 || n < 1) return 0;
  return (size_t)lstm64_scratch(nullptr, T, b, m, n, nullptr) * 8;
}
size_t linrec_qrnn_scratch_bytes_f64(int64_t T, int64_t b, int64_t m, int64_t n, int64_t k) {
  if (T < 1 || b < 1 || m < 1 || n < 1 || k < 1) return 0;
  return (size_t)qrnn64_scratch(nullptr, T, b, m, n, nullptr) * 8;
}

int linrec_gilr_forward_f64(const linrec_gilr_params_f64* p, const double* x, const double* h0, double* h,
                            double* g, double* i, int64_t T, int64_t b, int64_t m, int64_t n, int mode,
                            void* scratch, size_t scratch_bytes, void* stream) {
  DRC(check64(T, b, m, n, mode, x));
  if (!p || !p->U || !p->V || !p->b_g || !p->b_z || !h || !g || !i)
    return err64(LINREC_ERR_VALUE, "gilr_forward: parameters, h and the cache (g, i) must not be NULL");
  DRC(check_scratch64(scratch, scratch_bytes, gilr64_scratch(nullptr, T, b, m, n, nullptr)));
  Gilr64 s;
  gilr64_scratch(static_cast<double*>(scratch), T, b, m, n, &s);
  return gilr64_forward(p, x, h0, h, g, i, s.pre, s.imp, T, b, m, n, mode, static_cast<cudaStream_t>(stream));
}

int linrec_gilr_backward_f64(const linrec_gilr_params_f64* p, const double* x, const double* h0, const double* g,
                             const double* i, const double* h, const double* dh, linrec_gilr_grads_f64* grads,
                             double* dx, double* dh0, int64_t T, int64_t b, int64_t m, int64_t n, int mode,
                             void* scratch, size_t scratch_bytes, void* stream) {
  DRC(check64(T, b, m, n, mode, x));
  if (!p || !p->U || !p->V || !g || !i || !h || !dh || !grads || !dx)
    return err64(LINREC_ERR_VALUE, "gilr_backward: parameters, cache, d_h, grads and dx must not be NULL");
  DRC(check_scratch64(scratch, scratch_bytes, gilr64_scratch(nullptr, T, b, m, n, nullptr)));
  Gilr64 s;
  gilr64_scratch(static_cast<double*>(scratch), T, b, m, n, &s);
  return gilr64_backward(p, x, h0, g, i, h, dh, grads, dx, dh0 ? dh0 : s.dh0, s.G, s.dpre, s.part, s.split, T, b,
                         m, n, mode, static_cast<cudaStream_t>(stream));
}

int linrec_gilr_lstm_forward_f64(const linrec_gilr_lstm_params_f64* p, const double* x, const double* htil0,
                                 const double* c0, double* h, const linrec_gilr_lstm_cache_f64* cache, int64_t T,
                                 int64_t b, int64_t m, int64_t n, int mode, void* scratch, size_t scratch_bytes,
                                 void* stream) {
  DRC(check64(T, b, m, n, mode, x));
  if (!p || !p->U || !p->V || !p->bias || !p->surrogate.U || !p->surrogate.V || !p->surrogate.b_g ||
      !p->surrogate.b_z || !h || !cache || !cache->sg || !cache->si || !cache->htil || !cache->gates || !cache->c)
    return err64(LINREC_ERR_VALUE, "gilr_lstm_forward: parameters, h and every cache buffer must not be NULL");
  DRC(check_scratch64(scratch, scratch_bytes, lstm64_scratch(nullptr, T, b, m, n, nullptr)));
  Lstm64 s;
  lstm64_scratch(static_cast<double*>(scratch), T, b, m, n, &s);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t R = T * b, BN = b * n, N = R * n;
  // surrogate (htil lands one row block after htil0: rows 0..T-1 are htil_prev)
  if (htil0) DTRY(cudaMemcpyAsync(cache->htil, htil0, sizeof(double) * BN, cudaMemcpyDeviceToDevice, st));
  else DTRY(cudaMemsetAsync(cache->htil, 0, sizeof(double) * BN, st));
  DRC(gilr64_forward(&p->surrogate, x, htil0, cache->htil + BN, cache->sg, cache->si, s.pre_s, s.imp_s, T, b, m, n,
                     mode, st));
  // gates = act(x V^T + htil_prev U^T + bias)   (:262-285)
  DRC(affine64(x, m, p->V, m, s.pre, 4 * n, R, 4 * n, m, false, st));
  DRC(affine64(cache->htil, n, p->U, n, s.pre, 4 * n, R, 4 * n, n, true, st));
  k_lstm_gates64<<<grid64(N), 256, 0, st>>>(s.pre, p->bias, cache->gates, s.iz, R, n);
  DTRY(cudaGetLastError());
  DRC(linrec_scan_f64(cache->gates, s.iz, c0, cache->c, T, BN, mode, nullptr, st));
  k_mul64<<<grid64(N), 256, 0, st>>>(cache->gates + 2 * N, cache->c, h, N);
  DTRY(cudaGetLastError());
  return LINREC_OK;
}

int linrec_gilr_lstm_backward_f64(const linrec_gilr_lstm_params_f64* p, const double* x, const double* htil0,
                                  const double* c0, const linrec_gilr_lstm_cache_f64* cache, const double* dh,
                                  linrec_gilr_lstm_grads_f64* grads, double* dx, double* dhtil0, double* dc0,
                                  int64_t T, int64_t b, int64_t m, int64_t n, int mode, void* scratch,
                                  size_t scratch_bytes, void* stream) {
  DRC(check64(T, b, m, n, mode, x));
  if (!p || !p->U || !p->V || !p->surrogate.U || !p->surrogate.V || !cache || !cache->sg || !cache->si ||
      !cache->htil || !cache->gates || !cache->c || !dh || !grads || !dx)
    return err64(LINREC_ERR_VALUE, "gilr_lstm_backward: parameters, cache, d_h, grads and dx must not be NULL");
  DRC(check_scratch64(scratch, scratch_bytes, lstm64_scratch(nullptr, T, b, m, n, nullptr)));
  Lstm64 s;
  lstm64_scratch(static_cast<double*>(scratch), T, b, m, n, &s);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t R = T * b, BN = b * n, N = R * n;
  const double* gates = cache->gates;
  // dc = dh * o; cell scan backward -> diz, dc0 (df = c_{t-1} diz in dpre)   (:312-324)
  k_mul64<<<grid64(N), 256, 0, st>>>(dh, gates + 2 * N, s.dc, N);
  DTRY(cudaGetLastError());
  DRC(linrec_scan_backward_f64(gates, c0, cache->c, s.dc, nullptr, s.diz, dc0 ? dc0 : s.tmp0, T, BN, mode, nullptr,
                               st));
  k_lstm_dpre64<<<grid64(N), 256, 0, st>>>(gates, c0, s.diz, dh, cache->c, s.dpre, R, n, b);
  DTRY(cudaGetLastError());
  DRC(bgrad64(s.dpre, 4 * n, R, 4 * n, s.part, grads->bias, st));
  // dU += dpre^T htil_prev, dV += dpre^T x   (:344-351)
  if (grads->U) DRC(wgrad64(s.dpre, 4 * n, cache->htil, n, grads->U, n, R, 4 * n, n, s.split, st));
  if (grads->V) DRC(wgrad64(s.dpre, 4 * n, x, m, grads->V, m, R, 4 * n, m, s.split, st));
  // dhp = dpre U (gradient w.r.t. htil_prev); the row block after the last is 0
  DRC(igrad64(s.dpre, 4 * n, p->U, n, s.dhp, n, R, 4 * n, n, false, st));
  DTRY(cudaMemsetAsync(s.dhp + N, 0, sizeof(double) * BN, st));
  // surrogate backward on d_htil[t] = dhp[t+1]   (:356-363)
  DRC(gilr64_backward(&p->surrogate, x, htil0, cache->sg, cache->si, cache->htil + BN, s.dhp + BN, &grads->surrogate,
                      nullptr, s.tmp1, s.G, s.dpre_s, s.part, s.split, T, b, m, n, mode, st));
  // dx = dpre V + dg U_s + di V_s   (:352-355, :364)
  DRC(igrad64(s.dpre, 4 * n, p->V, m, dx, m, R, 4 * n, m, false, st));
  DRC(igrad64(s.dpre_s, 2 * n, p->surrogate.U, m, dx, m, R, n, m, true, st));
  DRC(igrad64(s.dpre_s + n, 2 * n, p->surrogate.V, m, dx, m, R, n, m, true, st));
  // htil0 feeds the surrogate scan and the t = 1 gate input   (:364-370)
  if (dhtil0) {
    k_add64<<<grid64(BN), 256, 0, st>>>(s.tmp1, s.dhp, dhtil0, BN);
    DTRY(cudaGetLastError());
  }
  return LINREC_OK;
}

int linrec_qrnn_forward_f64(const double* W, const double* bias, const double* x, const double* c0, double* h,
                            double* gates, double* c, int64_t T, int64_t b, int64_t m, int64_t n, int64_t k, int mode,
                            void* scratch, size_t scratch_bytes, void* stream) {
  DRC(check64(T, b, m, n, mode, x));
  if (k < 1) return err64(LINREC_ERR_SHAPE, "qrnn_init: window must be >= 1");
  if (k > T) return err64(LINREC_ERR_SHAPE, "qrnn_forward: filter window exceeds sequence length");
  if (!W || !bias || !h || !gates || !c)
    return err64(LINREC_ERR_VALUE, "qrnn_forward: W, bias, h, gates and c must not be NULL");
  DRC(check_scratch64(scratch, scratch_bytes, qrnn64_scratch(nullptr, T, b, m, n, nullptr)));
  Qrnn64 s;
  qrnn64_scratch(static_cast<double*>(scratch), T, b, m, n, &s);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t R = T * b, N = R * n;
  // pre[r] = sum_s x[r - s b] W_s^T: tap s adds into rows s*b.. (:466-470)
  for (int64_t tap = 0; tap < k; ++tap)
    DRC(affine64(x, m, W + tap * 3 * n * m, m, s.pre + tap * b * 3 * n, 3 * n, R - tap * b, 3 * n, m, tap > 0, st));
  k_qrnn_gates64<<<grid64(N), 256, 0, st>>>(s.pre, bias, gates, s.imp, R, n);
  DTRY(cudaGetLastError());
  DRC(linrec_scan_f64(gates, s.imp, c0, c, T, b * n, mode, nullptr, st));
  k_mul64<<<grid64(N), 256, 0, st>>>(gates + N, c, h, N);
  DTRY(cudaGetLastError());
  return LINREC_OK;
}

int linrec_qrnn_backward_f64(const double* W, const double* x, const double* c0, const double* gates, const double* c,
                             const double* dh, double* dW, double* dbias, double* dx, double* dc0, int64_t T,
                             int64_t b, int64_t m, int64_t n, int64_t k, int mode, void* scratch,
                             size_t scratch_bytes, void* stream) {
  DRC(check64(T, b, m, n, mode, x));
  if (k < 1 || k > T) return err64(LINREC_ERR_SHAPE, "qrnn_backward: window must be in [1, T]");
  if (!W || !gates || !c || !dh || !dx)
    return err64(LINREC_ERR_VALUE, "qrnn_backward: W, gates, c, d_h and dx must not be NULL");
  DRC(check_scratch64(scratch, scratch_bytes, qrnn64_scratch(nullptr, T, b, m, n, nullptr)));
  Qrnn64 s;
  qrnn64_scratch(static_cast<double*>(scratch), T, b, m, n, &s);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t R = T * b, N = R * n;
  // dc = dh * o; cell scan backward   (:510-521)
  k_mul64<<<grid64(N), 256, 0, st>>>(dh, gates + N, s.dc, N);
  DTRY(cudaGetLastError());
  DRC(linrec_scan_backward_f64(gates, c0, c, s.dc, nullptr, s.dimp, dc0 ? dc0 : s.tmp0, T, b * n, mode, nullptr,
                               st));
  k_qrnn_dpre64<<<grid64(N), 256, 0, st>>>(gates, c0, s.dimp, dh, c, s.dpre, R, n, b);
  DTRY(cudaGetLastError());
  DRC(bgrad64(s.dpre, 3 * n, R, 3 * n, s.part, dbias, st));
  // dW_s += dpre[s b ..]^T x[.. R - s b];  dx[r] = sum_s dpre[r + s b] W_s   (:536-543)
  for (int64_t tap = 0; tap < k; ++tap) {
    const double* d = s.dpre + tap * b * 3 * n;
    const double* Ws = W + tap * 3 * n * m;
    if (dW) DRC(wgrad64(d, 3 * n, x, m, dW + tap * 3 * n * m, m, R - tap * b, 3 * n, m, s.split, st));
    DRC(igrad64(d, 3 * n, Ws, m, dx, m, R - tap * b, 3 * n, m, tap > 0, st));
  }
  return LINREC_OK;
}

}  // extern "C"
