// CTA-local scans for short sequences (T <= 4096): one CTA owns VEC channels
// over the WHOLE sequence, so the scan needs no cross-CTA communication at
// all -- no look-back, no workspace, one launch.  This is the regime of the
// reference's correctness config (C1: T = 4096, W = 256) and of the paper's
// kernel table (b = 1, m <= 128, T <= 4096), where the
// chained scan's 96-row tiles leave most SMs idle and its per-tile look-back
// latency dominates (C1: 43-tile chains over 2 columns).
//
// Thread i of the NT threads holds R consecutive rows of its VEC channels in
// registers (loaded once, 128-bit), reduces them to an affine pair (A = prod
// of decays, B = zero-seeded result -- the reference's chunk_summary,
// recurrence.hpp:114-131, at thread granularity), the CTA scans the pairs
// (warp shuffles, then the warp totals through shared memory), and each
// thread re-scans its rows from its exclusive carry (the reference's phase 3,
// recurrence.hpp:232-237) and stores them.  The backward runs the same in
// reverse time on G_t = mu_t G_{t+1} + dh_t (mu_t = lam_{t+1}, lam_next at the
// end) with dx = G, dlam = h_{t-1} G and dh0 = lam_0 G_0 fused into the
// re-scan (recurrence.hpp:283-348).  Fixed association: deterministic.
#include "chain_impl.cuh"

namespace linrec_dev {

// Inclusive scan of (A, B) pairs over the CTA's threads in processing order
// (REV: from the last thread to the first); returns this thread's EXCLUSIVE
// pair (the composition of every earlier thread's pair).
template <class S, int VEC, int NT, bool REV>
__device__ __forceinline__ void cta_exclusive(S (&A)[VEC], S (&B)[VEC], S (*sA)[VEC], S (*sB)[VEC],
                                              S (&Ae)[VEC], S (&Be)[VEC]) {
  constexpr int NWP = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // warp-level inclusive scan in processing order
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      const S ap = REV ? __shfl_down_sync(0xffffffffu, A[v], off) : __shfl_up_sync(0xffffffffu, A[v], off);
      const S bp = REV ? __shfl_down_sync(0xffffffffu, B[v], off) : __shfl_up_sync(0xffffffffu, B[v], off);
      if (REV ? lane + off < 32 : lane >= off) {
        B[v] = fma_(A[v], bp, B[v]);
        A[v] = mul_(A[v], ap);
      }
    }
  }
  // exclusive within the warp
  S ae[VEC], be[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    const S ap = REV ? __shfl_down_sync(0xffffffffu, A[v], 1) : __shfl_up_sync(0xffffffffu, A[v], 1);
    const S bp = REV ? __shfl_down_sync(0xffffffffu, B[v], 1) : __shfl_up_sync(0xffffffffu, B[v], 1);
    const bool first = REV ? lane == 31 : lane == 0;
    ae[v] = first ? S(1) : ap;
    be[v] = first ? S(0) : bp;
  }
  // warp totals (the last lane in processing order holds them)
  if (lane == (REV ? 0 : 31)) {
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      sA[warp][v] = A[v];
      sB[warp][v] = B[v];
    }
  }
  __syncthreads();
  // compose the totals of the warps before this one (processing order), then
  // this thread's in-warp prefix: exclusive = in-warp o (earlier warps)
  S wa[VEC], wb[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) { wa[v] = S(1); wb[v] = S(0); }
#pragma unroll
  for (int i = 0; i < NWP; ++i) {
    const int w = REV ? NWP - 1 - i : i;
    if (REV ? w > warp : w < warp) {
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        wb[v] = fma_(sA[w][v], wb[v], sB[w][v]);
        wa[v] = mul_(sA[w][v], wa[v]);
      }
    }
  }
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    Be[v] = fma_(ae[v], wb[v], be[v]);
    Ae[v] = mul_(ae[v], wa[v]);
  }
}

template <class S, int VEC, int R, int NT>
__global__ void __launch_bounds__(NT) k_local_fwd(const S* __restrict__ lam, const S* __restrict__ x,
                                                  const S* __restrict__ h0, S* __restrict__ h, int T, int64_t W) {
  using IO = VecIO<S, VEC>;
  __shared__ S sA[NT / 32][VEC], sB[NT / 32][VEC];
  const int64_t ch = (int64_t)blockIdx.x * VEC;
  const int t0 = threadIdx.x * R;
  S l[R][VEC], xv[R][VEC];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    if (t0 + i < T) {
      IO::load_stream(lam + (int64_t)(t0 + i) * W + ch, l[i]);
      IO::load_stream(x + (int64_t)(t0 + i) * W + ch, xv[i]);
    } else {
#pragma unroll
      for (int v = 0; v < VEC; ++v) { l[i][v] = S(1); xv[i][v] = S(0); }
    }
  }
  S A[VEC], B[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) { A[v] = l[0][v]; B[v] = xv[0][v]; }
#pragma unroll
  for (int i = 1; i < R; ++i)
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      B[v] = fma_(l[i][v], B[v], xv[i][v]);
      A[v] = mul_(l[i][v], A[v]);
    }
  S Ae[VEC], Be[VEC];
  cta_exclusive<S, VEC, NT, false>(A, B, sA, sB, Ae, Be);
  S c[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) c[v] = fma_(Ae[v], h0 != nullptr ? h0[ch + v] : S(0), Be[v]);
#pragma unroll
  for (int i = 0; i < R; ++i) {
#pragma unroll
    for (int v = 0; v < VEC; ++v) c[v] = fma_(l[i][v], c[v], xv[i][v]);
    if (t0 + i < T) IO::store_stream(h + (int64_t)(t0 + i) * W + ch, c);
  }
}

template <class S, int VEC, int R, int NT>
__global__ void __launch_bounds__(NT)
    k_local_bwd(const S* __restrict__ lam, const S* __restrict__ h0, const S* __restrict__ h,
                const S* __restrict__ dh, const S* __restrict__ lam_next, const S* __restrict__ g_next,
                S* __restrict__ dlam, S* __restrict__ dx, S* __restrict__ dh0, int T, int64_t W) {
  using IO = VecIO<S, VEC>;
  __shared__ S sA[NT / 32][VEC], sB[NT / 32][VEC];
  const int64_t ch = (int64_t)blockIdx.x * VEC;
  const int t0 = threadIdx.x * R;
  // mu_t = lam_{t+1} (lam_next, or 0, at the end), dh_t, h_{t-1} (h0 at t = 0)
  S mu[R][VEC], d[R][VEC], hp[R][VEC];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int t = t0 + i;
    if (t < T) {
      if (t + 1 < T) {
        IO::load_stream(lam + (int64_t)(t + 1) * W + ch, mu[i]);
      } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) mu[i][v] = lam_next != nullptr ? lam_next[ch + v] : S(0);
      }
      IO::load_stream(dh + (int64_t)t * W + ch, d[i]);
      if (t > 0) {
        IO::load_stream(h + (int64_t)(t - 1) * W + ch, hp[i]);
      } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) hp[i][v] = h0 != nullptr ? h0[ch + v] : S(0);
      }
    } else {
#pragma unroll
      for (int v = 0; v < VEC; ++v) { mu[i][v] = S(1); d[i][v] = S(0); hp[i][v] = S(0); }
    }
  }
  S A[VEC], B[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) { A[v] = mu[R - 1][v]; B[v] = d[R - 1][v]; }
#pragma unroll
  for (int i = R - 2; i >= 0; --i)
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      B[v] = fma_(mu[i][v], B[v], d[i][v]);
      A[v] = mul_(mu[i][v], A[v]);
    }
  S Ae[VEC], Be[VEC];
  cta_exclusive<S, VEC, NT, true>(A, B, sA, sB, Ae, Be);
  S g[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) g[v] = fma_(Ae[v], g_next != nullptr ? g_next[ch + v] : S(0), Be[v]);
#pragma unroll
  for (int i = R - 1; i >= 0; --i) {
    S dl[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      g[v] = fma_(mu[i][v], g[v], d[i][v]);
      dl[v] = mul_(hp[i][v], g[v]);
    }
    const int t = t0 + i;
    if (t < T) {
      IO::store_stream(dx + (int64_t)t * W + ch, g);
      if (dlam != nullptr) IO::store_stream(dlam + (int64_t)t * W + ch, dl);
      if (t == 0 && dh0 != nullptr) {
        S l0[VEC], r[VEC];
        IO::load_cg(lam + ch, l0);
#pragma unroll
        for (int v = 0; v < VEC; ++v) r[v] = mul_(l0[v], g[v]);
        IO::store_cg(dh0 + ch, r);
      }
    }
  }
}

}  // namespace linrec_dev

namespace linrec_impl {

namespace {
// (rows per thread, threads): the smallest R of 1, 2, 4, 8, 16 with R * NT >= T
template <class S, int VEC, int NT, bool FWD>
cudaError_t dispatch_local(int R, const FwdCall<S>* f, const BwdCall<S>* b, cudaStream_t st) {
  const int64_t W = FWD ? f->W : b->W;
  const dim3 grid((unsigned)(W / VEC));
#define LOCAL_CASE(RR)                                                                                     \
  case RR:                                                                                                 \
    if constexpr (FWD)                                                                                     \
      linrec_dev::k_local_fwd<S, VEC, RR, NT><<<grid, NT, 0, st>>>(f->lam, f->x, f->h0, f->h, (int)f->T, W); \
    else                                                                                                   \
      linrec_dev::k_local_bwd<S, VEC, RR, NT><<<grid, NT, 0, st>>>(b->lam, b->h0, b->h, b->dh, b->lam_next, \
                                                                   b->g_next, b->dlam, b->dx, b->dh0,      \
                                                                   (int)b->T, W);                          \
    break;
  switch (R) {
    LOCAL_CASE(1)
    LOCAL_CASE(2)
    LOCAL_CASE(4)
    LOCAL_CASE(8)
    LOCAL_CASE(16)
    default:
      return cudaErrorInvalidConfiguration;
  }
#undef LOCAL_CASE
  return cudaGetLastError();
}

int local_rows(int64_t T, int nt) {
  int r = 1;
  while ((int64_t)r * nt < T) r <<= 1;
  return r;
}
}  // namespace

// Forward: 256 threads x up to 16 rows; backward (three arrays in
// registers): 512 threads x up to 8 rows.  Both cover T <= 4096.
constexpr int kLocalFwdNT = 256, kLocalBwdNT = 512;

// Short, narrow problems (latency-bound for the chained scan): T <= 4096 and
// at most 2^21 elements (C1 is 2^20).  LINREC_LOCAL=0 disables the path,
// LINREC_LOCAL_MAX overrides the element bound (tuning).
template <class S>
bool local_scan_ok(int64_t T, int64_t W, bool vec_ok) {
  static const int on = env_int("LINREC_LOCAL", 1);
  static const int64_t cap = env_int("LINREC_LOCAL_MAX", 1 << 21);
  const int64_t ctas = vec_ok ? W / Tuning<S>::VEC : W;
  return on != 0 && T >= 1 && T <= 4096 && T * W <= cap && ctas <= 65535;
}

template <class S>
cudaError_t launch_local_fwd(const FwdCall<S>& c, bool vec_ok, cudaStream_t st) {
  constexpr int V = Tuning<S>::VEC;
  const int R = local_rows(c.T, kLocalFwdNT);
  if (vec_ok) return dispatch_local<S, V, kLocalFwdNT, true>(R, &c, nullptr, st);
  return dispatch_local<S, 1, kLocalFwdNT, true>(R, &c, nullptr, st);
}

template <class S>
cudaError_t launch_local_bwd(const BwdCall<S>& c, bool vec_ok, cudaStream_t st) {
  constexpr int V = Tuning<S>::VEC;
  const int R = local_rows(c.T, kLocalBwdNT);
  if (R > 8) return cudaErrorInvalidConfiguration;
  if (vec_ok) return dispatch_local<S, V, kLocalBwdNT, false>(R, nullptr, &c, st);
  return dispatch_local<S, 1, kLocalBwdNT, false>(R, nullptr, &c, st);
}

template bool local_scan_ok<float>(int64_t, int64_t, bool);
template bool local_scan_ok<double>(int64_t, int64_t, bool);
template cudaError_t launch_local_fwd<float>(const FwdCall<float>&, bool, cudaStream_t);
template cudaError_t launch_local_fwd<double>(const FwdCall<double>&, bool, cudaStream_t);
template cudaError_t launch_local_bwd<float>(const BwdCall<float>&, bool, cudaStream_t);
template cudaError_t launch_local_bwd<double>(const BwdCall<double>&, bool, cudaStream_t);

}  // namespace linrec_impl
