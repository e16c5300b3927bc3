// Cluster scans for short sequences over few channels (the paper's kernel
// table regime, and the reference's correctness config C1:
// T = 4096, W = 256).  The CTA-local scan (local_scan.cu) gives each CTA a
// channel vector over the whole sequence: at W = 256 that is 64 CTAs on 148
// SMs, every load a 16-byte piece of a different row.  Here a thread-block
// CLUSTER of CS CTAs splits the sequence instead, each CTA owning T/CS rows of
// a 32-channel column (128-byte row segments, 8 lanes x float4), and the CTAs
// exchange their chunk aggregates through distributed shared memory -- one
// cluster barrier, no global look-back, no workspace, one launch:
//
//   1. load R rows per thread (all loads in flight at once), reduce them to an
//      affine pair (A = prod of decays, B = zero-seeded result -- the
//      reference's chunk_summary, recurrence.hpp:114-131);
//   2. scan the pairs across the CTA (warp shuffles, warp totals in shared
//      memory) and publish the CTA's total in shared memory;
//   3. barrier.cluster (release / acquire); gather the totals of the
//      cluster's earlier CTAs (one DSMEM round trip) and fold them in rank
//      order onto h0: the carry entering this CTA (the reference's phase 2,
//      recurrence.hpp:219-231);
//   4. re-scan the rows from each thread's exclusive carry and store (phase 3,
//      :232-237); a second cluster barrier keeps every CTA's shared memory
//      alive until the later ranks have read it.
// The backward runs the same in reverse time (ranks, warps and lanes in
// descending order) on G_t = mu_t G_{t+1} + dh_t with dx = G, dlam = h_{t-1} G
// and dh0 = lam_0 G_0 fused into the re-scan (recurrence.hpp:283-348).  Fixed
// association: deterministic.
#include <cooperative_groups.h>

#include "chain_impl.cuh"

namespace cg = cooperative_groups;

namespace linrec_dev {

// Programmatic dependent launch: the kernels are launched with programmatic
// stream serialisation, so the next kernel in the stream may be scheduled
// while this one runs (its launch and prologue overlap this kernel); every
// kernel waits for its predecessor's completion and memory flush before
// touching global memory (griddepcontrol.wait), and lets its successor launch
// once all of its own CTAs are resident (launch_dependents at entry).
__device__ __forceinline__ void pdl_wait_and_release_successor() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Exclusive (A, B) of this thread's slot within its CTA, in processing order
// (REV: descending slots), and -- for threads tid < CPB -- the CTA total of
// channel tid into tA / tB.  Slots: warp w, lane group g = lane / Q.
template <class S, int VEC, int Q, bool REV>
__device__ __forceinline__ void cta_slot_exclusive(S (&A)[VEC], S (&B)[VEC], S (*sA)[Q * VEC], S (*sB)[Q * VEC],
                                                   S* tA, S* tB, S (&Ae)[VEC], S (&Be)[VEC]) {
  constexpr int G = 32 / Q, CPB = Q * VEC, NW = 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, q = lane % Q, g = lane / Q;
  // in-warp inclusive scan over the G lane groups (processing order)
#pragma unroll
  for (int off = 1; off < G; off <<= 1)
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      const S ap = REV ? __shfl_down_sync(0xffffffffu, A[v], off * Q) : __shfl_up_sync(0xffffffffu, A[v], off * Q);
      const S bp = REV ? __shfl_down_sync(0xffffffffu, B[v], off * Q) : __shfl_up_sync(0xffffffffu, B[v], off * Q);
      if (REV ? g + off < G : g >= off) {
        B[v] = fma_(A[v], bp, B[v]);
        A[v] = mul_(A[v], ap);
      }
    }
  S ae[VEC], be[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    ae[v] = S(1);
    be[v] = S(0);
    if (G > 1) {
      const S ap = REV ? __shfl_down_sync(0xffffffffu, A[v], Q) : __shfl_up_sync(0xffffffffu, A[v], Q);
      const S bp = REV ? __shfl_down_sync(0xffffffffu, B[v], Q) : __shfl_up_sync(0xffffffffu, B[v], Q);
      if (REV ? g < G - 1 : g > 0) {
        ae[v] = ap;
        be[v] = bp;
      }
    }
  }
  if (g == (REV ? 0 : G - 1)) {  // the warp's total for its channels
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      sA[warp][q * VEC + v] = A[v];
      sB[warp][q * VEC + v] = B[v];
    }
  }
  __syncthreads();
  S wa[VEC], wb[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) { wa[v] = S(1); wb[v] = S(0); }
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    const int w = REV ? NW - 1 - i : i;
    if (REV ? w > warp : w < warp)
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        wb[v] = fma_(sA[w][q * VEC + v], wb[v], sB[w][q * VEC + v]);
        wa[v] = mul_(sA[w][q * VEC + v], wa[v]);
      }
  }
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    Be[v] = fma_(ae[v], wb[v], be[v]);
    Ae[v] = mul_(ae[v], wa[v]);
  }
  if ((int)threadIdx.x < CPB) {  // CTA total of channel tid, all warps in processing order
    const int c = threadIdx.x;
    S ta = S(1), tb = S(0);
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      const int w = REV ? NW - 1 - i : i;
      tb = fma_(sA[w][c], tb, sB[w][c]);
      ta = mul_(sA[w][c], ta);
    }
    tA[c] = ta;
    tB[c] = tb;
  }
}

// Carry entering this CTA for each of its CPB channels: `seed` folded
// through the totals (tA, tB) of the cluster's ranks before this one in
// processing order (REV: ranks CS-1 .. rank+1).  The remote totals are
// gathered in ONE distributed-shared-memory round trip (every thread loads
// its share into rA / rB), then threads tid < CPB fold them from local shared
// memory and leave the carry in sC.  Ends with this CTA's arrival on the
// second cluster barrier (its own totals may still be read by others).
template <class S, int CPB, int CS, bool REV>
__device__ __forceinline__ void cluster_carry(cg::cluster_group& cl, int rank, const S* tA, const S* tB,
                                              S (*rA)[CPB], S (*rB)[CPB], S* sC, const S* seed, int64_t col0,
                                              int64_t W) {
  for (int e = threadIdx.x; e < CS * CPB; e += blockDim.x) {
    const int r = e / CPB, c = e % CPB;
    if (REV ? r > rank : r < rank) {
      rA[r][c] = cl.map_shared_rank(tA, r)[c];
      rB[r][c] = cl.map_shared_rank(tB, r)[c];
    }
  }
  __syncthreads();
  cluster_arrive_release();  // done reading the other CTAs' shared memory
  if ((int)threadIdx.x < CPB) {
    const int c = threadIdx.x;
    S v = (seed != nullptr && col0 + c < W) ? seed[col0 + c] : S(0);
    if (REV) {
      for (int r = CS - 1; r > rank; --r) v = fma_(rA[r][c], v, rB[r][c]);
    } else {
      for (int r = 0; r < rank; ++r) v = fma_(rA[r][c], v, rB[r][c]);
    }
    sC[c] = v;
  }
  __syncthreads();
}

template <class S, int VEC, int Q, int R, int CS>
__global__ void __launch_bounds__(256) k_cluster_fwd(const S* __restrict__ lam, const S* __restrict__ x,
                                                     const S* __restrict__ h0, S* __restrict__ h, int T, int64_t W) {
  pdl_wait_and_release_successor();
  constexpr int G = 32 / Q, CPB = Q * VEC, RC = 8 * G * R;
  using IO = VecIO<S, VEC>;
  __shared__ S sA[8][CPB], sB[8][CPB];
  __shared__ S tA[CPB], tB[CPB];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, q = lane % Q, g = lane / Q;
  const int64_t ch = (int64_t)(blockIdx.x / CS) * CPB + q * VEC;
  const bool valid = ch < W;
  const int t0 = rank * RC + (warp * G + g) * R;
  S l[R][VEC], xv[R][VEC];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    if (valid && t0 + i < T) {
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
  cta_slot_exclusive<S, VEC, Q, false>(A, B, sA, sB, tA, tB, Ae, Be);
  cluster_arrive_release();  // this CTA's total is visible to the cluster
  cluster_wait_acquire();
  // carry entering this CTA: h0 folded through the totals of ranks 0 .. rank-1
  __shared__ S rA[CS][CPB], rB[CS][CPB], sC[CPB];
  cluster_carry<S, CPB, CS, false>(cl, rank, tA, tB, rA, rB, sC, h0, (int64_t)(blockIdx.x / CS) * CPB, W);
  S c[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) c[v] = fma_(Ae[v], sC[q * VEC + v], Be[v]);
#pragma unroll
  for (int i = 0; i < R; ++i) {
#pragma unroll
    for (int v = 0; v < VEC; ++v) c[v] = fma_(l[i][v], c[v], xv[i][v]);
    if (valid && t0 + i < T) IO::store_stream(h + (int64_t)(t0 + i) * W + ch, c);
  }
  cluster_wait_acquire();  // no CTA leaves while a later rank may still read its totals
}

template <class S, int VEC, int Q, int R, int CS>
__global__ void __launch_bounds__(256)
    k_cluster_bwd(const S* __restrict__ lam, const S* __restrict__ h0, const S* __restrict__ h,
                  const S* __restrict__ dh, const S* __restrict__ lam_next, const S* __restrict__ g_next,
                  S* __restrict__ dlam, S* __restrict__ dx, S* __restrict__ dh0, int T, int64_t W) {
  pdl_wait_and_release_successor();
  constexpr int G = 32 / Q, CPB = Q * VEC, RC = 8 * G * R;
  using IO = VecIO<S, VEC>;
  __shared__ S sA[8][CPB], sB[8][CPB];
  __shared__ S tA[CPB], tB[CPB];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, q = lane % Q, g = lane / Q;
  const int64_t ch = (int64_t)(blockIdx.x / CS) * CPB + q * VEC;
  const bool valid = ch < W;
  const int t0 = rank * RC + (warp * G + g) * R;
  // mu_t = lam_{t+1} (lam_next, or 0, at the end), dh_t, h_{t-1} (h0 at t = 0)
  S mu[R][VEC], d[R][VEC], hp[R][VEC];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int t = t0 + i;
    if (valid && t < T) {
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
  cta_slot_exclusive<S, VEC, Q, true>(A, B, sA, sB, tA, tB, Ae, Be);
  cluster_arrive_release();
  cluster_wait_acquire();
  // carry entering from above: g_next folded through ranks CS-1 .. rank+1
  __shared__ S rA[CS][CPB], rB[CS][CPB], sC[CPB];
  cluster_carry<S, CPB, CS, true>(cl, rank, tA, tB, rA, rB, sC, g_next, (int64_t)(blockIdx.x / CS) * CPB, W);
  S gc[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) gc[v] = fma_(Ae[v], sC[q * VEC + v], Be[v]);
#pragma unroll
  for (int i = R - 1; i >= 0; --i) {
    S dl[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      gc[v] = fma_(mu[i][v], gc[v], d[i][v]);
      dl[v] = mul_(hp[i][v], gc[v]);
    }
    const int t = t0 + i;
    if (valid && t < T) {
      IO::store_stream(dx + (int64_t)t * W + ch, gc);
      if (dlam != nullptr) IO::store_stream(dlam + (int64_t)t * W + ch, dl);
      if (t == 0 && dh0 != nullptr) {
        S l0[VEC], r0[VEC];
        IO::load_cg(lam + ch, l0);
#pragma unroll
        for (int v = 0; v < VEC; ++v) r0[v] = mul_(l0[v], gc[v]);
        IO::store_cg(dh0 + ch, r0);
      }
    }
  }
  cluster_wait_acquire();
}

}  // namespace linrec_dev

namespace linrec_impl {

namespace {

// Cluster shape: Q lanes across channels (8: 32-channel columns of 128-byte
// row segments; 1 when W has fewer than 8 vectors), CS CTAs per cluster
// (16 where the GPU schedules non-portable 16-CTA clusters, else 8), R rows
// per thread: the smallest of 1, 2, 4, 8 with CS * 8 * (32/Q) * R >= T (the
// backward holds three arrays of R rows in registers).
struct ClusterShape {
  int q = 0, cs = 0, r = 0;
  int64_t ncols = 0;
};

template <class S>
int cluster_rows(int64_t T, int q, int cs) {
  const int64_t slots = (int64_t)cs * 8 * (32 / q);
  int r = 1;
  while (r <= 8 && (int64_t)r * slots < T) r <<= 1;
  return r <= 8 ? r : 0;
}

template <class Kern>
bool cluster16_ok(Kern k) {
  if (cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(16);
  cfg.blockDim = dim3(256);
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeClusterDimension;
  at.val.clusterDim.x = 16;
  at.val.clusterDim.y = 1;
  at.val.clusterDim.z = 1;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return n >= 1;
}

template <class S, int VEC, int Q, int R, int CS, bool FWD>
cudaError_t launch_cluster_kernel(const FwdCall<S>* f, const BwdCall<S>* b, int64_t ncols, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(ncols * CS));
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  static const bool pdl = env_int("LINREC_PDL", 1) != 0;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 2 : 1;
  if constexpr (FWD) {
    auto k = linrec_dev::k_cluster_fwd<S, VEC, Q, R, CS>;
    if (CS > 8) {
      const cudaError_t e = func_attr_once(reinterpret_cast<const void*>(k),
                                           cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    return cudaLaunchKernelEx(&cfg, k, f->lam, f->x, f->h0, f->h, (int)f->T, f->W);
  } else {
    auto k = linrec_dev::k_cluster_bwd<S, VEC, Q, R, CS>;
    if (CS > 8) {
      const cudaError_t e = func_attr_once(reinterpret_cast<const void*>(k),
                                           cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    return cudaLaunchKernelEx(&cfg, k, b->lam, b->h0, b->h, b->dh, b->lam_next, b->g_next, b->dlam, b->dx, b->dh0,
                              (int)b->T, b->W);
  }
}

template <class S, int VEC, int Q, int CS, bool FWD>
cudaError_t dispatch_r(int r, const FwdCall<S>* f, const BwdCall<S>* b, int64_t ncols, cudaStream_t st) {
  switch (r) {
    case 1: return launch_cluster_kernel<S, VEC, Q, 1, CS, FWD>(f, b, ncols, st);
    case 2: return launch_cluster_kernel<S, VEC, Q, 2, CS, FWD>(f, b, ncols, st);
    case 4: return launch_cluster_kernel<S, VEC, Q, 4, CS, FWD>(f, b, ncols, st);
    case 8: return launch_cluster_kernel<S, VEC, Q, 8, CS, FWD>(f, b, ncols, st);
    default: return cudaErrorInvalidConfiguration;
  }
}

bool cluster16_supported() {
  static const bool ok = cluster16_ok(linrec_dev::k_cluster_fwd<float, 4, 8, 8, 16>);
  return ok;
}

template <class S>
ClusterShape cluster_shape(int64_t T, int64_t W) {
  constexpr int V = Tuning<S>::VEC;
  ClusterShape s;
  const int64_t nvec = W / V;
  s.q = nvec >= 8 ? 8 : 1;
  s.ncols = (nvec + s.q - 1) / s.q;
  // 8-CTA clusters when they cover T (measured faster than 16 at W = 4096,
  // T = 1024: 4.7 against 7.6 us), else 16 where the GPU schedules them
  static const int env_cs = env_int("LINREC_CLUSTER_CS", 0);
  s.cs = env_cs == 16 ? 16 : 8;
  s.r = cluster_rows<S>(T, s.q, s.cs);
  if (s.r == 0 && env_cs != 8 && cluster16_supported()) {
    s.cs = 16;
    s.r = cluster_rows<S>(T, s.q, s.cs);
  }
  if (s.cs == 16 && !cluster16_supported()) s.r = 0;
  return s;
}

}  // namespace

// fp32, 16-byte vectors, 512 <= T with a shape that covers T (<= 8 rows per
// thread), and too few channel vectors for the CTA-local scan to fill the GPU
// (W / 4 <= 2 x SMs).  Below T = 512 the CTA-local scan's single CTA barrier
// wins (scripts/bench_kernel.py, T = 256: 1.9-3.5 against 3.0-3.8 us).
// LINREC_CLUSTER=0 disables the path (comparison runs).
template <class S>
bool cluster_scan_ok(int64_t T, int64_t W, bool vec_ok) {
  static const int on = env_int("LINREC_CLUSTER", 1);
  if (!on || sizeof(S) != 4 || !vec_ok || T < 512 || T > (int64_t(1) << 30)) return false;
  const int64_t nvec = W / Tuning<S>::VEC;
  if (nvec > 2 * 148) return false;
  return cluster_shape<S>(T, W).r > 0;
}

template <class S>
cudaError_t launch_cluster_fwd(const FwdCall<S>& c, cudaStream_t st) {
  constexpr int V = Tuning<S>::VEC;
  const ClusterShape s = cluster_shape<S>(c.T, c.W);
  if (s.q == 8) {
    if (s.cs == 16) return dispatch_r<S, V, 8, 16, true>(s.r, &c, nullptr, s.ncols, st);
    return dispatch_r<S, V, 8, 8, true>(s.r, &c, nullptr, s.ncols, st);
  }
  if (s.cs == 16) return dispatch_r<S, V, 1, 16, true>(s.r, &c, nullptr, s.ncols, st);
  return dispatch_r<S, V, 1, 8, true>(s.r, &c, nullptr, s.ncols, st);
}

template <class S>
cudaError_t launch_cluster_bwd(const BwdCall<S>& c, cudaStream_t st) {
  constexpr int V = Tuning<S>::VEC;
  const ClusterShape s = cluster_shape<S>(c.T, c.W);
  if (s.q == 8) {
    if (s.cs == 16) return dispatch_r<S, V, 8, 16, false>(s.r, nullptr, &c, s.ncols, st);
    return dispatch_r<S, V, 8, 8, false>(s.r, nullptr, &c, s.ncols, st);
  }
  if (s.cs == 16) return dispatch_r<S, V, 1, 16, false>(s.r, nullptr, &c, s.ncols, st);
  return dispatch_r<S, V, 1, 8, false>(s.r, nullptr, &c, s.ncols, st);
}

template bool cluster_scan_ok<float>(int64_t, int64_t, bool);
template bool cluster_scan_ok<double>(int64_t, int64_t, bool);
template cudaError_t launch_cluster_fwd<float>(const FwdCall<float>&, cudaStream_t);
template cudaError_t launch_cluster_bwd<float>(const BwdCall<float>&, cudaStream_t);
// fp64 keeps the CTA-local scan (cluster_scan_ok<double> is false)
template <>
cudaError_t launch_cluster_fwd<double>(const FwdCall<double>&, cudaStream_t) {
  return cudaErrorNotSupported;
}
template <>
cudaError_t launch_cluster_bwd<double>(const BwdCall<double>&, cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace linrec_impl
