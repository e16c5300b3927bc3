// Peer-memory carry exchange of the sequence-sharded scan: the mailbox
// layout, system-scope release/acquire, and the two device halves that the
// stitch kernels fuse in (segment.cu):
//   publish_chunk   the virtual-segment fold (k_vseg_finalize) stores its
//                   32-channel chunk of the rank aggregate straight into the
//                   consumers' mailboxes; the last CTA to finish releases
//                   the flags
//   compose_chunk   the fix-up (k_fixup) folds the sources' aggregates for
//                   its channel column from its own mailbox into the
//                   incoming carry before fixing tiles; the last CTA to
//                   finish reading acknowledges the sources
// so the exchange costs no launch of its own (csrc/p2p.cu keeps the
// standalone publish / compose kernels of the same protocol).
//
// Every rank owns one mailbox (cudaMalloc'd, shared by CUDA IPC):
//   data[2 dirs][world][2][W]  the (A, B) aggregate rank q published for
//                              direction d, in slot [d][q]
//   flags[2][world]            epoch at which slot [d][q] became valid
//   acks[2][world]             epoch up to which rank q has consumed THIS
//                              rank's slot in q's mailbox (so a producer
//                              never overwrites an unread slot)
//   count[2][2]                per direction: CTAs of the fused publish /
//                              compose that finished (last-CTA detection)
#pragma once

#include <cstdint>

#include "launch.h"
#include "linrec_device.cuh"

namespace linrec_dev {
namespace p2p {

struct MboxLayout {
  int64_t W;
  int world;
  __host__ __device__ size_t data_floats() const { return (size_t)2 * world * 2 * W; }
  __host__ __device__ size_t flags_off() const { return (data_floats() * 4 + 255) / 256 * 256; }
  __host__ __device__ size_t acks_off() const { return flags_off() + (size_t)2 * world * 8; }
  __host__ __device__ size_t count_off() const { return acks_off() + (size_t)2 * world * 8; }
  __host__ __device__ size_t bytes() const { return count_off() + (size_t)4 * 8; }
  __device__ float* slot(void* base, int dir, int q) const {
    return reinterpret_cast<float*>(base) + ((size_t)dir * world + q) * 2 * W;
  }
  __device__ unsigned long long* flag(void* base, int dir, int q) const {
    return reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(base) + flags_off()) + dir * world + q;
  }
  __device__ unsigned long long* ack(void* base, int dir, int q) const {
    return reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(base) + acks_off()) + dir * world + q;
  }
  __device__ unsigned long long* count(void* base, int dir, int kind) const {
    return reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(base) + count_off()) + dir * 2 + kind;
  }
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void wait_geq(const unsigned long long* p, unsigned long long e) {
  if (ld_acquire_sys(p) >= e) return;
  SpinGuard g;
  while (ld_acquire_sys(p) < e) g.tick();
}

using linrec_impl::Exchange;
__device__ __forceinline__ MboxLayout layout(const Exchange& ex) { return MboxLayout{ex.W, ex.world}; }

// The CTA that completes this launch's grid-wide count -- called by thread 0
// after the CTA's part is done.  The last CTA resets the counter, so every
// launch counts from 0 whatever its grid size (T or W may change between
// steps on the same mailboxes); the next launch that uses the counter is
// stream-ordered after this one, so the reset cannot race with it.
__device__ __forceinline__ bool last_cta(unsigned long long* counter) {
  __threadfence_system();
  const unsigned long long old = atomicAdd(counter, 1ull);
  if (old + 1 != gridDim.x) return false;
  atomicExch(counter, 0ull);
  return true;
}

// Publish channels [j0, j0 + n) of agg [2][W] to every consumer; the whole
// CTA calls it (n <= blockDim.x).
__device__ __forceinline__ void publish_chunk(const Exchange& ex, const float* __restrict__ agg, int64_t j0, int n) {
  const MboxLayout L = layout(ex);
  void* own = ex.mboxes[ex.rank];
  for (int q = ex.q0; q < ex.q1; ++q) {
    if (q == ex.rank) continue;
    if (threadIdx.x == 0) wait_geq(L.ack(own, ex.dir, q), ex.epoch - 1);  // q read the previous epoch
    __syncthreads();
    float* dst = L.slot(ex.mboxes[q], ex.dir, ex.rank);
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      const int64_t j = j0 + t;
      dst[j] = ex.zero_a ? 0.f : __ldcg(agg + j);
      dst[ex.W + j] = __ldcg(agg + ex.W + j);
    }
  }
  __threadfence_system();  // every writer orders its peer stores before the flags
  __syncthreads();
  if (threadIdx.x == 0 && last_cta(L.count(own, ex.dir, 0)))
    for (int q = ex.q0; q < ex.q1; ++q)
      if (q != ex.rank) st_release_sys(L.flag(ex.mboxes[q], ex.dir, ex.rank), ex.epoch);
}

// Incoming carry of channels [j0, j0 + n) into out[0..n) (shared or global):
// wait for the sources' flags, fold them in the fixed order of k_compose
// (bit-identical to the all-gather path), acknowledge once every CTA of the
// grid has read its channels.  The whole CTA calls it.
__device__ __forceinline__ void compose_chunk(const Exchange& ex, int64_t j0, int n, float* out) {
  const MboxLayout L = layout(ex);
  void* own = ex.mboxes[ex.rank];
  if (threadIdx.x == 0)
    for (int q = ex.first; q != ex.last; q += ex.step) wait_geq(L.flag(own, ex.dir, q), ex.epoch);
  __syncthreads();
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const int64_t j = j0 + t;
    float c = 0.f;
    if (j < ex.W)
      for (int q = ex.first; q != ex.last; q += ex.step) {
        const float* s = L.slot(own, ex.dir, q);
        c = __fmaf_rn(__ldcg(s + j), c, __ldcg(s + ex.W + j));
      }
    out[t] = c;
  }
  __syncthreads();  // this CTA's slot reads are complete
  if (threadIdx.x == 0 && last_cta(L.count(own, ex.dir, 1)))
    for (int q = ex.first; q != ex.last; q += ex.step) st_release_sys(L.ack(ex.mboxes[q], ex.dir, ex.rank), ex.epoch);
}

}  // namespace p2p
}  // namespace linrec_dev
