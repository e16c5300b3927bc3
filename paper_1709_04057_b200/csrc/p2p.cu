// Carry exchange of the sequence-sharded scan over peer memory (NVLink /
// NVSwitch), replacing the NCCL all-gather of BASELINE.json's north star
// ("the GPUs exchange that tiny carry ... each GPU runs a local fix-up") with
// direct stores into the consumers' memory and a release/acquire flag --
// SURVEY.md 7, hard part 1(c).  Mailbox layout and protocol: p2p_impl.cuh.
// These are the standalone kernels; the sharded scan itself runs the same
// protocol fused into its stitch kernels (segment.cu).
// publish(d, e): for every consumer q, wait acks[d][q] >= e-1 (in the
//   producer's own mailbox), store the aggregate into q's slot [d][r],
//   fence.sys, st.release.sys q.flags[d][r] = e.
// compose(d, e): wait flags[d][q] >= e for the sources q in the fold (own
//   mailbox), fold them in the fixed order of k_compose (bit-identical to
//   the all-gather path), then st.release.sys q.acks[d][r] = e in each
//   source's mailbox.
// Every spin carries the library's 20 s watchdog (SpinGuard -> trap).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>

#include "launch.h"
#include "linrec_cuda.h"
#include "p2p_impl.cuh"

namespace linrec_dev {
namespace p2p {

// One CTA: agg [2][W] -> slot [dir][rank] of every consumer in [q0, q1).
__global__ void k_publish(const float* __restrict__ agg, MboxLayout L, int rank, int dir, unsigned long long epoch,
                          void* const* __restrict__ mboxes, int q0, int q1) {
  void* own = mboxes[rank];
  for (int q = q0; q < q1; ++q) {
    if (q == rank) continue;
    if (threadIdx.x == 0) wait_geq(L.ack(own, dir, q), epoch - 1);  // q has read the previous epoch
    __syncthreads();
    float* dst = L.slot(mboxes[q], dir, rank);
    for (int64_t i = threadIdx.x; i < 2 * L.W; i += blockDim.x) dst[i] = agg[i];
  }
  __threadfence_system();  // every writer orders its peer stores before the flags
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = q0; q < q1; ++q)
      if (q != rank) st_release_sys(L.flag(mboxes[q], dir, rank), epoch);
  }
}

// out[j] = fold over sources q = first, first+step, ... (!= last) of
// c = A_q c + B_q from seed (0 if null); A/B from the own mailbox, or from
// `local` (this rank's aggregate) for q == rank.  Acks each source.
__global__ void k_compose_p2p(MboxLayout L, int rank, int dir, unsigned long long epoch,
                              void* const* __restrict__ mboxes, const float* __restrict__ local, int64_t first,
                              int64_t last, int64_t step, const float* __restrict__ seed, float* __restrict__ out) {
  void* own = mboxes[rank];
  if (threadIdx.x == 0)
    for (int64_t q = first; q != last; q += step)
      if (q != rank) wait_geq(L.flag(own, dir, (int)q), epoch);
  __syncthreads();
  const int64_t W = L.W;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < W; j += (int64_t)gridDim.x * blockDim.x) {
    float c = seed != nullptr ? seed[j] : 0.f;
    for (int64_t q = first; q != last; q += step) {
      const float* s = q == rank ? local : L.slot(own, dir, (int)q);
      c = __fmaf_rn(s[j], c, s[W + j]);
    }
    out[j] = c;
  }
}

// Acks after every CTA of the compose has read the slots (separate tiny
// launch on the same stream, so stream order is the barrier).
__global__ void k_ack(MboxLayout L, int rank, int dir, unsigned long long epoch, void* const* __restrict__ mboxes,
                      int64_t first, int64_t last, int64_t step) {
  if (threadIdx.x != 0) return;
  for (int64_t q = first; q != last; q += step)
    if (q != rank) st_release_sys(L.ack(mboxes[q], dir, rank), epoch);
}

}  // namespace p2p
}  // namespace linrec_dev

namespace {
int perr(int code, const std::string& m) { return linrec_impl::set_error(code, m.c_str()); }
#define PTRY(expr)                                                                                          \
  do {                                                                                                      \
    cudaError_t e_ = (expr);                                                                                \
    if (e_ != cudaSuccess) return perr(LINREC_ERR_CUDA, std::string("linrec: CUDA error in ") + #expr + ": " + \
                                                            cudaGetErrorString(e_));                        \
  } while (0)
}  // namespace

extern "C" {

size_t linrec_p2p_mailbox_bytes(int64_t W, int world) {
  if (W < 1 || world < 1) return 0;
  return linrec_dev::p2p::MboxLayout{W, world}.bytes();
}

int linrec_ipc_alloc(size_t bytes, void** ptr, unsigned char* handle64) {
  if (!ptr || !handle64 || bytes == 0) return perr(LINREC_ERR_VALUE, "ipc_alloc: bytes, ptr and handle required");
  PTRY(cudaMalloc(ptr, bytes));
  PTRY(cudaMemset(*ptr, 0, bytes));
  // cudaMemset is asynchronous for device memory: finish it before a peer
  // can open the handle and publish into the mailbox (its epoch-1 flag
  // would otherwise be wiped by the pending zero-fill).
  PTRY(cudaDeviceSynchronize());
  cudaIpcMemHandle_t h;
  PTRY(cudaIpcGetMemHandle(&h, *ptr));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle64, &h, 64);
  return LINREC_OK;
}

int linrec_ipc_open(const unsigned char* handle64, void** ptr) {
  if (!ptr || !handle64) return perr(LINREC_ERR_VALUE, "ipc_open: handle and ptr required");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, 64);
  PTRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return LINREC_OK;
}

int linrec_ipc_close(void* ptr) {
  if (ptr) PTRY(cudaIpcCloseMemHandle(ptr));
  return LINREC_OK;
}

int linrec_ipc_free(void* ptr) {
  if (ptr) PTRY(cudaFree(ptr));
  return LINREC_OK;
}

int linrec_p2p_publish_f32(const float* agg, int64_t W, int world, int rank, int dir, uint64_t epoch,
                           void* const* mboxes, int q0, int q1, void* stream) {
  if (!agg || !mboxes || W < 1 || world < 1 || rank < 0 || rank >= world || (dir != 0 && dir != 1) || epoch < 1 ||
      q0 < 0 || q1 > world)
    return perr(LINREC_ERR_VALUE, "p2p_publish: invalid arguments");
  linrec_dev::p2p::k_publish<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      agg, linrec_dev::p2p::MboxLayout{W, world}, rank, dir, (unsigned long long)epoch, mboxes, q0, q1);
  PTRY(cudaGetLastError());
  return LINREC_OK;
}

int linrec_p2p_compose_f32(int64_t W, int world, int rank, int dir, uint64_t epoch, void* const* mboxes,
                           const float* local, int64_t first, int64_t last, int64_t step, const float* seed,
                           float* out, void* stream) {
  if (!mboxes || !out || W < 1 || world < 1 || rank < 0 || rank >= world || (dir != 0 && dir != 1) || epoch < 1 ||
      (step != 1 && step != -1))
    return perr(LINREC_ERR_VALUE, "p2p_compose: invalid arguments");
  const linrec_dev::p2p::MboxLayout L{W, world};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t blocks = (W + 255) / 256;
  linrec_dev::p2p::k_compose_p2p<<<(unsigned)(blocks < 64 ? blocks : 64), 256, 0, st>>>(
      L, rank, dir, (unsigned long long)epoch, mboxes, local, first, last, step, seed, out);
  PTRY(cudaGetLastError());
  linrec_dev::p2p::k_ack<<<1, 32, 0, st>>>(L, rank, dir, (unsigned long long)epoch, mboxes, first, last, step);
  PTRY(cudaGetLastError());
  return LINREC_OK;
}

}  // extern "C"
