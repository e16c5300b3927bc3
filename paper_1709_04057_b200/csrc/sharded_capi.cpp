// Sequence-sharded scan behind the C ABI (include/linrec_cuda.h,
// "sequence-sharded scan"): the per-rank orchestration of
// paper_1709_04057_b200/sharded.py (SequenceShardedScan, peer-memory
// exchange) in C++, so a C/C++ host runs the whole multi-GPU step -- the
// reference's phase-2/3 stitch (recurrence.hpp:219-237) lifted from chunks
// to ranks.  Per direction and step a rank launches two kernels: the segment
// scan (which also publishes the rank aggregate into the consumers'
// mailboxes over NVLink) and the compose + fix-up (which acquires the
// sources' aggregates).  No collective, no host synchronisation.
#include "linrec_cuda.h"

#include <cuda_runtime.h>

#include <cstring>
#include <new>
#include <string>
#include <vector>

namespace linrec_impl {
int set_error(int code, const char* msg);
}

struct linrec_sharded {
  int64_t T = 0, W = 0, row0 = 0, rows = 0;
  int world = 1, rank = 0, device = 0;
  int64_t tile_f = 0, tile_b = 0;
  uint64_t epoch[2] = {0, 0};
  // device buffers (one allocation)
  void* block = nullptr;
  float *seg_prod_f = nullptr, *seg_prod_b = nullptr, *agg = nullptr, *c_in = nullptr, *y_in = nullptr;
  float *ones = nullptr, *zeros = nullptr, *dh0_loc = nullptr;
  void** mboxes = nullptr;  // device array [world]
  bool have_carry = false;  // c_in holds the row before the segment (a forward ran)
};

namespace {
int err(int code, const std::string& m) { return linrec_impl::set_error(code, m.c_str()); }
#define STRY(expr)                                                                                         \
  do {                                                                                                     \
    cudaError_t e_ = (expr);                                                                               \
    if (e_ != cudaSuccess) return err(LINREC_ERR_CUDA, std::string("linrec: CUDA error in ") + #expr + ": " + \
                                                           cudaGetErrorString(e_));                        \
  } while (0)

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int d) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != d) cudaSetDevice(d);
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

linrec_exchange_t exchange(const linrec_sharded* s, int dir) {
  linrec_exchange_t e;
  e.mboxes = s->mboxes;
  e.world = s->world;
  e.rank = s->rank;
  e.epoch = s->epoch[dir];
  const int r = s->rank, R = s->world;
  if (dir == 0) {  // forward: publish to r+1..R-1, fold 0..r-1
    e.consumers_first = r + 1;
    e.consumers_last = R;
    e.sources_first = 0;
    e.sources_last = r;
    e.sources_step = 1;
    e.zero_a = r == 0;  // h0 is already inside rank 0's aggregate
  } else {  // backward: publish to 0..r-1, fold R-1..r+1
    e.consumers_first = 0;
    e.consumers_last = r;
    e.sources_first = R - 1;
    e.sources_last = r;
    e.sources_step = -1;
    e.zero_a = 0;
  }
  return e;
}
}  // namespace

extern "C" {

void linrec_sharded_bounds(int64_t T, int world, int rank, int64_t* row0, int64_t* rows) {
  // contiguous, sizes differing by at most one, longer segments first
  // (plan_chunks' rule, recurrence.hpp:61-80, applied to ranks)
  if (world < 1 || rank < 0 || rank >= world || T < 0) {
    if (row0) *row0 = 0;
    if (rows) *rows = 0;
    return;
  }
  const int64_t base = T / world, rem = T % world;
  if (row0) *row0 = rank * base + (rank < rem ? rank : rem);
  if (rows) *rows = base + (rank < rem ? 1 : 0);
}

int linrec_sharded_create(linrec_sharded_t* out, int64_t T, int64_t W, int world, int rank,
                          void* const* mboxes, int device) {
  if (!out) return err(LINREC_ERR_VALUE, "sharded_create: out required");
  *out = nullptr;
  if (T < 1 || W < 1) return err(LINREC_ERR_SHAPE, "Tensor3 dimensions must be >= 1");
  if (world < 1 || rank < 0 || rank >= world) return err(LINREC_ERR_VALUE, "sharded_create: invalid world / rank");
  if (T < world) return err(LINREC_ERR_SHAPE, "sharded_create: every rank needs at least one step (T >= world)");
  if (W % 4 != 0) return err(LINREC_ERR_VALUE, "sharded_create: the peer-memory exchange needs W % 4 == 0 (fp32)");
  if (!mboxes) return err(LINREC_ERR_VALUE, "sharded_create: mailboxes required");
  for (int q = 0; q < world; ++q)
    if (!mboxes[q]) return err(LINREC_ERR_VALUE, "sharded_create: every rank's mailbox must be mapped");
  DevGuard dg(device);
  linrec_sharded* s = new (std::nothrow) linrec_sharded();
  if (!s) return err(LINREC_ERR_INTERNAL, "sharded_create: out of host memory");
  s->T = T;
  s->W = W;
  s->world = world;
  s->rank = rank;
  s->device = device;
  linrec_sharded_bounds(T, world, rank, &s->row0, &s->rows);
  s->tile_f = linrec_segment_tile_rows(s->rows, W, 4, 0);
  s->tile_b = linrec_segment_tile_rows(s->rows, W, 4, 1);
  const int64_t nf = linrec_segment_prod_rows(s->rows, W, 4, 0);
  const int64_t nb = linrec_segment_prod_rows(s->rows, W, 4, 1);
  // [seg_prod_f | seg_prod_b | agg 2W | c_in | y_in | ones | zeros | dh0_loc] floats, then world pointers
  const size_t nfloats = size_t(nf + nb) * W + size_t(7) * W;
  const size_t bytes = nfloats * 4 + size_t(world) * sizeof(void*) + 256;
  cudaError_t e = cudaMalloc(&s->block, bytes);
  if (e != cudaSuccess) {
    delete s;
    return err(LINREC_ERR_CUDA, std::string("sharded_create: cudaMalloc: ") + cudaGetErrorString(e));
  }
  float* f = static_cast<float*>(s->block);
  s->seg_prod_f = f;
  f += nf * W;
  s->seg_prod_b = f;
  f += nb * W;
  s->agg = f;
  f += 2 * W;
  s->c_in = f;
  f += W;
  s->y_in = f;
  f += W;
  s->ones = f;
  f += W;
  s->zeros = f;
  f += W;
  s->dh0_loc = f;
  f += W;
  s->mboxes = reinterpret_cast<void**>((reinterpret_cast<uintptr_t>(f) + 255) & ~uintptr_t(255));
  std::vector<float> one(size_t(W), 1.0f);
  if ((e = cudaMemset(s->block, 0, bytes)) == cudaSuccess &&
      (e = cudaMemcpy(s->ones, one.data(), size_t(W) * 4, cudaMemcpyHostToDevice)) == cudaSuccess)
    e = cudaMemcpy(s->mboxes, mboxes, size_t(world) * sizeof(void*), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(s->block);
    delete s;
    return err(LINREC_ERR_CUDA, std::string("sharded_create: ") + cudaGetErrorString(e));
  }
  *out = s;
  return LINREC_OK;
}

int linrec_sharded_destroy(linrec_sharded_t s) {
  if (!s) return LINREC_OK;
  DevGuard dg(s->device);
  STRY(cudaDeviceSynchronize());
  STRY(cudaFree(s->block));
  delete s;
  return LINREC_OK;
}

int linrec_sharded_rows(linrec_sharded_t s, int64_t* row0, int64_t* rows) {
  if (!s) return err(LINREC_ERR_VALUE, "sharded_rows: null context");
  if (row0) *row0 = s->row0;
  if (rows) *rows = s->rows;
  return LINREC_OK;
}

int linrec_sharded_scan_f32(linrec_sharded_t s, const float* lam, const float* x, const float* h0, float* h,
                            linrec_workspace_t ws, void* stream) {
  if (!s) return err(LINREC_ERR_VALUE, "sharded_scan: null context");
  if (!lam || !x || !h) return err(LINREC_ERR_VALUE, "sharded_scan: decays, impulses and h are required");
  DevGuard dg(s->device);
  s->epoch[0] += 1;
  const linrec_exchange_t ex = exchange(s, 0);
  int rc = linrec_segment_scan_exchange_f32(lam, x, s->rank == 0 ? h0 : nullptr, h, s->seg_prod_f, s->agg, s->rows,
                                            s->W, &ex, ws, stream);
  if (rc) return rc;
  // every rank: the fix-up also stitches the segment's own virtual segments;
  // c_in receives the carry entering the segment (kept for the backward)
  rc = linrec_segment_fixup_exchange_f32(lam, h, s->seg_prod_f, s->c_in, s->rows, s->W, s->tile_f, &ex, stream);
  if (rc) return rc;
  s->have_carry = true;  // (rank 0's row before the segment is h0 itself)
  return LINREC_OK;
}

int linrec_sharded_scan_backward_f32(linrec_sharded_t s, const float* lam, const float* h0, const float* hprev,
                                     const float* h, const float* dh, float* dlam, float* dx, float* dh0,
                                     linrec_workspace_t ws, void* stream) {
  if (!s) return err(LINREC_ERR_VALUE, "sharded_scan_backward: null context");
  if (!lam || !h || !dh || !dlam || !dx)
    return err(LINREC_ERR_VALUE, "sharded_scan_backward: decays, h, d_h, d_decays and d_impulses are required");
  const int r = s->rank, R = s->world;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DevGuard dg(s->device);
  if (!hprev) {
    if (r == 0) hprev = h0 ? h0 : s->zeros;
    else if (s->have_carry) hprev = s->c_in;
    else
      return err(LINREC_ERR_VALUE,
                 "sharded_scan_backward: pass hprev (h at the row before this rank's segment) or run the forward "
                 "first");
  }
  const float* lam_next = r < R - 1 ? s->ones : nullptr;  // the next rank's decay travels in its carry
  if (r == R - 1) STRY(cudaMemsetAsync(s->y_in, 0, size_t(s->W) * 4, st));
  s->epoch[1] += 1;
  const linrec_exchange_t ex = exchange(s, 1);
  int rc = linrec_segment_scan_backward_exchange_f32(lam, hprev, h, dh, lam_next, dlam, dx, s->dh0_loc,
                                                     s->seg_prod_b, s->agg, s->rows, s->W, &ex, ws, stream);
  if (rc) return rc;
  rc = linrec_segment_fixup_backward_exchange_f32(lam, hprev, h, lam_next, s->seg_prod_b, s->y_in, dlam, dx, s->rows,
                                                  s->W, s->tile_b, &ex, stream);
  if (rc) return rc;
  if (r == 0 && dh0)  // dh0 = A'_0 * y_in + B'_0 from rank 0's own aggregate
    return linrec_compose_carries_f32(s->agg, 0, 1, 1, s->y_in, dh0, s->W, stream);
  return LINREC_OK;
}

}  // extern "C"
