/*
 * linrec_cuda.h -- C ABI of the B200 (sm_100a) linear-recurrence scan.
 *
 *     h_t = lam_t (*) h_{t-1} + x_t            (forward scan)
 *     G_t = lam_{t+1} (*) G_{t+1} + dh_t        (reverse-time backward scan)
 *     dx_t = G_t,  dlam_t = h_{t-1} (*) G_t,  dh0 = lam_1 (*) G_1
 *
 * This is the drop-in boundary for the reference's recurrence hot path
 * (/root/reference/proj/include/linrec/recurrence.hpp and its pybind11
 * module proj/bindings/linrec_py.cpp).  Every entry point below names the
 * reference interface it replaces.  Plain pointers and sizes only: no C++,
 * no torch, no CUDA headers in the signatures (`stream` is a cudaStream_t
 * passed as void*, NULL = legacy default stream).
 *
 * Layout (tensor.hpp:3-7, :49-75): every [T, batch, features] tensor is
 * time-major, C-contiguous, so step t is the contiguous slab [t*W, (t+1)*W)
 * with W = batch*features.  The library only sees (T, W).  [batch, features]
 * tensors (h0, dh0) are W contiguous values.
 *
 * Ownership: the caller owns every data buffer.  The library owns only the
 * look-back workspace (flags + chunk carries), either an explicit
 * linrec_workspace_t or a per-(device, stream) default one.
 *
 * Errors: every function returns a linrec_status; a thread-local message is
 * available from linrec_last_error().  Codes mirror the reference's error
 * classes (bindings map them back to the same Python exceptions):
 *   LINREC_ERR_SHAPE  -> ContractViolation / RuntimeError (recurrence.hpp:39-51, tensor.hpp:58)
 *   LINREC_ERR_DTYPE  -> TypeError  (linrec_py.cpp:24-29, :82-89)
 *   LINREC_ERR_VALUE  -> ValueError (linrec_py.cpp:35-37, :71-80)
 *   LINREC_ERR_CUDA   -> RuntimeError (no CPU fallback exists)
 *   LINREC_ERR_NONFINITE -> ContractViolation with the reference's
 *                       "non-finite value in <name> at [t=.., b=.., n=..]"
 *                       message (recurrence.hpp:133-163)
 *
 * Determinism: for fixed (T, W, dtype, mode) the results are bit-identical
 * run to run (the decoupled look-back applies chunk carries in a fixed
 * order).  mode LINREC_SERIAL is additionally bit-identical
 * to the reference's scan_serial / ScanMode::Serial backward on an
 * FMA-contracting x86-64 build.
 */
#ifndef LINREC_CUDA_H_
#define LINREC_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define LINREC_ABI_VERSION 1

typedef enum linrec_status {
  LINREC_OK = 0,
  LINREC_ERR_SHAPE = 1,
  LINREC_ERR_DTYPE = 2,
  LINREC_ERR_VALUE = 3,
  LINREC_ERR_CUDA = 4,
  LINREC_ERR_NONFINITE = 5,
  LINREC_ERR_INTERNAL = 6
} linrec_status;

/* ScanMode (recurrence.hpp:25).  LINREC_SERIAL runs the per-channel serial
 * kernel (bit-exact anchor); LINREC_PARALLEL the single-pass chained scan. */
typedef enum linrec_mode { LINREC_SERIAL = 0, LINREC_PARALLEL = 1 } linrec_mode;

typedef struct linrec_workspace* linrec_workspace_t;

/* ---- library ---------------------------------------------------------- */
int linrec_abi_version(void);
const char* linrec_last_error(void);
/* Number of CUDA devices visible (0 when none); never falls back to a CPU. */
int linrec_device_count(void);

/* Kernel selection for LINREC_PARALLEL.  AUTO (default) runs the persistent
 * TMA-fed kernels whenever rows are 16-byte aligned and W is a multiple of
 * the vector width, else the register-tiled kernels; REGISTER forces the
 * latter (testing / comparison).  Process-wide. */
typedef enum linrec_kernel_policy { LINREC_KERNEL_AUTO = 0, LINREC_KERNEL_REGISTER = 1 } linrec_kernel_policy;
int linrec_set_kernel_policy(int policy);

/* Device memory for callers without their own allocator (the Python
 * bindings' DeviceArray).  Stream-ordered on `stream`. */
int linrec_device_malloc(void** ptr, size_t bytes, int device, void* stream);
int linrec_device_free(void* ptr, int device, void* stream);

/* ---- workspace --------------------------------------------------------- *
 * Look-back state for the chained scans: a control block (epoch, ticket and
 * retirement counters), per-chunk status flags and per-chunk carries.  Grows
 * on demand, stream-ordered.  One workspace must not be used by two streams
 * concurrently; ws == NULL in the scan calls selects a library-owned
 * workspace keyed by (current device, stream). */
int linrec_workspace_create(linrec_workspace_t* ws, int device);
int linrec_workspace_destroy(linrec_workspace_t ws);
/* Bytes a chained scan of (T, W) in `dtype_bytes` (4 or 8) needs. */
size_t linrec_workspace_bytes(int64_t T, int64_t W, int dtype_bytes);

/* ---- forward scan, device pointers ------------------------------------- *
 * Replaces linrec::scan_serial (recurrence.hpp:169-179), scan_parallel
 * (:193-245) and scan (:255-263) -- and the compute of linrec.scan,
 * linrec_py.cpp:91-116.  lam, x, h: [T][W]; h0: [W] or NULL (= zeros,
 * linrec_py.cpp:98-100).  Asynchronous on `stream`.  T >= 1, W >= 1. */
int linrec_scan_f32(const float* lam, const float* x, const float* h0,
                    float* h, int64_t T, int64_t W, int mode,
                    linrec_workspace_t ws, void* stream);
int linrec_scan_f64(const double* lam, const double* x, const double* h0,
                    double* h, int64_t T, int64_t W, int mode,
                    linrec_workspace_t ws, void* stream);

/* ---- backward scan, device pointers ------------------------------------ *
 * Replaces linrec::scan_backward / detail::scan_backward_impl
 * (recurrence.hpp:283-377) and the compute of linrec.scan_backward
 * (linrec_py.cpp:118-140).  Inputs lam, h, dh: [T][W]; h0: [W] or NULL.
 * Outputs dlam, dx: [T][W]; dh0: [W].  Does not read x (the reference does
 * not either, recurrence.hpp:273-282).  No reversed copies are made.
 * dlam may be NULL (device entry points only): it is then not written --
 * callers that fold dlam = h_{t-1} * dx into their own pass (the layers)
 * save its 4 B/element store. */
int linrec_scan_backward_f32(const float* lam, const float* h0,
                             const float* h, const float* dh, float* dlam,
                             float* dx, float* dh0, int64_t T, int64_t W,
                             int mode, linrec_workspace_t ws, void* stream);
int linrec_scan_backward_f64(const double* lam, const double* h0,
                             const double* h, const double* dh, double* dlam,
                             double* dx, double* dh0, int64_t T, int64_t W,
                             int mode, linrec_workspace_t ws, void* stream);

/* Segment form of the backward scan (no reference counterpart: it is what
 * the reference's phase-2/phase-3 stitching does across chunk boundaries,
 * recurrence.hpp:219-237, lifted to the caller so a sequence can be split
 * across host chunks or GPUs).  The segment [0,T) is followed by a row whose
 * decay is lam_next[W] and whose gradient state is g_next[W] (both NULL =
 * the true end of the sequence, G_T := 0).  G_{T-1} = lam_next*g_next +
 * dh_{T-1} is evaluated as one fused multiply-add, as in the unsplit scan,
 * so LINREC_SERIAL stays bit-exact when chained. */
/* Gated adjoint (fused layer backward): scan_backward on d_h * gate
 * elementwise, for a layer whose output is h = gate * c of the recurrence's
 * state c -- GILR-LSTM's h = o * c (layers.hpp:312-324: dc = dh * o into
 * scan_backward) and QRNN's (layers.hpp:510-521).  The product is taken as the adjoint is staged
 * into shared memory (no dc array); dh0 and dlam (nullable) as
 * linrec_scan_backward_f32. */
int linrec_scan_backward_gated_f32(const float* lam, const float* h0,
                                   const float* h, const float* dh,
                                   const float* gate, float* dlam, float* dx,
                                   float* dh0, int64_t T, int64_t W, int mode,
                                   linrec_workspace_t ws, void* stream);
int linrec_scan_backward_segment_f32(const float* lam, const float* h0,
                                     const float* h, const float* dh,
                                     const float* lam_next,
                                     const float* g_next, float* dlam,
                                     float* dx, float* dh0, int64_t T,
                                     int64_t W, int mode,
                                     linrec_workspace_t ws, void* stream);
int linrec_scan_backward_segment_f64(const double* lam, const double* h0,
                                     const double* h, const double* dh,
                                     const double* lam_next,
                                     const double* g_next, double* dlam,
                                     double* dx, double* dh0, int64_t T,
                                     int64_t W, int mode,
                                     linrec_workspace_t ws, void* stream);

/* ---- host-pointer entry points (the numpy boundary) --------------------- *
 * Same semantics with HOST buffers: the call stages T-chunks host->device,
 * scans each chunk seeded with the previous chunk's carry, and copies results
 * back, overlapping the three on separate streams (full-duplex PCIe/C2C).
 * Page-locked (pinned) buffers run fully asynchronous; pageable buffers work
 * but are staged by the driver.  Synchronous: returns when the outputs are in
 * host memory.  `device` selects the GPU. */
int linrec_scan_host_f32(const float* lam, const float* x, const float* h0,
                         float* h, int64_t T, int64_t W, int mode,
                         int device);
int linrec_scan_host_f64(const double* lam, const double* x,
                         const double* h0, double* h, int64_t T, int64_t W,
                         int mode, int device);
int linrec_scan_backward_host_f32(const float* lam, const float* h0,
                                  const float* h, const float* dh,
                                  float* dlam, float* dx, float* dh0,
                                  int64_t T, int64_t W, int mode, int device);
int linrec_scan_backward_host_f64(const double* lam, const double* h0,
                                  const double* h, const double* dh,
                                  double* dlam, double* dx, double* dh0,
                                  int64_t T, int64_t W, int mode, int device);

/* ---- channel sharding of host arrays ---------------------- *
 * Channels are independent (recurrence.hpp:109: the inner loop of scan_span
 * runs over j), so a [T][W] problem splits into column blocks with no
 * communication.  *_columns: scan columns [c0, c1) of the FULL host arrays
 * (row stride W; h0 / dh0 are full [W] rows) on `device`, staging the strided
 * block with 2-D copies; only those columns of the outputs are written.
 * *_multi: split the columns over `ndev` devices (linrec_column_block: blocks
 * of multiples of 4 channels where W allows, longer first), one host thread
 * per device, each with its own streams -- the single-process form of the
 * channel-sharded multi-GPU scan.  Replaces: scan / scan_backward over host
 * Tensor3 (recurrence.hpp:255-263, :352-363) for the channel-parallel case. */
int linrec_scan_host_columns_f32(const float* lam, const float* x,
                                 const float* h0, float* h, int64_t T,
                                 int64_t W, int64_t c0, int64_t c1, int mode,
                                 int device);
int linrec_scan_host_columns_f64(const double* lam, const double* x,
                                 const double* h0, double* h, int64_t T,
                                 int64_t W, int64_t c0, int64_t c1, int mode,
                                 int device);
int linrec_scan_backward_host_columns_f32(const float* lam, const float* h0,
                                          const float* h, const float* dh,
                                          float* dlam, float* dx, float* dh0,
                                          int64_t T, int64_t W, int64_t c0,
                                          int64_t c1, int mode, int device);
int linrec_scan_backward_host_columns_f64(const double* lam,
                                          const double* h0, const double* h,
                                          const double* dh, double* dlam,
                                          double* dx, double* dh0, int64_t T,
                                          int64_t W, int64_t c0, int64_t c1,
                                          int mode, int device);
int linrec_scan_host_multi_f32(const float* lam, const float* x,
                               const float* h0, float* h, int64_t T, int64_t W,
                               int mode, const int* devices, int ndev);
int linrec_scan_host_multi_f64(const double* lam, const double* x,
                               const double* h0, double* h, int64_t T,
                               int64_t W, int mode, const int* devices,
                               int ndev);
int linrec_scan_backward_host_multi_f32(const float* lam, const float* h0,
                                        const float* h, const float* dh,
                                        float* dlam, float* dx, float* dh0,
                                        int64_t T, int64_t W, int mode,
                                        const int* devices, int ndev);
int linrec_scan_backward_host_multi_f64(const double* lam, const double* h0,
                                        const double* h, const double* dh,
                                        double* dlam, double* dx, double* dh0,
                                        int64_t T, int64_t W, int mode,
                                        const int* devices, int ndev);
/* FNV-1a 64-bit hash of host bytes, continuing from h (start: 0xcbf29ce484222325):
 * the input checksum of the reference's bench_kernel protocol
 * (bench.hpp:69-85 fnv1a64 / checksum_inputs), so a GPU bench row can be
 * matched to the reference's row on identical inputs. */
uint64_t linrec_fnv1a64(const void* data, size_t len, uint64_t h);
/* Column block [c0, c1) of device d of n under channel sharding. */
int linrec_column_block(int64_t W, int n, int d, int64_t* c0, int64_t* c1);

/* Page-locked host memory from a caching allocator (blocks are recycled by
 * size; at most a quarter of RAM stays pinned while idle).  Host buffers
 * from here run the host entry points above at full link speed: the Python
 * module allocates its numpy results with it (linrec_py.cpp:56-69 returns
 * fresh arrays; these are fresh too, just page-locked). */
int linrec_host_alloc(void** ptr, size_t bytes);
int linrec_host_free(void* ptr);

/* ---- finite screening (recurrence.hpp:133-163) -------------------------- *
 * Index of the first non-finite element of v[n] (device pointer), or -1.
 * Synchronous on `stream`. */
int linrec_first_nonfinite_f32(const float* v, int64_t n, int64_t* index,
                               void* stream);
int linrec_first_nonfinite_f64(const double* v, int64_t n, int64_t* index,
                               void* stream);

/* screen_finite (recurrence.hpp:133-155) of a device tensor
 * [T][batch][features] (T = 0: a [batch][features] tensor such as h0): OK,
 * or LINREC_ERR_NONFINITE with the reference's message
 * "non-finite value in <name> at [t=<1-based step>, b=<batch>, n=<feature>]"
 * ("[b=.., n=..]" for T = 0) naming the FIRST non-finite element in memory
 * order.  The check_finite option of scan_serial / scan_parallel / scan /
 * scan_backward (recurrence.hpp:169-377) is this screen on decays, impulses
 * and initial (forward) or decays and d_h (backward, :292-296) before the
 * scan; include/linrec/cuda_scan.hpp exposes it under those names.
 * Synchronous on `stream`. */
int linrec_screen_finite_f32(const float* v, int64_t T, int64_t batch,
                             int64_t features, const char* name,
                             void* stream);
int linrec_screen_finite_f64(const double* v, int64_t T, int64_t batch,
                             int64_t features, const char* name,
                             void* stream);

/* Kernels one linrec_scan_* (backward = 0) / linrec_scan_backward_* call
 * launches for this shape and mode with 16-byte aligned buffers (1; 2 when
 * the sequence is split into virtual segments: scan and fix-up; 5 with the
 * decay-adaptive stitch); -1 for invalid arguments.  For launch accounting
 * (bench.py's gpu_launches). */
int linrec_scan_kernel_count(int64_t T, int64_t W, int dtype_bytes, int backward, int mode);
/* The kernel family that call runs (static string): "serial" (per-channel),
 * "cluster" (thread-block cluster over a short sequence), "local" (CTA-local),
 * "tma" (persistent TMA-fed chained scan), "chained" (register chained scan);
 * NULL for invalid arguments.  For reports (bench.py's roofline kernel). */
const char* linrec_scan_kernel_name(int64_t T, int64_t W, int dtype_bytes, int backward, int mode);

/* ---- the reference's chunked scan with an explicit plan ----------------- *
 * scan_parallel(decays, impulses, initial, plan, pool, check_finite,
 * summaries) (recurrence.hpp:193-245) and scan_backward(in, h, d_h, plan,
 * pool) (:365-377) on the device: the reference's three phases (chunk
 * summaries, sequential stitch, seeded chunk re-scans) in its per-channel
 * operation order, so h and the ScanSummaries P, R, C [chunks][W]
 * (:186-191; each nullable) are bit-identical to the reference's for the
 * same plan.  bounds: HOST array of `chunks` (start, end) 1-based inclusive
 * pairs, checked like validate_plan (:84-94, same messages); plan_chunks
 * (:61-80) is linrec.plan_chunks.  The backward scans the reversed image
 * with the plan (ScanMode::Parallel).  Device pointers, stream-ordered; the
 * default parallel mode (linrec_scan_*) is the faster single-pass scan. */
int linrec_scan_plan_f32(const float* lam, const float* x, const float* h0, float* h, int64_t T, int64_t W,
                         const int64_t* bounds, int64_t chunks, float* P, float* R, float* C, void* stream);
int linrec_scan_plan_f64(const double* lam, const double* x, const double* h0, double* h, int64_t T, int64_t W,
                         const int64_t* bounds, int64_t chunks, double* P, double* R, double* C, void* stream);
int linrec_scan_backward_plan_f32(const float* lam, const float* h0, const float* h, const float* dh, float* dlam,
                                  float* dx, float* dh0, int64_t T, int64_t W, const int64_t* bounds,
                                  int64_t chunks, void* stream);
int linrec_scan_backward_plan_f64(const double* lam, const double* h0, const double* h, const double* dh,
                                  double* dlam, double* dx, double* dh0, int64_t T, int64_t W,
                                  const int64_t* bounds, int64_t chunks, void* stream);

/* ---- sequence sharding across GPUs (BASELINE.json north_star) ----------- *
 * A sequence split into contiguous T-segments, one per rank.  Forward, rank r
 * (segment [S, E)):
 *   1. linrec_segment_scan_*: single-pass scan of the segment seeded with h0
 *      on rank 0 and with 0 elsewhere, split internally into virtual
 *      segments whose stitch is left to step 4; it writes seg_prod (the decay
 *      products entering each chain position, plus the virtual segments'
 *      aggregates) and agg[2][W] = (prod lam over the segment, zero-carry
 *      state at its last row);
 *   2. all-gather of agg over the ranks (NCCL, the caller's communicator);
 *   3. linrec_compose_carries_*: c_in = fold of the aggregates of ranks
 *      0..r-1 (c = A_q*c + B_q from 0; rank 0 publishes A = 0);
 *   4. linrec_segment_fixup_* on EVERY rank (c_in = NULL on rank 0): one
 *      pass adding P_t * (virtual-segment carry + scale * c_in) on the tiles
 *      whose entering correction is non-zero (exact: past the underflow the
 *      correction is 0).
 * Backward, reverse time, with lam_next = a row of ones on every rank but the
 * last (the decay linking to the next rank is applied through the carry):
 *   1. linrec_segment_scan_backward_* (hprev = the true h row before the
 *      segment) writes dlam, dx, seg_prod, agg = (A', B') = (lam_S * prod mu,
 *      lam_S * G_S) and dh0 = B'; 2. all-gather agg; 3. compose ranks
 *      R-1 .. r+1 into y_in; 4. linrec_segment_fixup_backward_* on every
 *      rank (y_in = NULL on the last) adds P'_t*y to dx and h_{t-1}*P'_t*y to
 *      dlam; rank 0's dh0 = A'_0*y_in + B'_0 (compose with seed y_in).
 * seg_prod holds linrec_segment_prod_rows(...) rows of W values (the decay
 * products entering each chain position of the scan's virtual segments, then
 * those segments' aggregates, from which the fix-up folds each virtual
 * segment's carry); pass linrec_segment_tile_rows(...) to the fix-up.  Buffers 16-byte aligned when
 * W is a multiple of 4 (fp32) / 2 (fp64). */
int64_t linrec_segment_prod_rows(int64_t T, int64_t W, int dtype_bytes, int backward);
int64_t linrec_segment_tile_rows(int64_t T, int64_t W, int dtype_bytes, int backward);
int linrec_segment_scan_f32(const float* lam, const float* x, const float* h0, float* h, float* seg_prod,
                            float* agg, int64_t T, int64_t W, linrec_workspace_t ws, void* stream);
int linrec_segment_scan_f64(const double* lam, const double* x, const double* h0, double* h, double* seg_prod,
                            double* agg, int64_t T, int64_t W, linrec_workspace_t ws, void* stream);
int linrec_segment_scan_backward_f32(const float* lam, const float* hprev, const float* h, const float* dh,
                                     const float* lam_next, float* dlam, float* dx, float* dh0,
                                     float* seg_prod, float* agg, int64_t T, int64_t W, linrec_workspace_t ws,
                                     void* stream);
int linrec_segment_scan_backward_f64(const double* lam, const double* hprev, const double* h, const double* dh,
                                     const double* lam_next, double* dlam, double* dx, double* dh0,
                                     double* seg_prod, double* agg, int64_t T, int64_t W,
                                     linrec_workspace_t ws, void* stream);
int linrec_compose_carries_f32(const float* aggs, int64_t first, int64_t last, int64_t step, const float* seed,
                               float* out, int64_t W, void* stream);
int linrec_compose_carries_f64(const double* aggs, int64_t first, int64_t last, int64_t step, const double* seed,
                               double* out, int64_t W, void* stream);
int linrec_segment_fixup_f32(const float* lam, float* h, const float* seg_prod, const float* c_in, int64_t T,
                             int64_t W, int64_t tile_rows, void* stream);
int linrec_segment_fixup_f64(const double* lam, double* h, const double* seg_prod, const double* c_in,
                             int64_t T, int64_t W, int64_t tile_rows, void* stream);
int linrec_segment_fixup_backward_f32(const float* lam, const float* hprev, const float* h, const float* lam_next,
                                      const float* seg_prod, const float* y_in, float* dlam, float* dx, int64_t T,
                                      int64_t W, int64_t tile_rows, void* stream);
int linrec_segment_fixup_backward_f64(const double* lam, const double* hprev, const double* h,
                                      const double* lam_next, const double* seg_prod, const double* y_in,
                                      double* dlam, double* dx, int64_t T, int64_t W, int64_t tile_rows,
                                      void* stream);

/* The same steps with the carry exchange fused into the stitch kernels over
 * peer memory (the mailboxes of linrec_ipc_alloc / linrec_p2p_mailbox_bytes
 * below): the scan's virtual-segment fold stores this rank's aggregate
 * straight into the consumers' mailboxes and releases their flags; the
 * fix-up acquires the sources' flags, folds their aggregates into the
 * incoming carry in-kernel (also written to c_in / y_in when non-NULL) and
 * acknowledges them -- no all-gather and no compose launch.  fp32.
 * Forward: consumers = ranks r+1..R-1, sources = 0..r-1 (step 1), zero_a on
 * rank 0; backward: consumers = 0..r-1, sources = R-1..r+1 (step -1).  Every
 * rank calls every step (empty ranges are fine); epoch advances by one per
 * step and direction. */
typedef struct {
  void* const* mboxes;  /* DEVICE array [world] of every rank's mailbox, mapped in this process */
  int world, rank;
  uint64_t epoch;
  int consumers_first, consumers_last;             /* [first, last) */
  int sources_first, sources_last, sources_step;   /* first, first+step, ... != last */
  int zero_a;                                      /* publish A = 0 */
} linrec_exchange_t;
int linrec_segment_scan_exchange_f32(const float* lam, const float* x, const float* h0, float* h, float* seg_prod,
                                     float* agg, int64_t T, int64_t W, const linrec_exchange_t* ex,
                                     linrec_workspace_t ws, void* stream);
int linrec_segment_scan_backward_exchange_f32(const float* lam, const float* hprev, const float* h, const float* dh,
                                              const float* lam_next, float* dlam, float* dx, float* dh0,
                                              float* seg_prod, float* agg, int64_t T, int64_t W,
                                              const linrec_exchange_t* ex, linrec_workspace_t ws, void* stream);
int linrec_segment_fixup_exchange_f32(const float* lam, float* h, const float* seg_prod, float* c_in, int64_t T,
                                      int64_t W, int64_t tile_rows, const linrec_exchange_t* ex, void* stream);
int linrec_segment_fixup_backward_exchange_f32(const float* lam, const float* hprev, const float* h,
                                               const float* lam_next, const float* seg_prod, float* y_in,
                                               float* dlam, float* dx, int64_t T, int64_t W, int64_t tile_rows,
                                               const linrec_exchange_t* ex, void* stream);

/* ---- sequence-sharded scan: one call per rank and step ------------------- *
 * The whole sharded step of SURVEY.md 8e for a C/C++ host (the Python
 * driver paper_1709_04057_b200/sharded.py runs the same sequence): T rows of
 * a [T][W] fp32 problem split into `world` contiguous segments
 * (linrec_sharded_bounds: plan_chunks' rule, recurrence.hpp:61-80, applied
 * to ranks), rank r owning rows [row0, row0 + rows) on its own GPU.  Each
 * direction runs the segment scan (which publishes the rank's (A, B)
 * aggregate into the consumers' mailboxes over NVLink) and the compose +
 * fix-up (which acquires the sources' aggregates) -- the reference's
 * phase-2/3 stitch (recurrence.hpp:219-237) across ranks, with no
 * collective and no host synchronisation.
 *   mboxes: HOST array [world] of every rank's mailbox mapped in this
 *   process (own: linrec_ipc_alloc of linrec_p2p_mailbox_bytes(W, world);
 *   peers: linrec_ipc_open of their handles, exchanged out of band).
 *   Requirements: T >= world, W % 4 == 0, 16-byte aligned buffers.
 * Every rank calls every step in the same order (epochs advance per call).
 * scan: lam, x, h [rows][W] of this rank; h0 [W] read on rank 0 only (NULL =
 * zeros).  scan_backward: lam, h, dh -> dlam, dx [rows][W]; hprev = h at the
 * row before the segment (NULL: rank 0 uses h0, the others the carry their
 * last forward computed); dh0 [W] written on rank 0 only (others may pass
 * NULL).  Stream-ordered on `stream`; the context is not thread-safe. */
typedef struct linrec_sharded* linrec_sharded_t;
void linrec_sharded_bounds(int64_t T, int world, int rank, int64_t* row0, int64_t* rows);
int linrec_sharded_create(linrec_sharded_t* ctx, int64_t T, int64_t W, int world, int rank, void* const* mboxes,
                          int device);
int linrec_sharded_destroy(linrec_sharded_t ctx);
int linrec_sharded_rows(linrec_sharded_t ctx, int64_t* row0, int64_t* rows);
int linrec_sharded_scan_f32(linrec_sharded_t ctx, const float* lam, const float* x, const float* h0, float* h,
                            linrec_workspace_t ws, void* stream);
int linrec_sharded_scan_backward_f32(linrec_sharded_t ctx, const float* lam, const float* h0, const float* hprev,
                                     const float* h, const float* dh, float* dlam, float* dx, float* dh0,
                                     linrec_workspace_t ws, void* stream);

/* ---- layer building block: tcgen05 GEMM ---------------------------------- *
 * C[M][N] (row-major, pitch ldc) (+)= sum_k A(m,k) * B(n,k) on the sm_100a
 * tensor cores (kind::tf32 MMAs, fp32 accumulate in TMEM).  A is K-major
 * ([M][K], pitch lda) when a_mn == 0, MN-major ([K][M], pitch lda) when 1;
 * likewise B.  precision LINREC_PREC_FP32 runs 3xTF32 (hi/lo operand split,
 * fp32-grade results), LINREC_PREC_TF32 one TF32 pass.  k_splits > 1 splits
 * K across CTA pairs and reduces the partials (scratch: at least
 * linrec_gemm_scratch_bytes(M, N, k_splits)) in a fixed order (deterministic).  Pitches and pointers must be 16-byte
 * aligned.  The dense transforms of the reference's layers
 * (tensor.hpp:104-141 gemm_nn/nt/tn, :249-308) map onto it. */
#define LINREC_PREC_FP32 0
#define LINREC_PREC_TF32 1
int linrec_gemm_f32(const float* A, int a_mn, int64_t lda, const float* B, int b_mn, int64_t ldb, float* C,
                    int64_t ldc, int64_t M, int64_t N, int64_t K, int accumulate, int precision, int k_splits,
                    float* scratch, void* stream);
/* split count the layers pick for an M x N x K product (fills the persistent
 * grid of CTA pairs) and the scratch a given split count needs. */
int linrec_gemm_splits(int64_t M, int64_t N, int64_t K);
size_t linrec_gemm_scratch_bytes(int64_t M, int64_t N, int k_splits);

/* ---- GILR and GILR-LSTM layers (layers.hpp:23-375) ------------------------ *
 * The paper's recurrent layers on the GPU: gate projections on the tensor
 * cores (linrec_gemm_f32 with fused activation epilogues), recurrences on the
 * chained scans above.  All buffers are caller-owned device memory, fp32,
 * time-major [T][b][.] C-contiguous (x: [T][b][m], activations [T][b][n]),
 * parameters row-major exactly as GilrParams / GilrLstmParams
 * (layers.hpp:30-40, :146-160): gate blocks f, i, o, z stacked along rows.
 * m and n must be multiples of 4 (16-byte TMA rows).  Parameter gradients
 * ACCUMULATE into the grads buffers (the reference's += semantics,
 * tensor.hpp:272-296); dx is overwritten.  `scratch` is device memory of at
 * least linrec_gilr[_lstm]_scratch_bytes(); `precision` is LINREC_PREC_FP32
 * (3xTF32, the default) or LINREC_PREC_TF32; `mode` is the ScanMode of the
 * recurrences.  NULL h0 / htil0 / c0 mean zeros; NULL dh0 / dhtil0 / dc0 are
 * not written. */
#define LINREC_ACT_TANH 0     /* Activation::Tanh     (common.hpp:49-71) */
#define LINREC_ACT_IDENTITY 1 /* Activation::Identity */
#define LINREC_ACT_RELU 2     /* Activation::Relu     */

typedef struct linrec_gilr_params_f32 { /* GilrParams<float> (layers.hpp:30-40) */
  const float* U;   /* [n][m] gate weights */
  const float* V;   /* [n][m] candidate weights */
  const float* b_g; /* [n] gate bias */
  const float* b_z; /* [n] candidate bias */
  int act;          /* candidate activation, LINREC_ACT_* */
} linrec_gilr_params_f32;

typedef struct linrec_gilr_grads_f32 { /* GilrGrads<float> (layers.hpp:66-76) */
  float* U;
  float* V;
  float* b_g;
  float* b_z;
} linrec_gilr_grads_f32;

typedef struct linrec_gilr_lstm_params_f32 { /* GilrLstmParams<float> (layers.hpp:146-160) */
  linrec_gilr_params_f32 surrogate; /* m -> n; its act must be tanh in the reference init */
  const float* U;                   /* [4n][n], applied to htil_{t-1} */
  const float* V;                   /* [4n][m], applied to x_t */
  const float* bias;                /* [4n] */
} linrec_gilr_lstm_params_f32;

typedef struct linrec_gilr_lstm_grads_f32 { /* GilrLstmGrads<float> (layers.hpp:192-211) */
  linrec_gilr_grads_f32 surrogate;
  float* U;
  float* V;
  float* bias;
} linrec_gilr_lstm_grads_f32;

/* GilrLstmCache<float> (layers.hpp:183-188), device buffers:
 *   sg, si   [T][b][n]     surrogate gate / candidate (GilrCache::g, ::i)
 *   htil     [T+1][b][n]   row 0 = htil0, rows 1..T = surrogate output, so
 *                          rows 0..T-1 are htil_prev (detail::shift_right)
 *   gates    [4][T][b][n]  activated f, i, o, z planes (the reference keeps
 *                          them interleaved as [T][b][4n])
 *   c        [T][b][n]     cell state */
typedef struct linrec_gilr_lstm_cache_f32 {
  float* sg;
  float* si;
  float* htil;
  float* gates;
  float* c;
} linrec_gilr_lstm_cache_f32;

/* Per-stage timing of the layer calls on the calling thread: between
 * linrec_profile_begin() and linrec_profile_end(), every stage of
 * linrec_gilr*_f32 records a CUDA event on the call's stream;
 * linrec_profile_end() synchronizes them and writes one line per stage,
 * "<stage> <total ms> <count>\n", in first-seen order (summed over calls). */
int linrec_profile_begin(void);
int linrec_profile_end(char* out, size_t cap);

size_t linrec_gilr_scratch_bytes(int64_t T, int64_t b, int64_t m, int64_t n);
size_t linrec_gilr_lstm_scratch_bytes(int64_t T, int64_t b, int64_t m, int64_t n);

/* gilr_forward (layers.hpp:78-100): h [T][b][n]; g, i (the cache) [T][b][n]. */
int linrec_gilr_forward_f32(const linrec_gilr_params_f32* p, const float* x, const float* h0, float* h, float* g,
                            float* i, int64_t T, int64_t b, int64_t m, int64_t n, int mode, int precision,
                            void* scratch, size_t scratch_bytes, void* stream);
/* gilr_backward (layers.hpp:102-133). */
int linrec_gilr_backward_f32(const linrec_gilr_params_f32* p, const float* x, const float* h0, const float* g,
                             const float* i, const float* h, const float* dh, linrec_gilr_grads_f32* grads,
                             float* dx, float* dh0, int64_t T, int64_t b, int64_t m, int64_t n, int mode,
                             int precision, void* scratch, size_t scratch_bytes, void* stream);
/* gilr_lstm_forward (layers.hpp:245-293): h [T][b][n]; fills the cache. */
int linrec_gilr_lstm_forward_f32(const linrec_gilr_lstm_params_f32* p, const float* x, const float* htil0,
                                 const float* c0, float* h, const linrec_gilr_lstm_cache_f32* cache, int64_t T,
                                 int64_t b, int64_t m, int64_t n, int mode, int precision, void* scratch,
                                 size_t scratch_bytes, void* stream);
/* gilr_lstm_backward (layers.hpp:295-375). */
int linrec_gilr_lstm_backward_f32(const linrec_gilr_lstm_params_f32* p, const float* x, const float* htil0,
                                  const float* c0, const linrec_gilr_lstm_cache_f32* cache, const float* dh,
                                  linrec_gilr_lstm_grads_f32* grads, float* dx, float* dhtil0, float* dc0,
                                  int64_t T, int64_t b, int64_t m, int64_t n, int mode, int precision,
                                  void* scratch, size_t scratch_bytes, void* stream);

/* ---- QRNN (layers.hpp:376-548) ------------------------------------------- *
 * [f o z]_t = act(sum_{s<k} W_s x_{t-s} + b), c_t = f c_{t-1} + (1-f) z,
 * h_t = o c_t.  W: the k taps packed [k][3n][m] (QrnnParams::W[s] at
 * W + s*3n*m), bias [3n] (blocks f, o, z).  Cache (QrnnCache :420-423):
 * gates [3][T][b][n] activated f, o, z planes, c [T][b][n].  dW (packed like
 * W) and dbias accumulate; dx is overwritten.  1 <= k <= T. */
size_t linrec_qrnn_scratch_bytes(int64_t T, int64_t b, int64_t m, int64_t n, int64_t k);
int linrec_qrnn_forward_f32(const float* W, const float* bias, const float* x, const float* c0, float* h,
                            float* gates, float* c, int64_t T, int64_t b, int64_t m, int64_t n, int64_t k, int mode,
                            int precision, void* scratch, size_t scratch_bytes, void* stream);
int linrec_qrnn_backward_f32(const float* W, const float* x, const float* c0, const float* gates, const float* c,
                             const float* dh, float* dW, float* dbias, float* dx, float* dc0, int64_t T, int64_t b,
                             int64_t m, int64_t n, int64_t k, int mode, int precision, void* scratch,
                             size_t scratch_bytes, void* stream);

/* ---- the same layers in double precision ---------------------------------- *
 * layers.hpp is templated on S and proj/tests/test_layers.cpp runs it in
 * double.  Same buffers, layouts, NULL rules and accumulate semantics as the
 * _f32 entry points above (caches: gates as activated planes); the
 * projections run on a CUDA-core fp64 GEMM (linrec_gemm_f64, no tensor-core
 * fp64 operand type on the tcgen05 TF32 path) and the recurrences on
 * linrec_scan_f64 / linrec_scan_backward_f64.  m and n may be any width.
 * No precision argument: every product is fp64. */
typedef struct linrec_gilr_params_f64 { /* GilrParams<double> (layers.hpp:30-40) */
  const double* U;
  const double* V;
  const double* b_g;
  const double* b_z;
  int act;
} linrec_gilr_params_f64;

typedef struct linrec_gilr_grads_f64 { /* GilrGrads<double> (layers.hpp:66-76) */
  double* U;
  double* V;
  double* b_g;
  double* b_z;
} linrec_gilr_grads_f64;

typedef struct linrec_gilr_lstm_params_f64 { /* GilrLstmParams<double> (layers.hpp:146-160) */
  linrec_gilr_params_f64 surrogate;
  const double* U;
  const double* V;
  const double* bias;
} linrec_gilr_lstm_params_f64;

typedef struct linrec_gilr_lstm_grads_f64 { /* GilrLstmGrads<double> (layers.hpp:192-211) */
  linrec_gilr_grads_f64 surrogate;
  double* U;
  double* V;
  double* bias;
} linrec_gilr_lstm_grads_f64;

typedef struct linrec_gilr_lstm_cache_f64 { /* GilrLstmCache<double> (layers.hpp:183-188) */
  double* sg;
  double* si;
  double* htil;
  double* gates;
  double* c;
} linrec_gilr_lstm_cache_f64;

/* C[M][N] (+)= sum_k A(m,k) * B(n,k) in fp64 on the CUDA cores; operand
 * layouts as linrec_gemm_f32 (a_mn / b_mn select MN-major). */
int linrec_gemm_f64(const double* A, int a_mn, int64_t lda, const double* B, int b_mn, int64_t ldb, double* C,
                    int64_t ldc, int64_t M, int64_t N, int64_t K, int accumulate, void* stream);

size_t linrec_gilr_scratch_bytes_f64(int64_t T, int64_t b, int64_t m, int64_t n);
size_t linrec_gilr_lstm_scratch_bytes_f64(int64_t T, int64_t b, int64_t m, int64_t n);
size_t linrec_qrnn_scratch_bytes_f64(int64_t T, int64_t b, int64_t m, int64_t n, int64_t k);
int linrec_gilr_forward_f64(const linrec_gilr_params_f64* p, const double* x, const double* h0, double* h,
                            double* g, double* i, int64_t T, int64_t b, int64_t m, int64_t n, int mode,
                            void* scratch, size_t scratch_bytes, void* stream);
int linrec_gilr_backward_f64(const linrec_gilr_params_f64* p, const double* x, const double* h0, const double* g,
                             const double* i, const double* h, const double* dh, linrec_gilr_grads_f64* grads,
                             double* dx, double* dh0, int64_t T, int64_t b, int64_t m, int64_t n, int mode,
                             void* scratch, size_t scratch_bytes, void* stream);
int linrec_gilr_lstm_forward_f64(const linrec_gilr_lstm_params_f64* p, const double* x, const double* htil0,
                                 const double* c0, double* h, const linrec_gilr_lstm_cache_f64* cache, int64_t T,
                                 int64_t b, int64_t m, int64_t n, int mode, void* scratch, size_t scratch_bytes,
                                 void* stream);
int linrec_gilr_lstm_backward_f64(const linrec_gilr_lstm_params_f64* p, const double* x, const double* htil0,
                                  const double* c0, const linrec_gilr_lstm_cache_f64* cache, const double* dh,
                                  linrec_gilr_lstm_grads_f64* grads, double* dx, double* dhtil0, double* dc0,
                                  int64_t T, int64_t b, int64_t m, int64_t n, int mode, void* scratch,
                                  size_t scratch_bytes, void* stream);
int linrec_qrnn_forward_f64(const double* W, const double* bias, const double* x, const double* c0, double* h,
                            double* gates, double* c, int64_t T, int64_t b, int64_t m, int64_t n, int64_t k, int mode,
                            void* scratch, size_t scratch_bytes, void* stream);
int linrec_qrnn_backward_f64(const double* W, const double* x, const double* c0, const double* gates, const double* c,
                             const double* dh, double* dW, double* dbias, double* dx, double* dc0, int64_t T,
                             int64_t b, int64_t m, int64_t n, int64_t k, int mode, void* scratch,
                             size_t scratch_bytes, void* stream);

/* ---- training loop (training.hpp) ----------------------------------------- *
 * The reference's synthetic long-dependency task: generate_batch (:30-43)
 * from the reference Rng's counter-based splitmix64 stream (rng.hpp:21-27;
 * `counter` = draws taken so far, the batch takes b*T), one-hot x [T][b][p]
 * and labels [b] on the device; the readout + softmax cross-entropy of
 * model_forward / softmax_loss (:160-222) with loss_acc = (mean loss,
 * accuracy) as two device doubles -- means over b_total rows (b_total > b
 * when this rank holds b of a data-parallel global batch: the ranks' loss,
 * accuracy and gradients then SUM to the global ones); its backward (:229-240, dW_out / db_out
 * accumulate, d_hlast = the gradient of the last step); and
 * clip_global_norm + Adam (:248-288) fused over one flat parameter buffer with
 * fp64 moments (norm_out: device double, pre-clip norm; may be NULL). */
int linrec_synthetic_batch_f32(uint64_t seed, uint64_t counter, int64_t T, int64_t b, int64_t p, float* x,
                               int32_t* labels, void* stream);
int linrec_readout_loss_f32(const float* h_last, const float* W_out, const float* b_out, const int32_t* labels,
                            float* logits, float* d_logits, double* loss_acc, int64_t b, int64_t n, int64_t b_total,
                            void* stream);
int linrec_readout_backward_f32(const float* d_logits, const float* h_last, const float* W_out, float* dW_out,
                                float* db_out, float* d_hlast, int64_t b, int64_t n, void* stream);
size_t linrec_adam_scratch_bytes(void);
int linrec_clip_adam_f32(float* params, float* grads, double* m, double* v, int64_t count, double lr, double beta1,
                         double beta2, double eps, int64_t step, double clip_norm, double* norm_out, void* scratch,
                         size_t scratch_bytes, void* stream);

/* ---- sequence-sharding carry exchange over peer memory -------------------- *
 * The NCCL all-gather of the carries (linrec_segment_* above) replaced by
 * direct stores into the consumers' memory over NVLink plus release/acquire
 * flags (csrc/p2p.cu).  Each rank allocates one mailbox of
 * linrec_p2p_mailbox_bytes(W, world) with linrec_ipc_alloc (cudaMalloc +
 * cudaIpcGetMemHandle, 64-byte handle), exchanges handles out of band, opens
 * the peers' with linrec_ipc_open and passes a DEVICE array of the world
 * mailbox pointers (own at index rank).  dir 0 = forward, 1 = backward;
 * epoch = 1, 2, ... per call, equal on all ranks.
 * publish: this rank's aggregate agg [2][W] -> slot [dir][rank] of ranks
 *   [q0, q1) (waits until each consumer acked epoch-1).
 * compose: out = fold over sources first, first+step, ... != last of
 *   c = A_q c + B_q from seed (NULL = 0), q == rank taken from `local`;
 *   waits for the sources' flags, then acks them -- the same fold, in the
 *   same order, as linrec_compose_carries_f32. */
size_t linrec_p2p_mailbox_bytes(int64_t W, int world);
int linrec_ipc_alloc(size_t bytes, void** ptr, unsigned char* handle64);
int linrec_ipc_open(const unsigned char* handle64, void** ptr);
int linrec_ipc_close(void* ptr);
int linrec_ipc_free(void* ptr);
int linrec_p2p_publish_f32(const float* agg, int64_t W, int world, int rank, int dir, uint64_t epoch,
                           void* const* mboxes, int q0, int q1, void* stream);
int linrec_p2p_compose_f32(int64_t W, int world, int rank, int dir, uint64_t epoch, void* const* mboxes,
                           const float* local, int64_t first, int64_t last, int64_t step, const float* seed,
                           float* out, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* LINREC_CUDA_H_ */
