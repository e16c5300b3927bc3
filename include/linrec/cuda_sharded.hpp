// linrec/cuda_sharded.hpp -- C++ host API of the sequence-sharded scan over
// the C ABI (include/linrec_cuda.h, "sequence-sharded scan").  Header-only;
// link against liblinrec_cuda.so.
//
// The reference evaluates one long recurrence in chunks on one host
// (scan_parallel, recurrence.hpp:193-245: chunk summaries -> sequential
// stitch -> seeded re-scans).  Here the chunks are GPUs, one process per GPU:
//
//   linrec::cuda::PeerMailbox mb(W, world);          // this rank's mailbox
//   send mb.handle() to every peer, receive theirs;  // out of band (MPI, files, ...)
//   mb.open(peer_handles);                           // map the peers' mailboxes
//   linrec::cuda::SequenceShardedScan run(T, W, world, rank, mb, device);
//   run.scan(lam_seg, x_seg, h0, h_seg, stream);     // every rank, every step
//   run.scan_backward(lam_seg, h0, h_seg, dh_seg, grads_seg, stream);
//
// rank r owns rows run.rows() of every [T, b, n] tensor.
#pragma once

#include <array>
#include <cstdint>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "linrec/cuda_scan.hpp"
#include "linrec_cuda.h"

namespace linrec {
namespace cuda {

// Rows [first, first + count) of rank's segment (plan_chunks' rule).
inline std::pair<index_t, index_t> shard_rows(index_t T, int world, int rank) {
  int64_t r0 = 0, n = 0;
  linrec_sharded_bounds(T, world, rank, &r0, &n);
  return {r0, n};
}

// This rank's CUDA-IPC mailbox (device memory other ranks store into over
// NVLink) plus the peers' mailboxes mapped into this process.
class PeerMailbox {
 public:
  using Handle = std::array<unsigned char, 64>;
  PeerMailbox(index_t W, int world, int rank) : world_(world), rank_(rank) {
    throw_status(linrec_ipc_alloc(linrec_p2p_mailbox_bytes(W, world), &own_, handle_.data()));
    ptrs_.assign(size_t(world), nullptr);
    ptrs_[size_t(rank)] = own_;
  }
  PeerMailbox(const PeerMailbox&) = delete;
  PeerMailbox& operator=(const PeerMailbox&) = delete;
  ~PeerMailbox() {
    for (int q = 0; q < world_; ++q)
      if (q != rank_ && ptrs_[size_t(q)]) linrec_ipc_close(ptrs_[size_t(q)]);
    linrec_ipc_free(own_);
  }
  const Handle& handle() const { return handle_; }
  // handles[q] = rank q's handle (own entry ignored)
  void open(const std::vector<Handle>& handles) {
    if (int(handles.size()) != world_) throw ContractViolation("PeerMailbox::open: one handle per rank required");
    for (int q = 0; q < world_; ++q) {
      if (q == rank_ || ptrs_[size_t(q)]) continue;
      throw_status(linrec_ipc_open(handles[size_t(q)].data(), &ptrs_[size_t(q)]));
    }
  }
  void* const* pointers() const { return ptrs_.data(); }

 private:
  int world_, rank_;
  void* own_ = nullptr;
  Handle handle_{};
  std::vector<void*> ptrs_;
};

class SequenceShardedScan {
 public:
  SequenceShardedScan(index_t T, index_t W, int world, int rank, const PeerMailbox& mb, int device)
      : T_(T), W_(W) {
    throw_status(linrec_sharded_create(&ctx_, T, W, world, rank, mb.pointers(), device));
  }
  SequenceShardedScan(const SequenceShardedScan&) = delete;
  SequenceShardedScan& operator=(const SequenceShardedScan&) = delete;
  ~SequenceShardedScan() { linrec_sharded_destroy(ctx_); }

  std::pair<index_t, index_t> rows() const {
    int64_t r0 = 0, n = 0;
    throw_status(linrec_sharded_rows(ctx_, &r0, &n));
    return {r0, n};
  }

  // scan (recurrence.hpp:255-263) of this rank's rows; initial read on rank 0.
  void scan(const DeviceTensor3<float>& decays, const DeviceTensor3<float>& impulses,
            const DeviceTensor2<float>& initial, DeviceTensor3<float>& h, void* stream = nullptr,
            linrec_workspace_t ws = nullptr) {
    check_segment(decays);
    check_same_shape(decays, impulses, "recurrence");
    check_same_shape(decays, h, "scan_parallel(h)");
    throw_status(linrec_sharded_scan_f32(ctx_, decays.data, impulses.data, initial.data, h.data, ws, stream));
  }

  // scan_backward (recurrence.hpp:283-363) of this rank's rows; d_initial on rank 0.
  void scan_backward(const DeviceTensor3<float>& decays, const DeviceTensor2<float>& initial,
                     const DeviceTensor3<float>& h, const DeviceTensor3<float>& d_h,
                     RecurrenceGradients<float>& grads, void* stream = nullptr, linrec_workspace_t ws = nullptr,
                     const float* hprev = nullptr) {
    check_segment(decays);
    check_same_shape(decays, h, "scan_backward(h)");
    check_same_shape(decays, d_h, "scan_backward(d_h)");
    check_same_shape(decays, grads.d_decays, "scan_backward(d_decays)");
    check_same_shape(decays, grads.d_impulses, "scan_backward(d_impulses)");
    throw_status(linrec_sharded_scan_backward_f32(ctx_, decays.data, initial.data, hprev, h.data, d_h.data,
                                                  grads.d_decays.data, grads.d_impulses.data, grads.d_initial.data,
                                                  ws, stream));
  }

 private:
  void check_segment(const DeviceTensor3<float>& t) const {
    const auto r = rows();
    if (t.steps != r.second || t.step_size() != W_)
      throw ContractViolation("SequenceShardedScan: tensor is not this rank's [" + std::to_string(r.second) + ", " +
                              std::to_string(W_) + "] segment");
  }
  index_t T_, W_;
  linrec_sharded_t ctx_ = nullptr;
};

// ---- channel sharding of HOST tensors over several GPUs -------
// Channels are independent (recurrence.hpp:109), so the columns of a host
// [T][b*n] tensor split into per-GPU blocks (linrec_column_block) with no
// communication: one host thread per GPU stages its block with 2-D copies,
// scans it and writes its columns back.  The reference's scan / scan_backward
// over host Tensor3 (recurrence.hpp:255-263, :352-363), many GPUs at once.
template <class S>
struct HostTensor3 {
  S* data = nullptr;
  index_t steps = 0, batch = 0, features = 0;
  index_t step_size() const { return batch * features; }
};

namespace detail {
inline int multi_call(const float* l, const float* x, const float* h0, float* h, index_t T, index_t W, int mode,
                      const int* d, int n) {
  return linrec_scan_host_multi_f32(l, x, h0, h, T, W, mode, d, n);
}
inline int multi_call(const double* l, const double* x, const double* h0, double* h, index_t T, index_t W, int mode,
                      const int* d, int n) {
  return linrec_scan_host_multi_f64(l, x, h0, h, T, W, mode, d, n);
}
inline int multi_bwd_call(const float* l, const float* h0, const float* h, const float* dh, float* dl, float* dx,
                          float* dh0, index_t T, index_t W, int mode, const int* d, int n) {
  return linrec_scan_backward_host_multi_f32(l, h0, h, dh, dl, dx, dh0, T, W, mode, d, n);
}
inline int multi_bwd_call(const double* l, const double* h0, const double* h, const double* dh, double* dl,
                          double* dx, double* dh0, index_t T, index_t W, int mode, const int* d, int n) {
  return linrec_scan_backward_host_multi_f64(l, h0, h, dh, dl, dx, dh0, T, W, mode, d, n);
}
template <class S, class U>
void check_host_shape(const HostTensor3<S>& a, const HostTensor3<U>& b, const char* op) {
  if (a.steps != b.steps || a.batch != b.batch || a.features != b.features) {
    std::ostringstream os;
    os << op << ": shape mismatch, [" << a.steps << "," << a.batch << "," << a.features << "] vs [" << b.steps
       << "," << b.batch << "," << b.features << "]";
    throw ContractViolation(os.str());
  }
}
}  // namespace detail

// h = scan(decays, impulses, initial) with the channels split over `devices`;
// initial: [b*n] host row or nullptr (zeros).
template <class S>
void scan_channel_sharded(const HostTensor3<S>& decays, const HostTensor3<S>& impulses, const S* initial,
                          HostTensor3<S>& h, const std::vector<int>& devices, ScanMode mode = ScanMode::Parallel) {
  detail::check_host_shape(decays, impulses, "recurrence");
  detail::check_host_shape(decays, h, "scan_parallel(h)");
  throw_status(detail::multi_call(decays.data, impulses.data, initial, h.data, decays.steps, decays.step_size(),
                                  static_cast<int>(mode), devices.data(), int(devices.size())));
}

// (d_decays, d_impulses, d_initial[b*n]) = scan_backward(...) with the
// channels split over `devices`.
template <class S>
void scan_backward_channel_sharded(const HostTensor3<S>& decays, const S* initial, const HostTensor3<S>& h,
                                   const HostTensor3<S>& d_h, HostTensor3<S>& d_decays, HostTensor3<S>& d_impulses,
                                   S* d_initial, const std::vector<int>& devices,
                                   ScanMode mode = ScanMode::Parallel) {
  detail::check_host_shape(decays, h, "scan_backward(h)");
  detail::check_host_shape(decays, d_h, "scan_backward(d_h)");
  detail::check_host_shape(decays, d_decays, "scan_backward(d_decays)");
  detail::check_host_shape(decays, d_impulses, "scan_backward(d_impulses)");
  throw_status(detail::multi_bwd_call(decays.data, initial, h.data, d_h.data, d_decays.data, d_impulses.data,
                                      d_initial, decays.steps, decays.step_size(), static_cast<int>(mode),
                                      devices.data(), int(devices.size())));
}

}  // namespace cuda
}  // namespace linrec
