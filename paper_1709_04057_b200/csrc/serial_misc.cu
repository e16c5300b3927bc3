// Serial (bit-exact) kernels, plan construction, workspace init and the
// finite screen.
#include "chain_impl.cuh"

namespace linrec_impl {

template <class S>
ChainPlan plan_chain(bool forward, int64_t T, int64_t W, bool vec_ok) {
  return forward ? plan_chain_dir<S, true>(T, W, vec_ok) : plan_chain_dir<S, false>(T, W, vec_ok);
}
template ChainPlan plan_chain<float>(bool, int64_t, int64_t, bool);
template ChainPlan plan_chain<double>(bool, int64_t, int64_t, bool);

namespace {
constexpr int kSerialU = 8;
constexpr int kSerialThreads = 128;
}  // namespace

template <class S>
cudaError_t launch_serial_fwd(const FwdCall<S>& c, bool vec_ok, cudaStream_t st) {
  constexpr int V = Tuning<S>::VEC;
  const int vec = vec_ok ? V : 1;
  const int64_t threads = (c.W + vec - 1) / vec;
  const dim3 grid((unsigned)((threads + kSerialThreads - 1) / kSerialThreads));
  if (vec_ok)
    linrec_dev::k_serial_fwd<S, V, kSerialU><<<grid, kSerialThreads, 0, st>>>(c.lam, c.x, c.h0, c.h, c.T, c.W);
  else
    linrec_dev::k_serial_fwd<S, 1, kSerialU><<<grid, kSerialThreads, 0, st>>>(c.lam, c.x, c.h0, c.h, c.T, c.W);
  return cudaGetLastError();
}

template <class S>
cudaError_t launch_serial_bwd(const BwdCall<S>& c, bool vec_ok, cudaStream_t st) {
  constexpr int V = Tuning<S>::VEC;
  const int vec = vec_ok ? V : 1;
  const int64_t threads = (c.W + vec - 1) / vec;
  const dim3 grid((unsigned)((threads + kSerialThreads - 1) / kSerialThreads));
  if (vec_ok)
    linrec_dev::k_serial_bwd<S, V, kSerialU><<<grid, kSerialThreads, 0, st>>>(
        c.lam, c.h0, c.h, c.dh, c.lam_next, c.g_next, c.dlam, c.dx, c.dh0, c.T, c.W);
  else
    linrec_dev::k_serial_bwd<S, 1, kSerialU><<<grid, kSerialThreads, 0, st>>>(
        c.lam, c.h0, c.h, c.dh, c.lam_next, c.g_next, c.dlam, c.dx, c.dh0, c.T, c.W);
  return cudaGetLastError();
}

template cudaError_t launch_serial_fwd<float>(const FwdCall<float>&, bool, cudaStream_t);
template cudaError_t launch_serial_fwd<double>(const FwdCall<double>&, bool, cudaStream_t);
template cudaError_t launch_serial_bwd<float>(const BwdCall<float>&, bool, cudaStream_t);
template cudaError_t launch_serial_bwd<double>(const BwdCall<double>&, bool, cudaStream_t);

namespace {
__global__ void k_ws_init(linrec_dev::Ctrl* c) {
  c->epoch = 1u;
  c->ticket = 0ull;
  c->retired = 0ull;
}

// First non-finite index: grid-stride min-reduction.
template <class S>
__global__ void k_first_nonfinite(const S* __restrict__ v, int64_t n,
                                  unsigned long long* out) {
  unsigned long long best = ~0ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!isfinite(v[i])) {
      best = (unsigned long long)i;
      break;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long b = __shfl_xor_sync(0xffffffffu, best, o);
    best = b < best ? b : best;
  }
  if ((threadIdx.x & 31) == 0 && best != ~0ull) atomicMin(out, best);
}
}  // namespace

cudaError_t launch_ws_init(void* ctrl, cudaStream_t st) {
  k_ws_init<<<1, 1, 0, st>>>(reinterpret_cast<linrec_dev::Ctrl*>(ctrl));
  return cudaGetLastError();
}

template <class S>
cudaError_t first_nonfinite(const S* v, int64_t n, int64_t* index, cudaStream_t st) {
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMallocAsync(&d, sizeof(*d), st);
  if (e != cudaSuccess) return e;
  unsigned long long h = ~0ull;
  e = cudaMemcpyAsync(d, &h, sizeof(h), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && n > 0) {
    const int64_t blocks = (n + 255) / 256;
    k_first_nonfinite<S><<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, st>>>(v, n, d);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  *index = (h == ~0ull) ? -1 : (int64_t)h;
  return e;
}
template cudaError_t first_nonfinite<float>(const float*, int64_t, int64_t*, cudaStream_t);
template cudaError_t first_nonfinite<double>(const double*, int64_t, int64_t*, cudaStream_t);

}  // namespace linrec_impl
