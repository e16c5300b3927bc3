// Developer probe: per-CTA timeline of the stitch fix-up (fixup_chain) on
// synthetic C4-rank-shaped data (T rows x 128 channels, decays U(0.05,0.95)),
// with globaltimer stamps at the start and end of every CTA.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//     -Ipaper_1709_04057_b200/csrc scripts/dev/fixup_timeline.cu -o build/fixup_timeline
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "fixup_impl.cuh"

using namespace linrec_dev;

template <bool REV>
__global__ void __launch_bounds__(256, REV ? 1 : 2)
k_probe(FixupArgs<float> f, const float* carry, const float* scale, int64_t ncols, int walkers,
        unsigned long long* stamps) {
  __shared__ float s_wp[8][128];
  const unsigned long long t0 = globaltimer_ns();
  const int64_t col = blockIdx.x % ncols;
  const int j = (int)((blockIdx.x / ncols) % walkers);
  const int64_t vseg = (blockIdx.x / ncols) / walkers;
  fixup_chain<float, 4, 32, REV, CtaSync>(f, vseg, col, j, walkers, carry + vseg * f.W, scale, s_wp);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    stamps[3 * blockIdx.x] = t0;
    stamps[3 * blockIdx.x + 1] = globaltimer_ns();
    stamps[3 * blockIdx.x + 2] = smid;
  }
}

int main(int argc, char** argv) {
  const int64_t T = argc > 1 ? atoll(argv[1]) : 131072, W = 128, rows = 96;
  const int rev = argc > 2 ? atoi(argv[2]) : 0;
  const int walkers = argc > 3 ? atoi(argv[3]) : 2;
  const int evict = argc > 4 ? atoi(argv[4]) : 1;  // 0: warm L2/TLB, 1: 512 MB memset, 2: memset of a 48 MB buffer
  const int64_t target = rev ? 64 : 256;
  const int64_t ntt_total = (T + rows - 1) / rows;
  int64_t nseg = target;
  if (nseg > ntt_total / 8) nseg = ntt_total / 8;
  const int64_t ntt = (ntt_total + nseg - 1) / nseg, tseg = ntt * rows;
  nseg = (T + tseg - 1) / tseg;
  std::mt19937 rng(1);
  std::uniform_real_distribution<float> U(0.05f, 0.95f), V(-1.f, 1.f);
  std::vector<float> lam(T * W), out(T * W), sp(nseg * ntt * W), carry(nseg * W);
  for (auto& v : lam) v = U(rng);
  for (auto& v : out) v = V(rng);
  for (auto& v : carry) v = V(rng);
  for (int64_t s = 0; s < nseg; ++s)
    for (int64_t c = 0; c < W; ++c) {
      float P = 1.f;
      for (int64_t p = 0; p < ntt; ++p) {
        sp[(s * ntt + p) * W + c] = P;
        const int64_t tile = rev ? ntt - 1 - p : p;
        for (int64_t r = 0; r < rows; ++r) {
          const int64_t t = s * tseg + tile * rows + (rev ? rows - 1 - r : r);
          if (t < T && t + (rev ? 1 : 0) < T) P *= lam[(t + (rev ? 1 : 0)) * W + c];
        }
      }
    }
  float *d_lam, *d_out, *d_out1, *d_h, *d_sp, *d_carry;
  unsigned long long* d_st;
  const int64_t nct = nseg * walkers;
  cudaMalloc(&d_lam, T * W * 4); cudaMalloc(&d_out, T * W * 4); cudaMalloc(&d_out1, T * W * 4);
  cudaMalloc(&d_h, T * W * 4); cudaMalloc(&d_sp, sp.size() * 4); cudaMalloc(&d_carry, carry.size() * 4);
  cudaMalloc(&d_st, nct * 3 * 8);
  cudaMemcpy(d_lam, lam.data(), T * W * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_out, out.data(), T * W * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_out1, out.data(), T * W * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_h, out.data(), T * W * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_sp, sp.data(), sp.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_carry, carry.data(), carry.size() * 4, cudaMemcpyHostToDevice);
  FixupArgs<float> f{d_lam, rev ? d_h : nullptr, d_h, nullptr, d_sp, d_out, rev ? d_out1 : nullptr,
                     T, W, rows, nseg, tseg, ntt};
  void* big;
  cudaMalloc(&big, 512 << 20);
  for (int it = 0; it < 3; ++it) {
    if (evict == 1) cudaMemset(big, it, 512 << 20);  // evict L2 (and the TLB entries of these buffers)
    if (evict == 2) cudaMemset(big, it, 48 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    if (rev) k_probe<true><<<nct, 256>>>(f, d_carry, nullptr, 1, walkers, d_st);
    else k_probe<false><<<nct, 256>>>(f, d_carry, nullptr, 1, walkers, d_st);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> st(nct * 3);
    cudaMemcpy(st.data(), d_st, st.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long lo = ~0ull, hi = 0, maxd = 0, sumd = 0;
    for (int64_t b = 0; b < nct; ++b) {
      lo = std::min(lo, st[3 * b]); hi = std::max(hi, st[3 * b + 1]);
      maxd = std::max(maxd, st[3 * b + 1] - st[3 * b]); sumd += st[3 * b + 1] - st[3 * b];
    }
    printf("T=%lld rev=%d nseg=%lld ntt=%lld walkers=%d CTAs=%lld: event %.1f us, first start->last end %.1f us, "
           "CTA max %.1f us mean %.1f us\n", (long long)T, rev, (long long)nseg, (long long)ntt, walkers,
           (long long)nct, ms * 1000, (hi - lo) / 1e3, maxd / 1e3, sumd / 1e3 / nct);
    if (it == 2)
      for (int64_t b = 0; b < nct && b < 12; ++b)
        printf("  CTA %lld sm %llu start +%.2f us dur %.2f us\n", (long long)b, st[3 * b + 2],
               (st[3 * b] - lo) / 1e3, (st[3 * b + 1] - st[3 * b]) / 1e3);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
