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
k_probe(FixupArgs<float> f, const float* carry, const float* vagg, int64_t ncols, int walkers,
        unsigned long long* stamps) {
  __shared__ float s_wp[8][128];
  __shared__ float s_fa[8 * 128], s_fb[8 * 128], s_own[128];
  const unsigned long long t0 = globaltimer_ns();
  const int64_t col = blockIdx.x % ncols;
  const int j = (int)((blockIdx.x / ncols) % walkers);
  const int64_t vseg = (blockIdx.x / ncols) / walkers;
  Carries<float> cr{carry, nullptr, nullptr};
  if (vagg != nullptr) {  // the in-CTA fold of the segment carry (k_fixup's fold mode)
    float c[4], sc[4];
    fold_carry<float, 4, 32, REV, CtaSync>(f, vagg, vseg, col, s_fa, s_fb, c, sc);
    if (threadIdx.x < 32)
      for (int v = 0; v < 4; ++v) s_own[threadIdx.x * 4 + v] = c[v];
    __syncthreads();
    cr.rows = nullptr;
    cr.own = s_own - col * 128;
  }
  const unsigned long long t1 = globaltimer_ns();
  fixup_chain<float, 4, 32, REV, CtaSync>(f, vseg, col, j, walkers, cr, s_wp);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    stamps[4 * blockIdx.x] = t0;
    stamps[4 * blockIdx.x + 1] = globaltimer_ns();
    stamps[4 * blockIdx.x + 2] = smid;
    stamps[4 * blockIdx.x + 3] = t1;
  }
}

int main(int argc, char** argv) {
  const int64_t T = argc > 1 ? atoll(argv[1]) : 131072, W = 128, rows = 96;
  const int rev = argc > 2 ? atoi(argv[2]) : 0;
  const int walkers = argc > 3 ? atoi(argv[3]) : 2;
  const int evict = argc > 4 ? atoi(argv[4]) : 1;  // 0: warm L2/TLB, 1: 512 MB memset, 2: memset of a 48 MB buffer
  const int fold = argc > 5 ? atoi(argv[5]) : 0;   // 1: fold the carries from segment aggregates in-CTA
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
  cudaMalloc(&d_st, nct * 4 * 8);
  std::vector<float> vagg(nseg * 2 * W);
  for (int64_t sg = 0; sg < nseg; ++sg)
    for (int64_t c = 0; c < W; ++c) {
      vagg[(sg * 2) * W + c] = 0.5f * U(rng);  // decay product of the segment
      vagg[(sg * 2 + 1) * W + c] = V(rng);     // its zero-carry end state
    }
  float* d_vagg;
  cudaMalloc(&d_vagg, vagg.size() * 4);
  cudaMemcpy(d_vagg, vagg.data(), vagg.size() * 4, cudaMemcpyHostToDevice);
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
    if (rev) k_probe<true><<<nct, 256>>>(f, d_carry, fold ? d_vagg : nullptr, 1, walkers, d_st);
    else k_probe<false><<<nct, 256>>>(f, d_carry, fold ? d_vagg : nullptr, 1, walkers, d_st);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> st(nct * 4);
    cudaMemcpy(st.data(), d_st, st.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long lo = ~0ull, hi = 0, maxd = 0, sumd = 0, sumf = 0, maxf = 0;
    for (int64_t b = 0; b < nct; ++b) {
      lo = std::min(lo, st[4 * b]); hi = std::max(hi, st[4 * b + 1]);
      maxd = std::max(maxd, st[4 * b + 1] - st[4 * b]); sumd += st[4 * b + 1] - st[4 * b];
      maxf = std::max(maxf, st[4 * b + 3] - st[4 * b]); sumf += st[4 * b + 3] - st[4 * b];
    }
    printf("T=%lld rev=%d fold=%d nseg=%lld ntt=%lld walkers=%d CTAs=%lld: event %.1f us, first start->last end "
           "%.1f us, CTA max %.1f us mean %.1f us (fold part max %.1f mean %.1f)\n", (long long)T, rev, fold,
           (long long)nseg, (long long)ntt, walkers, (long long)nct, ms * 1000, (hi - lo) / 1e3, maxd / 1e3,
           sumd / 1e3 / nct, maxf / 1e3, sumf / 1e3 / nct);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
