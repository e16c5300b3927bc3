/*
 * linrec CPU oracle -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's recurrence core
 * (/root/reference/proj/include/linrec/recurrence.hpp) used as the parity
 * checker for the CUDA path.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library; the
 * product (paper_1709_04057_b200/) never links or calls it.
 *
 * Parity pinning: every function below is checked bit-for-bit against the
 * reference itself compiled from /root/reference (oracle/_ref, see
 * oracle/Makefile) and against the reference's frozen golden vectors
 * (tests/test_oracle.py, tests/golden/).
 *
 * Arithmetic: the reference is built with -O3 -march=native in GNU C++ mode
 * (proj/CMakeLists.txt:34-41), where GCC contracts `a*b + c` into a fused
 * multiply-add.  This file is compiled with -ffp-contract=off and spells the
 * contractions out with fma()/fmaf(), so its bits do not depend on compiler
 * flags and equal the reference's on any FMA-capable x86-64 host.
 *
 * Layout: time-major row-major [T][W], W = batch * features; step t is the
 * contiguous slab [t*W, (t+1)*W) (tensor.hpp:49-75).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t index_t;

/* plan_chunks -- recurrence.hpp:61-80.  Writes p (start,end) pairs, 1-based
 * inclusive, into bounds[2p]; returns p, or -1 on contract violation
 * (T < 1 or workers < 1, recurrence.hpp:64-66). */
index_t oracle_plan_chunks(index_t T, int workers, index_t* bounds) {
  if (T < 1 || workers < 1) return -1;
  const index_t p = (index_t)workers < T ? (index_t)workers : T;
  const index_t base = T / p, rem = T % p;
  index_t start = 1;
  for (index_t i = 0; i < p; ++i) {
    const index_t len = base + (i < rem ? 1 : 0);
    if (bounds) {
      bounds[2 * i] = start;
      bounds[2 * i + 1] = start + len - 1;
    }
    start += len;
  }
  return p;
}

/* predicted_speedup -- bench.hpp:61-65: p*T / (3*(T + log2 p)). */
double oracle_predicted_speedup(int p, index_t T) {
  if (p < 1 || T < 1) return -1.0;
  return (double)p * (double)T / (3.0 * ((double)T + log2((double)p)));
}

#define DEFINE_ORACLE(S, SUF, FMA)                                              \
  /* detail::scan_span -- recurrence.hpp:101-112 (rows t0..t1 inclusive). */   \
  static void scan_span_##SUF(const S* lam, const S* x, const S* seed, S* out,  \
                              index_t t0, index_t t1, index_t W) {              \
    const S* prev = seed;                                                       \
    for (index_t t = t0; t <= t1; ++t) {                                        \
      const S* l = lam + t * W;                                                 \
      const S* v = x + t * W;                                                   \
      S* o = out + t * W;                                                       \
      for (index_t j = 0; j < W; ++j) o[j] = FMA(l[j], prev[j], v[j]);          \
      prev = o;                                                                 \
    }                                                                           \
  }                                                                             \
                                                                                \
  /* scan_serial -- recurrence.hpp:169-179.  h0 == NULL means zeros            \
   * (bindings/linrec_py.cpp:98-100). */                                        \
  void oracle_scan_serial_##SUF(const S* lam, const S* x, const S* h0, S* h,    \
                                index_t T, index_t W) {                         \
    S* zero = NULL;                                                             \
    if (!h0) {                                                                  \
      zero = (S*)calloc((size_t)W, sizeof(S));                                  \
      h0 = zero;                                                                \
    }                                                                           \
    scan_span_##SUF(lam, x, h0, h, 0, T - 1, W);                                \
    free(zero);                                                                 \
  }                                                                             \
                                                                                \
  /* scan_parallel -- recurrence.hpp:193-245 with the three phases executed    \
   * in order (the thread pool never changes bits: disjoint writes, fixed      \
   * plan, test_recurrence.cpp:173-183).  bounds: p (s,e) 1-based pairs.       \
   * P, R, C: optional [p][W] outputs (ScanSummaries, recurrence.hpp:186-191). \
   */                                                                         \
  void oracle_scan_parallel_##SUF(const S* lam, const S* x, const S* h0, S* h,  \
                                  index_t T, index_t W, const index_t* bounds,  \
                                  index_t p, S* P_out, S* R_out, S* C_out) {    \
    (void)T;                                                                    \
    S* zero = NULL;                                                             \
    if (!h0) {                                                                  \
      zero = (S*)calloc((size_t)W, sizeof(S));                                  \
      h0 = zero;                                                                \
    }                                                                           \
    S* P = P_out ? P_out : (S*)malloc(sizeof(S) * (size_t)(p * W));             \
    S* R = R_out ? R_out : (S*)malloc(sizeof(S) * (size_t)(p * W));             \
    S* C = C_out ? C_out : (S*)malloc(sizeof(S) * (size_t)(p * W));             \
    /* phase 1: chunk_summary, recurrence.hpp:114-131 / :212-217 */             \
    for (index_t i = 0; i < p; ++i) {                                           \
      S* Pi = P + i * W;                                                        \
      S* Ri = R + i * W;                                                        \
      for (index_t j = 0; j < W; ++j) {                                         \
        Pi[j] = (S)1;                                                           \
        Ri[j] = (S)0;                                                           \
      }                                                                         \
      for (index_t t = bounds[2 * i] - 1; t <= bounds[2 * i + 1] - 1; ++t) {    \
        const S* l = lam + t * W;                                               \
        const S* v = x + t * W;                                                 \
        for (index_t j = 0; j < W; ++j) {                                       \
          Ri[j] = FMA(l[j], Ri[j], v[j]);                                       \
          Pi[j] = Pi[j] * l[j];                                                 \
        }                                                                       \
      }                                                                         \
    }                                                                           \
    /* phase 2: C_i = P_i * C_{i-1} + R_i, C_{-1} = h0 (:219-230) */            \
    {                                                                           \
      const S* prev = h0;                                                       \
      for (index_t i = 0; i < p; ++i) {                                         \
        for (index_t j = 0; j < W; ++j)                                         \
          C[i * W + j] = FMA(P[i * W + j], prev[j], R[i * W + j]);              \
        prev = C + i * W;                                                       \
      }                                                                         \
    }                                                                           \
    /* phase 3: seeded chunk scans (:232-237) */                                \
    for (index_t i = 0; i < p; ++i) {                                           \
      const S* seed = (i == 0) ? h0 : C + (i - 1) * W;                          \
      scan_span_##SUF(lam, x, seed, h, bounds[2 * i] - 1,                       \
                      bounds[2 * i + 1] - 1, W);                                \
    }                                                                           \
    if (!P_out) free(P);                                                        \
    if (!R_out) free(R);                                                        \
    if (!C_out) free(C);                                                        \
    free(zero);                                                                 \
  }                                                                             \
                                                                                \
  /* scan_backward_impl -- recurrence.hpp:283-348.  The reversed image         \
   * rev_dec[0]=0, rev_dec[s]=lam[T-s], rev_imp[s]=dh[T-1-s] (:305-318) is     \
   * scanned serially (bounds == NULL) or with the chunk plan, then            \
   * dx_t = G_t, dlam_t = h_{t-1} G_t (h0 at t=1), dh0 = lam_1 G_1            \
   * (:331-346).  h0 == NULL means zeros. */                                    \
  void oracle_scan_backward_##SUF(const S* lam, const S* h0, const S* h,        \
                                  const S* dh, S* dlam, S* dx, S* dh0,          \
                                  index_t T, index_t W, const index_t* bounds,  \
                                  index_t p) {                                  \
    S* zero = (S*)calloc((size_t)W, sizeof(S));                                 \
    if (!h0) h0 = zero;                                                         \
    S* rev_dec = (S*)calloc((size_t)(T * W), sizeof(S));                        \
    S* rev_imp = (S*)malloc(sizeof(S) * (size_t)(T * W));                       \
    S* g_rev = (S*)malloc(sizeof(S) * (size_t)(T * W));                         \
    for (index_t s = 0; s < T; ++s) {                                           \
      if (s > 0) memcpy(rev_dec + s * W, lam + (T - s) * W, sizeof(S) * W);     \
      memcpy(rev_imp + s * W, dh + (T - 1 - s) * W, sizeof(S) * W);             \
    }                                                                           \
    if (bounds)                                                                 \
      oracle_scan_parallel_##SUF(rev_dec, rev_imp, zero, g_rev, T, W, bounds,   \
                                 p, NULL, NULL, NULL);                          \
    else                                                                        \
      scan_span_##SUF(rev_dec, rev_imp, zero, g_rev, 0, T - 1, W);              \
    for (index_t t = 0; t < T; ++t) {                                           \
      const S* G = g_rev + (T - 1 - t) * W;                                     \
      const S* hprev = (t == 0) ? h0 : h + (t - 1) * W;                         \
      for (index_t j = 0; j < W; ++j) {                                         \
        dx[t * W + j] = G[j];                                                   \
        dlam[t * W + j] = hprev[j] * G[j];                                      \
      }                                                                         \
    }                                                                           \
    {                                                                           \
      const S* G1 = g_rev + (T - 1) * W;                                        \
      for (index_t j = 0; j < W; ++j) dh0[j] = lam[j] * G1[j];                  \
    }                                                                           \
    free(rev_dec);                                                              \
    free(rev_imp);                                                              \
    free(g_rev);                                                                \
    free(zero);                                                                 \
  }                                                                             \
                                                                                \
  /* First non-finite element, or -1 (tensor.hpp:310-319, recurrence.hpp:133-  \
   * 144 report it as [t=idx/W+1, b, n]). */                                    \
  index_t oracle_first_nonfinite_##SUF(const S* v, index_t n) {                 \
    for (index_t i = 0; i < n; ++i)                                             \
      if (!isfinite(v[i])) return i;                                            \
    return -1;                                                                  \
  }

DEFINE_ORACLE(float, f32, fmaf)
DEFINE_ORACLE(double, f64, fma)

/* Widened serial scan (fp64 arithmetic on fp32 data) -- the "error also
 * bounded against an fp64 serial scan" check of BASELINE.json north_star and
 * tests/python/test_smoke.py:17-26 (reference_scan accumulates in float64). */
void oracle_scan_serial_f32_wide(const float* lam, const float* x,
                                 const float* h0, double* h, index_t T,
                                 index_t W) {
  double* prev = (double*)calloc((size_t)W, sizeof(double));
  if (h0)
    for (index_t j = 0; j < W; ++j) prev[j] = h0[j];
  for (index_t t = 0; t < T; ++t)
    for (index_t j = 0; j < W; ++j) {
      prev[j] = (double)lam[t * W + j] * prev[j] + (double)x[t * W + j];
      h[t * W + j] = prev[j];
    }
  free(prev);
}

/* Widened backward (fp64 arithmetic on fp32 data): G, dlam, dx, dh0 as above
 * but accumulated in double. */
void oracle_scan_backward_f32_wide(const float* lam, const float* h0,
                                   const float* h, const float* dh,
                                   double* dlam, double* dx, double* dh0,
                                   index_t T, index_t W) {
  double* G = (double*)calloc((size_t)W, sizeof(double));
  for (index_t t = T - 1; t >= 0; --t)
    for (index_t j = 0; j < W; ++j) {
      const double mu = (t + 1 < T) ? (double)lam[(t + 1) * W + j] : 0.0;
      G[j] = mu * G[j] + (double)dh[t * W + j];
      dx[t * W + j] = G[j];
      const double hp = t == 0 ? (h0 ? (double)h0[j] : 0.0)
                               : (double)h[(t - 1) * W + j];
      dlam[t * W + j] = hp * G[j];
    }
  for (index_t j = 0; j < W; ++j) dh0[j] = (double)lam[j] * G[j];
  free(G);
}

/* splitmix64 counter RNG -- rng.hpp:15-52, frozen by test_rng.cpp:210-223.
 * state[0] = seed, state[1] = counter. */
uint64_t oracle_rng_next_u64(uint64_t* state) {
  uint64_t z = state[0] + (++state[1]) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t oracle_rng_split(uint64_t seed, uint64_t stream) {
  uint64_t z = seed ^ (0xD1B54A32D192ED03ULL * (stream + 1));
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* Fill v[n] with S(lo + (hi-lo)*u), u = (next>>11)*2^-53 (rng.hpp:33-36,
 * fill_uniform rng.hpp:63-66). */
void oracle_rng_fill_f32(uint64_t* state, float* v, index_t n, double lo,
                         double hi) {
  for (index_t i = 0; i < n; ++i) {
    const double u = (double)(oracle_rng_next_u64(state) >> 11) * 0x1.0p-53;
    v[i] = (float)fma(hi - lo, u, lo); /* contracted as in the -march build */
  }
}

void oracle_rng_fill_f64(uint64_t* state, double* v, index_t n, double lo,
                         double hi) {
  for (index_t i = 0; i < n; ++i) {
    const double u = (double)(oracle_rng_next_u64(state) >> 11) * 0x1.0p-53;
    v[i] = fma(hi - lo, u, lo);
  }
}

/* fnv1a64 over bytes -- bench.hpp:69-76 (input checksum of the bench). */
uint64_t oracle_fnv1a64(const void* data, size_t len, uint64_t h) {
  const unsigned char* p = (const unsigned char*)data;
  for (size_t i = 0; i < len; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}
