/*
 * GILR and GILR-LSTM layers -- CPU oracle, TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of /root/reference/proj/include/linrec/layers.hpp:
 *   gilr_forward       :78-100    gilr_backward       :102-133
 *   gilr_lstm_forward  :245-293   gilr_lstm_backward  :295-375
 *   qrnn_forward       :449-494   qrnn_backward       :496-548
 * with the dense transforms of tensor.hpp (affine :249-270,
 * accumulate_weight_grad :272-284, accumulate_bias_grad :286-296,
 * accumulate_input_grad :298-308) written as loops and the recurrence as the
 * serial scan of linrec_oracle.c (ScanMode::Serial).  The reference's GEMMs
 * are Eigen blocked products whose summation order is unspecified, so this
 * oracle is pinned to the reference by tolerance: forward against the
 * reference's own per-step layer oracle (tests/support/layer_oracles.hpp,
 * compiled into oracle/_ref), backward against central finite differences
 * exactly as proj/tests/test_layers.cpp:162-239 does.
 *
 * Layout: x [T][b][m] and every activation [T][b][n] time-major, flattened to
 * R = T*b rows.  Parameters row-major as in GilrParams / GilrLstmParams
 * (layers.hpp:28-40, :148-165): surrogate U, V [n][m], b_g, b_z [n];
 * gate U [4n][n], V [4n][m], bias [4n] (blocks f, i, o, z).
 * Gradients ACCUMULATE into the provided buffers, as in the reference.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t index_t;

/* Activation (common.hpp:49-71): 0 = tanh, 1 = identity, 2 = relu. */
#define DEFINE_LAYERS(S, SUF, FMA, EXP, TANH)                                         \
  static S sig_##SUF(S z) { return (S)1 / ((S)1 + EXP(-z)); }                         \
  static S act_##SUF(int a, S z) { return a == 0 ? TANH(z) : a == 1 ? z : (z > 0 ? z : (S)0); } \
  static S dact_##SUF(int a, S v) {                                                   \
    return a == 0 ? (S)1 - v * v : a == 1 ? (S)1 : (v > 0 ? (S)1 : (S)0);             \
  }                                                                                   \
  /* out[r][j] (+)= sum_k x[r][k] * w[j][k]  (+ bias[j] when !acc), affine :249 */    \
  static void affine_##SUF(const S* x, index_t R, index_t K, const S* w, index_t N,    \
                           const S* bias, S* out, int acc) {                          \
    for (index_t r = 0; r < R; ++r)                                                   \
      for (index_t j = 0; j < N; ++j) {                                               \
        S s = 0;                                                                      \
        for (index_t k = 0; k < K; ++k) s += x[r * K + k] * w[j * K + k];             \
        if (acc) out[r * N + j] += s;                                                 \
        else out[r * N + j] = s + (bias ? bias[j] : (S)0);                            \
      }                                                                               \
  }                                                                                   \
  /* dw[j][k] += sum_r d[r][j] * x[r][k]   (accumulate_weight_grad :272) */           \
  static void wgrad_##SUF(const S* d, index_t R, index_t N, const S* x, index_t K, S* dw) { \
    for (index_t j = 0; j < N; ++j)                                                   \
      for (index_t k = 0; k < K; ++k) {                                               \
        S s = 0;                                                                      \
        for (index_t r = 0; r < R; ++r) s += d[r * N + j] * x[r * K + k];             \
        dw[j * K + k] += s;                                                           \
      }                                                                               \
  }                                                                                   \
  static void bgrad_##SUF(const S* d, index_t R, index_t N, S* db) {                  \
    for (index_t j = 0; j < N; ++j) {                                                 \
      S s = 0;                                                                        \
      for (index_t r = 0; r < R; ++r) s += d[r * N + j];                              \
      db[j] += s;                                                                     \
    }                                                                                 \
  }                                                                                   \
  /* dx[r][k] (+)= sum_j d[r][j] * w[j][k]   (accumulate_input_grad :298) */          \
  static void igrad_##SUF(const S* d, index_t R, index_t N, const S* w, index_t K, S* dx, int acc) { \
    for (index_t r = 0; r < R; ++r)                                                   \
      for (index_t k = 0; k < K; ++k) {                                               \
        S s = 0;                                                                      \
        for (index_t j = 0; j < N; ++j) s += d[r * N + j] * w[j * K + k];             \
        dx[r * K + k] = acc ? dx[r * K + k] + s : s;                                  \
      }                                                                               \
  }                                                                                   \
  static void scan_##SUF(const S* lam, const S* imp, const S* h0, S* h, index_t T, index_t W) { \
    for (index_t j = 0; j < W; ++j) {                                                 \
      S prev = h0 ? h0[j] : (S)0;                                                     \
      for (index_t t = 0; t < T; ++t) {                                               \
        prev = FMA(lam[t * W + j], prev, imp[t * W + j]);                             \
        h[t * W + j] = prev;                                                          \
      }                                                                               \
    }                                                                                 \
  }                                                                                   \
  /* recurrence.hpp:283-348 serial: returns dlam, G (= d impulses), dh0 */            \
  static void scan_bwd_##SUF(const S* lam, const S* h0, const S* h, const S* dh, S* dlam, S* G, \
                             S* dh0, index_t T, index_t W) {                          \
    for (index_t j = 0; j < W; ++j) {                                                 \
      S g = 0;                                                                        \
      for (index_t t = T - 1; t >= 0; --t) {                                          \
        const S mu = t + 1 < T ? lam[(t + 1) * W + j] : (S)0;                         \
        g = FMA(mu, g, dh[t * W + j]);                                                \
        G[t * W + j] = g;                                                             \
        dlam[t * W + j] = (t == 0 ? (h0 ? h0[j] : (S)0) : h[(t - 1) * W + j]) * g;    \
      }                                                                               \
      if (dh0) dh0[j] = lam[j] * g;                                                   \
    }                                                                                 \
  }                                                                                   \
                                                                                      \
  /* gilr_forward :78-100.  Writes g, i (activated), h. */                            \
  void oracle_gilr_forward_##SUF(const S* x, const S* U, const S* V, const S* bg,     \
                                 const S* bz, const S* h0, int act, S* g, S* i, S* h,  \
                                 index_t T, index_t b, index_t m, index_t n) {        \
    const index_t R = T * b;                                                          \
    affine_##SUF(x, R, m, U, n, bg, g, 0);                                            \
    affine_##SUF(x, R, m, V, n, bz, i, 0);                                            \
    S* imp = (S*)malloc(sizeof(S) * (size_t)(R * n));                                 \
    for (index_t k = 0; k < R * n; ++k) {                                             \
      g[k] = sig_##SUF(g[k]);                                                         \
      i[k] = act_##SUF(act, i[k]);                                                    \
      imp[k] = ((S)1 - g[k]) * i[k];                                                  \
    }                                                                                 \
    scan_##SUF(g, imp, h0, h, T, b * n);                                              \
    free(imp);                                                                        \
  }                                                                                   \
                                                                                      \
  /* gilr_backward :102-133.  Accumulates dU, dV, dbg, dbz; writes dx; dh0. */        \
  void oracle_gilr_backward_##SUF(const S* x, const S* U, const S* V, const S* h0, int act, \
                                  const S* g, const S* i, const S* h, const S* dh,    \
                                  S* dU, S* dV, S* dbg, S* dbz, S* dx, S* dh0,        \
                                  index_t T, index_t b, index_t m, index_t n) {       \
    const index_t R = T * b, N = R * n;                                               \
    S* dl = (S*)malloc(sizeof(S) * (size_t)N);                                        \
    S* G = (S*)malloc(sizeof(S) * (size_t)N);                                         \
    S* dg = (S*)malloc(sizeof(S) * (size_t)N);                                        \
    S* di = (S*)malloc(sizeof(S) * (size_t)N);                                        \
    scan_bwd_##SUF(g, h0, h, dh, dl, G, dh0, T, b * n);                               \
    for (index_t k = 0; k < N; ++k) {                                                 \
      dg[k] = (dl[k] - G[k] * i[k]) * g[k] * ((S)1 - g[k]);                           \
      di[k] = G[k] * ((S)1 - g[k]) * dact_##SUF(act, i[k]);                           \
    }                                                                                 \
    wgrad_##SUF(dg, R, n, x, m, dU);                                                  \
    bgrad_##SUF(dg, R, n, dbg);                                                       \
    wgrad_##SUF(di, R, n, x, m, dV);                                                  \
    bgrad_##SUF(di, R, n, dbz);                                                       \
    igrad_##SUF(dg, R, n, U, m, dx, 0);                                               \
    igrad_##SUF(di, R, n, V, m, dx, 1);                                               \
    free(dl); free(G); free(dg); free(di);                                            \
  }                                                                                   \
                                                                                      \
  /* gilr_lstm_forward :245-293.  Writes h; caches (may be NULL): the surrogate's \
   * sg, si, htil; gates [R][4n] activated (f,i,o,z); c. */                           \
  void oracle_gilr_lstm_forward_##SUF(                                                \
      const S* x, const S* sU, const S* sV, const S* sbg, const S* sbz, const S* U,   \
      const S* V, const S* bias, const S* htil0, const S* c0, S* h, S* sg, S* si,     \
      S* htil, S* gates, S* c, index_t T, index_t b, index_t m, index_t n) {          \
    const index_t R = T * b, N = R * n, BN = b * n;                                   \
    S* hp = (S*)malloc(sizeof(S) * (size_t)N);                                        \
    S* f = (S*)malloc(sizeof(S) * (size_t)N);                                         \
    S* iz = (S*)malloc(sizeof(S) * (size_t)N);                                        \
    oracle_gilr_forward_##SUF(x, sU, sV, sbg, sbz, htil0, 0, sg, si, htil, T, b, m, n); \
    for (index_t k = 0; k < BN; ++k) hp[k] = htil0 ? htil0[k] : (S)0;                 \
    memcpy(hp + BN, htil, sizeof(S) * (size_t)(N - BN));                              \
    affine_##SUF(x, R, m, V, 4 * n, bias, gates, 0);                                  \
    affine_##SUF(hp, R, n, U, 4 * n, bias, gates, 1);                                 \
    for (index_t r = 0; r < R; ++r) {                                                 \
      S* gr = gates + r * 4 * n;                                                      \
      for (index_t j = 0; j < 3 * n; ++j) gr[j] = sig_##SUF(gr[j]);                   \
      for (index_t j = 3 * n; j < 4 * n; ++j) gr[j] = TANH(gr[j]);                    \
      for (index_t j = 0; j < n; ++j) {                                               \
        f[r * n + j] = gr[j];                                                         \
        iz[r * n + j] = gr[n + j] * gr[3 * n + j];                                    \
      }                                                                               \
    }                                                                                 \
    scan_##SUF(f, iz, c0, c, T, BN);                                                  \
    for (index_t r = 0; r < R; ++r)                                                   \
      for (index_t j = 0; j < n; ++j) h[r * n + j] = gates[r * 4 * n + 2 * n + j] * c[r * n + j]; \
    free(hp); free(f); free(iz);                                                      \
  }                                                                                   \
                                                                                      \
  /* gilr_lstm_backward :295-375.  Accumulates the 7 parameter gradients,       \
   * writes dx, dhtil0, dc0. */                                                       \
  void oracle_gilr_lstm_backward_##SUF(                                               \
      const S* x, const S* sU, const S* sV, const S* U, const S* V, const S* htil0,   \
      const S* c0, const S* sg, const S* si, const S* htil, const S* gates, const S* c, \
      const S* dh, S* dsU, S* dsV, S* dsbg, S* dsbz, S* dU, S* dV, S* dbias, S* dx,   \
      S* dhtil0, S* dc0, index_t T, index_t b, index_t m, index_t n) {                \
    const index_t R = T * b, N = R * n, BN = b * n;                                   \
    S* dc = (S*)malloc(sizeof(S) * (size_t)N);                                        \
    S* dO = (S*)malloc(sizeof(S) * (size_t)N);                                        \
    S* f = (S*)malloc(sizeof(S) * (size_t)N);                                         \
    S* df = (S*)malloc(sizeof(S) * (size_t)N);                                        \
    S* diz = (S*)malloc(sizeof(S) * (size_t)N);                                       \
    S* dpre = (S*)malloc(sizeof(S) * (size_t)(4 * N));                                \
    S* hp = (S*)malloc(sizeof(S) * (size_t)N);                                        \
    S* dhp = (S*)malloc(sizeof(S) * (size_t)N);                                       \
    S* dht = (S*)malloc(sizeof(S) * (size_t)N);                                       \
    S* dxs = (S*)malloc(sizeof(S) * (size_t)(R * m));                                 \
    S* dh0s = (S*)malloc(sizeof(S) * (size_t)BN);                                     \
    for (index_t r = 0; r < R; ++r)                                                   \
      for (index_t j = 0; j < n; ++j) {                                               \
        const S* gr = gates + r * 4 * n;                                              \
        dO[r * n + j] = dh[r * n + j] * c[r * n + j];                                 \
        dc[r * n + j] = dh[r * n + j] * gr[2 * n + j];                                \
        f[r * n + j] = gr[j];                                                         \
      }                                                                               \
    scan_bwd_##SUF(f, c0, c, dc, df, diz, dc0, T, BN);                                \
    for (index_t r = 0; r < R; ++r) {                                                 \
      const S* gr = gates + r * 4 * n;                                                \
      S* o = dpre + r * 4 * n;                                                        \
      for (index_t j = 0; j < n; ++j) {                                               \
        const S fv = gr[j], iv = gr[n + j], ov = gr[2 * n + j], zv = gr[3 * n + j];   \
        const S dfj = df[r * n + j], dizj = diz[r * n + j];                           \
        o[j] = dfj * fv * ((S)1 - fv);                                                \
        o[n + j] = dizj * zv * iv * ((S)1 - iv);                                      \
        o[2 * n + j] = dO[r * n + j] * ov * ((S)1 - ov);                              \
        o[3 * n + j] = dizj * iv * ((S)1 - zv * zv);                                  \
      }                                                                               \
    }                                                                                 \
    for (index_t k = 0; k < BN; ++k) hp[k] = htil0 ? htil0[k] : (S)0;                 \
    memcpy(hp + BN, htil, sizeof(S) * (size_t)(N - BN));                              \
    wgrad_##SUF(dpre, R, 4 * n, hp, n, dU);                                           \
    wgrad_##SUF(dpre, R, 4 * n, x, m, dV);                                            \
    bgrad_##SUF(dpre, R, 4 * n, dbias);                                               \
    igrad_##SUF(dpre, R, 4 * n, V, m, dx, 0);                                         \
    igrad_##SUF(dpre, R, 4 * n, U, n, dhp, 0);                                        \
    memcpy(dht, dhp + BN, sizeof(S) * (size_t)(N - BN));                              \
    memset(dht + (N - BN), 0, sizeof(S) * (size_t)BN);                                \
    oracle_gilr_backward_##SUF(x, sU, sV, htil0, 0, sg, si, htil, dht, dsU, dsV, dsbg, dsbz, \
                               dxs, dh0s, T, b, m, n);                                \
    for (index_t k = 0; k < R * m; ++k) dx[k] += dxs[k];                              \
    if (dhtil0)                                                                       \
      for (index_t k = 0; k < BN; ++k) dhtil0[k] = dh0s[k] + dhp[k];                  \
    free(dc); free(dO); free(f); free(df); free(diz); free(dpre); free(hp);           \
    free(dhp); free(dht); free(dxs); free(dh0s);                                      \
  }                                                                                      \
                                                                                      \
  /* qrnn_forward :449-494.  W: k taps packed [k][3n][m] (QrnnParams::W).        \
   * Writes h; gates [R][3n] activated (f, o, z), c (QrnnCache :420-423). */         \
  void oracle_qrnn_forward_##SUF(const S* x, const S* W, const S* bias, const S* c0,  \
                                 S* h, S* gates, S* c, index_t T, index_t b,          \
                                 index_t m, index_t n, index_t k) {                   \
    const index_t R = T * b, N = R * n;                                               \
    S* f = (S*)malloc(sizeof(S) * (size_t)N);                                         \
    S* imp = (S*)malloc(sizeof(S) * (size_t)N);                                       \
    for (index_t r = 0; r < R; ++r)                                                   \
      for (index_t j = 0; j < 3 * n; ++j) gates[r * 3 * n + j] = bias[j];             \
    /* tap s: rows s*b.. accumulate x rows 0.. against W_s (:468-470) */              \
    for (index_t s = 0; s < k && s < T; ++s)                                          \
      affine_##SUF(x, (T - s) * b, m, W + s * 3 * n * m, 3 * n, (const S*)0,          \
                   gates + s * b * 3 * n, 1);                                         \
    for (index_t r = 0; r < R; ++r) {                                                 \
      S* gr = gates + r * 3 * n;                                                      \
      for (index_t j = 0; j < 2 * n; ++j) gr[j] = sig_##SUF(gr[j]);                   \
      for (index_t j = 2 * n; j < 3 * n; ++j) gr[j] = TANH(gr[j]);                    \
      for (index_t j = 0; j < n; ++j) {                                               \
        f[r * n + j] = gr[j];                                                         \
        imp[r * n + j] = ((S)1 - gr[j]) * gr[2 * n + j];                              \
      }                                                                               \
    }                                                                                 \
    scan_##SUF(f, imp, c0, c, T, b * n);                                              \
    for (index_t r = 0; r < R; ++r)                                                   \
      for (index_t j = 0; j < n; ++j) h[r * n + j] = gates[r * 3 * n + n + j] * c[r * n + j]; \
    free(f); free(imp);                                                               \
  }                                                                                   \
                                                                                      \
  /* qrnn_backward :496-548.  Accumulates dW (packed [k][3n][m]) and dbias;      \
   * writes dx and dc0. */                                                            \
  void oracle_qrnn_backward_##SUF(const S* x, const S* W, const S* c0, const S* gates, \
                                  const S* c, const S* dh, S* dW, S* dbias, S* dx,    \
                                  S* dc0, index_t T, index_t b, index_t m, index_t n, \
                                  index_t k) {                                        \
    const index_t R = T * b, N = R * n;                                               \
    S* dc = (S*)malloc(sizeof(S) * (size_t)N);                                        \
    S* dO = (S*)malloc(sizeof(S) * (size_t)N);                                        \
    S* f = (S*)malloc(sizeof(S) * (size_t)N);                                         \
    S* df = (S*)malloc(sizeof(S) * (size_t)N);                                        \
    S* dimp = (S*)malloc(sizeof(S) * (size_t)N);                                      \
    S* dpre = (S*)malloc(sizeof(S) * (size_t)(3 * N));                                \
    for (index_t r = 0; r < R; ++r)                                                   \
      for (index_t j = 0; j < n; ++j) {                                               \
        const S* gr = gates + r * 3 * n;                                              \
        dO[r * n + j] = dh[r * n + j] * c[r * n + j];                                 \
        dc[r * n + j] = dh[r * n + j] * gr[n + j];                                    \
        f[r * n + j] = gr[j];                                                         \
      }                                                                               \
    scan_bwd_##SUF(f, c0, c, dc, df, dimp, dc0, T, b * n);                            \
    for (index_t r = 0; r < R; ++r) {                                                 \
      const S* gr = gates + r * 3 * n;                                                \
      S* o = dpre + r * 3 * n;                                                        \
      for (index_t j = 0; j < n; ++j) {                                               \
        const S fv = gr[j], ov = gr[n + j], zv = gr[2 * n + j];                       \
        const S dfj = df[r * n + j], dij = dimp[r * n + j];                           \
        o[j] = (dfj - dij * zv) * fv * ((S)1 - fv);                                   \
        o[n + j] = dO[r * n + j] * ov * ((S)1 - ov);                                  \
        o[2 * n + j] = dij * ((S)1 - fv) * ((S)1 - zv * zv);                          \
      }                                                                               \
    }                                                                                 \
    bgrad_##SUF(dpre, R, 3 * n, dbias);                                               \
    for (index_t q = 0; q < R * m; ++q) dx[q] = 0;                                    \
    for (index_t s = 0; s < k && s < T; ++s) {                                        \
      const index_t nr = (T - s) * b;                                                 \
      wgrad_##SUF(dpre + s * b * 3 * n, nr, 3 * n, x, m, dW + s * 3 * n * m);         \
      igrad_##SUF(dpre + s * b * 3 * n, nr, 3 * n, W + s * 3 * n * m, m, dx, 1);      \
    }                                                                                 \
    free(dc); free(dO); free(f); free(df); free(dimp); free(dpre);                    \
  }

DEFINE_LAYERS(double, f64, fma, exp, tanh)
DEFINE_LAYERS(float, f32, fmaf, expf, tanhf)
