/*
 * hgca_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline leg).
 *
 * Plain-C restatement of the reference's two attention loops
 *   _core.attend_dense    /root/reference/pkg/src/tierkv/_core.pyx:22-84
 *   _core.attend_indexed  /root/reference/pkg/src/tierkv/_core.pyx:87-150
 * with the same loop order and the same double-precision arithmetic:
 *   s = sum_c (double)q[c] * (double)k[c]   (sequential in c, _core.pyx:61-63)
 *   s *= scale; m = running max              (_core.pyx:64-67)
 *   w = exp(s - m); z += w; acc[c] += w*v    (_core.pyx:71-76, j sequential)
 *   out = (real)(acc/z); lse = m + log(z); weights = (real)(w/z)  (_core.pyx:77-82)
 * Built with -ffp-contract=off so acc += w*v is a separately rounded multiply
 * and add, exactly like the reference's -O3 x86-64 (no FMA) Cython build.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load this library. The product path never calls it.
 *
 * Multi-head helpers (or_*_heads) run the identical per-head loops under an
 * OpenMP parallel-for over independent heads: the per-head arithmetic is
 * unchanged, so results are bit-identical to the serial loops.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define DEF_DENSE(NAME, REAL)                                                              \
  static void NAME##_one(const REAL* q, const REAL* k, const REAL* v, int64_t nq,         \
                         int64_t nkv, int64_t d, double scale, int keep_w, REAL* out,     \
                         double* lse, REAL* wts, double* scores, double* acc) {          \
    for (int64_t i = 0; i < nq; ++i) {                                                     \
      if (nkv == 0) {                                                                      \
        for (int64_t c = 0; c < d; ++c) out[i * d + c] = (REAL)0;                          \
        lse[i] = -INFINITY;                                                                \
        continue;                                                                          \
      }                                                                                    \
      double m = -INFINITY;                                                                \
      for (int64_t j = 0; j < nkv; ++j) {                                                  \
        double s = 0.0;                                                                    \
        for (int64_t c = 0; c < d; ++c) s += (double)q[i * d + c] * (double)k[j * d + c]; \
        s *= scale;                                                                        \
        scores[j] = s;                                                                     \
        if (s > m) m = s;                                                                  \
      }                                                                                    \
      double z = 0.0;                                                                      \
      for (int64_t c = 0; c < d; ++c) acc[c] = 0.0;                                        \
      for (int64_t j = 0; j < nkv; ++j) {                                                  \
        double w = exp(scores[j] - m);                                                     \
        scores[j] = w;                                                                     \
        z += w;                                                                            \
        for (int64_t c = 0; c < d; ++c) acc[c] += w * (double)v[j * d + c];                \
      }                                                                                    \
      for (int64_t c = 0; c < d; ++c) out[i * d + c] = (REAL)(acc[c] / z);                 \
      lse[i] = m + log(z);                                                                 \
      if (keep_w)                                                                          \
        for (int64_t j = 0; j < nkv; ++j) wts[i * nkv + j] = (REAL)(scores[j] / z);        \
    }                                                                                      \
  }

#define DEF_INDEXED(NAME, REAL)                                                            \
  static void NAME##_one(const REAL* q, const REAL* k, const REAL* v, const int64_t* idx, \
                         int64_t n, int64_t nq, int64_t d, double scale, int keep_w,      \
                         REAL* out, double* lse, REAL* wts, double* scores, double* acc) { \
    for (int64_t i = 0; i < nq; ++i) {                                                     \
      if (n == 0) {                                                                        \
        for (int64_t c = 0; c < d; ++c) out[i * d + c] = (REAL)0;                          \
        lse[i] = -INFINITY;                                                                \
        continue;                                                                          \
      }                                                                                    \
      double m = -INFINITY;                                                                \
      for (int64_t j = 0; j < n; ++j) {                                                    \
        const REAL* kr = k + idx[j] * d;                                                   \
        double s = 0.0;                                                                    \
        for (int64_t c = 0; c < d; ++c) s += (double)q[i * d + c] * (double)kr[c];        \
        s *= scale;                                                                        \
        scores[j] = s;                                                                     \
        if (s > m) m = s;                                                                  \
      }                                                                                    \
      double z = 0.0;                                                                      \
      for (int64_t c = 0; c < d; ++c) acc[c] = 0.0;                                        \
      for (int64_t j = 0; j < n; ++j) {                                                    \
        double w = exp(scores[j] - m);                                                     \
        scores[j] = w;                                                                     \
        z += w;                                                                            \
        const REAL* vr = v + idx[j] * d;                                                   \
        for (int64_t c = 0; c < d; ++c) acc[c] += w * (double)vr[c];                       \
      }                                                                                    \
      for (int64_t c = 0; c < d; ++c) out[i * d + c] = (REAL)(acc[c] / z);                 \
      lse[i] = m + log(z);                                                                 \
      if (keep_w)                                                                          \
        for (int64_t j = 0; j < n; ++j) wts[i * n + j] = (REAL)(scores[j] / z);            \
    }                                                                                      \
  }

DEF_DENSE(dense_f32, float)
DEF_DENSE(dense_f64, double)
DEF_INDEXED(indexed_f32, float)
DEF_INDEXED(indexed_f64, double)

/* Stacked-head dense attention: q [H,nq,d], k/v [H,nkv,d] (_core.pyx:22-84). */
#define DEF_DENSE_API(NAME, REAL)                                                           \
  int NAME(const REAL* q, const REAL* k, const REAL* v, int64_t H, int64_t nq, int64_t nkv, \
           int64_t d, double scale, int keep_w, REAL* out, double* lse, REAL* wts,          \
           int threads) {                                                                   \
    int64_t h;                                                                              \
    _Pragma("omp parallel for schedule(dynamic, 1) num_threads(threads) if (threads > 1)")  \
    for (h = 0; h < H; ++h) {                                                               \
      double* scores = (double*)malloc(sizeof(double) * (nkv > 0 ? nkv : 1));              \
      double* acc = (double*)malloc(sizeof(double) * (d > 0 ? d : 1));                      \
      dense_##REAL##_wrap(q + h * nq * d, k + h * nkv * d, v + h * nkv * d, nq, nkv, d,     \
                          scale, keep_w, out + h * nq * d, lse + h * nq,                    \
                          keep_w ? wts + h * nq * nkv : 0, scores, acc);                    \
      free(scores);                                                                         \
      free(acc);                                                                            \
    }                                                                                       \
    return 0;                                                                               \
  }

#define dense_float_wrap dense_f32_one
#define dense_double_wrap dense_f64_one
#define indexed_float_wrap indexed_f32_one
#define indexed_double_wrap indexed_f64_one

DEF_DENSE_API(or_attend_dense_f32, float)
DEF_DENSE_API(or_attend_dense_f64, double)

/* Single-head gathered attention: q [nq,d], k/v [M,d], idx [n] (_core.pyx:87-150). */
int or_attend_indexed_f32(const float* q, const float* k, const float* v, const int64_t* idx,
                          int64_t n, int64_t nq, int64_t d, double scale, int keep_w,
                          float* out, double* lse, float* wts) {
  double* scores = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
  double* acc = (double*)malloc(sizeof(double) * (d > 0 ? d : 1));
  indexed_f32_one(q, k, v, idx, n, nq, d, scale, keep_w, out, lse, wts, scores, acc);
  free(scores);
  free(acc);
  return 0;
}

int or_attend_indexed_f64(const double* q, const double* k, const double* v, const int64_t* idx,
                          int64_t n, int64_t nq, int64_t d, double scale, int keep_w,
                          double* out, double* lse, double* wts) {
  double* scores = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
  double* acc = (double*)malloc(sizeof(double) * (d > 0 ? d : 1));
  indexed_f64_one(q, k, v, idx, n, nq, d, scale, keep_w, out, lse, wts, scores, acc);
  free(scores);
  free(acc);
  return 0;
}

/*
 * The engine's decode-mode sparse loop (engine.py:139-148: one attend_indexed
 * per head over that head's entries) for many heads at once:
 *   q [T,nq,d] (one query block per task), archive k/v for task t at
 *   k + kv_off[t]*d, idx_cat concatenated per-task index lists with
 *   idx_off[T+1]. Tasks are independent, so OpenMP over tasks does not change
 *   any per-task result.
 */
int or_attend_indexed_tasks_f32(const float* q, const float* k, const float* v,
                                const int64_t* kv_off, const int64_t* idx_cat,
                                const int64_t* idx_off, int64_t T, int64_t nq, int64_t d,
                                double scale, int keep_w, float* out, double* lse, float* wts,
                                const int64_t* wts_off, int threads) {
  int64_t t;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads) if (threads > 1)
  for (t = 0; t < T; ++t) {
    int64_t n = idx_off[t + 1] - idx_off[t];
    double* scores = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
    double* acc = (double*)malloc(sizeof(double) * (d > 0 ? d : 1));
    indexed_f32_one(q + t * nq * d, k + kv_off[t] * d, v + kv_off[t] * d, idx_cat + idx_off[t],
                    n, nq, d, scale, keep_w, out + t * nq * d, lse + t * nq,
                    keep_w ? wts + wts_off[t] : 0, scores, acc);
    free(scores);
    free(acc);
  }
  return 0;
}
