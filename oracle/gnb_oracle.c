/*
 * gnb_oracle.c -- C restatement of the reference hot path.
 * TEST / CPU-BASELINE INFRASTRUCTURE ONLY: loaded by tests/, smoke() and
 * bench.py's cpu_baseline / --impl reference legs.  The product
 * (paper_1905_13746_b200, libgnb.so) never links or calls it.
 *
 * Parity is pinned: tests/test_oracle_c.py checks it bit-for-bit against
 * oracle/oracle.py, which is checked against golden vectors produced by the
 * reference itself (tests/golden/make_golden.py).
 *
 * Built with -ffp-contract=off: `acc = acc + x * ll` is a multiply then an
 * add, exactly the reference's `score_m += n * ll_m`
 * (pkg/src/groupnb/classifier.py:143-147).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  const void* x;
  int x_type; /* 0 int32, 1 uint16, 2 uint8 (same counts, narrower storage) */
  int64_t lo, hi, ldx;
  int32_t F, C, width, limit;
  const int32_t* size;
  const int32_t* route;
  const double* prior; /* [S][C] */
  const double* ll;    /* [S][C][F] */
  int32_t* label;
  double* logpost;     /* nullable [N][C] */
} pred_job;

static void finish_row(const pred_job* j, int64_t r, const double* acc) {
  int best = 0;
  for (int c = 1; c < j->C; ++c)
    if (acc[c] > acc[best]) best = c; /* strict: ties -> lowest index (benign) */
  j->label[r] = best;
  if (j->logpost)
    for (int c = 0; c < j->C; ++c) j->logpost[r * j->C + c] = acc[c];
}

/* log_posterior + predict + _classify_slice (classifier.py:132-158,
 * engine.py:187-206) for rows [lo, hi).  Four rows that share a model are
 * scored together so 4*C independent accumulator chains overlap; each chain
 * is still the reference's exact sequence of multiply-then-add in feature
 * order.  One body per storage type. */
#define DEFINE_PREDICT_ROWS(NAME, T)                                                    \
  static void* NAME(void* arg) {                                                        \
    const pred_job* j = (const pred_job*)arg;                                           \
    const int C = j->C, F = j->F;                                                       \
    const T* X = (const T*)j->x;                                                        \
    int64_t r = j->lo;                                                                  \
    while (r < j->hi) {                                                                 \
      int64_t rows[4];                                                                  \
      int nr = 0, s = -1;                                                               \
      while (r < j->hi && nr < 4) {                                                     \
        const int32_t sz = j->size[r];                                                  \
        if (sz < 0 || sz >= j->limit) {                                                 \
          j->label[r] = -1;                                                             \
          if (j->logpost)                                                               \
            for (int c = 0; c < C; ++c) j->logpost[r * C + c] = __builtin_nan("");     \
          ++r;                                                                          \
          continue;                                                                     \
        }                                                                               \
        const int rs = j->route[sz / j->width];                                         \
        if (nr > 0 && rs != s) break;                                                   \
        s = rs;                                                                         \
        rows[nr++] = r++;                                                               \
      }                                                                                 \
      if (nr == 0) continue;                                                            \
      double acc[4][16];                                                                \
      const T* xr[4];                                                                   \
      for (int i = 0; i < nr; ++i) {                                                    \
        xr[i] = X + rows[i] * j->ldx;                                                   \
        for (int c = 0; c < C; ++c) acc[i][c] = j->prior[s * C + c];                    \
      }                                                                                 \
      const double* ll = j->ll + (int64_t)s * C * F;                                    \
      if (nr == 4) {                                                                    \
        for (int f = 0; f < F; ++f) {                                                   \
          const double x0 = xr[0][f], x1 = xr[1][f], x2 = xr[2][f], x3 = xr[3][f];      \
          for (int c = 0; c < C; ++c) {                                                 \
            const double w = ll[(int64_t)c * F + f];                                    \
            acc[0][c] = acc[0][c] + x0 * w;                                             \
            acc[1][c] = acc[1][c] + x1 * w;                                             \
            acc[2][c] = acc[2][c] + x2 * w;                                             \
            acc[3][c] = acc[3][c] + x3 * w;                                             \
          }                                                                             \
        }                                                                               \
      } else {                                                                          \
        for (int i = 0; i < nr; ++i)                                                    \
          for (int f = 0; f < F; ++f) {                                                 \
            const double x = xr[i][f];                                                  \
            for (int c = 0; c < C; ++c) acc[i][c] = acc[i][c] + x * ll[(int64_t)c * F + f]; \
          }                                                                             \
      }                                                                                 \
      for (int i = 0; i < nr; ++i) finish_row(j, rows[i], acc[i]);                      \
    }                                                                                   \
    return NULL;                                                                        \
  }

DEFINE_PREDICT_ROWS(predict_rows_i32, int32_t)
DEFINE_PREDICT_ROWS(predict_rows_u16, uint16_t)
DEFINE_PREDICT_ROWS(predict_rows_u8, uint8_t)

static void* predict_rows(void* arg) {
  const pred_job* j = (const pred_job*)arg;
  return j->x_type == 2 ? predict_rows_u8(arg)
         : j->x_type == 1 ? predict_rows_u16(arg)
                          : predict_rows_i32(arg);
}

int oracle_predict_typed(const void* x, int32_t x_type, int64_t n, int32_t F, int64_t ldx,
                         const int32_t* size, int32_t width, int32_t limit,
                         const int32_t* route, int32_t C, const double* prior, const double* ll,
                         int32_t* label, double* logpost, int32_t threads) {
  if (C < 2 || C > 16 || threads < 1 || x_type < 0 || x_type > 2) return 1;
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  pred_job jobs[256];
  int started[256];
  const int64_t per = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    pred_job j = {x, x_type, t * per, (t + 1) * per < n ? (t + 1) * per : n, ldx, F, C,
                  width, limit, size, route, prior, ll, label, logpost};
    jobs[t] = j;
    started[t] = 0;
    if (jobs[t].lo >= jobs[t].hi) continue;
    if (threads > 1 && pthread_create(&tid[t], NULL, predict_rows, &jobs[t]) == 0)
      started[t] = 1;
    else
      predict_rows(&jobs[t]);
  }
  for (int t = 0; t < threads; ++t)
    if (started[t]) pthread_join(tid[t], NULL);
  return 0;
}

int oracle_predict(const int32_t* x, int64_t n, int32_t F, int64_t ldx, const int32_t* size,
                   int32_t width, int32_t limit, const int32_t* route, int32_t C,
                   const double* prior, const double* ll, int32_t* label, double* logpost,
                   int32_t threads) {
  return oracle_predict_typed(x, 0, n, F, ldx, size, width, limit, route, C, prior, ll, label,
                              logpost, threads);
}

/* Segmented sums (features.py:48-53, classifier.py:94-101, corpus.py:302-305)
 * plus sums of squares; exact 64-bit integers. */
int oracle_fit_stats(const int32_t* x, int64_t n, int32_t V, int64_t ldx, const int32_t* size,
                     const int32_t* label, int32_t width, int32_t limit, int32_t C,
                     int64_t* S, int64_t* Q, int64_t* cnt, int64_t* status) {
  const int64_t G = limit / width;
  memset(S, 0, sizeof(int64_t) * G * C * V);
  if (Q) memset(Q, 0, sizeof(int64_t) * G * C * V);
  memset(cnt, 0, sizeof(int64_t) * G * C);
  status[0] = status[1] = 0;
  for (int64_t r = 0; r < n; ++r) {
    if (size[r] < 0 || size[r] >= limit) {
      ++status[1];
      continue;
    }
    if (label[r] < 0 || label[r] >= C) {
      ++status[0];
      continue;
    }
    const int64_t key = (int64_t)(size[r] / width) * C + label[r];
    ++cnt[key];
    const int32_t* row = x + r * ldx;
    int64_t* s = S + key * V;
    int64_t* q = Q ? Q + key * V : NULL;
    for (int v = 0; v < V; ++v) {
      s[v] += row[v];
      if (q) q[v] += (int64_t)row[v] * row[v];
    }
  }
  return 0;
}
