/*
 * pgo.c -- float64 CPU ORACLE of one SGD step of the Polyglot/SENNA window
 * ranking LM.  TEST INFRASTRUCTURE ONLY (see pgo.h for who may call it).
 *
 * Written to be read against the sources, not to be fast:
 *   - no blocking, fusion or reordering beyond the definitions;
 *   - the corrupt window is evaluated from scratch (no shared-context
 *     shortcut), reading SURVEY.md §8(c) step 2;
 *   - embedding gradients are emitted as 2n unmerged rows per active example
 *     ("duplicates NOT pre-merged") and applied by the serial
 *     k-order index_add ("Given a row of W indexed by I, this
 *     operation adds the corresponding row of Y to it ... for each row indexed
 *     by I", the serial baseline).
 * Every function cites the passage it follows.  Parity pins: tests/test_oracle_*.py.
 */
#include "pgo.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

enum { PGO_OK = 0, PGO_EINVAL = 1, PGO_ERANGE = 2, PGO_EDIVERGED = 6 };

static int64_t g_bad_pos = -1, g_bad_val = 0;

void pgo_last_bad(int64_t* position, int64_t* value) {
  if (position) *position = g_bad_pos;
  if (value) *value = g_bad_val;
}

static int check_shape(int64_t V, int d, int n, int h) {
  if (V < 2 || d < 1 || n < 1 || h < 1 || V > 2147483647LL) return PGO_EINVAL;
  return PGO_OK;
}

/* Index validation before any mutation ("index error reporting
 * offending position and value"; "w never left partially
 * updated").  idx is checked first in flat order, then corr. */
static int check_indices(int64_t V, int n, const int32_t* idx,
                         const int32_t* corr, int64_t B) {
  for (int64_t i = 0; i < B * n; ++i)
    if (idx[i] < 0 || idx[i] >= V) {
      g_bad_pos = i; g_bad_val = idx[i];
      return PGO_ERANGE;
    }
  if (corr)
    for (int64_t k = 0; k < B; ++k)
      if (corr[k] < 0 || corr[k] >= V) {
        g_bad_pos = B * n + k; g_bad_val = corr[k];
        return PGO_ERANGE;
      }
  return PGO_OK;
}

/* ---------------------------------------------------------------------- */
/* Initialisation, reading G10 / SURVEY.md §8(c) step 7:                   */
/*   the i-th output of a SplitMix64 stream keyed by (seed, tensor id);    */
/*   u = (x >> 40) * 2^-24 in [0,1); value = float((2u - 1) * r), widened. */
/*   r = 0.5 for C (fan_in 1), 0.5/(n*d) for W1, 0.5/h for w2; biases 0.   */
/*   ("uniform in [-0.5/fan_in, +0.5/fan_in] ... biases zero") */
/* ---------------------------------------------------------------------- */
static uint64_t splitmix64_output(uint64_t state_after_increment) {
  uint64_t z = state_after_increment;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static void fill_uniform(double* out, int64_t count, uint64_t seed,
                         uint64_t tensor_id, double r) {
  uint64_t state = seed ^ (0x632BE59BD9B4E019ULL * (tensor_id + 1));
  for (int64_t i = 0; i < count; ++i) {
    state += 0x9E3779B97F4A7C15ULL;               /* SplitMix64 increment */
    uint64_t x = splitmix64_output(state);
    double u = (double)(x >> 40) * (1.0 / 16777216.0);
    float v = (float)((2.0 * u - 1.0) * r);
    out[i] = (double)v;
  }
}

int pgo_init_params(int64_t V, int d, int n, int h, uint64_t seed,
                    double* C, double* W1, double* b1, double* w2, double* b2) {
  if (check_shape(V, d, n, h)) return PGO_EINVAL;
  fill_uniform(C, V * d, seed, 0, 0.5);
  fill_uniform(W1, (int64_t)n * d * h, seed, 1, 0.5 / (double)(n * d));
  fill_uniform(w2, h, seed, 2, 0.5 / (double)h);
  for (int u = 0; u < h; ++u) b1[u] = 0.0;
  *b2 = 0.0;
  return PGO_OK;
}

/* ---------------------------------------------------------------------- */
/* Score of one window (hardtanh per north_star / G1):    */
/*   x = concat_p C[t_p];  a = W1^T x + b1;  z = clamp(a,-1,1);            */
/*   s = w2 . z + b2.                                                       */
/* ---------------------------------------------------------------------- */
static double hardtanh(double a) { return a < -1.0 ? -1.0 : (a > 1.0 ? 1.0 : a); }

/* Nonlinearity switch: 0 = hardtanh (north_star,
 * G1), 1 = tanh.  Process-wide; test infrastructure. */
static int g_act = 0;
int pgo_set_activation(int act) {
  if (act != 0 && act != 1) return PGO_EINVAL;
  g_act = act;
  return PGO_OK;
}
/* Batch reduction (reading G4 / SURVEY.md §8(f) NEXT-2): 0 = mean (default:
 * L = (1/B) sum l_k, gradients likewise), 1 = sum (L = sum l_k, the reading
 * PAPER.md:197-198 hints at).  Process-wide; test infrastructure. */
static int g_sum = 0;
int pgo_set_reduction(int sum) {
  if (sum != 0 && sum != 1) return PGO_EINVAL;
  g_sum = sum;
  return PGO_OK;
}
static double batch_scale(int64_t B) { return g_sum ? 1.0 : 1.0 / (double)B; }

static double act_f(double a) { return g_act ? tanh(a) : hardtanh(a); }
/* f'(a): hardtanh' = 1 strictly inside (-1, 1), 0 at and beyond +-1 (G2);
 * tanh' = 1 - tanh(a)^2. */
static double act_d(double a) {
  if (g_act) { const double t = tanh(a); return 1.0 - t * t; }
  return fabs(a) < 1.0 ? 1.0 : 0.0;
}

static void build_window(int d, int n, const double* C, const int32_t* tokens,
                         double* x) {
  for (int p = 0; p < n; ++p)
    for (int j = 0; j < d; ++j) x[p * d + j] = C[(int64_t)tokens[p] * d + j];
}

static double score_window(int d, int n, int h, const double* W1,
                           const double* b1, const double* w2, double b2,
                           const double* x, double* a) {
  double s = b2;
  for (int u = 0; u < h; ++u) {
    double acc = b1[u];
    for (int i = 0; i < n * d; ++i) acc += x[i] * W1[(int64_t)i * h + u];
    a[u] = acc;
    s += w2[u] * act_f(acc);
  }
  return s;
}

/* The true window and its corrupted copy: block c = floor(n/2) is replaced
 * by the corrupt centre word (reading G5). */
static void corrupt_tokens(int n, const int32_t* tokens, int32_t corr_word,
                           int32_t* out) {
  for (int p = 0; p < n; ++p) out[p] = tokens[p];
  out[n / 2] = corr_word;
}

int pgo_forward(int64_t V, int d, int n, int h, const double* C,
                const double* W1, const double* b1, const double* w2,
                const double* b2, const int32_t* idx, const int32_t* corr,
                int64_t B, double* a_out, double* a_corr_out, double* s_out,
                double* s_corr_out, double* loss_out) {
  if (check_shape(V, d, n, h) || B < 1) return PGO_EINVAL;
  int rc = check_indices(V, n, idx, corr, B);
  if (rc) return rc;
  double* x = malloc(sizeof(double) * n * d);
  double* a = malloc(sizeof(double) * h);
  int32_t* tk = malloc(sizeof(int32_t) * n);
  double hinge_sum = 0.0;
  for (int64_t k = 0; k < B; ++k) {
    build_window(d, n, C, idx + k * n, x);
    double s = score_window(d, n, h, W1, b1, w2, *b2, x, a);
    if (a_out) memcpy(a_out + k * h, a, sizeof(double) * h);
    corrupt_tokens(n, idx + k * n, corr[k], tk);
    build_window(d, n, C, tk, x);
    double sc = score_window(d, n, h, W1, b1, w2, *b2, x, a);
    if (a_corr_out) memcpy(a_corr_out + k * h, a, sizeof(double) * h);
    if (s_out) s_out[k] = s;
    if (s_corr_out) s_corr_out[k] = sc;
    double m = 1.0 - s + sc;
    hinge_sum += m > 0.0 ? m : 0.0;
  }
  if (loss_out) *loss_out = hinge_sum * batch_scale(B);  /* mean (reading G4) or sum */
  free(x); free(a); free(tk);
  return PGO_OK;
}

int pgo_score(int64_t V, int d, int n, int h, const double* C, const double* W1,
              const double* b1, const double* w2, const double* b2,
              const int32_t* idx, int64_t B, double* scores) {
  if (check_shape(V, d, n, h) || B < 1) return PGO_EINVAL;
  int rc = check_indices(V, n, idx, NULL, B);
  if (rc) return rc;
  double* x = malloc(sizeof(double) * n * d);
  double* a = malloc(sizeof(double) * h);
  for (int64_t k = 0; k < B; ++k) {
    build_window(d, n, C, idx + k * n, x);
    scores[k] = score_window(d, n, h, W1, b1, w2, *b2, x, a);
  }
  free(x); free(a);
  return PGO_OK;
}

/* ---------------------------------------------------------------------- */
/* Backward.  Gradients of       */
/* inv_batch * sum_k max(0, m_k) w.r.t. every parameter, all at the        */
/* pre-step parameters.  For each k with m > 0 (G3: subgradient 0 at 0):   */
/*   g = -inv_batch (d m/d s = -1), g' = +inv_batch (d m/d s' = +1)         */
/*   delta  = g  * w2 .* f'(a)   (hardtanh: [|a| < 1], G2; tanh: 1 - z^2)  */
/*   delta' = g' * w2 .* f'(a')                                             */
/*   dW1 += x delta^T + x' delta'^T;  db1 += delta + delta';                */
/*   dw2 += g z + g' z';  db2 += g + g'                                     */
/*   dx = W1 delta, dx' = W1 delta'  -> 2n rows (idx[k][p], dx_p) then      */
/*   (corrupted tokens[p], dx'_p), unmerged.                  */
/* rows must hold 2*n*B entries and Y 2*n*B*d.                              */
/* ---------------------------------------------------------------------- */
int pgo_backward(int64_t V, int d, int n, int h, const double* C,
                 const double* W1, const double* b1, const double* w2,
                 const double* b2, const int32_t* idx, const int32_t* corr,
                 int64_t B, double inv_batch, double* dW1, double* db1,
                 double* dw2, double* db2, int32_t* rows, double* Y,
                 int64_t* nrows) {
  if (check_shape(V, d, n, h) || B < 1) return PGO_EINVAL;
  int rc = check_indices(V, n, idx, corr, B);
  if (rc) return rc;
  const int nd = n * d;
  memset(dW1, 0, sizeof(double) * nd * h);
  memset(db1, 0, sizeof(double) * h);
  memset(dw2, 0, sizeof(double) * h);
  *db2 = 0.0;
  double* x = malloc(sizeof(double) * nd);
  double* xc = malloc(sizeof(double) * nd);
  double* a = malloc(sizeof(double) * h);
  double* ac = malloc(sizeof(double) * h);
  double* delta = malloc(sizeof(double) * h);
  double* deltac = malloc(sizeof(double) * h);
  int32_t* tk = malloc(sizeof(int32_t) * n);
  int64_t r = 0;
  for (int64_t k = 0; k < B; ++k) {
    const int32_t* t = idx + k * n;
    corrupt_tokens(n, t, corr[k], tk);
    build_window(d, n, C, t, x);
    build_window(d, n, C, tk, xc);
    double s = score_window(d, n, h, W1, b1, w2, *b2, x, a);
    double sc = score_window(d, n, h, W1, b1, w2, *b2, xc, ac);
    double m = 1.0 - s + sc;
    if (!(m > 0.0)) continue;                      /* inactive hinge */
    double g = -inv_batch, gc = +inv_batch;
    for (int u = 0; u < h; ++u) {
      delta[u] = g * w2[u] * act_d(a[u]);
      deltac[u] = gc * w2[u] * act_d(ac[u]);
    }
    for (int i = 0; i < nd; ++i)
      for (int u = 0; u < h; ++u)
        dW1[(int64_t)i * h + u] += x[i] * delta[u] + xc[i] * deltac[u];
    for (int u = 0; u < h; ++u) {
      db1[u] += delta[u] + deltac[u];
      dw2[u] += g * act_f(a[u]) + gc * act_f(ac[u]);
    }
    *db2 += g + gc;
    /* dx = W1 delta (true window), then dx' = W1 delta' (corrupt window) */
    for (int pass = 0; pass < 2; ++pass) {
      const int32_t* toks = pass == 0 ? t : tk;
      const double* dl = pass == 0 ? delta : deltac;
      for (int p = 0; p < n; ++p) {
        rows[r] = toks[p];
        for (int j = 0; j < d; ++j) {
          double acc = 0.0;
          for (int u = 0; u < h; ++u)
            acc += W1[(int64_t)(p * d + j) * h + u] * dl[u];
          Y[r * d + j] = acc;
        }
        ++r;
      }
    }
  }
  *nrows = r;
  free(x); free(xc); free(a); free(ac); free(delta); free(deltac); free(tk);
  return PGO_OK;
}

/* ---------------------------------------------------------------------- */
/* Serial scatter-add, the paper's operation in the      */
/* order of its Python baseline:         */
/*   for k = 0..n-1 in sequence: W[I[k], :] += Y[k, :]                     */
/* ---------------------------------------------------------------------- */
int pgo_index_add(double* W, int64_t rows, int cols, const double* Y,
                  const int32_t* I, int64_t n) {
  if (rows < 0 || cols < 1 || n < 0) return PGO_EINVAL;
  for (int64_t k = 0; k < n; ++k)
    if (I[k] < 0 || I[k] >= rows) {
      g_bad_pos = k; g_bad_val = I[k];
      return PGO_ERANGE;
    }
  for (int64_t k = 0; k < n; ++k)
    for (int j = 0; j < cols; ++j) W[(int64_t)I[k] * cols + j] += Y[k * cols + j];
  return PGO_OK;
}

int pgo_index_add_f32(float* W, int64_t rows, int cols, const float* Y,
                      const int32_t* I, int64_t n) {
  if (rows < 0 || cols < 1 || n < 0) return PGO_EINVAL;
  for (int64_t k = 0; k < n; ++k)
    if (I[k] < 0 || I[k] >= rows) {
      g_bad_pos = k; g_bad_val = I[k];
      return PGO_ERANGE;
    }
  for (int64_t k = 0; k < n; ++k)
    for (int j = 0; j < cols; ++j) W[(int64_t)I[k] * cols + j] += Y[k * cols + j];
  return PGO_OK;
}

/* ---------------------------------------------------------------------- */
/* sgd_update ("[OP] sgd_update ... post: dense params       */
/* updated as theta -= lr * grad theta; embedding table updated via          */
/* index_add(C, -lr * values, indices)"):                                    */
/*   theta -= lr * grad for W1, b1, w2, b2;                                  */
/*   C: serial index_add of (-lr * Y) over the rows in emission order.       */
/* lr > 0 ("pre: lr > 0"); an out-of-range row leaves every      */
/* parameter unchanged (checked before anything is written).                 */
/* ---------------------------------------------------------------------- */
int pgo_sgd_update(int64_t V, int d, int n, int h, double* C, double* W1,
                   double* b1, double* w2, double* b2, double lr,
                   const double* dW1, const double* db1, const double* dw2,
                   double db2, const int32_t* rows, const double* Y,
                   int64_t nrows) {
  if (check_shape(V, d, n, h) || nrows < 0 || !(lr > 0.0) || !isfinite(lr))
    return PGO_EINVAL;
  for (int64_t k = 0; k < nrows; ++k)
    if (rows[k] < 0 || rows[k] >= V) {
      g_bad_pos = k; g_bad_val = rows[k];
      return PGO_ERANGE;
    }
  for (int64_t i = 0; i < (int64_t)n * d * h; ++i) W1[i] -= lr * dW1[i];
  for (int u = 0; u < h; ++u) {
    b1[u] -= lr * db1[u];
    w2[u] -= lr * dw2[u];
  }
  *b2 -= lr * db2;
  double* scaled = malloc(sizeof(double) * (nrows > 0 ? nrows : 1) * d);
  for (int64_t i = 0; i < nrows * d; ++i) scaled[i] = -lr * Y[i];
  int rc = pgo_index_add(C, V, d, scaled, rows, nrows);
  free(scaled);
  return rc;
}

/* ---------------------------------------------------------------------- */
/* One SGD step (reading G8: every gradient and the       */
/* returned loss use the pre-step parameters, then all updates apply).     */
/* A non-finite loss leaves every parameter unchanged.        */
/* ---------------------------------------------------------------------- */
int pgo_train_step(int64_t V, int d, int n, int h, double* C, double* W1,
                   double* b1, double* w2, double* b2, const int32_t* idx,
                   const int32_t* corr, int64_t B, double lr,
                   double* loss_out) {
  if (check_shape(V, d, n, h) || B < 1 || !(lr > 0.0) || !isfinite(lr))
    return PGO_EINVAL;
  int rc = check_indices(V, n, idx, corr, B);
  if (rc) return rc;
  double loss;
  rc = pgo_forward(V, d, n, h, C, W1, b1, w2, b2, idx, corr, B, NULL, NULL,
                   NULL, NULL, &loss);
  if (rc) return rc;
  if (loss_out) *loss_out = loss;
  if (!isfinite(loss)) return PGO_EDIVERGED;
  const int64_t nd = (int64_t)n * d;
  double* dW1 = malloc(sizeof(double) * nd * h);
  double* db1 = malloc(sizeof(double) * h);
  double* dw2 = malloc(sizeof(double) * h);
  double db2;
  int32_t* rows = malloc(sizeof(int32_t) * 2 * n * B);
  double* Y = malloc(sizeof(double) * 2 * n * B * d);
  int64_t nrows = 0;
  rc = pgo_backward(V, d, n, h, C, W1, b1, w2, b2, idx, corr, B,
                    batch_scale(B), dW1, db1, dw2, &db2, rows, Y, &nrows);
  if (!rc)
    rc = pgo_sgd_update(V, d, n, h, C, W1, b1, w2, b2, lr, dW1, db1, dw2, db2,
                      rows, Y, nrows);
  free(dW1); free(db1); free(dw2); free(rows); free(Y);
  return rc;
}

/* ---------------------------------------------------------------------- */
/* G-rank data-parallel emulation: the batch is split    */
/* into `world` contiguous equal shards; each shard's gradients are scaled */
/* by 1/B_global; dense gradients are summed in rank order and the sparse  */
/* rows concatenated in rank order; then one update as above.  In exact    */
/* arithmetic this equals pgo_train_step on the whole batch.               */
/* ---------------------------------------------------------------------- */
int pgo_train_step_dp(int64_t V, int d, int n, int h, double* C, double* W1,
                      double* b1, double* w2, double* b2, const int32_t* idx,
                      const int32_t* corr, int64_t B, int world, double lr,
                      double* loss_out) {
  if (check_shape(V, d, n, h) || B < 1 || world < 1 || B % world != 0 ||
      !(lr > 0.0) || !isfinite(lr))
    return PGO_EINVAL;
  int rc = check_indices(V, n, idx, corr, B);
  if (rc) return rc;
  const int64_t Bl = B / world, nd = (int64_t)n * d;
  double loss = 0.0;
  for (int g = 0; g < world; ++g) {
    double lg;
    pgo_forward(V, d, n, h, C, W1, b1, w2, b2, idx + g * Bl * n, corr + g * Bl,
                Bl, NULL, NULL, NULL, NULL, &lg);
    loss += g_sum ? lg : lg * (double)Bl / (double)B;
  }
  if (loss_out) *loss_out = loss;
  if (!isfinite(loss)) return PGO_EDIVERGED;
  double* dW1 = calloc(nd * h, sizeof(double));
  double* db1 = calloc(h, sizeof(double));
  double* dw2 = calloc(h, sizeof(double));
  double db2 = 0.0;
  double* gW1 = malloc(sizeof(double) * nd * h);
  double* gb1 = malloc(sizeof(double) * h);
  double* gw2 = malloc(sizeof(double) * h);
  double gb2;
  int32_t* rows = malloc(sizeof(int32_t) * 2 * n * B);
  double* Y = malloc(sizeof(double) * 2 * n * B * d);
  int64_t nrows = 0;
  for (int g = 0; g < world; ++g) {
    int64_t nr = 0;
    pgo_backward(V, d, n, h, C, W1, b1, w2, b2, idx + g * Bl * n, corr + g * Bl,
                 Bl, batch_scale(B), gW1, gb1, gw2, &gb2, rows + nrows,
                 Y + nrows * d, &nr);
    nrows += nr;
    for (int64_t i = 0; i < nd * h; ++i) dW1[i] += gW1[i];
    for (int u = 0; u < h; ++u) { db1[u] += gb1[u]; dw2[u] += gw2[u]; }
    db2 += gb2;
  }
  rc = pgo_sgd_update(V, d, n, h, C, W1, b1, w2, b2, lr, dW1, db1, dw2, db2,
                    rows, Y, nrows);
  free(dW1); free(db1); free(dw2); free(gW1); free(gb1); free(gw2);
  free(rows); free(Y);
  return rc;
}
