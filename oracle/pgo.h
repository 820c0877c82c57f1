/*
 * pgo.h -- float64 CPU ORACLE for one SGD step of the Polyglot/SENNA window
 * ranking language model (arXiv:1404.1521).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, constant or helper with the CUDA product path
 * (paper_1404_1521_b200/csrc, include/pg.h); the two are independent
 * implementations of the same written definition.
 *
 * What it computes (PAPER.md gives no formulas; the readings are SURVEY.md
 * §8(c) and DESIGN.md "Readings"):
 *   x_k   = concat_p C[idx[k][p]]                       (gather dual)
 *   x'_k  = x_k with block c=floor(n/2) := C[corr[k]]
 *   a     = W1^T x + b1,  z = hardtanh(a) = clamp(a,-1,1) (BASELINE.json north_star)
 *           or z = tanh(a) after pgo_set_activation(1)
 *   s     = w2 . z + b2,  m = 1 - s + s',  l = max(0, m)
 *   L     = (1/B) sum_k l_k                              (reading G4)
 *   backward by hand, subgradient 0 at |a|=1 and at m=0  (readings G2, G3)
 *   update: dense theta -= lr*grad; embedding rows by the serial k-order
 *   scatter-add C[I[j]] += -lr*Y[j]                      (
 *                                                          SPEC.md:61-69)
 *
 * Layouts (all row-major, caller-owned):
 *   C  [V][d]      W1 [n*d][h] (row p*d+j is input feature j of window slot p)
 *   b1 [h]  w2 [h]  b2 [1]
 *   idx [B][n] int32, corr [B] int32.
 * Status codes: 0 ok, 1 invalid argument, 2 index out of range (no mutation),
 * 6 non-finite loss (no mutation).  On status 2 the first offending flat
 * position and its value are available from pgo_last_bad().
 */
#ifndef PGO_H
#define PGO_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

int pgo_init_params(int64_t V, int d, int n, int h, uint64_t seed,
                    double* C, double* W1, double* b1, double* w2, double* b2);

int pgo_forward(int64_t V, int d, int n, int h,
                const double* C, const double* W1, const double* b1,
                const double* w2, const double* b2,
                const int32_t* idx, const int32_t* corr, int64_t B,
                double* a_out, double* a_corr_out,   /* [B][h] or NULL */
                double* s_out, double* s_corr_out,   /* [B] or NULL */
                double* loss_out);                   /* mean hinge, or NULL */

int pgo_backward(int64_t V, int d, int n, int h,
                 const double* C, const double* W1, const double* b1,
                 const double* w2, const double* b2,
                 const int32_t* idx, const int32_t* corr, int64_t B,
                 double inv_batch,
                 double* dW1, double* db1, double* dw2, double* db2,
                 int32_t* rows, double* Y, int64_t* nrows);

int pgo_score(int64_t V, int d, int n, int h,
              const double* C, const double* W1, const double* b1,
              const double* w2, const double* b2,
              const int32_t* idx, int64_t B, double* scores);

/* theta -= lr * grad (dense), C via serial index_add of -lr * Y. */
int pgo_sgd_update(int64_t V, int d, int n, int h,
                   double* C, double* W1, double* b1, double* w2, double* b2,
                   double lr, const double* dW1, const double* db1,
                   const double* dw2, double db2,
                   const int32_t* rows, const double* Y, int64_t nrows);

int pgo_train_step(int64_t V, int d, int n, int h,
                   double* C, double* W1, double* b1, double* w2, double* b2,
                   const int32_t* idx, const int32_t* corr, int64_t B,
                   double lr, double* loss_out);

int pgo_train_step_dp(int64_t V, int d, int n, int h,
                      double* C, double* W1, double* b1, double* w2, double* b2,
                      const int32_t* idx, const int32_t* corr, int64_t B,
                      int world, double lr, double* loss_out);

int pgo_index_add(double* W, int64_t rows, int cols, const double* Y,
                  const int32_t* I, int64_t n);
int pgo_index_add_f32(float* W, int64_t rows, int cols, const float* Y,
                      const int32_t* I, int64_t n);

void pgo_last_bad(int64_t* position, int64_t* value);
/* 0 = hardtanh (default), 1 = tanh; process-wide. */
int pgo_set_activation(int act);
/* 0 = mean over the batch (default, reading G4), 1 = sum; process-wide. */
int pgo_set_reduction(int sum);

#ifdef __cplusplus
}
#endif
#endif
