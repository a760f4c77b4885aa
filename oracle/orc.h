/*
 * oracle/orc.h -- C-ABI of the CPU ORACLE (liborc.so), TEST INFRASTRUCTURE ONLY.
 *
 * The host "oracle twins" of the product entry points: same arrays, same layout
 * (column-major matrices, symmetric matrices packed lower, [instance][stage][element]), host
 * pointers, FP64.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg load this library; it shares no code with paper_2509_16370_b200/csrc.
 * Ownership: the caller allocates every buffer; the oracle allocates only its own scratch.
 * Threads: POSIX threads over contiguous instance ranges (instances are independent).
 */
#ifndef ORC_H
#define ORC_H
#include <stdint.h>

/* per-instance status words (the product's RR_ST_* values) */
#define ORC_OK 0
#define ORC_G_NOT_PD 1      /* G_i = B_iᵀW_iB_i + R_i not positive definite at stage (status >> 8) */
#define ORC_S_NOT_PD 2      /* S_i = I + δV_i not positive definite                              */
#define ORC_NONFINITE 3
#define OIPM_NONPOS_SLACK 4 /* ipm: s or z not strictly positive                                  */
#define OIPM_LS_FAILED 5    /* ipm: no Armijo step within max_backtracks                          */

/* Tier T2: the regularized Riccati recursion of P:613-625, literally (Cholesky of S_i and G_i),
 * forward sweep P:496-509 / P:640-644 and duals y_i = V_i x_i + v_i, for `batch`
 * instances of the rr_problem arrays; V, v, K, k may be NULL.  Returns 0, or -1 on invalid
 * dimensions.  rr_oracle.c. */
int orc_rr_solve(int nx, int nu, int N, int64_t batch, int nthreads, const double* A, const double* B,
                 const double* Q, const double* M, const double* R, const double* q, const double* r,
                 const double* c, const double* QN, const double* qN, const double* c0, const double* delta,
                 double* x, double* u, double* y, double* V, double* v, double* K, double* k, int32_t* status);

/* Cholesky S = LLᵀ of an n×n column-major SPD matrix (L lower, column-major); 0 or -1 (not PD). */
int orc_chol(int n, const double* S, double* L);
/* b ← (LLᵀ)⁻¹ b */
void orc_chol_solve(int n, const double* L, double* b);

/* One regularized-IPM step (rows a1-a8): condense, T2, expand, merit and
 * D, fraction-to-boundary + Armijo line search (reading R12),
 * in-place update.  ipm_oracle.c. */
typedef struct {
  int nx, nu, N, ng, ngN, nc, ncN, model; /* model: 0 LQ, 1 cart-pole, 2 quadrotor (reading R19) */
  int64_t batch;
  /* stage data at the iterate */
  const double *s0, *fval, *gradf, *gradfN, *Q, *M, *R, *QN, *A, *B, *dres;
  const double *ce, *Ce, *ceN, *CeN, *gv, *Gj, *gvN, *GjN, *model_params;
  /* iterate (updated in place) */
  double *x, *u, *s, *z, *sN, *zN, *y, *lam, *lamN;
  const double *mu, *eta;
  /* params */
  double tau, armijo_c, beta;
  int max_backtracks;
  /* results */
  double *dx, *du, *ds, *dsN, *dy, *dlam, *dlamN, *dz, *dzN;
  double *alpha_p, *alpha_d, *D, *D_closed, *merit0, *merit_acc;
  int32_t *n_backtracks, *status;
} orc_ipm_args;

int orc_ipm_step(const orc_ipm_args* a, int nthreads);
/* 𝒜 at step length alpha along the direction in a->dx.. for instance b (before the update). */
double orc_ipm_merit(const orc_ipm_args* a, int64_t b, double alpha);

/* the built-in models' explicit-Euler steps x⁺ = d(x, u) (reading R19) */
void orc_cartpole_step(const double* prm, const double* x, const double* u, double* xn);
void orc_quadrotor_step(const double* prm, const double* x, const double* u, double* xn);

#endif
