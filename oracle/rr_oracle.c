/*
 * oracle/rr_oracle.c -- CPU ORACLE, TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct FP64 implementation of the regularized Riccati
 * recursion of arXiv 2509.16370 ("tier T2" in DESIGN.md).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load this library.  It shares no code, header or constant with the CUDA path
 * (paper_2509_16370_b200/csrc); the only common thing is the documented array
 * layout of the inputs.
 *
 * Paper citations: P:n = line n of the paper's PAPER.md.
 *   Regularized LQR system  [P Cᵀ; C −δI][x; y] = −[s; c]        §1.4
 *   Simplified recursion (W, G, g, H, h, K, k, V, v)             §2,
 *   Ansatz u_i = K_i x_i + k_i and forward pass                   §2,
 *   x_0 = (I + δV_0)⁻¹(c_0 − δ v_0)                               §2,
 *   x_{i+1} = (I+δV_{i+1})⁻¹(A_i x_i + B_i u_i + c_{i+1} − δ v_{i+1})  (rewrite of
 *            the ansatz row −A_i x_i − B_i u_i + F_{i+1} x_{i+1} = −f_{i+1}, P:501-504,
 *            with F = I + δV, f = δ v − c)
 *   y_i = V_i x_i + v_i                                           §2,
 * Readings: c has N+1 blocks c_0..c_N (R1)
 * parenthesisation read as P:618-624 (R3); (I+δV)⁻¹ and G⁻¹ applied through
 * Cholesky factorizations (R9); V_i symmetrized as (V+Vᵀ)/2 (R10); δ = 0 accepted (R6).
 *
 * Layout (the C-ABI's documented layout, restated here independently):
 *   column-major matrices, symmetric matrices packed lower (LAPACK 'L' packed),
 *   per-operand arrays indexed [instance][stage][element].
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "orc.h"

static int64_t sym_size(int n) { return (int64_t)n * (n + 1) / 2; }

/* packed lower, column-major: element (r, c) with r >= c */
static int64_t pidx(int n, int r, int c) {
  if (r < c) { int t = r; r = c; c = t; }
  return (int64_t)c * (2 * n - c - 1) / 2 + r;
}

static void unpack_sym(int n, const double* P, double* F) {
  for (int c = 0; c < n; ++c)
    for (int r = 0; r < n; ++r) F[r + c * n] = P[pidx(n, r, c)];
}

static void pack_sym(int n, const double* F, double* P) {
  for (int c = 0; c < n; ++c)
    for (int r = c; r < n; ++r) P[pidx(n, r, c)] = F[r + c * n];
}

/* Cholesky S = L Lᵀ of a full n×n SPD matrix; L full (upper part zero).
 * Returns 0 on success, 1 if a pivot is not strictly positive. */
int orc_chol(int n, const double* S, double* L) {
  memset(L, 0, sizeof(double) * n * n);
  for (int j = 0; j < n; ++j) {
    double d = S[j + j * n];
    for (int k = 0; k < j; ++k) d -= L[j + k * n] * L[j + k * n];
    if (!(d > 0.0)) return 1;
    double ljj = sqrt(d);
    L[j + j * n] = ljj;
    for (int i = j + 1; i < n; ++i) {
      double s = S[i + j * n];
      for (int k = 0; k < j; ++k) s -= L[i + k * n] * L[j + k * n];
      L[i + j * n] = s / ljj;
    }
  }
  return 0;
}

/* Solve (L Lᵀ) x = b in place (forward then backward substitution). */
void orc_chol_solve(int n, const double* L, double* b) {
  for (int i = 0; i < n; ++i) {
    double s = b[i];
    for (int k = 0; k < i; ++k) s -= L[i + k * n] * b[k];
    b[i] = s / L[i + i * n];
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int k = i + 1; k < n; ++k) s -= L[k + i * n] * b[k];
    b[i] = s / L[i + i * n];
  }
}

/* C = op(A) * op(B) with plain loops. ta/tb: 0 = as stored, 1 = transposed.
 * A is (ta ? k×m : m×k), B is (tb ? n×k : k×n), C is m×n; all column-major. */
static void mm(int m, int n, int k, int ta, const double* A, int tb, const double* B, double* C) {
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i) {
      double s = 0.0;
      for (int l = 0; l < k; ++l) {
        double a = ta ? A[l + i * k] : A[i + l * m];
        double b = tb ? B[j + l * n] : B[l + j * k];
        s += a * b;
      }
      C[i + j * m] = s;
    }
}

/* y = op(A) x; A is m×n column-major (ta = 1 → y = Aᵀ x, length n). */
static void mv(int m, int n, int ta, const double* A, const double* x, double* y) {
  int rows = ta ? n : m, cols = ta ? m : n;
  for (int i = 0; i < rows; ++i) {
    double s = 0.0;
    for (int l = 0; l < cols; ++l) s += (ta ? A[l + i * m] : A[i + l * m]) * x[l];
    y[i] = s;
  }
}

typedef struct {
  int nx, nu, N;
  const double *A, *B, *Q, *M, *R, *q, *r, *c, *QN, *qN, *c0, *delta;
  double *x, *u, *y, *V, *v, *K, *k;
  int32_t* status;
} orc_rr_args;

static int all_finite(const double* a, int n) {
  for (int i = 0; i < n; ++i)
    if (!isfinite(a[i])) return 0;
  return 1;
}

/* One instance of the regularized LQR solve, literal Eq. (RR),
 * forward pass and dual recovery.
 * Outputs: x[(N+1)n], u[N m], y[(N+1)n]; optionally the policy V[(N+1)sym(n)],
 * v[(N+1)n], K[N m n] (column-major m×n), k[N m].  Returns the status word. */
static int32_t rr_solve_one(const orc_rr_args* a, int64_t b) {
  const int n = a->nx, m = a->nu, N = a->N;
  const int64_t sn = sym_size(n), sm = sym_size(m);
  const double* A = a->A + b * N * n * n;
  const double* B = a->B + b * N * n * m;
  const double* Q = a->Q + b * N * sn;
  const double* M = a->M + b * N * n * m;
  const double* R = a->R + b * N * sm;
  const double* q = a->q + b * N * n;
  const double* r = a->r + b * N * m;
  const double* c = a->c + b * N * n; /* c[i] = c_{i+1} */
  const double* QN = a->QN + b * sn;
  const double* qN = a->qN + b * n;
  const double* c0 = a->c0 + b * n;
  const double delta = a->delta[b];
  double* x = a->x + b * (N + 1) * n;
  double* u = a->u + b * N * m;
  double* y = a->y + b * (N + 1) * n;

  /* full storage of the whole policy for this instance */
  double* Vs = (double*)malloc(sizeof(double) * (N + 1) * n * n);
  double* vs = (double*)malloc(sizeof(double) * (N + 1) * n);
  double* Ks = (double*)malloc(sizeof(double) * (N > 0 ? N : 1) * m * n);
  double* ks = (double*)malloc(sizeof(double) * (N > 0 ? N : 1) * m);
  double* S = (double*)malloc(sizeof(double) * n * n);
  double* L = (double*)malloc(sizeof(double) * n * n);
  double* W = (double*)malloc(sizeof(double) * n * n);
  double* WA = (double*)malloc(sizeof(double) * n * n);
  double* WB = (double*)malloc(sizeof(double) * n * m);
  double* G = (double*)malloc(sizeof(double) * m * m);
  double* LG = (double*)malloc(sizeof(double) * m * m);
  double* H = (double*)malloc(sizeof(double) * m * n);
  double* Vi = (double*)malloc(sizeof(double) * n * n);
  double* KtH = (double*)malloc(sizeof(double) * n * n);
  double* Rf = (double*)malloc(sizeof(double) * m * m);
  double* Qf = (double*)malloc(sizeof(double) * n * n);
  double* e = (double*)malloc(sizeof(double) * n);
  double* g = (double*)malloc(sizeof(double) * n);
  double* h = (double*)malloc(sizeof(double) * m);
  double* t = (double*)malloc(sizeof(double) * n);
  double* t2 = (double*)malloc(sizeof(double) * n);
  double* tm = (double*)malloc(sizeof(double) * m);
  int32_t st = ORC_OK;

  /* V_N = Q_N, v_N = q_N  (f_N = z_N, F_N = I + δQ_N; P:511-512 with P:566-567) */
  unpack_sym(n, QN, Vs + (int64_t)N * n * n);
  memcpy(vs + (int64_t)N * n, qN, sizeof(double) * n);

  for (int i = N - 1; i >= 0 && st == ORC_OK; --i) {
    const double* Vn = Vs + (int64_t)(i + 1) * n * n;
    const double* vn = vs + (int64_t)(i + 1) * n;
    const double* Ai = A + (int64_t)i * n * n;
    const double* Bi = B + (int64_t)i * n * m;
    const double* Mi = M + (int64_t)i * n * m;
    const double* qi = q + (int64_t)i * n;
    const double* ri = r + (int64_t)i * m;
    const double* cn = c + (int64_t)i * n; /* c_{i+1} */
    double* Ki = Ks + (int64_t)i * m * n;
    double* ki = ks + (int64_t)i * m;

    /* W_i = (I + δ V_{i+1})⁻¹ V_{i+1} */
    for (int jj = 0; jj < n * n; ++jj) S[jj] = delta * Vn[jj];
    for (int d = 0; d < n; ++d) S[d + d * n] += 1.0;
    if (orc_chol(n, S, L)) { st = ORC_S_NOT_PD | (i << 8); break; }
    for (int col = 0; col < n; ++col) {
      memcpy(W + col * n, Vn + col * n, sizeof(double) * n);
      orc_chol_solve(n, L, W + col * n);
    }
    /* G_i = Bᵀ W B + R */
    mm(n, m, n, 0, W, 0, Bi, WB);
    mm(m, m, n, 1, Bi, 0, WB, G);
    unpack_sym(m, R + (int64_t)i * sm, Rf);
    for (int jj = 0; jj < m * m; ++jj) G[jj] += Rf[jj];
    /* g_i = v_{i+1} + W (c_{i+1} − δ v_{i+1}) */
    for (int d = 0; d < n; ++d) e[d] = cn[d] - delta * vn[d];
    mv(n, n, 0, W, e, t);
    for (int d = 0; d < n; ++d) g[d] = vn[d] + t[d];
    /* H_i = Bᵀ W A + Mᵀ */
    mm(n, n, n, 0, W, 0, Ai, WA);
    mm(m, n, n, 1, Bi, 0, WA, H);
    for (int rr = 0; rr < m; ++rr)
      for (int cc = 0; cc < n; ++cc) H[rr + cc * m] += Mi[cc + rr * n];
    /* h_i = r + Bᵀ g */
    mv(n, m, 1, Bi, g, tm);
    for (int d = 0; d < m; ++d) h[d] = ri[d] + tm[d];
    /* K_i = −G⁻¹ H,  k_i = −G⁻¹ h */
    if (orc_chol(m, G, LG)) { st = ORC_G_NOT_PD | (i << 8); break; }
    for (int col = 0; col < n; ++col) {
      for (int d = 0; d < m; ++d) Ki[d + col * m] = H[d + col * m];
      orc_chol_solve(m, LG, Ki + col * m);
      for (int d = 0; d < m; ++d) Ki[d + col * m] = -Ki[d + col * m];
    }
    memcpy(ki, h, sizeof(double) * m);
    orc_chol_solve(m, LG, ki);
    for (int d = 0; d < m; ++d) ki[d] = -ki[d];
    /* V_i = Aᵀ W A + Q + Kᵀ H, symmetrized (reading R10) */
    mm(n, n, n, 1, Ai, 0, WA, Vi);
    unpack_sym(n, Q + (int64_t)i * sn, Qf);
    mm(n, n, m, 1, Ki, 0, H, KtH);
    double* Vo = Vs + (int64_t)i * n * n;
    for (int cc = 0; cc < n; ++cc)
      for (int rr = 0; rr < n; ++rr) Vo[rr + cc * n] = Vi[rr + cc * n] + Qf[rr + cc * n] + KtH[rr + cc * n];
    for (int cc = 0; cc < n; ++cc)
      for (int rr = cc + 1; rr < n; ++rr) {
        double s = 0.5 * (Vo[rr + cc * n] + Vo[cc + rr * n]);
        Vo[rr + cc * n] = s;
        Vo[cc + rr * n] = s;
      }
    /* v_i = q + Aᵀ g + Kᵀ h */
    mv(n, n, 1, Ai, g, t);
    mv(m, n, 1, Ki, h, t2);
    double* vo = vs + (int64_t)i * n;
    for (int d = 0; d < n; ++d) vo[d] = qi[d] + t[d] + t2[d];
  }

  if (st == ORC_OK) {
    /* x_0 = (I + δV_0)⁻¹ (c_0 − δ v_0) */
    for (int jj = 0; jj < n * n; ++jj) S[jj] = delta * Vs[jj];
    for (int d = 0; d < n; ++d) S[d + d * n] += 1.0;
    if (orc_chol(n, S, L)) st = ORC_S_NOT_PD;
    else {
      for (int d = 0; d < n; ++d) x[d] = c0[d] - delta * vs[d];
      orc_chol_solve(n, L, x);
    }
  }
  for (int i = 0; i < N && st == ORC_OK; ++i) {
    const double* xi = x + (int64_t)i * n;
    double* ui = u + (int64_t)i * m;
    double* xn = x + (int64_t)(i + 1) * n;
    const double* Vn = Vs + (int64_t)(i + 1) * n * n;
    const double* vn = vs + (int64_t)(i + 1) * n;
    /* u_i = K_i x_i + k_i */
    mv(m, n, 0, Ks + (int64_t)i * m * n, xi, tm);
    for (int d = 0; d < m; ++d) ui[d] = tm[d] + ks[(int64_t)i * m + d];
    /* x_{i+1} = (I + δV_{i+1})⁻¹ (A x + B u + c_{i+1} − δ v_{i+1}) */
    mv(n, n, 0, A + (int64_t)i * n * n, xi, t);
    mv(n, m, 0, B + (int64_t)i * n * m, ui, t2);
    for (int d = 0; d < n; ++d) xn[d] = t[d] + t2[d] + c[(int64_t)i * n + d] - delta * vn[d];
    for (int jj = 0; jj < n * n; ++jj) S[jj] = delta * Vn[jj];
    for (int d = 0; d < n; ++d) S[d + d * n] += 1.0;
    if (orc_chol(n, S, L)) { st = ORC_S_NOT_PD | ((i + 1) << 8); break; }
    orc_chol_solve(n, L, xn);
  }
  if (st == ORC_OK) {
    /* y_i = V_i x_i + v_i */
    for (int i = 0; i <= N; ++i) {
      mv(n, n, 0, Vs + (int64_t)i * n * n, x + (int64_t)i * n, t);
      for (int d = 0; d < n; ++d) y[(int64_t)i * n + d] = t[d] + vs[(int64_t)i * n + d];
    }
    if (!all_finite(x, (N + 1) * n) || !all_finite(u, N * m) || !all_finite(y, (N + 1) * n))
      st = ORC_NONFINITE;
  }
  if (st != ORC_OK) {
    for (int64_t d = 0; d < (int64_t)(N + 1) * n; ++d) { x[d] = NAN; y[d] = NAN; }
    for (int64_t d = 0; d < (int64_t)N * m; ++d) u[d] = NAN;
  }
  if (a->V) for (int i = 0; i <= N; ++i) pack_sym(n, Vs + (int64_t)i * n * n, a->V + (b * (N + 1) + i) * sn);
  if (a->v) memcpy(a->v + b * (N + 1) * n, vs, sizeof(double) * (N + 1) * n);
  if (a->K) memcpy(a->K + b * N * m * n, Ks, sizeof(double) * N * m * n);
  if (a->k) memcpy(a->k + b * N * m, ks, sizeof(double) * N * m);

  free(Vs); free(vs); free(Ks); free(ks); free(S); free(L); free(W); free(WA); free(WB);
  free(G); free(LG); free(H); free(Vi); free(KtH); free(Rf); free(Qf); free(e); free(g);
  free(h); free(t); free(t2); free(tm);
  return st;
}

typedef struct {
  const orc_rr_args* a;
  int64_t begin, end;
} orc_range;

static void* rr_worker(void* p) {
  orc_range* rg = (orc_range*)p;
  for (int64_t b = rg->begin; b < rg->end; ++b) {
    int32_t st = rr_solve_one(rg->a, b);
    if (rg->a->status) rg->a->status[b] = st;
  }
  return NULL;
}

/* Batched oracle solve over `batch` instances with `nthreads` POSIX threads
 * (contiguous instance ranges; instances are independent).  Returns 0, or -1
 * on invalid arguments.  V, v, K, k may be NULL. */
int orc_rr_solve(int nx, int nu, int N, int64_t batch, int nthreads,
                 const double* A, const double* B, const double* Q, const double* M,
                 const double* R, const double* q, const double* r, const double* c,
                 const double* QN, const double* qN, const double* c0, const double* delta,
                 double* x, double* u, double* y, double* V, double* v, double* K, double* k,
                 int32_t* status) {
  if (nx < 1 || nu < 1 || N < 0 || batch < 0 || nthreads < 1) return -1;
  orc_rr_args a = {nx, nu, N, A, B, Q, M, R, q, r, c, QN, qN, c0, delta, x, u, y, V, v, K, k, status};
  if (nthreads > batch) nthreads = batch > 0 ? (int)batch : 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
  orc_range* rg = (orc_range*)malloc(sizeof(orc_range) * nthreads);
  for (int t = 0; t < nthreads; ++t) {
    rg[t].a = &a;
    rg[t].begin = batch * t / nthreads;
    rg[t].end = batch * (t + 1) / nthreads;
    pthread_create(&th[t], NULL, rr_worker, &rg[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th); free(rg);
  return 0;
}
