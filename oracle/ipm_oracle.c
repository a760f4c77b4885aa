/*
 * oracle/ipm_oracle.c -- CPU ORACLE of one regularized-IPM step, TEST INFRASTRUCTURE ONLY.
 * (Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it; it shares
 *  no code with the CUDA path.)
 *
 * One step of the regularized interior point method of §1.2 on the stagewise problem of §1.1,
 * in the paper's order (P:n = PAPER.md line n):
 *   condense (§1.3): Σ = (W + I/η)⁻¹ with W = Z⁻¹S, r_z = g + μ Z⁻¹e
 *     (Eq.(3×3) rhs); P̃ = P + GᵀΣG + η C_eᵀC_e; s̃ = ∇ₓL + GᵀΣ r_z + η C_eᵀ c_e;
 *     δ = 1/η
 *   regularized LQR (T2, rr_oracle.c) → Δx, Δu and Δy (the LQR y; reading R8)
 *   expand: Δz = Σ(GΔx + r_z), Δλ = η(C_eΔx + c_e),
 *           Δs = −Z⁻¹SΔz + μZ⁻¹e − s
 *   merit 𝒜, D = ∇ₓ𝒜·Δx + ∇ₛ𝒜·Δs (Theorem; also the closed form)
 *   line search over (x, s) with 𝒜 (mechanics = reading R12: fraction-to-boundary
 *   τ, Armijo c₁, backtracking β, ≤ max_backtracks; z uses α_d, y and λ use α_p)
 * Built-in models for the trial points (reading R19): 0 = LQ (linear d, g, c_e; cost quadratic
 * with Hessian P, so every trial value is exact), 1 = cart-pole (explicit-Euler cart-pole
 * dynamics evaluated at the trial point; costs quadratic; constraints linear), 2 = quadrotor
 * (explicit-Euler C5 quadrotor dynamics at the trial point; costs quadratic; constraints linear).
 */
#define _USE_MATH_DEFINES
#include <math.h>
#include <pthread.h>
#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "orc.h"

/* status codes and orc_ipm_args: orc.h */

static int64_t symn(int n) { return (int64_t)n * (n + 1) / 2; }
static int64_t pk(int n, int r, int c) {
  if (r < c) { int t = r; r = c; c = t; }
  return (int64_t)c * (2 * n - c - 1) / 2 + r;
}

/* cart-pole, explicit Euler (C4): state (p, θ, ṗ, θ̇), input F; θ measured from the
 * hanging position, φ = θ − π is the angle from upright used in the classic equations.
 * params: [dt, m_c, m_p, l (half length), g] */
static void cartpole_step(const double* prm, const double* x, const double* u, double* xn) {
  const double dt = prm[0], mc = prm[1], mp = prm[2], l = prm[3], g = prm[4];
  const double phi = x[1] - M_PI;
  const double sp = sin(phi), cp = cos(phi);
  const double th_d = x[3], F = u[0];
  const double mt = mc + mp;
  const double tmp = (F + mp * l * th_d * th_d * sp) / mt;
  const double thdd = (g * sp - cp * tmp) / (l * (4.0 / 3.0 - mp * cp * cp / mt));
  const double pdd = tmp - mp * l * thdd * cp / mt;
  xn[0] = x[0] + dt * x[2];
  xn[1] = x[1] + dt * x[3];
  xn[2] = x[2] + dt * pdd;
  xn[3] = x[3] + dt * thdd;
}

/* exported for tests (model pin against finite differences / the generator) */
void orc_cartpole_step(const double* prm, const double* x, const double* u, double* xn) {
  cartpole_step(prm, x, u, xn);
}

/* quadrotor, explicit Euler x+ = x + dt f(x, u) (SURVEY §8(d), C5 model).
 * state (p[3], ZYX Euler angles phi theta psi, world velocity v[3], body rates w[3]);
 * input (thrust T, torques tau[3]); params: [dt, mass, Jx, Jy, Jz, g].
 * f: p' = v;  (phi, theta, psi)' = W(phi, theta) w;  v' = R(phi, theta, psi) (0, 0, T/mass) - (0, 0, g)
 * with R = Rz(psi) Ry(theta) Rx(phi);  J w' = tau - w x (J w), J = diag(Jx, Jy, Jz). */
static void quadrotor_step(const double* prm, const double* x, const double* u, double* xn) {
  const double dt = prm[0], mass = prm[1], J[3] = {prm[2], prm[3], prm[4]}, g = prm[5];
  const double ph = x[3], th = x[4], ps = x[5];
  const double* v = x + 6;
  const double* w = x + 9;
  /* R = Rz(psi) Ry(theta) Rx(phi), written out as the product of the three elementary rotations */
  const double Rz[3][3] = {{cos(ps), -sin(ps), 0}, {sin(ps), cos(ps), 0}, {0, 0, 1}};
  const double Ry[3][3] = {{cos(th), 0, sin(th)}, {0, 1, 0}, {-sin(th), 0, cos(th)}};
  const double Rx[3][3] = {{1, 0, 0}, {0, cos(ph), -sin(ph)}, {0, sin(ph), cos(ph)}};
  double Ryx[3][3], R[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      Ryx[a][b] = 0.0;
      for (int k = 0; k < 3; ++k) Ryx[a][b] += Ry[a][k] * Rx[k][b];
    }
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      R[a][b] = 0.0;
      for (int k = 0; k < 3; ++k) R[a][b] += Rz[a][k] * Ryx[k][b];
    }
  /* Euler-angle rates: W = [[1, s_ph t_th, c_ph t_th], [0, c_ph, -s_ph], [0, s_ph / c_th, c_ph / c_th]] */
  const double W[3][3] = {{1.0, sin(ph) * tan(th), cos(ph) * tan(th)},
                          {0.0, cos(ph), -sin(ph)},
                          {0.0, sin(ph) / cos(th), cos(ph) / cos(th)}};
  double f[12];
  for (int a = 0; a < 3; ++a) f[a] = v[a];
  for (int a = 0; a < 3; ++a) f[3 + a] = W[a][0] * w[0] + W[a][1] * w[1] + W[a][2] * w[2];
  const double Tm = u[0] / mass;
  for (int a = 0; a < 3; ++a) f[6 + a] = R[a][2] * Tm - (a == 2 ? g : 0.0);
  /* w x (J w) */
  const double Jw[3] = {J[0] * w[0], J[1] * w[1], J[2] * w[2]};
  const double cr[3] = {w[1] * Jw[2] - w[2] * Jw[1], w[2] * Jw[0] - w[0] * Jw[2], w[0] * Jw[1] - w[1] * Jw[0]};
  for (int a = 0; a < 3; ++a) f[9 + a] = (u[1 + a] - cr[a]) / J[a];
  for (int a = 0; a < 12; ++a) xn[a] = x[a] + dt * f[a];
}

void orc_quadrotor_step(const double* prm, const double* x, const double* u, double* xn) {
  quadrotor_step(prm, x, u, xn);
}

/* y = Mat v, Mat rows×cols column-major */
static void matvec(int rows, int cols, const double* Mat, const double* v, double* y) {
  for (int r = 0; r < rows; ++r) {
    double s = 0.0;
    for (int c = 0; c < cols; ++c) s += Mat[r + (int64_t)c * rows] * v[c];
    y[r] = s;
  }
}
/* y = Matᵀ v */
static void matTvec(int rows, int cols, const double* Mat, const double* v, double* y) {
  for (int c = 0; c < cols; ++c) {
    double s = 0.0;
    for (int r = 0; r < rows; ++r) s += Mat[r + (int64_t)c * rows] * v[r];
    y[c] = s;
  }
}

/* per-instance views */
typedef struct {
  int n, m, N, ng, ngN, nc, ncN, nz;
  const double *s0, *gradf, *gradfN, *Q, *M, *R, *QN, *A, *B, *dres, *ce, *Ce, *ceN, *CeN, *gv, *Gj, *gvN, *GjN;
  double fval, mu, eta;
  double *x, *u, *s, *z, *sN, *zN, *y, *lam, *lamN;
  double *dx, *du, *ds, *dsN, *dy, *dlam, *dlamN, *dz, *dzN;
} inst_t;

static inst_t view(const orc_ipm_args* a, int64_t b) {
  inst_t I;
  const int n = a->nx, m = a->nu, N = a->N, nz = n + m;
  I.n = n; I.m = m; I.N = N; I.ng = a->ng; I.ngN = a->ngN; I.nc = a->nc; I.ncN = a->ncN; I.nz = nz;
  I.s0 = a->s0 + b * n;
  I.gradf = a->gradf + b * N * nz;
  I.gradfN = a->gradfN + b * n;
  I.Q = a->Q + b * N * symn(n); I.M = a->M + b * N * n * m; I.R = a->R + b * N * symn(m);
  I.QN = a->QN + b * symn(n);
  I.A = a->A + b * N * n * n; I.B = a->B + b * N * n * m; I.dres = a->dres + b * N * n;
  I.ce = a->ce ? a->ce + b * N * a->nc : NULL;
  I.Ce = a->Ce ? a->Ce + b * N * a->nc * nz : NULL;
  I.ceN = a->ceN ? a->ceN + b * a->ncN : NULL;
  I.CeN = a->CeN ? a->CeN + b * a->ncN * n : NULL;
  I.gv = a->gv ? a->gv + b * N * a->ng : NULL;
  I.Gj = a->Gj ? a->Gj + b * N * a->ng * nz : NULL;
  I.gvN = a->gvN ? a->gvN + b * a->ngN : NULL;
  I.GjN = a->GjN ? a->GjN + b * a->ngN * n : NULL;
  I.fval = a->fval[b]; I.mu = a->mu[b]; I.eta = a->eta[b];
  I.x = a->x + b * (N + 1) * n; I.u = a->u + b * N * m;
  I.s = a->s ? a->s + b * N * a->ng : NULL; I.z = a->z ? a->z + b * N * a->ng : NULL;
  I.sN = a->sN ? a->sN + b * a->ngN : NULL; I.zN = a->zN ? a->zN + b * a->ngN : NULL;
  I.y = a->y + b * (N + 1) * n;
  I.lam = a->lam ? a->lam + b * N * a->nc : NULL; I.lamN = a->lamN ? a->lamN + b * a->ncN : NULL;
  I.dx = a->dx + b * (N + 1) * n; I.du = a->du + b * N * m;
  I.ds = a->ds ? a->ds + b * N * a->ng : NULL; I.dsN = a->dsN ? a->dsN + b * a->ngN : NULL;
  I.dy = a->dy + b * (N + 1) * n;
  I.dlam = a->dlam ? a->dlam + b * N * a->nc : NULL; I.dlamN = a->dlamN ? a->dlamN + b * a->ncN : NULL;
  I.dz = a->dz ? a->dz + b * N * a->ng : NULL; I.dzN = a->dzN ? a->dzN + b * a->ngN : NULL;
  return I;
}

/* Stage "blocks" for stage i (i == N: terminal, x only): dimensions and pointers. */
typedef struct {
  int w;  /* width of the stage variable (n+m, or n at the terminal stage) */
  int ng, nc;
  const double *gv, *Gj, *ce, *Ce;
  double *s, *z, *lam, *ds, *dz, *dlam;
} stg_t;

static stg_t stage(const inst_t* I, int i) {
  stg_t S;
  if (i < I->N) {
    S.w = I->nz; S.ng = I->ng; S.nc = I->nc;
    S.gv = I->gv ? I->gv + (int64_t)i * I->ng : NULL;
    S.Gj = I->Gj ? I->Gj + (int64_t)i * I->ng * I->nz : NULL;
    S.ce = I->ce ? I->ce + (int64_t)i * I->nc : NULL;
    S.Ce = I->Ce ? I->Ce + (int64_t)i * I->nc * I->nz : NULL;
    S.s = I->s ? I->s + (int64_t)i * I->ng : NULL;
    S.z = I->z ? I->z + (int64_t)i * I->ng : NULL;
    S.lam = I->lam ? I->lam + (int64_t)i * I->nc : NULL;
    S.ds = I->ds ? I->ds + (int64_t)i * I->ng : NULL;
    S.dz = I->dz ? I->dz + (int64_t)i * I->ng : NULL;
    S.dlam = I->dlam ? I->dlam + (int64_t)i * I->nc : NULL;
  } else {
    S.w = I->n; S.ng = I->ngN; S.nc = I->ncN;
    S.gv = I->gvN; S.Gj = I->GjN; S.ce = I->ceN; S.Ce = I->CeN;
    S.s = I->sN; S.z = I->zN; S.lam = I->lamN; S.ds = I->dsN; S.dz = I->dzN; S.dlam = I->dlamN;
  }
  return S;
}

/* stage vector (x_i, u_i) of a trajectory */
static void stage_vec(const inst_t* I, const double* x, const double* u, int i, double* v) {
  memcpy(v, x + (int64_t)i * I->n, sizeof(double) * I->n);
  if (i < I->N) memcpy(v + I->n, u + (int64_t)i * I->m, sizeof(double) * I->m);
}

/* full stage Hessian block P_i (w×w, column-major) */
static void stage_P(const inst_t* I, int i, double* P) {
  const int n = I->n, m = I->m;
  if (i < I->N) {
    const int w = n + m;
    const double* Q = I->Q + (int64_t)i * symn(n);
    const double* M = I->M + (int64_t)i * n * m;
    const double* R = I->R + (int64_t)i * symn(m);
    for (int c = 0; c < w; ++c)
      for (int r = 0; r < w; ++r) {
        double v;
        if (r < n && c < n) v = Q[pk(n, r, c)];
        else if (r < n) v = M[r + (c - n) * n];
        else if (c < n) v = M[c + (r - n) * n];
        else v = R[pk(m, r - n, c - n)];
        P[r + c * w] = v;
      }
  } else {
    for (int c = 0; c < n; ++c)
      for (int r = 0; r < n; ++r) P[r + c * n] = I->QN[pk(n, r, c)];
  }
}

/* Augmented Barrier-Lagrangian 𝒜(x̄ + αΔx, s + αΔs; y, λ, z, μ, η) (reading R14: all
 * equality constraints -- initial state, dynamics, stage equalities -- are penalised).
 * Returns NAN if a slack is not positive. */
static double merit(const inst_t* I, const double* prm, int model, double alpha) {
  const int n = I->n, m = I->m, N = I->N;
  const double mu = I->mu, eta = I->eta;
  double* v = (double*)malloc(sizeof(double) * I->nz);
  double* dv = (double*)malloc(sizeof(double) * I->nz);
  double* Pv = (double*)malloc(sizeof(double) * I->nz * I->nz);
  double* t = (double*)malloc(sizeof(double) * (I->nz + 64));
  double f = I->fval, bar = 0.0, lin = 0.0, pen = 0.0;
  int ok = 1;
  for (int i = 0; i <= N; ++i) {
    stg_t S = stage(I, i);
    const double* gf = (i < N) ? I->gradf + (int64_t)i * I->nz : I->gradfN;
    stage_vec(I, I->dx, I->du, i, dv);
    stage_P(I, i, Pv);
    /* f(x̄ + αΔ) = f̄ + α ∇fᵀΔ + ½ α² ΔᵀPΔ (exact for the quadratic costs of the built-in models) */
    double gd = 0.0, dPd = 0.0;
    for (int r = 0; r < S.w; ++r) gd += gf[r] * dv[r];
    matvec(S.w, S.w, Pv, dv, t);
    for (int r = 0; r < S.w; ++r) dPd += dv[r] * t[r];
    f += alpha * gd + 0.5 * alpha * alpha * dPd;
    /* inequalities g(α) + s(α) (g linear) and the barrier */
    for (int e = 0; e < S.ng; ++e) {
      double gd_e = 0.0;
      for (int c = 0; c < S.w; ++c) gd_e += S.Gj[e + (int64_t)c * S.ng] * dv[c];
      const double sa = S.s[e] + alpha * S.ds[e];
      if (!(sa > 0.0)) ok = 0;
      const double ga = S.gv[e] + alpha * gd_e + sa;
      bar += log(sa);
      lin += S.z[e] * ga;
      pen += ga * ga;
    }
    /* stage equalities c_e(α) (linear) */
    for (int e = 0; e < S.nc; ++e) {
      double cd = 0.0;
      for (int c = 0; c < S.w; ++c) cd += S.Ce[e + (int64_t)c * S.nc] * dv[c];
      const double ca = S.ce[e] + alpha * cd;
      lin += S.lam[e] * ca;
      pen += ca * ca;
    }
  }
  /* dynamics / initial-state constraints: c_0 = s_0 − x_0, c_{i+1} = d_i(x_i, u_i) − x_{i+1} */
  for (int r = 0; r < n; ++r) {
    const double c0 = I->s0[r] - (I->x[r] + alpha * I->dx[r]);
    lin += I->y[r] * c0;
    pen += c0 * c0;
  }
  double* xa = (double*)malloc(sizeof(double) * n);
  double* ua = (double*)malloc(sizeof(double) * m);
  double* xn = (double*)malloc(sizeof(double) * n);
  for (int i = 0; i < N; ++i) {
    const double* Ai = I->A + (int64_t)i * n * n;
    const double* Bi = I->B + (int64_t)i * n * m;
    if (model == 1 || model == 2) {
      for (int r = 0; r < n; ++r) xa[r] = I->x[(int64_t)i * n + r] + alpha * I->dx[(int64_t)i * n + r];
      for (int r = 0; r < m; ++r) ua[r] = I->u[(int64_t)i * m + r] + alpha * I->du[(int64_t)i * m + r];
      if (model == 1) cartpole_step(prm, xa, ua, xn);
      else quadrotor_step(prm, xa, ua, xn);
    } else {
      /* linear model: d(x̄+αΔx, ū+αΔu) − x̄_{i+1} = dres_i + α(AΔx + BΔu) */
      matvec(n, n, Ai, I->dx + (int64_t)i * n, xa);
      matvec(n, m, Bi, I->du + (int64_t)i * m, xn);
      for (int r = 0; r < n; ++r) xn[r] = I->x[(int64_t)(i + 1) * n + r] + I->dres[(int64_t)i * n + r] + alpha * (xa[r] + xn[r]);
    }
    for (int r = 0; r < n; ++r) {
      const double ca = xn[r] - (I->x[(int64_t)(i + 1) * n + r] + alpha * I->dx[(int64_t)(i + 1) * n + r]);
      lin += I->y[(int64_t)(i + 1) * n + r] * ca;
      pen += ca * ca;
    }
  }
  free(xa); free(ua); free(xn); free(v); free(dv); free(Pv); free(t);
  if (!ok) return NAN;
  return f - mu * bar + lin + 0.5 * eta * pen;
}

typedef struct { const orc_ipm_args* a; int64_t begin, end; } ipm_range;

static int32_t ipm_step_one(const orc_ipm_args* a, int64_t b) {
  inst_t I = view(a, b);
  const int n = I.n, m = I.m, N = I.N, nz = I.nz;
  const double mu = I.mu, eta = I.eta;
  /* positivity of s, z (needed by log s and Z⁻¹S) */
  for (int i = 0; i <= N; ++i) {
    stg_t S = stage(&I, i);
    for (int e = 0; e < S.ng; ++e)
      if (!(S.s[e] > 0.0) || !(S.z[e] > 0.0)) {
        /* iterate untouched; direction NaN; steps 0; merit and D NaN */
        for (int64_t k = 0; k < (int64_t)(N + 1) * n; ++k) { I.dx[k] = NAN; I.dy[k] = NAN; }
        for (int64_t k = 0; k < (int64_t)N * m; ++k) I.du[k] = NAN;
        for (int q = 0; q <= N; ++q) {
          stg_t T = stage(&I, q);
          for (int f = 0; f < T.ng; ++f) { T.ds[f] = NAN; T.dz[f] = NAN; }
          for (int f = 0; f < T.nc; ++f) T.dlam[f] = NAN;
        }
        if (a->alpha_p) a->alpha_p[b] = 0.0;
        if (a->alpha_d) a->alpha_d[b] = 0.0;
        if (a->D) a->D[b] = NAN;
        if (a->D_closed) a->D_closed[b] = NAN;
        if (a->merit0) a->merit0[b] = NAN;
        if (a->merit_acc) a->merit_acc[b] = NAN;
        if (a->n_backtracks) a->n_backtracks[b] = 0;
        return OIPM_NONPOS_SLACK | (i << 8);
      }
  }
  /* ---- condense into a regularized LQR problem ---- */
  const int64_t sn = symn(n), sm = symn(m);
  double* Qt = (double*)calloc(N * sn + 1, sizeof(double));
  double* Mt = (double*)calloc(N * n * m + 1, sizeof(double));
  double* Rt = (double*)calloc(N * sm + 1, sizeof(double));
  double* qt = (double*)calloc(N * n + 1, sizeof(double));
  double* rt = (double*)calloc(N * m + 1, sizeof(double));
  double* QNt = (double*)calloc(sn, sizeof(double));
  double* qNt = (double*)calloc(n, sizeof(double));
  double* c0 = (double*)calloc(n, sizeof(double));
  double* P = (double*)malloc(sizeof(double) * nz * nz);
  double* sg = (double*)malloc(sizeof(double) * nz);
  double* tmp = (double*)malloc(sizeof(double) * nz);
  int maxg = a->ng > a->ngN ? a->ng : a->ngN;
  double* Sig = (double*)malloc(sizeof(double) * (maxg + 1));
  double* rz = (double*)malloc(sizeof(double) * (maxg + 1));
  for (int i = 0; i <= N; ++i) {
    stg_t S = stage(&I, i);
    const int w = S.w;
    stage_P(&I, i, P);
    /* ∇ₓL: ∇f + Cᵀy + Gᵀz + C_eᵀλ; (Cᵀy) at x_i = −y_i + A_iᵀ y_{i+1}, at u_i = B_iᵀ y_{i+1} */
    const double* gf = (i < N) ? I.gradf + (int64_t)i * nz : I.gradfN;
    for (int r = 0; r < w; ++r) sg[r] = gf[r];
    for (int r = 0; r < n; ++r) sg[r] -= I.y[(int64_t)i * n + r];
    if (i < N) {
      matTvec(n, n, I.A + (int64_t)i * n * n, I.y + (int64_t)(i + 1) * n, tmp);
      for (int r = 0; r < n; ++r) sg[r] += tmp[r];
      matTvec(n, m, I.B + (int64_t)i * n * m, I.y + (int64_t)(i + 1) * n, tmp);
      for (int r = 0; r < m; ++r) sg[n + r] += tmp[r];
    }
    if (S.ng > 0) {
      matTvec(S.ng, w, S.Gj, S.z, tmp);
      for (int r = 0; r < w; ++r) sg[r] += tmp[r];
    }
    if (S.nc > 0) {
      matTvec(S.nc, w, S.Ce, S.lam, tmp);
      for (int r = 0; r < w; ++r) sg[r] += tmp[r];
    }
    /* inequality fold: Σ = (s/z + 1/η)⁻¹, r_z = g + μ/z; P += GᵀΣG, s̃ += GᵀΣ r_z */
    for (int e = 0; e < S.ng; ++e) {
      Sig[e] = 1.0 / (S.s[e] / S.z[e] + 1.0 / eta);
      rz[e] = S.gv[e] + mu / S.z[e];
    }
    for (int c = 0; c < w; ++c)
      for (int r = 0; r < w; ++r) {
        double acc = 0.0;
        for (int e = 0; e < S.ng; ++e) acc += S.Gj[e + (int64_t)r * S.ng] * Sig[e] * S.Gj[e + (int64_t)c * S.ng];
        for (int e = 0; e < S.nc; ++e) acc += eta * S.Ce[e + (int64_t)r * S.nc] * S.Ce[e + (int64_t)c * S.nc];
        P[r + c * w] += acc;
      }
    for (int r = 0; r < w; ++r) {
      double acc = 0.0;
      for (int e = 0; e < S.ng; ++e) acc += S.Gj[e + (int64_t)r * S.ng] * Sig[e] * rz[e];
      for (int e = 0; e < S.nc; ++e) acc += eta * S.Ce[e + (int64_t)r * S.nc] * S.ce[e];
      sg[r] += acc;
    }
    /* scatter into the LQR stage */
    if (i < N) {
      for (int c = 0; c < n; ++c)
        for (int r = c; r < n; ++r) Qt[i * sn + pk(n, r, c)] = P[r + c * w];
      for (int c = 0; c < m; ++c)
        for (int r = 0; r < n; ++r) Mt[(int64_t)i * n * m + r + c * n] = P[r + (n + c) * w];
      for (int c = 0; c < m; ++c)
        for (int r = c; r < m; ++r) Rt[i * sm + pk(m, r, c)] = P[(n + r) + (n + c) * w];
      for (int r = 0; r < n; ++r) qt[(int64_t)i * n + r] = sg[r];
      for (int r = 0; r < m; ++r) rt[(int64_t)i * m + r] = sg[n + r];
    } else {
      for (int c = 0; c < n; ++c)
        for (int r = c; r < n; ++r) QNt[pk(n, r, c)] = P[r + c * n];
      for (int r = 0; r < n; ++r) qNt[r] = sg[r];
    }
  }
  for (int r = 0; r < n; ++r) c0[r] = I.s0[r] - I.x[r];
  const double delta = 1.0 / eta;
  int32_t st = 0;
  orc_rr_solve(n, m, N, 1, 1, I.A, I.B, Qt, Mt, Rt, qt, rt, I.dres, QNt, qNt, c0, &delta, I.dx, I.du, I.dy,
               NULL, NULL, NULL, NULL, &st);
  /* ---- expand ---- */
  double amax = 1.0, admax = 1.0;
  for (int i = 0; i <= N && st == 0; ++i) {
    stg_t S = stage(&I, i);
    stage_vec(&I, I.dx, I.du, i, tmp);
    for (int e = 0; e < S.ng; ++e) {
      double gd = 0.0;
      for (int c = 0; c < S.w; ++c) gd += S.Gj[e + (int64_t)c * S.ng] * tmp[c];
      const double sig = 1.0 / (S.s[e] / S.z[e] + 1.0 / eta);
      S.dz[e] = sig * (gd + S.gv[e] + mu / S.z[e]);
      S.ds[e] = -(S.s[e] / S.z[e]) * S.dz[e] + mu / S.z[e] - S.s[e];
      if (S.ds[e] < 0.0) { double t = a->tau * S.s[e] / (-S.ds[e]); if (t < amax) amax = t; }
      if (S.dz[e] < 0.0) { double t = a->tau * S.z[e] / (-S.dz[e]); if (t < admax) admax = t; }
    }
    for (int e = 0; e < S.nc; ++e) {
      double cd = 0.0;
      for (int c = 0; c < S.w; ++c) cd += S.Ce[e + (int64_t)c * S.nc] * tmp[c];
      S.dlam[e] = eta * (cd + S.ce[e]);
    }
  }
  double D = NAN, Dc = NAN, A0 = NAN, Aacc = NAN, alpha = 0.0;
  int nb = 0;
  if (st == 0) {
    /* D = ∇ₓ𝒜·Δx + ∇ₛ𝒜·Δs with ∇ₓ𝒜 = ∇f + Cᵀ(y+ηc) + C_eᵀ(λ+ηc_e) + Gᵀ(z+η(g+s)),
     *     ∇ₛ𝒜 = −μ/s + z + η(g+s)   (Lemma rhs) */
    double Dsum = 0.0, quadP = 0.0, quadS = 0.0, pen = 0.0;
    for (int i = 0; i <= N; ++i) {
      stg_t S = stage(&I, i);
      const double* gf = (i < N) ? I.gradf + (int64_t)i * nz : I.gradfN;
      stage_vec(&I, I.dx, I.du, i, tmp);
      stage_P(&I, i, P);
      for (int r = 0; r < S.w; ++r) Dsum += gf[r] * tmp[r];
      matvec(S.w, S.w, P, tmp, sg);
      for (int r = 0; r < S.w; ++r) quadP += tmp[r] * sg[r];
      for (int e = 0; e < S.ng; ++e) {
        double gd = 0.0;
        for (int c = 0; c < S.w; ++c) gd += S.Gj[e + (int64_t)c * S.ng] * tmp[c];
        const double gs = S.gv[e] + S.s[e];
        Dsum += (S.z[e] + eta * gs) * (gd + S.ds[e]) + (-mu / S.s[e]) * S.ds[e];
        quadS += S.z[e] / S.s[e] * S.ds[e] * S.ds[e];
        pen += (gd + S.ds[e]) * (gd + S.ds[e]);
      }
      for (int e = 0; e < S.nc; ++e) {
        double cd = 0.0;
        for (int c = 0; c < S.w; ++c) cd += S.Ce[e + (int64_t)c * S.nc] * tmp[c];
        Dsum += (S.lam[e] + eta * S.ce[e]) * cd;
        pen += cd * cd;
      }
    }
    /* dynamics rows: (CΔ)_0 = −Δx_0; (CΔ)_{i+1} = A_iΔx_i + B_iΔu_i − Δx_{i+1} */
    for (int r = 0; r < n; ++r) {
      const double cd = -I.dx[r];
      Dsum += (I.y[r] + eta * (I.s0[r] - I.x[r])) * cd;
      pen += cd * cd;
    }
    double* ad = (double*)malloc(sizeof(double) * n);
    double* bd = (double*)malloc(sizeof(double) * n);
    for (int i = 0; i < N; ++i) {
      matvec(n, n, I.A + (int64_t)i * n * n, I.dx + (int64_t)i * n, ad);
      matvec(n, m, I.B + (int64_t)i * n * m, I.du + (int64_t)i * m, bd);
      for (int r = 0; r < n; ++r) {
        const double cd = ad[r] + bd[r] - I.dx[(int64_t)(i + 1) * n + r];
        Dsum += (I.y[(int64_t)(i + 1) * n + r] + eta * I.dres[(int64_t)i * n + r]) * cd;
        pen += cd * cd;
      }
    }
    free(ad); free(bd);
    D = Dsum;
    Dc = -quadP - quadS - eta * pen;   /* Theorem closed form */
    /* ---- line search over (x, s) with 𝒜 (reading R12) ---- */
    A0 = merit(&I, a->model_params, a->model, 0.0);
    alpha = amax;
    int accepted = 0;
    for (nb = 0; nb <= a->max_backtracks; ++nb) {
      const double At = merit(&I, a->model_params, a->model, alpha);
      if (At <= A0 + a->armijo_c * alpha * D) { Aacc = At; accepted = 1; break; }
      alpha *= a->beta;
    }
    if (!accepted) { st = OIPM_LS_FAILED; alpha = 0.0; nb = a->max_backtracks + 1; }
    else {
      /* update: x, u, s, y, λ with α_p; z with α_d (reading R12) */
      for (int64_t e = 0; e < (int64_t)(N + 1) * n; ++e) { I.x[e] += alpha * I.dx[e]; I.y[e] += alpha * I.dy[e]; }
      for (int64_t e = 0; e < (int64_t)N * m; ++e) I.u[e] += alpha * I.du[e];
      for (int i = 0; i <= N; ++i) {
        stg_t S = stage(&I, i);
        for (int e = 0; e < S.ng; ++e) { S.s[e] += alpha * S.ds[e]; S.z[e] += admax * S.dz[e]; }
        for (int e = 0; e < S.nc; ++e) S.lam[e] += alpha * S.dlam[e];
      }
    }
  }
  if (a->alpha_p) a->alpha_p[b] = alpha;
  if (a->alpha_d) a->alpha_d[b] = (st == 0) ? admax : 0.0;
  if (a->D) a->D[b] = D;
  if (a->D_closed) a->D_closed[b] = Dc;
  if (a->merit0) a->merit0[b] = A0;
  if (a->merit_acc) a->merit_acc[b] = Aacc;
  if (a->n_backtracks) a->n_backtracks[b] = nb;
  free(Qt); free(Mt); free(Rt); free(qt); free(rt); free(QNt); free(qNt); free(c0); free(P);
  free(sg); free(tmp); free(Sig); free(rz);
  return st;
}

static void* ipm_worker(void* p) {
  ipm_range* rg = (ipm_range*)p;
  for (int64_t b = rg->begin; b < rg->end; ++b) {
    int32_t st = ipm_step_one(rg->a, b);
    if (rg->a->status) rg->a->status[b] = st;
  }
  return NULL;
}

/* Batched oracle IPM step.  The iterate arrays are updated in place. */
int orc_ipm_step(const orc_ipm_args* a, int nthreads) {
  if (a->nx < 1 || a->nu < 1 || a->N < 0 || a->batch < 0 || nthreads < 1) return -1;
  if (nthreads > a->batch) nthreads = a->batch > 0 ? (int)a->batch : 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
  ipm_range* rg = (ipm_range*)malloc(sizeof(ipm_range) * nthreads);
  for (int t = 0; t < nthreads; ++t) {
    rg[t].a = a;
    rg[t].begin = a->batch * t / nthreads;
    rg[t].end = a->batch * (t + 1) / nthreads;
    pthread_create(&th[t], NULL, ipm_worker, &rg[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th); free(rg);
  return 0;
}

/* The merit 𝒜 at step length alpha for instance b (tests: finite-difference slope of the Theorem). */
double orc_ipm_merit(const orc_ipm_args* a, int64_t b, double alpha) {
  inst_t I = view(a, b);
  return merit(&I, a->model_params, a->model, alpha);
}
