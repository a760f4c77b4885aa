// ipm_solve.cu -- device-resident batched regularized-IPM solve: repeated ipm_step
// (rows a1-a8) with per-instance μ / η updates, convergence masks and a report.
//
// Method: the regularized interior point method of §1.2; the step is ipm.cu.  The outer
// loop (when μ and η change, when to stop) is paper-silent ("can be used"); it follows
// SPEC's ipm_solve / update_parameters, reading R21:
//   iteration k, every running instance:
//     eval      problem data at the iterate: cost quadratic with Hessian P and constraints linear
//               (exact from the reference data at the initial iterate, reading R19); dynamics
//               linear (LQ), the cart-pole or the quadrotor model with analytic Jacobians
//     residuals r_stat = ||∇ₓL||∞, r_feas = max(||c||∞, ||c_e||∞, ||g+s||∞), r_comp = ||Sz − μ||∞,
//               r_comp0 = ||Sz||∞
//     stop      converged if max(r_stat, r_feas, r_comp0) <= tol and μ <= 10 μ_min; MAXITER at k = max
//     μ         if max(r_stat, r_feas, r_comp) <= κ μ:  μ <- max(μ_min, min(κ_μ μ, μ^θ_μ))
//     η         if k >= 5, r_feas > tol and r_feas > 0.9 r_feas(k−5):  η <- min(η_max, κ_η η)
//     step      one ipm_step over the device-built list of running instances (no host sync)
// B200 organisation: one thread per (instance, stage) for the evaluation, one warp per instance for
// the residual reductions and decisions (which also appends the instance to the active list with
// an atomic), and the ipm_step kernel launched over the list (CTAs past the count exit at once), so
// converged instances cost nothing.  All state lives in the caller's workspace.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "ipm.cuh"
#include "ipm_solve.cuh"
#include "rr_common.cuh"

namespace rrk {

namespace {

constexpr int WMAX = 16;  // n + m of every compiled ipm_step shape

struct SolveWs {  // views into the workspace (layout computed on the host)
  double *x_ref, *u_ref;
  double *fval, *fpart, *gradf, *gradfN, *dres, *gv, *gvN, *ce, *ceN, *A, *B;
  double *mu, *eta, *hist;
  double *dx, *du, *ds, *dsN, *dy, *dlam, *dlamN, *dz, *dzN, *alpha_p, *alpha_d, *D, *merit0, *merit_acc;
  int32_t *nbt, *stepst, *state, *iters, *list, *count;
  double* step_ws;
  int64_t step_ws_bytes;
};

struct Layout {
  int64_t bytes = 0;
  int64_t step_ws = 0;
  template <typename T>
  int64_t take(int64_t count) {  // 256-byte aligned sub-buffers
    const int64_t off = bytes;
    bytes += ((count * (int64_t)sizeof(T) + 255) / 256) * 256;
    return off;
  }
};

// Build (or size, when base == nullptr) the workspace views.
int64_t carve(const ipm_dims& d, char* base, SolveWs* w) {
  const int64_t b = d.batch, N = d.N, n = d.nx, m = d.nu, wd = n + m;
  Layout L;
  auto D = [&](double** p, int64_t cnt) {
    const int64_t off = L.take<double>(cnt);
    if (base) *p = reinterpret_cast<double*>(base + off);
  };
  auto I = [&](int32_t** p, int64_t cnt) {
    const int64_t off = L.take<int32_t>(cnt);
    if (base) *p = reinterpret_cast<int32_t*>(base + off);
  };
  SolveWs t{};
  SolveWs* v = base ? w : &t;
  D(&v->x_ref, b * (N + 1) * n);
  D(&v->u_ref, b * N * m);
  D(&v->fval, b);
  D(&v->fpart, b * (N + 1));
  D(&v->gradf, b * N * wd);
  D(&v->gradfN, b * n);
  D(&v->dres, b * N * n);
  D(&v->gv, b * N * d.ng);
  D(&v->gvN, b * d.ngN);
  D(&v->ce, b * N * d.nc);
  D(&v->ceN, b * d.ncN);
  const bool nl = d.model != IPM_MODEL_LQ;  // nonlinear model: Jacobians re-evaluated at every iterate
  D(&v->A, nl ? b * N * n * n : 0);
  D(&v->B, nl ? b * N * n * m : 0);
  D(&v->mu, b);
  D(&v->eta, b);
  D(&v->hist, b * 5);
  D(&v->dx, b * (N + 1) * n);
  D(&v->du, b * N * m);
  D(&v->ds, b * N * d.ng);
  D(&v->dsN, b * d.ngN);
  D(&v->dy, b * (N + 1) * n);
  D(&v->dlam, b * N * d.nc);
  D(&v->dlamN, b * d.ncN);
  D(&v->dz, b * N * d.ng);
  D(&v->dzN, b * d.ngN);
  D(&v->alpha_p, b);
  D(&v->alpha_d, b);
  D(&v->D, b);
  D(&v->merit0, b);
  D(&v->merit_acc, b);
  I(&v->nbt, b);
  I(&v->stepst, b);
  I(&v->state, b);
  I(&v->iters, b);
  I(&v->list, b);
  I(&v->count, 1);
  const int64_t sw = ipm_ws_bytes(d);
  if (sw < 0) return -1;
  const int64_t off = L.take<char>(sw);
  if (base) {
    v->step_ws = reinterpret_cast<double*>(base + off);
    v->step_ws_bytes = sw;
  }
  return L.bytes + 256;
}

__device__ __forceinline__ int pk(int n, int r, int c) { return r >= c ? pidx(n, r, c) : pidx(n, c, r); }

// ---- initialisation: reference iterate, μ / η, state ----
__global__ void solve_init_kernel(ipm_dims d, ipm_iterate it, SolveWs w) {
  const int64_t b = d.batch, N = d.N, n = d.nx, m = d.nu;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = tid; e < b * (N + 1) * n; e += nt) w.x_ref[e] = it.x[e];
  for (int64_t e = tid; e < b * N * m; e += nt) w.u_ref[e] = it.u[e];
  for (int64_t e = tid; e < b; e += nt) {
    w.mu[e] = it.mu[e];
    w.eta[e] = it.eta[e];
    w.state[e] = -1;
    w.iters[e] = 0;
    w.stepst[e] = 0;
  }
  for (int64_t e = tid; e < b * 5; e += nt) w.hist[e] = 0.0;
}

// ---- cart-pole explicit-Euler step and its Jacobians (model of DESIGN.md §4 / reading R19) ----
// x = (p, θ, ṗ, θ̇), θ from the hanging position (φ = θ − π from upright in the classic equations).
__device__ void cartpole_eval(const double* prm, const double* x, double F, double* xn, double* A, double* Bv) {
  const double dt = prm[0], mc = prm[1], mp = prm[2], l = prm[3], g = prm[4];
  const double phi = x[1] - M_PI;
  double sp, cp;
  sincos(phi, &sp, &cp);
  const double thd = x[3], mt = mc + mp;
  const double tmp = (F + mp * l * thd * thd * sp) / mt;
  const double den = l * (4.0 / 3.0 - mp * cp * cp / mt);
  const double num = g * sp - cp * tmp;
  const double thdd = num / den;
  const double pdd = tmp - mp * l * thdd * cp / mt;
  xn[0] = x[0] + dt * x[2];
  xn[1] = x[1] + dt * x[3];
  xn[2] = x[2] + dt * pdd;
  xn[3] = x[3] + dt * thdd;
  // derivatives with respect to θ (= φ), θ̇ and F
  const double tmp_p = mp * l * thd * thd * cp / mt, tmp_w = 2.0 * mp * l * thd * sp / mt, tmp_F = 1.0 / mt;
  const double den_p = 2.0 * l * mp * cp * sp / mt;
  const double num_p = g * cp + sp * tmp - cp * tmp_p, num_w = -cp * tmp_w, num_F = -cp * tmp_F;
  const double thdd_p = (num_p * den - num * den_p) / (den * den), thdd_w = num_w / den, thdd_F = num_F / den;
  const double k = mp * l / mt;
  const double pdd_p = tmp_p - k * (thdd_p * cp - thdd * sp), pdd_w = tmp_w - k * thdd_w * cp,
               pdd_F = tmp_F - k * thdd_F * cp;
  // A column-major 4×4 (I + dt ∂f/∂x), B 4×1
  for (int e = 0; e < 16; ++e) A[e] = (e % 5 == 0) ? 1.0 : 0.0;
  A[0 + 2 * 4] = dt;           // ∂p⁺/∂ṗ
  A[1 + 3 * 4] = dt;           // ∂θ⁺/∂θ̇
  A[2 + 1 * 4] = dt * pdd_p;   // ∂ṗ⁺/∂θ
  A[2 + 3 * 4] = dt * pdd_w;   // ∂ṗ⁺/∂θ̇
  A[3 + 1 * 4] = dt * thdd_p;  // ∂θ̇⁺/∂θ
  A[3 + 3 * 4] += dt * thdd_w; // ∂θ̇⁺/∂θ̇
  Bv[0] = 0.0;
  Bv[1] = 0.0;
  Bv[2] = dt * pdd_F;
  Bv[3] = dt * thdd_F;
}

// ---- quadrotor explicit-Euler step x⁺ = x + dt f(x, u) and its Jacobians (SURVEY §8(d) C5 model) ----
// x = (p, φ θ ψ ZYX Euler angles, world velocity v, body rates ω), u = (T, τ); prm [dt, mass, Jx, Jy, Jz, g].
// A = I + dt ∂f/∂x (column-major 12×12), B = dt ∂f/∂u (column-major 12×4), derivatives written out.
__device__ void quadrotor_eval(const double* prm, const double* x, const double* u, double* xn, double* A,
                               double* B) {
  const double dt = prm[0], mass = prm[1], Jx = prm[2], Jy = prm[3], Jz = prm[4], g = prm[5];
  double sph, cph, sth, cth, sps, cps;
  sincos(x[3], &sph, &cph);
  sincos(x[4], &sth, &cth);
  sincos(x[5], &sps, &cps);
  const double wx = x[9], wy = x[10], wz = x[11], T = u[0], Tm = T / mass;
  const double tth = sth / cth, ic = 1.0 / cth;
  const double a1 = sph * wy + cph * wz;  // W row terms
  const double a2 = cph * wy - sph * wz;
  const double r0 = cps * sth * cph + sps * sph, r1 = sps * sth * cph - cps * sph, r2 = cth * cph;  // R e₃
  double f[12];
  f[0] = x[6];
  f[1] = x[7];
  f[2] = x[8];
  f[3] = wx + tth * a1;
  f[4] = a2;
  f[5] = ic * a1;
  f[6] = r0 * Tm;
  f[7] = r1 * Tm;
  f[8] = r2 * Tm - g;
  f[9] = (u[1] - (Jz - Jy) * wy * wz) / Jx;
  f[10] = (u[2] - (Jx - Jz) * wz * wx) / Jy;
  f[11] = (u[3] - (Jy - Jx) * wx * wy) / Jz;
  for (int r = 0; r < 12; ++r) xn[r] = x[r] + dt * f[r];
  for (int e = 0; e < 144; ++e) A[e] = (e % 13 == 0) ? 1.0 : 0.0;
  for (int e = 0; e < 48; ++e) B[e] = 0.0;
  auto a = [&](int r, int c, double v) { A[r + 12 * c] += dt * v; };
  for (int k = 0; k < 3; ++k) a(k, 6 + k, 1.0);  // ṗ = v
  // φ̇ = ωx + tanθ (sφ ωy + cφ ωz)
  a(3, 3, tth * a2);
  a(3, 4, ic * ic * a1);
  a(3, 9, 1.0);
  a(3, 10, tth * sph);
  a(3, 11, tth * cph);
  // θ̇ = cφ ωy − sφ ωz
  a(4, 3, -a1);
  a(4, 10, cph);
  a(4, 11, -sph);
  // ψ̇ = (sφ ωy + cφ ωz) / cθ
  a(5, 3, ic * a2);
  a(5, 4, ic * tth * a1);
  a(5, 10, ic * sph);
  a(5, 11, ic * cph);
  // v̇ = R(φ, θ, ψ) e₃ T/m − g e₃
  a(6, 3, (-cps * sth * sph + sps * cph) * Tm);
  a(6, 4, cps * cth * cph * Tm);
  a(6, 5, (-sps * sth * cph + cps * sph) * Tm);
  a(7, 3, (-sps * sth * sph - cps * cph) * Tm);
  a(7, 4, sps * cth * cph * Tm);
  a(7, 5, r0 * Tm);
  a(8, 3, -cth * sph * Tm);
  a(8, 4, -sth * cph * Tm);
  // ω̇ = J⁻¹(τ − ω × Jω)
  a(9, 10, -(Jz - Jy) * wz / Jx);
  a(9, 11, -(Jz - Jy) * wy / Jx);
  a(10, 9, -(Jx - Jz) * wz / Jy);
  a(10, 11, -(Jx - Jz) * wx / Jy);
  a(11, 9, -(Jy - Jx) * wy / Jz);
  a(11, 10, -(Jy - Jx) * wx / Jz);
  B[6 + 12 * 0] = dt * r0 / mass;
  B[7 + 12 * 0] = dt * r1 / mass;
  B[8 + 12 * 0] = dt * r2 / mass;
  B[9 + 12 * 1] = dt / Jx;
  B[10 + 12 * 2] = dt / Jy;
  B[11 + 12 * 3] = dt / Jz;
}

// ---- evaluation: one thread per (instance, stage 0..N) of the running instances ----
__global__ void solve_eval_kernel(ipm_dims d, ipm_stage_data ref, ipm_iterate it, SolveWs w) {
  const int N = d.N, n = d.nx, m = d.nu, wd = n + m, ng = d.ng, nc = d.nc;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= d.batch * (int64_t)(N + 1)) return;
  const int64_t b = t / (N + 1);
  const int i = (int)(t % (N + 1));
  if (w.state[b] != -1) return;
  const int64_t sN = N;
  double dz[WMAX];
#pragma unroll
  for (int r = 0; r < WMAX; ++r) dz[r] = 0.0;
  const int wi = (i < N) ? wd : n;
  for (int r = 0; r < n; ++r) dz[r] = it.x[(b * (sN + 1) + i) * n + r] - w.x_ref[(b * (sN + 1) + i) * n + r];
  if (i < N)
    for (int r = 0; r < m; ++r) dz[n + r] = it.u[(b * sN + i) * m + r] - w.u_ref[(b * sN + i) * m + r];
  // gradient and f: ∇f = ∇f_ref + P Δ, f-part = ∇f_refᵀΔ + ½ ΔᵀPΔ
  const int sn = n * (n + 1) / 2, sm = m * (m + 1) / 2;
  const double* gref = (i < N) ? ref.gradf + (b * sN + i) * wd : ref.gradfN + b * n;
  double* gout = (i < N) ? w.gradf + (b * sN + i) * wd : w.gradfN + b * n;
  double fp = 0.0;
  for (int r = 0; r < wi; ++r) {
    double pr = 0.0;
    for (int c = 0; c < wi; ++c) {
      double P;
      if (i == N) P = ref.QN[b * sn + pk(n, r, c)];
      else if (r < n && c < n) P = ref.Q[(b * sN + i) * sn + pk(n, r, c)];
      else if (r < n) P = ref.M[(b * sN + i) * n * m + r + (c - n) * n];
      else if (c < n) P = ref.M[(b * sN + i) * n * m + c + (r - n) * n];
      else P = ref.R[(b * sN + i) * sm + pk(m, r - n, c - n)];
      pr = fma(P, dz[c], pr);
    }
    gout[r] = gref[r] + pr;
    fp += dz[r] * (gref[r] + 0.5 * pr);
  }
  w.fpart[b * (sN + 1) + i] = fp;
  // linear constraints: g = g_ref + G Δ, c_e = c_e,ref + C_e Δ
  const int ngi = (i < N) ? ng : d.ngN, nci = (i < N) ? nc : d.ncN;
  for (int k = 0; k < ngi; ++k) {
    const double* G = (i < N) ? ref.Gj + (b * sN + i) * ng * wd : ref.GjN + b * d.ngN * n;
    double v = (i < N) ? ref.gv[(b * sN + i) * ng + k] : ref.gvN[b * d.ngN + k];
    for (int r = 0; r < wi; ++r) v = fma(G[k + r * ngi], dz[r], v);
    if (i < N) w.gv[(b * sN + i) * ng + k] = v;
    else w.gvN[b * d.ngN + k] = v;
  }
  for (int k = 0; k < nci; ++k) {
    const double* C = (i < N) ? ref.Ce + (b * sN + i) * nc * wd : ref.CeN + b * d.ncN * n;
    double v = (i < N) ? ref.ce[(b * sN + i) * nc + k] : ref.ceN[b * d.ncN + k];
    for (int r = 0; r < wi; ++r) v = fma(C[k + r * nci], dz[r], v);
    if (i < N) w.ce[(b * sN + i) * nc + k] = v;
    else w.ceN[b * d.ncN + k] = v;
  }
  if (i == N) return;
  // dynamics residual d_i(x_i, u_i) − x_{i+1} (and Jacobians for the cart-pole)
  const double* xi = it.x + (b * (sN + 1) + i) * n;
  const double* x1 = it.x + (b * (sN + 1) + i + 1) * n;
  double* dr = w.dres + (b * sN + i) * n;
  if (d.model == IPM_MODEL_CARTPOLE) {
    double xn[4], A[16], Bv[4];
    cartpole_eval(ref.model_params, xi, it.u[b * sN + i], xn, A, Bv);
    for (int r = 0; r < 4; ++r) dr[r] = xn[r] - x1[r];
    for (int e = 0; e < 16; ++e) w.A[(b * sN + i) * 16 + e] = A[e];
    for (int e = 0; e < 4; ++e) w.B[(b * sN + i) * 4 + e] = Bv[e];
  } else if (d.model == IPM_MODEL_QUADROTOR) {
    double xn[12], A[144], Bq[48];
    quadrotor_eval(ref.model_params, xi, it.u + (b * sN + i) * 4, xn, A, Bq);
    for (int r = 0; r < 12; ++r) dr[r] = xn[r] - x1[r];
    for (int e = 0; e < 144; ++e) w.A[(b * sN + i) * 144 + e] = A[e];
    for (int e = 0; e < 48; ++e) w.B[(b * sN + i) * 48 + e] = Bq[e];
  } else {
    const double* A = ref.A + (b * sN + i) * n * n;
    const double* B = ref.B + (b * sN + i) * n * m;
    const double* dx1r = w.x_ref + (b * (sN + 1) + i + 1) * n;
    for (int r = 0; r < n; ++r) {
      double v = ref.dres[(b * sN + i) * n + r] - (x1[r] - dx1r[r]);
      for (int c = 0; c < n; ++c) v = fma(A[r + c * n], dz[c], v);
      for (int c = 0; c < m; ++c) v = fma(B[r + c * n], dz[n + c], v);
      dr[r] = v;
    }
  }
}

// ---- residuals, decisions, active list: one warp per instance ----
__global__ void solve_kkt_kernel(ipm_dims d, ipm_stage_data ref, ipm_iterate it, SolveWs w, ipm_solve_settings S,
                                 ipm_solve_report rep, int k) {
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= d.batch) return;
  if (w.state[b] != -1) return;  // warp-uniform
  if (k > 0 && w.stepst[b] != 0) {  // the previous step failed: the instance ends with its status
    if (lane == 0) w.state[b] = w.stepst[b];
    return;
  }
  const int N = d.N, n = d.nx, m = d.nu, wd = n + m, ng = d.ng, nc = d.nc;
  const int64_t sN = N;
  const double mu = w.mu[b];
  const double* A = (d.model != IPM_MODEL_LQ) ? w.A : ref.A;
  const double* B = (d.model != IPM_MODEL_LQ) ? w.B : ref.B;
  double rs = 0.0, rf = 0.0, rc = 0.0, rc0 = 0.0, fsum = 0.0;
  bool bad = false;
  auto mx = [&](double& acc, double v) {
    bad |= !isfinite(v);
    acc = fmax(acc, fabs(v));
  };
  for (int i = lane; i <= N; i += 32) {
    fsum += w.fpart[b * (sN + 1) + i];
    const double* y0 = it.y + (b * (sN + 1) + i) * n;
    const int ngi = (i < N) ? ng : d.ngN, nci = (i < N) ? nc : d.ncN, wi = (i < N) ? wd : n;
    const double* G = (i < N) ? ref.Gj + (b * sN + i) * ng * wd : ref.GjN + b * d.ngN * n;
    const double* C = (i < N) ? ref.Ce + (b * sN + i) * nc * wd : ref.CeN + b * d.ncN * n;
    const double* z = (i < N) ? it.z + (b * sN + i) * ng : it.zN + b * d.ngN;
    const double* s = (i < N) ? it.s + (b * sN + i) * ng : it.sN + b * d.ngN;
    const double* lam = (i < N) ? it.lam + (b * sN + i) * nc : it.lamN + b * d.ncN;
    const double* gf = (i < N) ? w.gradf + (b * sN + i) * wd : w.gradfN + b * n;
    for (int r = 0; r < wi; ++r) {  // ∇ₓL row r of stage i: ∇f + Cᵀy + C_eᵀλ + Gᵀz
      double g = gf[r];
      if (r < n) g -= y0[r];
      if (i < N) {
        const double* y1 = y0 + n;
        if (r < n)
          for (int c = 0; c < n; ++c) g = fma(A[(b * sN + i) * n * n + c + r * n], y1[c], g);
        else
          for (int c = 0; c < n; ++c) g = fma(B[(b * sN + i) * n * m + c + (r - n) * n], y1[c], g);
      }
      for (int q = 0; q < ngi; ++q) g = fma(G[q + r * ngi], z[q], g);
      for (int q = 0; q < nci; ++q) g = fma(C[q + r * nci], lam[q], g);
      mx(rs, g);
    }
    for (int q = 0; q < ngi; ++q) {
      const double gvv = (i < N) ? w.gv[(b * sN + i) * ng + q] : w.gvN[b * d.ngN + q];
      mx(rf, gvv + s[q]);
      const double sz = s[q] * z[q];
      mx(rc, sz - mu);
      mx(rc0, sz);
    }
    for (int q = 0; q < nci; ++q) mx(rf, (i < N) ? w.ce[(b * sN + i) * nc + q] : w.ceN[b * d.ncN + q]);
    if (i < N)
      for (int r = 0; r < n; ++r) mx(rf, w.dres[(b * sN + i) * n + r]);
    if (i == 0)
      for (int r = 0; r < n; ++r) mx(rf, ref.s0[b * n + r] - it.x[b * (sN + 1) * n + r]);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    rs = fmax(rs, __shfl_xor_sync(RR_FULL_MASK, rs, off));
    rf = fmax(rf, __shfl_xor_sync(RR_FULL_MASK, rf, off));
    rc = fmax(rc, __shfl_xor_sync(RR_FULL_MASK, rc, off));
    rc0 = fmax(rc0, __shfl_xor_sync(RR_FULL_MASK, rc0, off));
    fsum += __shfl_xor_sync(RR_FULL_MASK, fsum, off);
  }
  bad = __any_sync(RR_FULL_MASK, bad);
  if (lane != 0) return;
  w.fval[b] = ref.fval[b] + fsum;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  if (rep.r_stat) rep.r_stat[b] = bad ? nan : rs;
  if (rep.r_feas) rep.r_feas[b] = bad ? nan : rf;
  if (rep.r_comp) rep.r_comp[b] = bad ? nan : rc0;
  if (bad) {
    w.state[b] = RR_ST_NONFINITE;
    return;
  }
  if (fmax(fmax(rs, rf), rc0) <= S.tol_kkt && mu <= 10.0 * S.mu_min) {
    w.state[b] = 0;
    return;
  }
  if (k == S.max_iters) {
    w.state[b] = RR_ST_MAXITER;
    return;
  }
  if (fmax(fmax(rs, rf), rc) <= S.kappa * mu) w.mu[b] = fmax(S.mu_min, fmin(S.kappa_mu * mu, pow(mu, S.theta_mu)));
  double* h = w.hist + b * 5 + (k % 5);
  if (k >= 5 && rf > S.tol_kkt && rf > 0.9 * *h) w.eta[b] = fmin(S.eta_max, S.kappa_eta * w.eta[b]);
  *h = rf;
  w.iters[b] += 1;
  w.list[atomicAdd(w.count, 1)] = (int32_t)b;
}

__global__ void solve_report_kernel(ipm_dims d, SolveWs w, ipm_solve_report rep) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= d.batch) return;
  if (rep.status) rep.status[b] = w.state[b];
  if (rep.iters) rep.iters[b] = w.iters[b];
  if (rep.mu) rep.mu[b] = w.mu[b];
  if (rep.eta) rep.eta[b] = w.eta[b];
}

}  // namespace

int64_t ipm_solve_ws_bytes(const ipm_dims& d) {
  if (!ipm_supported(d)) return -1;
  return carve(d, nullptr, nullptr);
}

cudaError_t ipm_solve_launch(const ipm_dims& d, const ipm_stage_data& data, const ipm_iterate& it,
                             const ipm_solve_settings& S, const ipm_solve_report& rep, void* workspace,
                             cudaStream_t s, bool* supported) {
  *supported = ipm_supported(d);
  if (!*supported) return cudaSuccess;
  SolveWs w{};
  carve(d, static_cast<char*>(workspace), &w);
  const int64_t b = d.batch;
  solve_init_kernel<<<(unsigned)std::min<int64_t>((b * (d.N + 1) * d.nx + 255) / 256 + 1, 148 * 16), 256, 0, s>>>(d, it, w);
  // the data ipm_step sees: constants from the reference, the rest from the evaluation
  ipm_stage_data cur = data;
  cur.fval = w.fval;
  cur.gradf = w.gradf;
  cur.gradfN = w.gradfN;
  cur.dres = w.dres;
  cur.gv = d.ng ? w.gv : nullptr;
  cur.gvN = d.ngN ? w.gvN : nullptr;
  cur.ce = d.nc ? w.ce : nullptr;
  cur.ceN = d.ncN ? w.ceN : nullptr;
  if (d.model != IPM_MODEL_LQ) {
    cur.A = w.A;
    cur.B = w.B;
  }
  ipm_iterate cit = it;
  cit.mu = w.mu;
  cit.eta = w.eta;
  IpmArgs a;
  a.d = d;
  if (S.linear_merit) a.d.model = IPM_MODEL_LQ;  // trial merits on the linearisation (reading R22)
  a.d_ = cur;
  a.it = cit;
  a.prm = S.step;
  a.r = ipm_result{w.dx, w.du, d.ng ? w.ds : nullptr, d.ngN ? w.dsN : nullptr, w.dy, d.nc ? w.dlam : nullptr,
                   d.ncN ? w.dlamN : nullptr, d.ng ? w.dz : nullptr, d.ngN ? w.dzN : nullptr, w.alpha_p, w.alpha_d,
                   w.D, w.merit0, w.merit_acc, w.nbt};
  a.ws = w.step_ws;
  a.status = w.stepst;
  a.list = w.list;
  a.count = w.count;
  const int64_t ev_threads = b * (int64_t)(d.N + 1);
  for (int k = 0; k <= S.max_iters; ++k) {
    cudaError_t e = cudaMemsetAsync(w.count, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
    solve_eval_kernel<<<(unsigned)((ev_threads + 127) / 128), 128, 0, s>>>(d, data, it, w);
    solve_kkt_kernel<<<(unsigned)((b * 32 + 127) / 128), 128, 0, s>>>(d, data, it, w, S, rep, k);
    if (k < S.max_iters) {
      bool sup = false;
      e = ipm_launch(a, s, &sup);
      if (e != cudaSuccess) return e;
    }
  }
  solve_report_kernel<<<(unsigned)((b + 127) / 128), 128, 0, s>>>(d, w, rep);
  return cudaGetLastError();
}

}  // namespace rrk
