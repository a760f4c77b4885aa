// ipm_user.cu -- the line search of the regularized IPM step with CALLER-evaluated trial values
// (general user models through ipm_direction + ipm_merit + ipm_update).
//
// ipm_direction (ipm.cu in direction-only mode) gives the step (rows a1-a7) with α_max, α_d, D and
// 𝒜(0); the caller evaluates its own model at (x̄ + αΔx, ū + αΔu) and ipm_merit returns
//   𝒜(α) = f − μ Σ log(s + αΔs) + yᵀc + λᵀc_e + zᵀ(g + s + αΔs)
//          + η/2 (‖c‖² + ‖c_e‖² + ‖g + s + αΔs‖²)                      (reading R14)
// with c = (s_0 − x_0 − αΔx_0, d_i(trial) − x_{i+1}(trial)) and the iterate's multipliers; ipm_update
// applies the accepted steps (x, u, s, y, λ with α_p; z with α_d, reading R12).
// One warp per instance for the merit (lanes over stages, warp reductions), one thread per element
// for the update.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ipm.cuh"
#include "rr_common.cuh"

namespace rrk {

namespace {

__global__ void ipm_merit_kernel(ipm_dims d, ipm_stage_data data, ipm_iterate it, ipm_result r, const double* alpha,
                                 ipm_trial_values tv, double* merit) {
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= d.batch) return;
  const int n = d.nx, N = d.N, ng = d.ng, nc = d.nc;
  const int64_t sN = N;
  const double al = alpha[b], mu = it.mu[b], eta = it.eta[b];
  double lin = 0.0, pen = 0.0, bar = 0.0;
  bool ok = true;
  for (int i = lane; i <= N; i += 32) {
    const bool term = (i == N);
    const int ngi = term ? d.ngN : ng, nci = term ? d.ncN : nc;
    const double* s = term ? it.sN + b * d.ngN : it.s + (b * sN + i) * ng;
    const double* ds = term ? r.dsN + b * d.ngN : r.ds + (b * sN + i) * ng;
    const double* z = term ? it.zN + b * d.ngN : it.z + (b * sN + i) * ng;
    const double* g = term ? tv.gvN + b * d.ngN : tv.gv + (b * sN + i) * ng;
    for (int e = 0; e < ngi; ++e) {
      const double sa = fma(al, ds[e], s[e]);
      ok &= sa > 0.0;
      bar += log(sa);
      const double ga = g[e] + sa;
      lin = fma(z[e], ga, lin);
      pen = fma(ga, ga, pen);
    }
    const double* lam = term ? it.lamN + b * d.ncN : it.lam + (b * sN + i) * nc;
    const double* ce = term ? tv.ceN + b * d.ncN : tv.ce + (b * sN + i) * nc;
    for (int e = 0; e < nci; ++e) {
      lin = fma(lam[e], ce[e], lin);
      pen = fma(ce[e], ce[e], pen);
    }
    if (!term) {  // dynamics row i+1: c = d_i(trial) − x_{i+1}(trial), multiplier y_{i+1}
      const double* y1 = it.y + (b * (sN + 1) + i + 1) * n;
      const double* c = tv.dres + (b * sN + i) * n;
      for (int e = 0; e < n; ++e) {
        lin = fma(y1[e], c[e], lin);
        pen = fma(c[e], c[e], pen);
      }
    }
    if (i == 0) {  // initial-state row: c_0 = s_0 − x_0(trial)
      for (int e = 0; e < n; ++e) {
        const double c0 = data.s0[b * n + e] - fma(al, r.dx[b * (sN + 1) * n + e], it.x[b * (sN + 1) * n + e]);
        lin = fma(it.y[b * (sN + 1) * n + e], c0, lin);
        pen = fma(c0, c0, pen);
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    lin += __shfl_xor_sync(RR_FULL_MASK, lin, off);
    pen += __shfl_xor_sync(RR_FULL_MASK, pen, off);
    bar += __shfl_xor_sync(RR_FULL_MASK, bar, off);
  }
  ok = __all_sync(RR_FULL_MASK, ok);
  if (lane == 0)
    merit[b] = ok ? tv.fval[b] - mu * bar + lin + 0.5 * eta * pen : __longlong_as_double(0x7ff8000000000000LL);
}

__global__ void ipm_axpy_kernel(double* x, const double* dx, const double* alpha, int64_t per, int64_t batch) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= per * batch) return;
  const double al = alpha[t / per];
  if (al != 0.0) x[t] = fma(al, dx[t], x[t]);
}

}  // namespace

cudaError_t ipm_merit_launch(const ipm_dims& d, const ipm_stage_data& data, const ipm_iterate& it, const ipm_result& r,
                             const double* alpha, const ipm_trial_values& tv, double* merit, cudaStream_t s) {
  ipm_merit_kernel<<<(unsigned)((d.batch * 32 + 127) / 128), 128, 0, s>>>(d, data, it, r, alpha, tv, merit);
  return cudaGetLastError();
}

cudaError_t ipm_update_launch(const ipm_dims& d, const ipm_iterate& it, const ipm_result& r, const double* alpha_p,
                              const double* alpha_d, cudaStream_t s) {
  const int64_t b = d.batch, N = d.N;
  struct V { double* x; const double* dx; const double* al; int64_t per; } vs[] = {
      {it.x, r.dx, alpha_p, (N + 1) * d.nx}, {it.y, r.dy, alpha_p, (N + 1) * d.nx}, {it.u, r.du, alpha_p, N * d.nu},
      {it.s, r.ds, alpha_p, N * d.ng},       {it.sN, r.dsN, alpha_p, d.ngN},        {it.lam, r.dlam, alpha_p, N * d.nc},
      {it.lamN, r.dlamN, alpha_p, d.ncN},    {it.z, r.dz, alpha_d, N * d.ng},       {it.zN, r.dzN, alpha_d, d.ngN}};
  for (const V& v : vs) {
    if (v.per == 0 || v.x == nullptr) continue;
    ipm_axpy_kernel<<<(unsigned)((v.per * b + 255) / 256), 256, 0, s>>>(v.x, v.dx, v.al, v.per, b);
  }
  return cudaGetLastError();
}

}  // namespace rrk
