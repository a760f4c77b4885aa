// ipm_model.cuh -- device pieces shared by the ipm_step kernels (ipm.cu, ipm_c4t.cu): the barrier
// log-sum accumulator and the built-in dynamics models of the merit's trial points (reading R19).
#pragma once
#include <cuda_runtime.h>
#include <math.h>

#include "rr.h"

namespace rrk {

// Σ log a_e accumulated as a running product m·2^k (frexp renormalisation after every factor, so no
// overflow/underflow for any positive normal factors), with a single log at the end: the barrier
// sums of 𝒜 cost one log per lane instead of one per slack.
struct LogAcc {
  double m = 1.0;
  int k = 0;
  __device__ __forceinline__ void add(double x) {
    int e;
    m = frexp(m * x, &e);
    k += e;
  }
  __device__ __forceinline__ double value() const { return log(m) + k * 0.69314718055994530942; }
};

// cart-pole, explicit Euler (C4); θ from the hanging position, φ = θ − π.
__device__ __forceinline__ void cartpole_step(const double* prm, const double* x, double u, double* xn) {
  const double dt = prm[0], mc = prm[1], mp = prm[2], l = prm[3], g = prm[4];
  const double phi = x[1] - 3.14159265358979323846;
  double sp, cp;
  sincos(phi, &sp, &cp);
  const double thd = x[3];
  const double imt = 1.0 / (mc + mp);  // one IEEE division per call instead of four
  const double tmp = (u + mp * l * thd * thd * sp) * imt;
  const double thdd = (g * sp - cp * tmp) / (l * (4.0 / 3.0 - mp * cp * cp * imt));
  const double pdd = tmp - mp * l * thdd * cp * imt;
  xn[0] = x[0] + dt * x[2];
  xn[1] = x[1] + dt * x[3];
  xn[2] = x[2] + dt * pdd;
  xn[3] = x[3] + dt * thdd;
}

// quadrotor, explicit Euler x⁺ = x + dt f(x, u) (SURVEY §8(d) C5 model): x = (p, ZYX Euler angles
// (φ, θ, ψ), world velocity v, body rates ω), u = (thrust T, torques τ); params [dt, mass, Jx, Jy, Jz, g].
// Euler-angle rates W(φ, θ)ω; acceleration R(φ, θ, ψ)[0, 0, T/m] − [0, 0, g] with R = Rz(ψ)Ry(θ)Rx(φ);
// Euler's equations J ω̇ = τ − ω × Jω for the diagonal inertia J.
__device__ __forceinline__ void quadrotor_step(const double* prm, const double* x, const double* u, double* xn) {
  const double dt = prm[0], mass = prm[1], Jx = prm[2], Jy = prm[3], Jz = prm[4], g = prm[5];
  double sph, cph, sth, cth, sps, cps;
  sincos(x[3], &sph, &cph);
  sincos(x[4], &sth, &cth);
  sincos(x[5], &sps, &cps);
  const double wx = x[9], wy = x[10], wz = x[11];
  const double tth = sth / cth;
  const double dphi = wx + sph * tth * wy + cph * tth * wz;
  const double dth = cph * wy - sph * wz;
  const double dpsi = (sph * wy + cph * wz) / cth;
  const double Tm = u[0] / mass;
  const double ax = (cps * sth * cph + sps * sph) * Tm;
  const double ay = (sps * sth * cph - cps * sph) * Tm;
  const double az = cth * cph * Tm - g;
  const double dwx = (u[1] - (Jz - Jy) * wy * wz) / Jx;
  const double dwy = (u[2] - (Jx - Jz) * wz * wx) / Jy;
  const double dwz = (u[3] - (Jy - Jx) * wx * wy) / Jz;
  xn[0] = x[0] + dt * x[6];
  xn[1] = x[1] + dt * x[7];
  xn[2] = x[2] + dt * x[8];
  xn[3] = x[3] + dt * dphi;
  xn[4] = x[4] + dt * dth;
  xn[5] = x[5] + dt * dpsi;
  xn[6] = x[6] + dt * ax;
  xn[7] = x[7] + dt * ay;
  xn[8] = x[8] + dt * az;
  xn[9] = wx + dt * dwx;
  xn[10] = wy + dt * dwy;
  xn[11] = wz + dt * dwz;
}

// x⁺ = d(x, u) of the built-in nonlinear models (their n, m are fixed; checked by ipm_supported)
template <int NX, int NU>
__device__ __forceinline__ void model_step(int model, const double* prm, const double* x, const double* u, double* xn) {
  if (model == IPM_MODEL_CARTPOLE) {
    cartpole_step(prm, x, u[0], xn);
    return;
  }
  if constexpr (NX >= 12 && NU >= 4) {
    if (model == IPM_MODEL_QUADROTOR) quadrotor_step(prm, x, u, xn);
  }
}

}  // namespace rrk
