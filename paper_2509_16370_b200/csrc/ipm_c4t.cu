// ipm_c4t.cu -- ipm_step (rows a1-a8) for the C4 shape with ONE THREAD per instance (sm_100a).
//
// SURVEY §8(d) proposes this shape for n_x ≤ 4 ("the whole stage fits in registers, so thread- or
// quad-lane-per-instance is the better shape"): every instance is one thread, its stage a handful of
// 4×4 / 5×5 register matrices, no intra-instance communication, the whole C4 batch one wave (16,384
// threads, 3.5 warps per SM).  Stage data go through two shared tiles per warp (coalesced 8-byte
// LDGSTS, transposed to element-major so each lane reads its column conflict-free), the forward
// record is [stage][entry][instance] in the workspace (coalesced, register-pipelined one stage
// ahead), the update streams the warp's contiguous iterate blocks.  MEASURED SLOWER than the
// lane-group kernel of ipm.cu on C4 (2.1 / 1.56 / 1.82 / 2.60 ms across the variants of
// DESIGN.md §7 against 1.22 ms): with one warp per scheduler every dependent FP64 chain (the 4-pivot
// S⁻¹ sweep, the model's sincos) and every global round trip is exposed.  Kept as an A/B variant
// behind RR_IPM_C4T=1 with its own parity tests (tests/test_ipm_c4t_gpu.py).
//
// Method (arXiv 2509.16370, P:n = PAPER.md line n) -- identical to ipm.cu, see there for the cites:
//   pass 1 (backward): condense (Σ = (S/Z + I/η)⁻¹, r_z = g + μ/z; P̃ = P + GᵀΣG, s̃ = ∇ₓℒ + GᵀΣr_z,
//     P:277-300), one step of Eq.(RR) with δ = 1/η, record Φ = S⁻¹(A + BK),
//     φ = S⁻¹(Bk + c − δv), K, k, V, v;
//   pass 2 (forward): Δx_{i+1} = ΦΔx_i + φ, Δu = KΔx + k, Δy = VΔx + v, expand
//     Δz, Δs, D = ∇𝒜·(Δx, Δs) and the merit polynomial,
//     fraction to the boundary;
//   pass 3: Armijo backtracking on 𝒜 (reading R12), trial dynamics through the model;
//   pass 4: in-place update.
// Shape: n = 4, m = 1, n_g = 4, n_c = 0 (terminal n_gN ≤ 4, n_cN = 0), IPM_MODEL_LQ or
// IPM_MODEL_CARTPOLE, all instances (no ipm_solve active list), 16-byte aligned operand bases.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include <type_traits>

#include "ipm.cuh"
#include "ipm_model.cuh"
#include "rr_common.cuh"

namespace rrk {

namespace {

constexpr int NX = 4, NZ = 5, NG = 4;  // n, n + m (m = 1), n_g
// forward record per stage (doubles), stored [stage][entry][instance]
constexpr int R_PHI = 0, R_phi = 16, R_K = 20, R_k = 24, R_V = 25, R_v = 35, RCP = 40;

__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void st2(double* p, double a, double b) {
  *reinterpret_cast<double2*>(p) = make_double2(a, b);
}

// Stage data of one (instance, stage) in registers
struct StageData {
  double A[NX][NX];  // A[r][c]
  double B[NX];
  double P[NZ][NZ];  // [[Q M]; [Mᵀ R]]
  double gf[NZ];
  double c[NX];      // dres = d_i(x̄_i, ū_i) − x̄_{i+1}
  double G[NG][NZ];  // G[e][c]
  double gv[NG], s[NG], z[NG];
  double yi[NX], yn[NX];
};

__device__ __forceinline__ double F_(const StageData& d, int r, int c) { return c < NX ? d.A[r][c] : d.B[r]; }

// Shared-memory staging of a warp's stage data: one tile per buffer, element k of lane q at k·SW + q
// (SW = 33: the coalesced-copy writes and the per-lane reads are both conflict-free).  The copy of
// an L-double chunk per instance walks the 32 chunks with consecutive lanes on consecutive global
// doubles (coalesced 8-byte LDGSTS, transposed on the shared side).
constexpr int SW = 33;
constexpr int E_A = 0, E_B = 16, E_Q = 20, E_M = 30, E_R = 34, E_gf = 35, E_c = 40, E_G = 44, E_gv = 64, E_s = 68,
              E_z = 72, E_y = 76, NE = 84;  // E_y: y_i | y_{i+1}
constexpr int BUF = NE * SW;

template <int L>
__device__ __forceinline__ void copy_arr(double* dst, const double* base, int64_t stride, int64_t off, int64_t inst0,
                                         int nact, int lane) {
  for (int f = lane; f < L * nact; f += nact) {
    const int q = f / L, o = f - q * L;
    cp_async8(dst + o * SW + q, base + (inst0 + q) * stride + off + o);
  }
}

__device__ __forceinline__ void issue_stage(const IpmArgs& a, double* buf, int64_t inst0, int nact, int lane, int64_t sN,
                                            int i) {
  copy_arr<16>(buf + E_A * SW, a.d_.A, sN * 16, (int64_t)i * 16, inst0, nact, lane);
  copy_arr<4>(buf + E_B * SW, a.d_.B, sN * 4, (int64_t)i * 4, inst0, nact, lane);
  copy_arr<10>(buf + E_Q * SW, a.d_.Q, sN * 10, (int64_t)i * 10, inst0, nact, lane);
  copy_arr<4>(buf + E_M * SW, a.d_.M, sN * 4, (int64_t)i * 4, inst0, nact, lane);
  copy_arr<1>(buf + E_R * SW, a.d_.R, sN, i, inst0, nact, lane);
  copy_arr<5>(buf + E_gf * SW, a.d_.gradf, sN * 5, (int64_t)i * 5, inst0, nact, lane);
  copy_arr<4>(buf + E_c * SW, a.d_.dres, sN * 4, (int64_t)i * 4, inst0, nact, lane);
  copy_arr<20>(buf + E_G * SW, a.d_.Gj, sN * 20, (int64_t)i * 20, inst0, nact, lane);
  copy_arr<4>(buf + E_gv * SW, a.d_.gv, sN * 4, (int64_t)i * 4, inst0, nact, lane);
  copy_arr<4>(buf + E_s * SW, a.it.s, sN * 4, (int64_t)i * 4, inst0, nact, lane);
  copy_arr<4>(buf + E_z * SW, a.it.z, sN * 4, (int64_t)i * 4, inst0, nact, lane);
  copy_arr<8>(buf + E_y * SW, a.it.y, (sN + 1) * 4, (int64_t)i * 4, inst0, nact, lane);
}

__device__ __forceinline__ void load_stage_smem(const double* buf, int lane, StageData& d) {
  auto E = [&](int k) { return buf[k * SW + lane]; };
#pragma unroll
  for (int c = 0; c < NX; ++c)
#pragma unroll
    for (int r = 0; r < NX; ++r) d.A[r][c] = E(E_A + r + 4 * c);
#pragma unroll
  for (int r = 0; r < NX; ++r) d.B[r] = E(E_B + r);
#pragma unroll
  for (int c = 0; c < NX; ++c)
#pragma unroll
    for (int r = 0; r < NX; ++r) d.P[r][c] = r >= c ? E(E_Q + pidx(NX, r, c)) : E(E_Q + pidx(NX, c, r));
#pragma unroll
  for (int r = 0; r < NX; ++r) {
    d.P[r][4] = E(E_M + r);
    d.P[4][r] = d.P[r][4];
  }
  d.P[4][4] = E(E_R);
#pragma unroll
  for (int e = 0; e < NZ; ++e) d.gf[e] = E(E_gf + e);
#pragma unroll
  for (int r = 0; r < NX; ++r) d.c[r] = E(E_c + r);
#pragma unroll
  for (int c = 0; c < NZ; ++c)
#pragma unroll
    for (int e = 0; e < NG; ++e) d.G[e][c] = E(E_G + e + 4 * c);
#pragma unroll
  for (int e = 0; e < NG; ++e) {
    d.gv[e] = E(E_gv + e);
    d.s[e] = E(E_s + e);
    d.z[e] = E(E_z + e);
  }
#pragma unroll
  for (int r = 0; r < NX; ++r) {
    d.yi[r] = E(E_y + r);
    d.yn[r] = E(E_y + 4 + r);
  }
}

// Σ = (s/z + 1/η)⁻¹ = zη/(sη + z), r_z = g + μ/z, over the first ng constraints
__device__ __forceinline__ void condense_duals(const double* s, const double* z, const double* g, int ng, double mu,
                                               double eta, double* sig, double* rz, int i, int& nonpos) {
#pragma unroll
  for (int e = 0; e < NG; ++e) {
    if (e < ng && (!(s[e] > 0.0) || !(z[e] > 0.0))) nonpos = min(nonpos, i);
    sig[e] = (e < ng) ? z[e] * eta * rcp_nr(fma(s[e], eta, z[e])) : 0.0;
    rz[e] = (e < ng) ? fma(mu, rcp_nr(z[e]), g[e]) : 0.0;
  }
}

// −(I + δV)⁻¹ by the symmetric sweep operator (S SPD with eigenvalues >= 1; reading R9)
__device__ __forceinline__ void inv_S(const double (&V)[NX][NX], double delta, double (&Si)[NX][NX], bool& notpd) {
  double A[NX][NX];
#pragma unroll
  for (int r = 0; r < NX; ++r)
#pragma unroll
    for (int c = 0; c < NX; ++c) A[r][c] = delta * V[r][c] + (r == c ? 1.0 : 0.0);
#pragma unroll
  for (int p = 0; p < NX; ++p) {
    const double d = A[p][p];
    notpd |= !(d > 0.0);
    const double id = rcp_nr(d);
    double col[NX];
#pragma unroll
    for (int r = 0; r < NX; ++r) col[r] = A[r][p];
#pragma unroll
    for (int r = 0; r < NX; ++r)
#pragma unroll
      for (int c = 0; c < NX; ++c) {
        if (r == p && c == p) A[r][c] = -id;
        else if (r == p) A[r][c] = col[c] * id;  // row p = column p (symmetry)
        else if (c == p) A[r][c] = col[r] * id;
        else A[r][c] = fma(-col[r] * id, col[c], A[r][c]);
      }
  }
#pragma unroll
  for (int r = 0; r < NX; ++r)
#pragma unroll
    for (int c = 0; c < NX; ++c) Si[r][c] = -A[r][c];
}

__global__ void __launch_bounds__(32) ipm_c4t_kernel(const IpmArgs a) {
  extern __shared__ __align__(16) double smem[];  // two stage tiles of the warp
  const int64_t inst = (int64_t)blockIdx.x * 32 + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int64_t inst0 = inst - lane;
  const int nact = (a.d.batch - inst0) < 32 ? (int)(a.d.batch - inst0) : 32;  // lanes 0..nact−1 hold instances
  if (lane >= nact) return;
  const unsigned mask = nact == 32 ? 0xffffffffu : ((1u << nact) - 1u);
  double* buf0 = smem;
  double* buf1 = smem + BUF;
  const int N = a.d.N, ngN = a.d.ngN;
  const int64_t sN = N, Bt = a.d.batch;
  const double mu = a.it.mu[inst], eta = a.it.eta[inst];
  const double delta = 1.0 / eta;  // P:387-394 (reading R15)
  double* rec0 = a.ws;             // [N][RCP][batch]
  auto R = [&](int i, int e) -> double* { return rec0 + ((int64_t)i * RCP + e) * Bt + inst; };
  int32_t st = 0;
  int nonpos = 0x7fffffff;
  const int model = a.d.model;

  // terminal condensed blocks: P̃_N = Q_N + G_NᵀΣ_N G_N, q̃_N = ∇f_N − y_N + G_Nᵀ(z_N + Σ_N r_z,N)
  double PN[NX][NX], qN[NX], GN[NG][NX], sNv[NG], zNv[NG], gNv[NG], sigN[NG], rzN[NG];
  {
    const double* QN = a.d_.QN + inst * 10;
#pragma unroll
    for (int c = 0; c < NX; ++c)
#pragma unroll
      for (int r = 0; r < NX; ++r) PN[r][c] = r >= c ? QN[pidx(NX, r, c)] : QN[pidx(NX, c, r)];
#pragma unroll
    for (int e = 0; e < NG; ++e) {
      const bool ok = e < ngN;
      sNv[e] = ok ? a.it.sN[inst * ngN + e] : 1.0;
      zNv[e] = ok ? a.it.zN[inst * ngN + e] : 1.0;
      gNv[e] = ok ? a.d_.gvN[inst * ngN + e] : 0.0;
#pragma unroll
      for (int c = 0; c < NX; ++c) GN[e][c] = ok ? a.d_.GjN[inst * ngN * NX + e + c * ngN] : 0.0;
    }
    condense_duals(sNv, zNv, gNv, ngN, mu, eta, sigN, rzN, N, nonpos);
#pragma unroll
    for (int j = 0; j < NX; ++j) {
      double v = a.d_.gradfN[inst * NX + j] - a.it.y[(inst * (sN + 1) + N) * NX + j];
#pragma unroll
      for (int e = 0; e < NG; ++e) v = fma(GN[e][j], fma(sigN[e], rzN[e], zNv[e]), v);
      qN[j] = v;
    }
  }
  double V[NX][NX], v[NX];
#pragma unroll
  for (int r = 0; r < NX; ++r) {
    v[r] = qN[r];
#pragma unroll
    for (int c = 0; c < NX; ++c) {
      double t = PN[r][c];
#pragma unroll
      for (int e = 0; e < NG; ++e) t = fma(GN[e][r], sigN[e] * GN[e][c], t);
      V[r][c] = t;
    }
  }

  // ================= pass 1: backward (condense + Eq.(RR)) =================
  if (N > 0) {
    issue_stage(a, buf0, inst0, nact, lane, sN, N - 1);
    cp_async_commit();
  }
  for (int i = N - 1; i >= 0; --i) {
    double* cur = ((N - 1 - i) & 1) ? buf1 : buf0;
    double* nxt = ((N - 1 - i) & 1) ? buf0 : buf1;
    if (i > 0) issue_stage(a, nxt, inst0, nact, lane, sN, i - 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp(mask);
    StageData d;
    load_stage_smem(cur, lane, d);
    __syncwarp(mask);  // every lane has read `cur` before it is refilled
    double sig[NG], rz[NG];
    condense_duals(d.s, d.z, d.gv, NG, mu, eta, sig, rz, i, nonpos);
    // P̃ = P + GᵀΣG;  s̃ = ∇f − (y_i; 0) + Fᵀy_{i+1} + Gᵀ(z + Σ r_z)
    double Pt[NZ][NZ], qt[NZ];
#pragma unroll
    for (int r = 0; r < NZ; ++r)
#pragma unroll
      for (int c = 0; c < NZ; ++c) {
        double t = d.P[r][c];
#pragma unroll
        for (int e = 0; e < NG; ++e) t = fma(d.G[e][r], sig[e] * d.G[e][c], t);
        Pt[r][c] = t;
      }
#pragma unroll
    for (int j = 0; j < NZ; ++j) {
      double t = d.gf[j] - (j < NX ? d.yi[j] : 0.0);
#pragma unroll
      for (int r = 0; r < NX; ++r) t = fma(F_(d, r, j), d.yn[r], t);
#pragma unroll
      for (int e = 0; e < NG; ++e) t = fma(d.G[e][j], fma(sig[e], rz[e], d.z[e]), t);
      qt[j] = t;
    }
    // S⁻¹, W = S⁻¹V, e = c − δv, g = v + W e
    bool notpd = false;
    double Si[NX][NX];
    inv_S(V, delta, Si, notpd);
    if (notpd && st == 0) st = mk_status(RR_ST_S_NOT_PD, i);
    double W[NX][NX], e_[NX], g[NX];
#pragma unroll
    for (int r = 0; r < NX; ++r) e_[r] = d.c[r] - delta * v[r];
#pragma unroll
    for (int r = 0; r < NX; ++r)
#pragma unroll
      for (int c = 0; c < NX; ++c) {
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < NX; ++k) t = fma(Si[r][k], V[k][c], t);
        W[r][c] = t;
      }
#pragma unroll
    for (int r = 0; r < NX; ++r) {
      double t = v[r];
#pragma unroll
      for (int k = 0; k < NX; ++k) t = fma(W[r][k], e_[k], t);
      g[r] = t;
    }
    // T = W F (NX × NZ);  U = Fᵀ T + P̃ (lower, mirrored);  b = s̃ + Fᵀ g
    double T[NX][NZ], U[NZ][NZ], b[NZ];
#pragma unroll
    for (int r = 0; r < NX; ++r)
#pragma unroll
      for (int c = 0; c < NZ; ++c) {
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < NX; ++k) t = fma(W[r][k], F_(d, k, c), t);
        T[r][c] = t;
      }
#pragma unroll
    for (int r = 0; r < NZ; ++r)
#pragma unroll
      for (int c = 0; c <= r; ++c) {
        double t = Pt[r][c];
#pragma unroll
        for (int k = 0; k < NX; ++k) t = fma(F_(d, k, r), T[k][c], t);
        U[r][c] = t;
        U[c][r] = t;
      }
#pragma unroll
    for (int j = 0; j < NZ; ++j) {
      double t = qt[j];
#pragma unroll
      for (int k = 0; k < NX; ++k) t = fma(F_(d, k, j), g[k], t);
      b[j] = t;
    }
    // u-block (m = 1): G = U_uu;  K = −G⁻¹H, k = −G⁻¹b_u;  V_i = U_xx + HᵀK, v_i = b_x + Hᵀk
    const double piv = U[4][4];
    if (!(piv > 0.0) && st == 0) st = mk_status(RR_ST_G_NOT_PD, i);
    const double ip = rcp_nr(piv);
    double K[NX];
#pragma unroll
    for (int j = 0; j < NX; ++j) K[j] = -U[4][j] * ip;
    const double k = -b[4] * ip;
#pragma unroll
    for (int r = 0; r < NX; ++r) {
#pragma unroll
      for (int c = 0; c < NX; ++c) V[r][c] = fma(U[r][4], K[c], U[r][c]);
      v[r] = fma(U[r][4], k, b[r]);
    }
    // Φ = S⁻¹(A + B K), φ = S⁻¹(B k + e)
    double Phi[NX][NX], phi[NX];
#pragma unroll
    for (int r = 0; r < NX; ++r) {
#pragma unroll
      for (int c = 0; c < NX; ++c) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < NX; ++q) t = fma(Si[r][q], fma(d.B[q], K[c], d.A[q][c]), t);
        Phi[r][c] = t;
      }
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < NX; ++q) t = fma(Si[r][q], fma(d.B[q], k, e_[q]), t);
      phi[r] = t;
    }
    // record [stage][entry][instance]
#pragma unroll
    for (int c = 0; c < NX; ++c)
#pragma unroll
      for (int r = 0; r < NX; ++r) *R(i, R_PHI + r + 4 * c) = Phi[r][c];
#pragma unroll
    for (int r = 0; r < NX; ++r) {
      *R(i, R_phi + r) = phi[r];
      *R(i, R_K + r) = K[r];
      *R(i, R_v + r) = v[r];
    }
    *R(i, R_k) = k;
#pragma unroll
    for (int c = 0; c < NX; ++c)
#pragma unroll
      for (int r = c; r < NX; ++r) *R(i, R_V + pidx(NX, r, c)) = V[r][c];
  }

  // ================= pass 2: forward + expand + merit/D accumulation =================
  // Δx_0 = (I + δV_0)⁻¹(c_0 − δ v_0), c_0 = s_0 − x̄_0
  double xr[NX], c0v[NX];
  {
    bool notpd = false;
    double Si[NX][NX];
    inv_S(V, delta, Si, notpd);
    if (notpd && st == 0) st = mk_status(RR_ST_S_NOT_PD, 0);
    double t[NX];
#pragma unroll
    for (int r = 0; r < NX; ++r) {
      c0v[r] = a.d_.s0[inst * NX + r] - a.it.x[inst * (sN + 1) * NX + r];
      t[r] = c0v[r] - delta * v[r];
    }
#pragma unroll
    for (int r = 0; r < NX; ++r) {
      double u = 0.0;
#pragma unroll
      for (int q = 0; q < NX; ++q) u = fma(Si[r][q], t[q], u);
      xr[r] = u;
    }
  }
  double sD = 0.0, sK0 = 0.0, sK1 = 0.0, sK2 = 0.0;
  LogAcc sLog;
  double amax = 1.0, admax = 1.0;
  const double tau = a.prm.tau;
  bool bad = false;
  // row 0 (initial state): c_0(α) = c_0 − αΔx_0
#pragma unroll
  for (int j = 0; j < NX; ++j) {
    const double y0 = a.it.y[inst * (sN + 1) * NX + j];
    const double c0 = c0v[j], cd = -xr[j];
    sD += (y0 + eta * c0) * cd;
    sK0 += y0 * c0 + 0.5 * eta * c0 * c0;
    sK1 += y0 * cd + eta * c0 * cd;
    sK2 += 0.5 * eta * cd * cd;
  }
  {
    double* dx = a.r.dx + inst * (sN + 1) * NX;
    st2(dx, xr[0], xr[1]);
    st2(dx + 2, xr[2], xr[3]);
  }
  // expansion of the inequalities of one stage + their merit terms
  auto expand_ineq = [&](const double (&Gd)[NG], const double* s, const double* z, const double* g, const double* sig,
                         const double* rz, int ng, double* ds_out, double* dz_out) {
#pragma unroll
    for (int e = 0; e < NG; ++e) {
      if (e >= ng) continue;
      const double dzv = sig[e] * (Gd[e] + rz[e]);
      const double iz = rcp_nr(z[e]);
      const double dsv = fma(-(s[e] * iz), dzv, fma(mu, iz, -s[e]));
      if (dsv < 0.0) amax = fmin(amax, tau * s[e] / (-dsv));
      if (dzv < 0.0) admax = fmin(admax, tau * z[e] / (-dzv));
      const double gs = g[e] + s[e], bq = Gd[e] + dsv;
      sD += (z[e] + eta * gs) * bq + (-mu * rcp_nr(s[e])) * dsv;
      sK0 += z[e] * gs + 0.5 * eta * gs * gs;
      sK1 += z[e] * bq + eta * gs * bq;
      sK2 += 0.5 * eta * bq * bq;
      sLog.add(s[e]);
      ds_out[e] = dsv;
      dz_out[e] = dzv;
      bad |= !isfinite(dsv) || !isfinite(dzv);
    }
  };
  // stage data through the shared tiles (one stage ahead); the record (coalesced: [stage][entry][instance])
  // in registers, its loads for stage i+1 issued before stage i's expansion work
  double rc[RCP - 1];
  if (N > 0) {
    issue_stage(a, buf0, inst0, nact, lane, sN, 0);
    cp_async_commit();
#pragma unroll
    for (int e = 0; e < RCP - 1; ++e) rc[e] = *R(0, e);
  }
  for (int i = 0; i < N; ++i) {
    double* cur = (i & 1) ? buf1 : buf0;
    double* nxt = (i & 1) ? buf0 : buf1;
    if (i + 1 < N) issue_stage(a, nxt, inst0, nact, lane, sN, i + 1);
    cp_async_commit();
    // Δu_i = KΔx_i + k,  Δx_{i+1} = ΦΔx_i + φ,  Δy_i = VΔx_i + v
    double du = rc[R_k], xn[NX], dy[NX];
#pragma unroll
    for (int q = 0; q < NX; ++q) du = fma(rc[R_K + q], xr[q], du);
#pragma unroll
    for (int r = 0; r < NX; ++r) {
      double t = rc[R_phi + r], y = rc[R_v + r];
#pragma unroll
      for (int q = 0; q < NX; ++q) {
        t = fma(rc[R_PHI + r + 4 * q], xr[q], t);
        y = fma(rc[R_V + (r >= q ? pidx(NX, r, q) : pidx(NX, q, r))], xr[q], y);
      }
      xn[r] = t;
      dy[r] = y;
    }
    if (i + 1 < N) {
#pragma unroll
      for (int e = 0; e < RCP - 1; ++e) rc[e] = *R(i + 1, e);
    }
    cp_async_wait<1>();
    __syncwarp(mask);
    StageData d;
    load_stage_smem(cur, lane, d);
    __syncwarp(mask);
    double sig[NG], rz[NG];
    condense_duals(d.s, d.z, d.gv, NG, mu, eta, sig, rz, i, nonpos);
    {
      double* dyo = a.r.dy + (inst * (sN + 1) + i) * NX;
      double* dxo = a.r.dx + (inst * (sN + 1) + i + 1) * NX;
      st2(dyo, dy[0], dy[1]);
      st2(dyo + 2, dy[2], dy[3]);
      st2(dxo, xn[0], xn[1]);
      st2(dxo + 2, xn[2], xn[3]);
      a.r.du[inst * sN + i] = du;
    }
#pragma unroll
    for (int r = 0; r < NX; ++r) bad |= !(isfinite(xn[r]) && isfinite(dy[r]));
    bad |= !isfinite(du);
    const double dzf[NZ] = {xr[0], xr[1], xr[2], xr[3], du};
    double Gd[NG];
#pragma unroll
    for (int e = 0; e < NG; ++e) {
      double t = 0.0;
#pragma unroll
      for (int c = 0; c < NZ; ++c) t = fma(d.G[e][c], dzf[c], t);
      Gd[e] = t;
    }
    double dso[NG], dzo[NG];
    expand_ineq(Gd, d.s, d.z, d.gv, sig, rz, NG, dso, dzo);
    {
      const int64_t si = inst * sN + i;
      st2(a.r.ds + si * 4, dso[0], dso[1]);
      st2(a.r.ds + si * 4 + 2, dso[2], dso[3]);
      st2(a.r.dz + si * 4, dzo[0], dzo[1]);
      st2(a.r.dz + si * 4 + 2, dzo[2], dzo[3]);
    }
    // cost: ∇fᵀΔ and ½ΔᵀPΔ
#pragma unroll
    for (int j = 0; j < NZ; ++j) {
      double pd = 0.0;
#pragma unroll
      for (int c = 0; c < NZ; ++c) pd = fma(d.P[j][c], dzf[c], pd);
      const double gd = d.gf[j] * dzf[j];
      sD += gd;
      sK1 += gd;
      sK2 += 0.5 * dzf[j] * pd;
    }
    // dynamics row i+1: (CΔ)_r = (FΔ)_r − Δx_{i+1,r};  c_{i+1} at the iterate
#pragma unroll
    for (int j = 0; j < NX; ++j) {
      double fd = 0.0;
#pragma unroll
      for (int c = 0; c < NZ; ++c) fd = fma(F_(d, j, c), dzf[c], fd);
      const double cd = fd - xn[j];
      sD += (d.yn[j] + eta * d.c[j]) * cd;
      if (model == IPM_MODEL_LQ) {
        sK0 += d.yn[j] * d.c[j] + 0.5 * eta * d.c[j] * d.c[j];
        sK1 += d.yn[j] * cd + eta * d.c[j] * cd;
        sK2 += 0.5 * eta * cd * cd;
      }
    }
#pragma unroll
    for (int r = 0; r < NX; ++r) xr[r] = xn[r];
  }
  // terminal: y_N = Ṽ_N x_N + ṽ_N (condensed terminal blocks), expansions on x_N, cost with Q_N
  {
    double dyN[NX];
#pragma unroll
    for (int j = 0; j < NX; ++j) {
      double t = qN[j];
#pragma unroll
      for (int r = 0; r < NX; ++r) {
        double pt = PN[j][r];
#pragma unroll
        for (int e = 0; e < NG; ++e) pt = fma(GN[e][j], sigN[e] * GN[e][r], pt);
        t = fma(pt, xr[r], t);
      }
      dyN[j] = t;
      bad |= !isfinite(t);
    }
    double* dyo = a.r.dy + (inst * (sN + 1) + N) * NX;
    st2(dyo, dyN[0], dyN[1]);
    st2(dyo + 2, dyN[2], dyN[3]);
    double Gd[NG];
#pragma unroll
    for (int e = 0; e < NG; ++e) {
      double t = 0.0;
#pragma unroll
      for (int c = 0; c < NX; ++c) t = fma(GN[e][c], xr[c], t);
      Gd[e] = t;
    }
    double dso[NG], dzo[NG];
    expand_ineq(Gd, sNv, zNv, gNv, sigN, rzN, ngN, dso, dzo);
#pragma unroll
    for (int e = 0; e < NG; ++e)
      if (e < ngN) {
        a.r.dsN[inst * ngN + e] = dso[e];
        a.r.dzN[inst * ngN + e] = dzo[e];
      }
#pragma unroll
    for (int j = 0; j < NX; ++j) {
      double pd = 0.0;
#pragma unroll
      for (int c = 0; c < NX; ++c) pd = fma(PN[j][c], xr[c], pd);
      const double gd = a.d_.gradfN[inst * NX + j] * xr[j];
      sD += gd;
      sK1 += gd;
      sK2 += 0.5 * xr[j] * pd;
    }
  }
  const double D = sD;
  const double K0 = sK0 + a.d_.fval[inst];
  const double K1 = sK1, K2 = sK2;
  const double Abase = K0 - mu * sLog.value();
  int32_t status = st;
  if (status == 0 && bad) status = RR_ST_NONFINITE;
  if (nonpos != 0x7fffffff) status = mk_status(RR_ST_NONPOS_SLACK, nonpos);
  // dynamics terms of 𝒜 at α = 0 through the built-in model (fused into the first trial when there is one)
  const bool fuse0 = model != IPM_MODEL_LQ && status == 0 && !a.direction_only;
  double A0 = Abase, sDyn0 = 0.0;
  const double* prm = a.d_.model_params;
  if (model != IPM_MODEL_LQ && !fuse0) {
    for (int i = 0; i < N; ++i) {
      const double* xb = a.it.x + (inst * (sN + 1) + i) * NX;
      const double* yb = a.it.y + (inst * (sN + 1) + i + 1) * NX;
      double xa[NX], xnm[NX];
#pragma unroll
      for (int r = 0; r < NX; ++r) xa[r] = xb[r];
      cartpole_step(prm, xa, a.it.u[inst * sN + i], xnm);
#pragma unroll
      for (int r = 0; r < NX; ++r) {
        const double cr = xnm[r] - xb[NX + r];
        sDyn0 += yb[r] * cr + 0.5 * eta * cr * cr;
      }
    }
    A0 = Abase + sDyn0;
  }

  // ================= pass 3: Armijo backtracking over (x, s) with 𝒜 =================
  double alpha = amax, Aacc = __longlong_as_double(0x7ff8000000000000LL);
  int nb = 0;
  bool accepted = false;
  if (status == 0 && !a.direction_only) {
    for (nb = 0; nb <= a.prm.max_backtracks; ++nb) {
      LogAcc sl;
      double sdyn = 0.0;
      bool pos = true;
      // stage i's loads were issued one stage ahead (x̄_i, Δx_i carried from the previous stage)
      const double* X = a.it.x + inst * (sN + 1) * NX;
      const double* DX = a.r.dx + inst * (sN + 1) * NX;
      const double* Y = a.it.y + inst * (sN + 1) * NX;
      const double* S = a.it.s + inst * sN * NG;
      const double* DS = a.r.ds + inst * sN * NG;
      double xb[NX], dxb[NX];
#pragma unroll
      for (int r = 0; r < NX; ++r) {
        xb[r] = X[r];
        dxb[r] = DX[r];
      }
      double sv[NG], dsv[NG];
#pragma unroll
      for (int e = 0; e < NG; ++e) {
        sv[e] = N > 0 ? S[e] : 0.0;
        dsv[e] = N > 0 ? DS[e] : 0.0;
      }
      for (int i = 0; i < N; ++i) {
        // next stage's slacks and this stage's x̄_{i+1}, Δx_{i+1}, ū_i, Δu_i, y_{i+1}
        double sn[NG], dsn[NG], xn1[NX], dxn1[NX], yb[NX];
        const double ub = a.it.u[inst * sN + i], dub = a.r.du[inst * sN + i];
#pragma unroll
        for (int e = 0; e < NG; ++e) {
          sn[e] = (i + 1 < N) ? S[(i + 1) * NG + e] : 0.0;
          dsn[e] = (i + 1 < N) ? DS[(i + 1) * NG + e] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < NX; ++r) {
          xn1[r] = X[(i + 1) * NX + r];
          dxn1[r] = DX[(i + 1) * NX + r];
          yb[r] = Y[(i + 1) * NX + r];
        }
#pragma unroll
        for (int e = 0; e < NG; ++e) {
          const double sa = fma(alpha, dsv[e], sv[e]);
          pos &= sa > 0.0;
          sl.add(sa);
        }
        if (model != IPM_MODEL_LQ) {
          double xa[NX], xnm[NX];
#pragma unroll
          for (int r = 0; r < NX; ++r) xa[r] = xb[r] + alpha * dxb[r];
          cartpole_step(prm, xa, ub + alpha * dub, xnm);
#pragma unroll
          for (int r = 0; r < NX; ++r) {
            const double cr = xnm[r] - (xn1[r] + alpha * dxn1[r]);
            sdyn += yb[r] * cr + 0.5 * eta * cr * cr;
          }
          if (fuse0 && nb == 0) {
            cartpole_step(prm, xb, ub, xnm);
#pragma unroll
            for (int r = 0; r < NX; ++r) {
              const double cr = xnm[r] - xn1[r];
              sDyn0 += yb[r] * cr + 0.5 * eta * cr * cr;
            }
          }
        }
#pragma unroll
        for (int r = 0; r < NX; ++r) {
          xb[r] = xn1[r];
          dxb[r] = dxn1[r];
        }
#pragma unroll
        for (int e = 0; e < NG; ++e) {
          sv[e] = sn[e];
          dsv[e] = dsn[e];
        }
      }
      for (int e = 0; e < ngN; ++e) {  // terminal slacks
        const double sa = fma(alpha, a.r.dsN[inst * ngN + e], a.it.sN[inst * ngN + e]);
        pos &= sa > 0.0;
        sl.add(sa);
      }
      if (fuse0 && nb == 0) A0 = Abase + sDyn0;
      const double At = K0 + alpha * (K1 + alpha * K2) - mu * sl.value() + sdyn;
      if (pos && At <= A0 + a.prm.armijo_c * alpha * D) {
        Aacc = At;
        accepted = true;
        break;
      }
      alpha *= a.prm.beta;
    }
    if (!accepted) {
      status = RR_ST_LS_FAILED;
      alpha = 0.0;
      nb = a.prm.max_backtracks + 1;
    }
  }

  // ================= pass 4: update the iterate in place =================
  // Warp-cooperative: the warp's consecutive instances own one contiguous block of every iterate
  // array ([b][...] layouts), so the warp streams the block with coalesced accesses; each element
  // takes its instance's step, shuffled from the owning lane (instances not accepted: untouched).
  {
    __syncwarp(mask);
    const double ap = accepted ? alpha : 0.0, ad = accepted ? admax : 0.0;
    const int acc = accepted ? 1 : 0;
    // units of W doubles (W = 2 when `per` is even: a unit never straddles two instances), 8 units
    // in flight per lane; the owner of element e is e / per, by a rounded reciprocal and one fix-up
    auto stream_w = [&](auto wtag, double* xv, const double* dv, int64_t per, bool dual) {
      constexpr int W = decltype(wtag)::value;
      const int64_t units = per * nact / W;
      double* xb = xv + inst0 * per;
      const double* db = dv + inst0 * per;
      const double inv = 1.0 / (double)per;
      for (int64_t u0 = 0; u0 < units; u0 += (int64_t)nact * 8) {  // lanes ≥ nact have exited
        double xa[8][W], da[8][W];
        int own[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int64_t u = u0 + lane + (int64_t)nact * k;
          own[k] = 0;
          if (u < units) {
            const int64_t e = u * W;
            int q = (int)((double)e * inv);
            if ((int64_t)(q + 1) * per <= e) ++q;
            else if ((int64_t)q * per > e) --q;
            own[k] = q;
            if constexpr (W == 2) {
              const double2 xv2 = ld2(xb + e), dv2 = ld2(db + e);
              xa[k][0] = xv2.x, xa[k][1] = xv2.y, da[k][0] = dv2.x, da[k][1] = dv2.y;
            } else {
              xa[k][0] = xb[e];
              da[k][0] = db[e];
            }
          }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int64_t u = u0 + lane + (int64_t)nact * k;
          const double st_ = __shfl_sync(mask, dual ? ad : ap, own[k]);
          const int ok = __shfl_sync(mask, acc, own[k]);
          if (u < units && ok) {
            if constexpr (W == 2) st2(xb + u * 2, fma(st_, da[k][0], xa[k][0]), fma(st_, da[k][1], xa[k][1]));
            else xb[u] = fma(st_, da[k][0], xa[k][0]);
          }
        }
      }
    };
    auto stream = [&](double* xv, const double* dv, int64_t per, bool dual) {
      if ((per & 1) == 0) stream_w(std::integral_constant<int, 2>{}, xv, dv, per, dual);
      else stream_w(std::integral_constant<int, 1>{}, xv, dv, per, dual);
    };
    stream(a.it.x, a.r.dx, (sN + 1) * NX, false);
    stream(a.it.y, a.r.dy, (sN + 1) * NX, false);
    stream(a.it.u, a.r.du, sN, false);
    stream(a.it.s, a.r.ds, sN * NG, false);
    stream(a.it.z, a.r.dz, sN * NG, true);
    if (ngN > 0) {
      stream(a.it.sN, a.r.dsN, ngN, false);
      stream(a.it.zN, a.r.dzN, ngN, true);
    }
  }
  a.status[inst] = status;
  {
    const bool ok = (status == 0);
    const bool searched = ok || status == RR_ST_LS_FAILED;
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    if (a.r.alpha_p) a.r.alpha_p[inst] = ok ? alpha : 0.0;
    if (a.r.alpha_d) a.r.alpha_d[inst] = ok ? admax : 0.0;
    if (a.r.D) a.r.D[inst] = searched ? D : nan;
    if (a.r.merit0) a.r.merit0[inst] = searched ? A0 : nan;
    if (a.r.merit_acc) a.r.merit_acc[inst] = ok ? Aacc : nan;
    if (a.r.n_backtracks) a.r.n_backtracks[inst] = searched ? nb : 0;
  }
  if ((status & 0xff) == RR_ST_NONPOS_SLACK) {  // direction undefined: NaN-fill
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    const int64_t nx1 = (sN + 1) * NX;
    for (int64_t e = 0; e < nx1; ++e) {
      a.r.dx[inst * nx1 + e] = nan;
      a.r.dy[inst * nx1 + e] = nan;
    }
    for (int64_t e = 0; e < sN; ++e) a.r.du[inst * sN + e] = nan;
    for (int64_t e = 0; e < sN * NG; ++e) {
      a.r.ds[inst * sN * NG + e] = nan;
      a.r.dz[inst * sN * NG + e] = nan;
    }
    for (int e = 0; e < ngN; ++e) {
      a.r.dsN[inst * ngN + e] = nan;
      a.r.dzN[inst * ngN + e] = nan;
    }
  }
}

}  // namespace

// The C4 shape on the thread-per-instance kernel when RR_IPM_C4T=1 (A/B; the lane-group kernel is the default).
bool ipm_c4t_applies(const IpmArgs& a) {
  const ipm_dims& d = a.d;
  if (!(d.nx == 4 && d.nu == 1 && d.ng == 4 && d.nc == 0 && d.ngN <= 4 && d.ncN == 0)) return false;
  if (d.model != IPM_MODEL_LQ && d.model != IPM_MODEL_CARTPOLE) return false;
  if (a.list != nullptr || !a.aligned16) return false;
  if (a.r.dx == nullptr || a.r.dy == nullptr || a.r.du == nullptr || a.r.ds == nullptr || a.r.dz == nullptr)
    return false;
  if (d.ngN > 0 && (a.r.dsN == nullptr || a.r.dzN == nullptr)) return false;
  const char* v = getenv("RR_IPM_C4T");  // opt-in: measured slower than the lane-group kernel
  return v != nullptr && v[0] == '1';
}

cudaError_t ipm_c4t_launch(const IpmArgs& a, cudaStream_t s) {
  const int64_t blocks = (a.d.batch + 31) / 32;  // one warp (32 instances) per CTA
  const int smb = (int)(sizeof(double) * 2 * BUF);
  cudaError_t e = cudaFuncSetAttribute(ipm_c4t_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smb);
  if (e != cudaSuccess) return e;
  if (blocks > 0) ipm_c4t_kernel<<<(unsigned)blocks, 32, smb, s>>>(a);
  return cudaGetLastError();
}

}  // namespace rrk
