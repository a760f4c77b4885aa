// rr_fused.cu -- fused regularized-Riccati factor + solve, one lane group per instance (sm_100a).
//
// Method (arXiv 2509.16370, P:n = PAPER.md line n):
//   backward sweep i = N-1..0 of Eq.(RR), forward sweep,
//   dual recovery y_i = V_i x_i + v_i.
//
// B200 design (kernel K1):
//   * One lane group of LG lanes (LG = 4, 8, 16 or 32; 32/LG instances per warp) owns one instance.
//     Lane j owns COLUMN j of the stage's (n+m)-wide matrices: F = [A B], T = W F, U = Fᵀ W F + P,
//     so the dense contractions are register-resident FMA loops fed by broadcast shared-memory reads.
//   * The stage inputs (A, B, Q, M, R, q, r, c) of stage i-1 stream into a double-buffered
//     per-instance shared-memory slot with cp.async while stage i computes.
//   * S = I + δV_{i+1} is factored by a right-looking Cholesky (pivot column broadcast through
//     shared memory); W = S⁻¹V, and later the closed-loop Φ_i = S⁻¹(A + B K_i) and
//     φ_i = S⁻¹(B k_i + c_{i+1} - δ v_{i+1}), are column-parallel triangular solves.
//   * G⁻¹H, G⁻¹h and the Schur complement AᵀWA + Q - HᵀG⁻¹H = V_i are ONE Gauss-Jordan
//     elimination of the u-block of U (pivot columns via warp shuffles), applied to the
//     right-hand side b = [q + Aᵀg; r + Bᵀg] as well, which yields v_i and -k_i (P:606-611,
//     the HᵀK = KᵀH identities make this the paper's V_i, v_i).  G is SPD (R PD), so Gauss-Jordan
//     without pivoting is the Cholesky-equivalent elimination (reading R9).
//   * The forward sweep is then x_{i+1} = Φ_i x_i + φ_i, u_i = K_i x_i + k_i, y_i = V_i x_i + v_i,
//     reading one per-stage record written by the backward sweep (no re-read of A, B, c and no
//     second Cholesky), so its serial chain per stage is one matrix-vector product.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rr_common.cuh"
#include "rr_fused.cuh"

namespace rrk {

template <int NX, int NU>
struct FusedLayout {
  static constexpr int NZ = NX + NU;
  static constexpr int STG = NX * NX + 2 * NX * NU + NX * (NX + 1) / 2 + NU * (NU + 1) / 2 + 2 * NX + NU;
  static constexpr int STG_PAD = (STG + 1) & ~1;
  // per-instance shared slot (doubles): 2 stage buffers | Lc | Wb | invd | vb | gb | vs | pad
  static constexpr int SLOT = 2 * STG_PAD + 2 * NX * NX + NX + NZ + 2 * NX;
  static constexpr int SLOT_PAD = (SLOT + 1) & ~1;
  // per-stage workspace record (doubles): Phi NX*NX | phi NX | K NU*NX | k NU | V NX*NX | v NX
  static constexpr int REC = 2 * NX * NX + NU * NX + NU + 2 * NX;
  static constexpr int REC_PAD = (REC + 1) & ~1;
};

template <int NX, int NU, int LG, int WARPS, bool EXACT>
__global__ void __launch_bounds__(WARPS * 32) rr_fused_kernel(const FusedArgs a) {
  using LY = FusedLayout<NX, NU>;
  constexpr int NZ = LY::NZ;
  constexpr int IPW = 32 / LG;
  static_assert(NZ <= LG, "lane group narrower than n+m");
  static_assert(32 % LG == 0, "lane group must divide the warp");

  const int n = EXACT ? NX : a.nx;
  const int m = EXACT ? NU : a.nu;
  const int N = a.N;
  const int sn = n * (n + 1) / 2, sm = m * (m + 1) / 2;
  // stage-record offsets inside a stage buffer (same element order as the global operands)
  const int oA = 0, oB = oA + n * n, oQ = oB + n * m, oM = oQ + sn, oR = oM + n * m, oq = oR + sm,
            orr = oq + n, oc = orr + m;

  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / LG, j = lane % LG, gbase = grp * LG;
  double* slot = smem + (warp * IPW + grp) * LY::SLOT_PAD;
  double* stg0 = slot;
  double* stg1 = slot + LY::STG_PAD;
  double* Lc = slot + 2 * LY::STG_PAD;  // Cholesky factor of S, column-major NX×NX (lower)
  double* Wb = Lc + NX * NX;            // W_i column-major NX×NX
  double* invd = Wb + NX * NX;          // 1 / L_kk
  double* vb = invd + NX;               // b vector (NZ)
  double* gb = vb + NZ;                 // g_i (NX)
  double* vs = gb + NX;                 // v_{i+1} (NX), then x (forward)

  int64_t inst = ((int64_t)blockIdx.x * WARPS + warp) * IPW + grp;
  const bool valid = inst < a.batch;
  if (!valid) inst = a.batch - 1;
  const double delta = a.p.delta[inst];
  const int64_t sN = (int64_t)N;
  double* rec0 = a.ws + inst * sN * LY::REC_PAD;

  int32_t st = 0;  // first failure seen by this lane (backward order)
  auto fail = [&](int code, int stage) {
    if (st == 0) st = mk_status(code, stage);
  };

  auto issue_stage = [&](int i, double* dst) {
    const int64_t s = inst * sN + i;
    copy_async(dst + oA, a.p.A + s * n * n, n * n, j, LG);
    copy_async(dst + oB, a.p.B + s * n * m, n * m, j, LG);
    copy_async(dst + oQ, a.p.Q + s * sn, sn, j, LG);
    copy_async(dst + oM, a.p.M + s * n * m, n * m, j, LG);
    copy_async(dst + oR, a.p.R + s * sm, sm, j, LG);
    copy_async(dst + oq, a.p.q + s * n, n, j, LG);
    copy_async(dst + orr, a.p.r + s * m, m, j, LG);
    copy_async(dst + oc, a.p.c + s * n, n, j, LG);
  };

  // ---- padded accessors (column s < NX: x-part, s >= NX: u-part a = s - NX) ----
  auto Fat = [&](const double* sb, int k, int s) -> double {  // F = [A B], NX rows, NZ cols
    if (k >= n) return 0.0;
    if (s < NX) return s < n ? sb[oA + k + s * n] : 0.0;
    const int u = s - NX;
    return u < m ? sb[oB + k + u * n] : 0.0;
  };
  auto Pat = [&](const double* sb, int s, int t) -> double {  // P = [[Q M]; [Mᵀ R]] padded
    if (s < NX && t < NX) {
      if (s >= n || t >= n) return 0.0;
      return s >= t ? sb[oQ + pidx(n, s, t)] : sb[oQ + pidx(n, t, s)];
    }
    if (s < NX) {  // t in u
      const int u = t - NX;
      return (s < n && u < m) ? sb[oM + s + u * n] : 0.0;
    }
    if (t < NX) {
      const int u = s - NX;
      return (t < n && u < m) ? sb[oM + t + u * n] : 0.0;
    }
    const int u = s - NX, w = t - NX;
    if (u < m && w < m) return u >= w ? sb[oR + pidx(m, u, w)] : sb[oR + pidx(m, w, u)];
    return u == w ? 1.0 : 0.0;
  };

  // ---- Cholesky of S = I + δV (lane j holds column j of V in Vc) into Lc / invd ----
  auto cholS = [&](const double (&Vc)[NX], int stage) {
    double Sc[NX];
#pragma unroll
    for (int r = 0; r < NX; ++r) Sc[r] = delta * Vc[r] + (r == j ? 1.0 : 0.0);
#pragma unroll
    for (int p = 0; p < NX; ++p) {
      if (j == p) {
        const double d = Sc[p];
        if (!(d > 0.0)) fail(RR_ST_S_NOT_PD, stage);
        const double ip = rsqrt(d);
        invd[p] = ip;
        Lc[p * NX + p] = d * ip;
#pragma unroll
        for (int r = p + 1; r < NX; ++r) Lc[p * NX + r] = Sc[r] * ip;
      }
      __syncwarp();
      if (j > p && j < NX) {
        const double ljp = Lc[p * NX + j];
#pragma unroll
        for (int r = p + 1; r < NX; ++r) Sc[r] = fma(-Lc[p * NX + r], ljp, Sc[r]);
      }
    }
  };
  // in-place solve (L Lᵀ) X = X with the factor in Lc / invd
  auto cholSolve = [&](double (&X)[NX]) {
#pragma unroll
    for (int k = 0; k < NX; ++k) {
      X[k] *= invd[k];
#pragma unroll
      for (int r = k + 1; r < NX; ++r) X[r] = fma(-Lc[k * NX + r], X[k], X[r]);
    }
#pragma unroll
    for (int k = NX - 1; k >= 0; --k) {
      X[k] *= invd[k];
#pragma unroll
      for (int r = 0; r < k; ++r) X[r] = fma(-Lc[r * NX + k], X[k], X[r]);
    }
  };

  // ---- carried state: Vc = column j of V_{i+1}; vs[] = v_{i+1} ----
  double Vc[NX];
  {
    const double* QN = a.p.QN + inst * sn;
#pragma unroll
    for (int r = 0; r < NX; ++r) {
      double val = 0.0;
      if (j < n && r < n) val = r >= j ? QN[pidx(n, r, j)] : QN[pidx(n, j, r)];
      Vc[r] = val;
    }
    if (j < n) vs[j] = a.p.qN[inst * n + j];
    else if (j < NX) vs[j] = 0.0;
    if (valid && a.f.V != nullptr && j < n) {
      double* Vo = a.f.V + (inst * (sN + 1) + N) * sn;
      for (int r = j; r < n; ++r) Vo[pidx(n, r, j)] = QN[pidx(n, r, j)];
    }
    if (valid && a.f.v != nullptr && j < n) a.f.v[(inst * (sN + 1) + N) * n + j] = a.p.qN[inst * n + j];
  }

  if (N > 0) {
    issue_stage(N - 1, stg0);
    cp_async_commit();
  }
  __syncwarp();

  for (int i = N - 1; i >= 0; --i) {
    const double* sb = ((N - 1 - i) & 1) ? stg1 : stg0;
    double* nb = ((N - 1 - i) & 1) ? stg0 : stg1;
    if (i > 0) issue_stage(i - 1, nb);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();

    // (1) S = I + δ V_{i+1} = L Lᵀ
    cholS(Vc, i);
    // (2) W_i = S⁻¹ V_{i+1}, column j
    double X[NX];
#pragma unroll
    for (int r = 0; r < NX; ++r) X[r] = Vc[r];
    cholSolve(X);
    // (3) W to shared; g_i = v_{i+1} + W (c_{i+1} - δ v_{i+1}); W symmetric: row j = X
    if (j < NX) {
#pragma unroll
      for (int r = 0; r < NX; ++r) Wb[j * NX + r] = X[r];
      double gj = (j < n) ? vs[j] : 0.0;
#pragma unroll
      for (int k = 0; k < NX; ++k) {
        const double e = (k < n) ? (sb[oc + k] - delta * vs[k]) : 0.0;
        gj = fma(X[k], e, gj);
      }
      gb[j] = gj;
    }
    __syncwarp();
    // (4) T = W F, column j (lane j's column of F in registers)
    double Fc[NX];
#pragma unroll
    for (int k = 0; k < NX; ++k) Fc[k] = (j < NZ) ? Fat(sb, k, j) : 0.0;
    double T[NX];
#pragma unroll
    for (int r = 0; r < NX; ++r) T[r] = 0.0;
#pragma unroll
    for (int k = 0; k < NX; ++k)
#pragma unroll
      for (int r = 0; r < NX; ++r) T[r] = fma(Wb[k * NX + r], Fc[k], T[r]);
    // (5) U = Fᵀ W F + P, column j  (blocks AᵀWA+Q, H = BᵀWA+Mᵀ, G = BᵀWB+R: P:617)
    double U[NZ];
#pragma unroll
    for (int s = 0; s < NZ; ++s) {
      double acc = (j < NZ) ? Pat(sb, s, j) : 0.0;
#pragma unroll
      for (int k = 0; k < NX; ++k) acc = fma(Fat(sb, k, s), T[k], acc);
      U[s] = acc;
    }
    // b_j = [q + Aᵀ g ; r + Bᵀ g]_j
    if (j < NZ) {
      double bj = (j < NX) ? ((j < n) ? sb[oq + j] : 0.0) : ((j - NX < m) ? sb[orr + j - NX] : 0.0);
#pragma unroll
      for (int k = 0; k < NX; ++k) bj = fma(Fc[k], gb[k], bj);
      vb[j] = bj;
    }
    __syncwarp();
    double b[NZ];
#pragma unroll
    for (int s = 0; s < NZ; ++s) b[s] = vb[s];
    // (6) Gauss-Jordan on the u-block: G⁻¹H, G⁻¹h, V_i = AᵀWA+Q-HᵀG⁻¹H, v_i
#pragma unroll
    for (int p = NX; p < NZ; ++p) {
      double colp[NZ];
#pragma unroll
      for (int s = 0; s < NZ; ++s) colp[s] = __shfl_sync(RR_FULL_MASK, U[s], gbase + p);
      const double piv = colp[p];
      if (!(piv > 0.0)) fail(RR_ST_G_NOT_PD, i);
      const double ip = 1.0 / piv;
      const double rp = U[p] * ip;
      const double bp = b[p] * ip;
#pragma unroll
      for (int s = 0; s < NZ; ++s) {
        if (s == p) continue;
        U[s] = fma(-colp[s], rp, U[s]);
        b[s] = fma(-colp[s], bp, b[s]);
      }
      U[p] = rp;
      b[p] = bp;
    }
    // now: lane j < n: U[0..NX) = V_i[:, j], U[NX..) = -K_i[:, j];  b = [v_i ; -k_i]
    // (7) closed loop for the forward sweep: Φ_i = S⁻¹(A + B K_i) (lanes j < NX),
    //     φ_i = S⁻¹(B k_i + c_{i+1} - δ v_{i+1}) (lane NX); S = I + δV_{i+1} still in Lc/invd.
    double t[NX];
#pragma unroll
    for (int r = 0; r < NX; ++r) {
      double base = 0.0;
      if (j < NX) base = Fc[r];
      else if (j == NX) base = (r < n) ? (sb[oc + r] - delta * vs[r]) : 0.0;
      t[r] = base;
    }
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const double coef = (j < NX) ? -U[NX + u] : ((j == NX) ? -b[NX + u] : 0.0);
#pragma unroll
      for (int r = 0; r < NX; ++r) t[r] = fma(Fat(sb, r, NX + u), coef, t[r]);
    }
    cholSolve(t);
    // (8) stores: workspace record i, optional factor outputs
    double* rec = rec0 + (int64_t)i * LY::REC_PAD;
    double* rPhi = rec;
    double* rphi = rPhi + NX * NX;
    double* rK = rphi + NX;
    double* rk = rK + NU * NX;
    double* rV = rk + NU;
    double* rv = rV + NX * NX;
    if (j < NX) {
#pragma unroll
      for (int r = 0; r < NX; ++r) {
        rPhi[j * NX + r] = t[r];
        rV[j * NX + r] = U[r];
      }
#pragma unroll
      for (int u = 0; u < NU; ++u) rK[j * NU + u] = -U[NX + u];
    } else if (j == NX) {
#pragma unroll
      for (int r = 0; r < NX; ++r) rphi[r] = t[r];
    }
    if (j == 0) {
#pragma unroll
      for (int r = 0; r < NX; ++r) rv[r] = b[r];
#pragma unroll
      for (int u = 0; u < NU; ++u) rk[u] = -b[NX + u];
    }
    if (valid) {
      if (a.f.V != nullptr && j < n) {
        double* Vo = a.f.V + (inst * (sN + 1) + i) * sn;
#pragma unroll
        for (int r = 0; r < NX; ++r)
          if (r >= j && r < n) Vo[pidx(n, r, j)] = U[r];
      }
      if (a.f.K != nullptr && j < n) {
        double* Ko = a.f.K + (inst * sN + i) * m * n;
#pragma unroll
        for (int u = 0; u < NU; ++u)
          if (u < m) Ko[j * m + u] = -U[NX + u];
      }
      if (j == 0) {
        if (a.f.v != nullptr) {
          double* vo = a.f.v + (inst * (sN + 1) + i) * n;
#pragma unroll
          for (int r = 0; r < NX; ++r)
            if (r < n) vo[r] = b[r];
        }
        if (a.f.k != nullptr) {
          double* ko = a.f.k + (inst * sN + i) * m;
#pragma unroll
          for (int u = 0; u < NU; ++u)
            if (u < m) ko[u] = -b[NX + u];
        }
      }
    }
    // (9) carry V_i, v_i
#pragma unroll
    for (int r = 0; r < NX; ++r) Vc[r] = (j < NX) ? U[r] : 0.0;
    __syncwarp();  // everyone done reading vs (v_{i+1}) and the stage buffer
    if (j == 0) {
#pragma unroll
      for (int r = 0; r < NX; ++r) vs[r] = b[r];
    }
    __syncwarp();
  }

  // ---- x_0 = (I + δV_0)⁻¹ (c_0 - δ v_0) ----
  cholS(Vc, 0);
  double xr[NX];  // x_i replicated in every lane of the group
  {
    double t0[NX];
#pragma unroll
    for (int r = 0; r < NX; ++r) t0[r] = (r < n) ? (a.p.c0[inst * n + r] - delta * vs[r]) : 0.0;
    cholSolve(t0);
#pragma unroll
    for (int r = 0; r < NX; ++r) xr[r] = t0[r];
  }

  // ---- status of the backward sweep, combined over the group ----
  int64_t key = status_key(st);
#pragma unroll
  for (int off = LG / 2; off > 0; off >>= 1) {
    const int64_t o = __shfl_xor_sync(RR_FULL_MASK, key, off);
    key = o > key ? o : key;
  }
  int32_t status = key < 0 ? 0 : (int32_t)(((key >> 8) << 8) | (key & 0xff));

  // ---- forward sweep: y_i = V_i x_i + v_i, u_i = K_i x_i + k_i, x_{i+1} = Φ_i x_i + φ_i ----
  bool bad = false;
  double* xo = a.s.x + inst * (sN + 1) * n;
  double* uo = a.s.u + inst * sN * m;
  double* yo = a.s.y + inst * (sN + 1) * n;
  const int ui = j - NX;  // control row owned by this lane (if 0 <= ui < m)
  // register prefetch of record i: row j of Φ, V (lanes < NX) or row ui of K (lanes NX..)
  double pr_Phi[NX], pr_V[NX], pr_phi = 0.0, pr_v = 0.0;
  auto load_rec = [&](int i) {
    const double* rec = rec0 + (int64_t)i * LY::REC_PAD;
    if (j < NX) {
#pragma unroll
      for (int k = 0; k < NX; ++k) {
        pr_Phi[k] = rec[k * NX + j];
        pr_V[k] = rec[NX * NX + NX + NU * NX + NU + k * NX + j];
      }
      pr_phi = rec[NX * NX + j];
      pr_v = rec[2 * NX * NX + NX + NU * NX + NU + j];
    } else if (ui >= 0 && ui < NU) {
#pragma unroll
      for (int k = 0; k < NX; ++k) pr_Phi[k] = rec[NX * NX + NX + k * NU + ui];
      pr_phi = rec[NX * NX + NX + NU * NX + ui];
    }
  };
  if (N > 0) load_rec(0);
  // store x_0 (lane j writes element j; xr is replicated so use a shuffle-free select)
  {
    double xj = 0.0;
#pragma unroll
    for (int r = 0; r < NX; ++r) xj = (r == j) ? xr[r] : xj;
    if (valid && j < n) xo[j] = xj;
    bad |= (j < n) && !isfinite(xj);
  }
  for (int i = 0; i < N; ++i) {
    double cPhi[NX], cV[NX];
#pragma unroll
    for (int k = 0; k < NX; ++k) {
      cPhi[k] = pr_Phi[k];
      cV[k] = pr_V[k];
    }
    const double cphi = pr_phi, cv = pr_v;
    if (i + 1 < N) load_rec(i + 1);
    double acc1 = cphi, acc2 = cv;
#pragma unroll
    for (int k = 0; k < NX; ++k) {
      acc1 = fma(cPhi[k], xr[k], acc1);
      acc2 = fma(cV[k], xr[k], acc2);
    }
    // lanes < NX: acc1 = x_{i+1}[j], acc2 = y_i[j];  lanes NX..: acc1 = u_i[ui]
    if (valid) {
      if (j < n) yo[(int64_t)i * n + j] = acc2;
      if (ui >= 0 && ui < m) uo[(int64_t)i * m + ui] = acc1;
      if (j < n) xo[(int64_t)(i + 1) * n + j] = acc1;
    }
    bad |= ((j < n) && !(isfinite(acc1) && isfinite(acc2))) || ((ui >= 0 && ui < m) && !isfinite(acc1));
#pragma unroll
    for (int r = 0; r < NX; ++r) xr[r] = __shfl_sync(RR_FULL_MASK, acc1, gbase + r);
  }
  // y_N = Q_N x_N + q_N
  {
    const double* QN = a.p.QN + inst * sn;
    if (j < n) {
      double acc = a.p.qN[inst * n + j];
#pragma unroll
      for (int k = 0; k < NX; ++k)
        if (k < n) acc = fma(k >= j ? QN[pidx(n, k, j)] : QN[pidx(n, j, k)], xr[k], acc);
      if (valid) yo[sN * n + j] = acc;
      bad |= !isfinite(acc);
    }
  }
  const unsigned anybad = __ballot_sync(RR_FULL_MASK, bad);
  const unsigned gmask = (LG == 32) ? 0xffffffffu : (((1u << LG) - 1u) << gbase);
  if (status == 0 && (anybad & gmask)) status = RR_ST_NONFINITE;
  if (valid && status != 0) {  // NaN-fill the failed instance's outputs
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    for (int64_t e = j; e < (sN + 1) * n; e += LG) {
      xo[e] = nan;
      yo[e] = nan;
    }
    for (int64_t e = j; e < sN * m; e += LG) uo[e] = nan;
  }
  if (valid && j == 0) a.status[inst] = status;
}

// ------------------------------------------------------------------------------------------
template <int NX, int NU, int LG, bool EXACT>
struct FusedCfg {
  static constexpr int WARPS = 4;
  static constexpr int IPB = WARPS * (32 / LG);  // instances per block
  static size_t smem_bytes() { return sizeof(double) * (size_t)IPB * FusedLayout<NX, NU>::SLOT_PAD; }
  static int64_t ws_doubles(int64_t batch, int N) { return batch * (int64_t)N * FusedLayout<NX, NU>::REC_PAD; }
  static cudaError_t launch(const FusedArgs& a, cudaStream_t s) {
    auto k = rr_fused_kernel<NX, NU, LG, WARPS, EXACT>;
    const size_t sm = smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    const int64_t blocks = (a.batch + IPB - 1) / IPB;
    k<<<(unsigned)blocks, WARPS * 32, sm, s>>>(a);
    return cudaGetLastError();
  }
};

// Shape dispatch: exact specialisations for the BASELINE configs, padded fallbacks otherwise.
template <typename F>
static bool dispatch_fused(int nx, int nu, F&& f) {
  if (nx == 12 && nu == 4) return f(FusedCfg<12, 4, 16, true>{});
  if (nx == 4 && nu == 1) return f(FusedCfg<4, 1, 8, true>{});
  if (nx == 2 && nu == 1) return f(FusedCfg<2, 1, 4, true>{});
  if (nx <= 2 && nu <= 2) return f(FusedCfg<2, 2, 4, false>{});
  if (nx <= 4 && nu <= 4) return f(FusedCfg<4, 4, 8, false>{});
  if (nx <= 8 && nu <= 8) return f(FusedCfg<8, 8, 16, false>{});
  if (nx <= 16 && nu <= 16) return f(FusedCfg<16, 16, 32, false>{});
  return false;
}

int64_t fused_workspace_bytes(int nx, int nu, int N, int64_t batch) {
  int64_t out = -1;
  dispatch_fused(nx, nu, [&](auto cfg) {
    out = 8 * decltype(cfg)::ws_doubles(batch, N) + 256;
    return true;
  });
  return out;
}

cudaError_t fused_launch(const FusedArgs& a, cudaStream_t s, bool* supported) {
  cudaError_t err = cudaSuccess;
  *supported = dispatch_fused(a.nx, a.nu, [&](auto cfg) {
    err = decltype(cfg)::launch(a, s);
    return true;
  });
  return err;
}

}  // namespace rrk
