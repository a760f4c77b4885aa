// rr_stage.cuh -- per-stage building blocks of the regularized Riccati recursion for one lane
// group (LG lanes) per instance; lane j owns COLUMN j of the stage's (n+m)-wide matrices.
// Used by the fused rr_factor_solve kernel (rr_fused.cu) and the fused ipm_step kernel (ipm.cu).
//
// Method: arXiv 2509.16370, Eq.(RR), forward sweep,
// duals.  P:n = PAPER.md line n.
//
// Per stage (all steps lane-parallel, pivots exchanged through a small shared "publish" buffer):
//   (1) S⁻¹ for S = I + δV_{i+1} by the symmetric sweep operator (Gauss-Jordan in place; S is SPD
//       with eigenvalues >= 1, so no pivoting is needed) -- the (I+δV)⁻¹ of P:616;
//   (2) W_i = S⁻¹ V_{i+1} (product), g_i = v_{i+1} + W(c_{i+1} − δv_{i+1})
//   (3) T = W F, U = Fᵀ T + P with F = [A B]: U holds AᵀWA+Q, H = BᵀWA+Mᵀ, G = BᵀWB+R
//   (4) Gauss-Jordan on the u-block of U and of b = [q + Aᵀg; r + Bᵀg]: the x-columns end as
//       [V_i; −K_i] and b as [v_i; −k_i] (P:621-624 with the HᵀK = KᵀH identities of P:606-611)
//   (5) closed loop for the forward sweep: Φ_i = S⁻¹(A + B K_i), φ_i = S⁻¹(B k_i + c_{i+1} − δv_{i+1})
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rr_common.cuh"

namespace rrk {

// Workspace record written by the backward sweep for the forward sweep, per (instance, stage):
//   Phi NX*NX (col-major) | phi NX | K NU*NX (col-major) | k NU | V packed lower sym(NX) | v NX
template <int NX, int NU>
struct Rec {
  static constexpr int PHI = 0;
  static constexpr int phi = NX * NX;
  static constexpr int K = phi + NX;
  static constexpr int k = K + NU * NX;
  static constexpr int V = k + NU;
  static constexpr int v = V + NX * (NX + 1) / 2;
  static constexpr int SIZE = v + NX;
  static constexpr int PAD = (SIZE + 1) & ~1;
};

// Per-instance shared-memory work area used by the stage step (doubles; all offsets even).
template <int NX, int NU>
struct Work {
  static constexpr int NZ = NX + NU;
  static constexpr int NZP = (NZ + 1) & ~1;
  static constexpr int Si = 0;              // S⁻¹ col-major NX×NX
  static constexpr int pub = Si + NX * NX;  // 2 × NZP pivot-publish buffers
  static constexpr int pq = pub + 2 * NZP;  // pivot column entries of processed u rows (NU, padded)
  static constexpr int vb = pq + ((NU + 1) & ~1);  // b vector (NZ)
  static constexpr int gb = vb + NZP;       // g_i (NX)
  static constexpr int vs = gb + NX;        // v_{i+1} (NX)
  static constexpr int Wb = vs + NX;        // W_i col-major NX×NX (last: the DMMA stage reuses it)
  static constexpr int SIZE = Wb + NX * NX;
  static constexpr int PAD = (SIZE + 1) & ~1;
};

template <int NX, int NU, int LG>
struct Stage {
  static constexpr int NZ = NX + NU;
  using WK = Work<NX, NU>;
  static_assert(NZ <= LG, "lane group narrower than n+m");
  static_assert(NX % 2 == 0, "vectorised smem/global accesses assume an even (padded) NX");

  // broadcast read of NX consecutive doubles (16-byte aligned) from shared memory
  __device__ static __forceinline__ void bcast(const double* src, double (&dst)[NX]) {
#pragma unroll
    for (int r = 0; r < NX; r += 2) {
      const double2 v = *reinterpret_cast<const double2*>(src + r);
      dst[r] = v.x;
      dst[r + 1] = v.y;
    }
  }
  __device__ static __forceinline__ void store_col(double* dst, const double (&src)[NX]) {
#pragma unroll
    for (int r = 0; r < NX; r += 2) reinterpret_cast<double2*>(dst)[r / 2] = make_double2(src[r], src[r + 1]);
  }

  // (1) wk[Si] = (I + δV)⁻¹ by the symmetric sweep operator; lane j holds column j of V in Vc.
  // Sweep on pivot p (A symmetric): Ã_pp = −1/A_pp, Ã_rp = A_rp/A_pp, Ã_pc = A_pc/A_pp,
  // Ã_rc = A_rc − A_rp A_pc / A_pp; after all pivots Ã = −A⁻¹.  Column p = row p (symmetry), so
  // the pivot column is published by every lane writing its own element p.
  __device__ static __forceinline__ void invS(const double (&Vc)[NX], double delta, int j, double* wk, int stage,
                                              int32_t& st) {
    double A[NX];
#pragma unroll
    for (int r = 0; r < NX; ++r) A[r] = delta * Vc[r] + (r == j ? 1.0 : 0.0);
    bool notpd = false;
#pragma unroll
    for (int p = 0; p < NX; ++p) {
      double col[NX];
      // pivot column = row p (symmetry): every lane publishes its element p, one broadcast read
      // (measured: 12 register shuffles per pivot are 9% slower on the C2 kernel than this)
      double* pb = wk + WK::pub + (p & 1) * WK::NZP;
      if (j < NX) pb[j] = A[p];
      __syncwarp();
      bcast(pb, col);
      const double d = col[p];
      notpd |= !(d > 0.0);
      const double id = rcp_nr(d);
      const double f = (A[p] - (j == p ? 1.0 : 0.0)) * id;
#pragma unroll
      for (int r = 0; r < NX; ++r)
        if (r != p) A[r] = fma(-col[r], f, A[r]);
      A[p] = (j == p) ? -id : f;
    }
    if (notpd && st == 0) st = mk_status(RR_ST_S_NOT_PD, stage);
    if (j < NX) {  // S⁻¹ is symmetric: write column j as row j (consecutive lanes, conflict-free)
#pragma unroll
      for (int r = 0; r < NX; ++r) wk[WK::Si + r * NX + j] = -A[r];
    }
    __syncwarp();
  }

  // X <- S⁻¹ X (S⁻¹ in wk[Si], broadcast columns)
  __device__ static __forceinline__ void mulSinv(double (&X)[NX], const double* wk) {
    double Y[NX];
#pragma unroll
    for (int r = 0; r < NX; ++r) Y[r] = 0.0;
#pragma unroll
    for (int k = 0; k < NX; ++k) {
      const double* Sk = wk + WK::Si + k * NX;
#pragma unroll
      for (int r = 0; r < NX; r += 2) {
        const double2 s2 = *reinterpret_cast<const double2*>(Sk + r);
        Y[r] = fma(s2.x, X[k], Y[r]);
        Y[r + 1] = fma(s2.y, X[k], Y[r + 1]);
      }
    }
#pragma unroll
    for (int r = 0; r < NX; ++r) X[r] = Y[r];
  }

  // One backward step of Eq.(RR) at stage i.
  //   F:    stage F = [A_i B_i] column-major (NX rows, ld NX; padded rows/cols zero), 16-byte aligned
  //   cv:   c_{i+1} (NX)
  //   Pcol: functor s -> P_i[s][j], P_i = [[Q M];[Mᵀ R]] (padded u-diagonal 1)
  //   qj:   j-th entry of (q_i; r_i)
  //   Vc:   in: column j of V_{i+1};  out: column j of V_i (lanes j < NX)
  //   wk[vs]: in: v_{i+1};  out: v_i
  //   rec:  workspace record for stage i (nullptr: not written)
  // Returns U (lanes j < NX: V_i column j | −K_i column j) and b (v_i | −k_i, replicated).
  template <typename PFun>
  __device__ static __forceinline__ void backward(const double* F, const double* cv, PFun&& Pcol, double qj,
                                                  double delta, int j, double* wk, double (&Vc)[NX],
                                                  double (&U)[NZ], double (&b)[NZ], double* rec, int stage,
                                                  int32_t& st) {
    // (1) S⁻¹
    invS(Vc, delta, j, wk, stage, st);
    // (2) W = S⁻¹ V_{i+1} (column j; W symmetric so also row j); g_i = v_{i+1} + W(c_{i+1} − δv_{i+1})
    double X[NX];
#pragma unroll
    for (int r = 0; r < NX; ++r) X[r] = Vc[r];
    mulSinv(X, wk);
    if (j < NX) {
      store_col(wk + WK::Wb + j * NX, X);
      double g0 = wk[WK::vs + j], g1 = 0.0;
#pragma unroll
      for (int k = 0; k < NX; ++k) {
        const double e = cv[k] - delta * wk[WK::vs + k];
        if (k & 1) g1 = fma(X[k], e, g1);
        else g0 = fma(X[k], e, g0);
      }
      wk[WK::gb + j] = g0 + g1;
    }
    __syncwarp();
    // (3) T = W F (column j), U = Fᵀ T + P (column j)
    const int jc = (j < NZ) ? j : 0;
    double Fc[NX];
#pragma unroll
    for (int k = 0; k < NX; k += 2) {
      const double2 f2 = *reinterpret_cast<const double2*>(F + jc * NX + k);
      Fc[k] = (j < NZ) ? f2.x : 0.0;
      Fc[k + 1] = (j < NZ) ? f2.y : 0.0;
    }
    double T[NX];
#pragma unroll
    for (int r = 0; r < NX; ++r) T[r] = 0.0;
#pragma unroll
    for (int k = 0; k < NX; ++k) {
      const double* Wk = wk + WK::Wb + k * NX;
#pragma unroll
      for (int r = 0; r < NX; r += 2) {
        const double2 w2 = *reinterpret_cast<const double2*>(Wk + r);
        T[r] = fma(w2.x, Fc[k], T[r]);
        T[r + 1] = fma(w2.y, Fc[k], T[r + 1]);
      }
    }
#pragma unroll
    for (int s = 0; s < NZ; ++s) {
      const double* Fs = F + s * NX;
      double a0 = Pcol(s), a1 = 0.0;
#pragma unroll
      for (int k = 0; k < NX; k += 2) {
        const double2 f2 = *reinterpret_cast<const double2*>(Fs + k);
        a0 = fma(f2.x, T[k], a0);
        a1 = fma(f2.y, T[k + 1], a1);
      }
      U[s] = a0 + a1;
    }
    // b_j = [q + Aᵀ g ; r + Bᵀ g]_j
    {
      double gk[NX];
      bcast(wk + WK::gb, gk);
      double b0 = qj, b1 = 0.0;
#pragma unroll
      for (int k = 0; k < NX; k += 2) {
        b0 = fma(Fc[k], gk[k], b0);
        b1 = fma(Fc[k + 1], gk[k + 1], b1);
      }
      if (j < NZ) wk[WK::vb + j] = b0 + b1;
    }
    __syncwarp();
#pragma unroll
    for (int s = 0; s < NZ; ++s) b[s] = wk[WK::vb + s];
    // (4) Gauss-Jordan on the u-block.  Pivot column p: rows in x and unprocessed u equal row p
    // (the unprocessed part is a symmetric Schur complement), published by every lane; rows of
    // already processed pivots come from lane p itself.
#pragma unroll
    for (int p = NX; p < NZ; ++p) {
      double* pb = wk + WK::pub + (p & 1) * WK::NZP;
      if (j < NZ) pb[j] = U[p];
      if (j == p) {
#pragma unroll
        for (int q = NX; q < p; ++q) wk[WK::pq + (q - NX)] = U[q];
      }
      __syncwarp();
      double col[NZ];
#pragma unroll
      for (int s = 0; s < NZ; ++s) col[s] = (s >= NX && s < p) ? wk[WK::pq + (s - NX)] : pb[s];
      const double piv = col[p];
      if (!(piv > 0.0) && st == 0) st = mk_status(RR_ST_G_NOT_PD, stage);
      const double ip = rcp_nr(piv);
      const double rp = U[p] * ip;
      const double bp = b[p] * ip;
#pragma unroll
      for (int s = 0; s < NZ; ++s) {
        if (s == p) continue;
        U[s] = fma(-col[s], rp, U[s]);
        b[s] = fma(-col[s], bp, b[s]);
      }
      U[p] = rp;
      b[p] = bp;
      __syncwarp();  // pq is rewritten by the next pivot
    }
    // lanes j < NX: U[0..NX) = V_i[:, j], U[NX..) = −K_i[:, j];  b = [v_i ; −k_i]
    // (5) Φ_i = S⁻¹(A + B K_i) (lanes j < NX);  φ_i = S⁻¹(B k_i + c_{i+1} − δ v_{i+1}) (lane NX)
    double t[NX];
#pragma unroll
    for (int r = 0; r < NX; ++r) t[r] = (j < NX) ? Fc[r] : ((j == NX) ? (cv[r] - delta * wk[WK::vs + r]) : 0.0);
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const double coef = (j < NX) ? -U[NX + u] : ((j == NX) ? -b[NX + u] : 0.0);
      const double* Fu = F + (NX + u) * NX;
#pragma unroll
      for (int r = 0; r < NX; r += 2) {
        const double2 f2 = *reinterpret_cast<const double2*>(Fu + r);
        t[r] = fma(f2.x, coef, t[r]);
        t[r + 1] = fma(f2.y, coef, t[r + 1]);
      }
    }
    mulSinv(t, wk);
    // (6) record for the forward sweep
    if (rec != nullptr) {
      using RC = Rec<NX, NU>;
      if (j < NX) {
        store_col(rec + RC::PHI + j * NX, t);
#pragma unroll
        for (int u = 0; u < NU; ++u) rec[RC::K + j * NU + u] = -U[NX + u];
        double* Vp = rec + RC::V + j * (2 * NX - j - 1) / 2;  // packed column j starts at row j
#pragma unroll
        for (int r = 0; r < NX; ++r)
          if (r >= j) Vp[r] = U[r];
      } else if (j == NX) {
        store_col(rec + RC::phi, t);
#pragma unroll
        for (int r = 0; r < NX; ++r) rec[RC::v + r] = b[r];
#pragma unroll
        for (int u = 0; u < NU; ++u) rec[RC::k + u] = -b[NX + u];
      }
    }
    // (7) carry V_i (lanes j < NX), v_i
#pragma unroll
    for (int r = 0; r < NX; ++r) Vc[r] = (j < NX) ? U[r] : 0.0;
    __syncwarp();  // all reads of vs (v_{i+1}), F, cv, Si done
    if (j == 0) {
#pragma unroll
      for (int r = 0; r < NX; ++r) wk[WK::vs + r] = b[r];
    }
    __syncwarp();
  }
};

}  // namespace rrk
