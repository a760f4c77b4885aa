// rr_stage_mma.cuh -- backward step of Eq.(RR) with the dense stage contractions on the FP64
// tensor-core path (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4), two instances per warp.
//
// Method: arXiv 2509.16370, Eq.(RR) and the forward-sweep quantities of P:496-509.
// Why: with one lane per column the SIMT products need one 128-bit shared-memory broadcast per
// two FMAs, which caps them at ~50% of the FP64 pipe (profiles/r01_*).  DMMA consumes register
// fragments with 8×8 reuse inside the unit (256 FMA per instruction), so the products run on
// the FP64 pipe with half the shared-memory traffic.  tcgen05 has no FP64 kind; DMMA runs on the
// same FP64 units (measured 37.1 TF/s vs 34.1 TF/s DFMA, profiles/r01_k0_fp64_probe.txt).
//
// Matrices are padded to 16×16 tiles (two 8-row × two 8-column DMMA tiles); valid extents:
// NX (states), NZ = NX + NU (stage columns), NX % 4 == 0 (K blocks of 4), NZ <= 16.
// Fragment layouts of m8n8k4.row.col.f64 (g = lane>>2, t = lane&3):
//   A (8×4): a = A[g][t];  B (4×8): b = B[t][g];  C (8×8): c0 = C[g][2t], c1 = C[g][2t+1].
// Per stage, lane group q (16 lanes, instance q of the warp) runs the SIMT parts; the whole warp
// runs the DMMA parts for instance 0 then instance 1:
//   (1) SIMT  S⁻¹ (symmetric sweep, rr_stage.cuh); Vs = [V_{i+1} | V_{i+1} e], e = c_{i+1} − δ v_{i+1}
//   (2) DMMA  [W | W e] = S⁻¹ Vs                       (W = (I+δV)⁻¹V; g = v + W e)
//   (3) SIMT  g, b = [q + Aᵀg; r + Bᵀg]
//   (4) DMMA  T = W F                                   (F = [A B])
//   (5) DMMA  U = Fᵀ T + P                              (AᵀWA+Q, H = BᵀWA+Mᵀ, G = BᵀWB+R)
//   (6) SIMT  Gauss-Jordan on the u-block of U and b    (−K_i, V_i, −k_i, v_i)
//   (7) SIMT  M = [A + B K_i | B k_i + c_{i+1} − δ v_{i+1}]
//   (8) DMMA  [Φ_i | φ_i] = S⁻¹ M -> workspace record (row-major, ld NX+2)
#pragma once
#include "rr_stage.cuh"

namespace rrk {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
#ifdef RR_DMMA_VOLATILE
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
#else
  // not volatile: a pure register operation, so the compiler may interleave independent chains
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
#endif
}

// Workspace record of the MMA kernel (per instance and stage):
//   S_{i+1}⁻¹ packed | K_i | k_i | V_i packed | v_i | e_i = c_{i+1} − δv_{i+1}
// forward: x⁺ = S⁻¹(A x + B u + e) with A, B re-read by TMA, so the backward needs no closed-loop
// products (measured 15.4 -> 14.6 ms on C2 against a [Φ | φ] record, round 1).
template <int NX, int NU>
struct RecM {
  static constexpr int S = 0;
  static constexpr int K = NX * (NX + 1) / 2;
  static constexpr int k = K + NU * NX;
  static constexpr int V = k + NU;
  static constexpr int v = V + NX * (NX + 1) / 2;
  static constexpr int e = v + NX;
  static constexpr int SIZE = e + NX;
  static constexpr int PAD = (SIZE + 1) & ~1;
};

// Per-instance work area of the MMA stage (doubles, even offsets).  The SIMT helpers of
// rr_stage.cuh address Si, pub, pq, vb, gb, vs through Work<NX, NU>; WorkM places X1/X2 over
// Work's (unused here) Wb slot and beyond so that the whole slot stays small.
template <int NX, int NU>
struct WorkM {
  static constexpr int NZ = NX + NU;
  using W = Work<NX, NU>;
  static_assert(W::Wb + NX * NX == W::SIZE, "Work<> must end with Wb");
  static constexpr int ULD = 18;                // U leading dimension: conflict-free C-fragment stores
  // one region per instance, reused within a stage: [V | Ve] rows (ld NX; the B operand of W = S⁻¹Vs),
  // then U (col-major, ld ULD; written once W is formed, read by the u-block elimination), then the
  // forward record staged for its TMA bulk store (after the elimination holds U in registers)
  static constexpr int X = W::Wb;
  static constexpr int X1 = X, X2 = X;
  static constexpr int XSZ = 16 * ULD;
  static_assert(XSZ >= NX * NX + NX && XSZ >= NZ * ULD - (ULD - NZ), "X must hold Vs and U");
  static constexpr int E = X + XSZ;             // e = c_{i+1} − δ v_{i+1} (NX, even)
  static constexpr int BP = E + ((NX + 1) & ~1);  // 2 publish slots for b_p in the u-block elimination
  static constexpr int SIZE = BP + 2;
  static constexpr int PAD = (SIZE + 1) & ~1;
};

// W and T live in shared memory row-major with a row stride of 16 doubles and the 16-byte column
// pairs XOR-swizzled by σ(r) = 4(r&1) + 2((r>>1)&1): C-fragment pair stores (c0, c1 adjacent), A-fragment
// loads (row r, column k) and B-fragment loads (row k, column n) are then all free of bank conflicts
// (each quarter-warp of 128-bit stores and each half-warp of 64-bit loads hits distinct banks).
__device__ __forceinline__ int swz16(int r, int c) {
  return 16 * r + 2 * ((c >> 1) ^ (4 * (r & 1) + 2 * ((r >> 1) & 1))) + (c & 1);
}

template <int NX, int NU>
struct StageMMA {
  static constexpr int NZ = NX + NU;
  static constexpr int LG = 16;
  static constexpr int KT = NX / 4;          // K blocks over the state dimension
  static constexpr int MT = (NX + 7) / 8;    // row tiles over states
  static constexpr int ZT = (NZ + 7) / 8;    // tiles over stage columns
  static constexpr int CT = (NX + 1 + 7) / 8;  // tiles over NX+1 columns ([W | We], [Φ | φ])
  static_assert(NX % 4 == 0 && NZ <= 16 && NX + 1 <= 16, "MMA stage needs NX % 4 == 0 and NX + NU <= 16");
  using ST = Stage<NX, NU, 16>;
  using WK = Work<NX, NU>;
  using WM = WorkM<NX, NU>;
  using RC = RecM<NX, NU>;

  // one backward step for the two instances of the warp.
  //   wkq[q]: work area of instance q; Fq/cvq: stage F / c_{i+1} of instance q (stage buffer)
  //   Pat(q, s, t): P_i[s][t] of instance q;  qjf(): this lane's entry of (q_i; r_i)
  //   wait_inputs(): waits for this stage's input copies (called after the S⁻¹ sweep, which needs
  //   none);  prefetch(): issues the next stage's input copies (called once the inputs are dead)
  // S⁻¹ = (I + δV)⁻¹ by the symmetric sweep operator on a 4 × 4 lane grid of 3 × 3 blocks (NX = 12):
  // lane (R, C) = (j / 4, j % 4) holds A[3R..3R+2][3C..3C+2].  Per pivot p the four lanes of block
  // column p / 3 publish their rows of column p (= row p by symmetry); every lane reads the 3 entries
  // of its rows and the 3 of its columns (8 distinct addresses per warp-wide load instead of the 12
  // broadcasts of the column-per-lane sweep), then updates its 9 entries.  V is read from Vs = X1
  // (column-major, written by the caller), S⁻¹ = −A is stored to wk[Si] (column-major, symmetric).
  __device__ static __forceinline__ void invS_grid(double* wk, double delta, int j, int stage, int32_t& st) {
    static_assert(NX == 12, "grid sweep is laid out for NX = 12 (4 x 4 lanes of 3 x 3 blocks)");
    const int R = j >> 2, C = j & 3;
    double a[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int k = 0; k < 3; ++k)
        a[i][k] = delta * wk[WM::X1 + (3 * C + k) * NX + 3 * R + i] + ((3 * R + i == 3 * C + k) ? 1.0 : 0.0);
    bool notpd = false;
#pragma unroll
    for (int p = 0; p < NX; ++p) {
      double* pb = wk + WK::pub + (p & 1) * WK::NZP;
      const int pc = p / 3, pk = p % 3;
      if (C == pc) {
#pragma unroll
        for (int i = 0; i < 3; ++i) pb[3 * R + i] = a[i][pk];
      }
      __syncwarp();
      double cr[3], cc[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        cr[i] = pb[3 * R + i];  // A[3R+i][p]
        cc[i] = pb[3 * C + i];  // A[p][3C+i] = A[3C+i][p]
      }
      const double d = pb[p];
      notpd |= !(d > 0.0);
      const double id = rcp_nr(d);
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const bool rp = (3 * R + i == p);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const bool cp = (3 * C + k == p);
          const double upd = fma(-cr[i] * id, cc[k], a[i][k]);
          a[i][k] = rp ? (cp ? -id : cc[k] * id) : (cp ? cr[i] * id : upd);
        }
      }
    }
    if (notpd && st == 0) st = mk_status(RR_ST_S_NOT_PD, stage);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int k = 0; k < 3; ++k) wk[WK::Si + (3 * C + k) * NX + 3 * R + i] = -a[i][k];
    __syncwarp();
  }

  // FAC = true: the factorization only (rr_factor): no Φ / φ, the u-block is eliminated with the
  // symmetric sweep operator (−G⁻¹ lands in the u-columns) and recq[q] points at factor record i
  // [V_i | S_i⁻¹ | K_i | G_i⁻¹] (record i+1 receives S_{i+1}⁻¹).
  // RT: element type of the records (double; float for the FP32 factor record of rr_factor,
  // RR_FLAG_FACTOR_FP32 -- FAC only)
  template <bool FAC = false, typename RT = double, typename PFun, typename QFun, typename WaitFn, typename PrefFn>
  __device__ static __forceinline__ void backward(double* const (&wkq)[2], const double* const (&Fq)[2],
                                                  const double* const (&cvq)[2], PFun&& Pat, QFun&& qjf,
                                                  WaitFn&& wait_inputs, PrefFn&& prefetch, double delta, int grp,
                                                  int j, int lane, double (&Vc)[NX], double (&U)[NZ],
                                                  double& bj, RT* const (&recq)[2], int stage,
                                                  int32_t& st) {
    double* wk = grp ? wkq[1] : wkq[0];
    const double* F = grp ? Fq[1] : Fq[0];
    const double* cv = grp ? cvq[1] : cvq[0];
    const int g = lane >> 2, t = lane & 3;
    // (1) S⁻¹ (no stage input needed), then Vs = [V | V e] (V symmetric: (V e)_j = column j · e)
#ifndef RR_REC_STG
    if (lane == 0) bulk_wait_read0();  // the previous stage's record bulk stores have read X (Vs goes there)
    __syncwarp();
#endif
#ifndef RR_INVS_GRID
#ifdef RR_AB_SKIP_INVS  // A/B probe only: cost of the SIMT S⁻¹ sweep (wrong results)
    if (j < NX) {
#pragma unroll
      for (int r = 0; r < NX; ++r) wk[WK::Si + r * NX + j] = (r == j) ? 1.0 : 0.0;
    }
    __syncwarp();
#else
    ST::invS(Vc, delta, j, wk, stage, st);
#endif
    if (j < NX) {
#pragma unroll
      for (int r = 0; r < NX; ++r) wk[WM::X1 + r * NX + j] = Vc[r];  // V symmetric: column j as row j
    }
#else  // 4 × 4 grid sweep: measured 6% slower on C2 (more scalar loads and selects per pivot)
    if (j < NX) {
#pragma unroll
      for (int r = 0; r < NX; ++r) wk[WM::X1 + r * NX + j] = Vc[r];
    }
    __syncwarp();
    invS_grid(wk, delta, j, stage, st);
#endif
    wait_inputs();
    if (j < NX) wk[WM::E + j] = cv[j] - delta * wk[WK::vs + j];  // e = c_{i+1} − δ v_{i+1}
    __syncwarp();
    if (j < NX) {
      double ek[NX];
      ST::bcast(wk + WM::E, ek);
      double ve0 = 0.0, ve1 = 0.0;
#pragma unroll
      for (int k = 0; k < NX; k += 2) {
        ve0 = fma(Vc[k], ek[k], ve0);
        ve1 = fma(Vc[k + 1], ek[k + 1], ve1);
      }
      wk[WM::X1 + NX * NX + j] = ve0 + ve1;  // column NX of Vs
    }
    __syncwarp();
    // (2)-(5) per instance q, in DMMA registers: [W | We] = S⁻¹ Vs, X = Fᵀ W, U = Fᵀ Xᵀ + P.
    // A C fragment holds C[g][2t], C[g][2t+1]; used with the contraction index permuted to
    // k-blocks {2t + 8kt} and {2t + 1 + 8kt} it IS the A fragment of C (row g, "column" t) and, for
    // a symmetric or transposed use, the B fragment -- so W and X never round-trip through shared
    // memory (the previous T = W F / U = Fᵀ T chain stored W and T and re-read both as fragments).
    // Only Fᵀ is loaded, as 128-bit pairs (k, k+1) straight from the TMA stage buffer.
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const double* Si = wkq[q] + WK::Si;
      const double* Vs = wkq[q] + WM::X1;
      double w[MT][CT][2];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < CT; ++nt) w[mt][nt][0] = w[mt][nt][1] = 0.0;
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) {
        double aS[MT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int r = 8 * mt + g;
          aS[mt] = (r < NX) ? Si[(4 * kt + t) * NX + r] : 0.0;
        }
#pragma unroll
        for (int nt = 0; nt < CT; ++nt) {
          const int col = 8 * nt + g;
          const double bv = (col <= NX) ? Vs[col * NX + 4 * kt + t] : 0.0;
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) dmma884(w[mt][nt][0], w[mt][nt][1], aS[mt], bv);
        }
      }
      // g = v + W e (column NX of [W | We]: tile nt = NX / 8, lanes 2t + e = NX % 8)
      if (2 * t == (NX & 7)) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int r = 8 * mt + g;
          if (r < NX) wkq[q][WK::gb + r] = wkq[q][WK::vs + r] + w[mt][NX >> 3][0];
        }
      }
      // Fᵀ A fragments, k permuted: fa[mt][kt][e] = Fᵀ[8mt + g][2t + e + 8kt] (zero outside NZ × NX)
      const double* Fx = Fq[q];
      double fa[ZT][2][2];
#pragma unroll
      for (int mt = 0; mt < ZT; ++mt)
#pragma unroll
        for (int kt = 0; kt < 2; ++kt) {
          const int mm = 8 * mt + g, k0 = 2 * t + 8 * kt;
          double2 f2 = make_double2(0.0, 0.0);
          if (mm < NZ && k0 < NX) f2 = *reinterpret_cast<const double2*>(Fx + mm * NX + k0);
          fa[mt][kt][0] = f2.x;
          fa[mt][kt][1] = f2.y;
        }
      // B fragments of W (symmetric): B[k][n] = W[n][k] = w[nt][kt][e] at k = 2t + e + 8kt, n = 8nt + g;
      // k >= NX (the We column and padding) excluded
      double x[ZT][MT][2];
#pragma unroll
      for (int mt = 0; mt < ZT; ++mt)
#pragma unroll
        for (int nt = 0; nt < MT; ++nt) x[mt][nt][0] = x[mt][nt][1] = 0.0;
#pragma unroll
      for (int kt = 0; kt < 2; ++kt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (8 * kt >= NX) continue;
#pragma unroll
          for (int nt = 0; nt < MT; ++nt) {
            const double wb = (2 * t + e + 8 * kt < NX) ? w[nt][kt][e] : 0.0;
#pragma unroll
            for (int mt = 0; mt < ZT; ++mt) dmma884(x[mt][nt][0], x[mt][nt][1], fa[mt][kt][e], wb);
          }
        }
      // U = Fᵀ Xᵀ + P: B[k][n] = X[n][k] = x[nt][kt][e] (own C fragment of X), C initialised with P
      double c[ZT][ZT][2];
#pragma unroll
      for (int mt = 0; mt < ZT; ++mt)
#pragma unroll
        for (int nt = 0; nt < ZT; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
#if defined(RR_NO_PTAB)
            const int r = 8 * mt + g, col = 8 * nt + 2 * t + e;
            c[mt][nt][e] = (r < NZ && col < NZ) ? Pat(q, r, col) : 0.0;
#elif !defined(RR_P_SIMT)
            c[mt][nt][e] = Pat(q, (mt * ZT + nt) * 2 + e);  // P-gather table (kernel)
#else
            c[mt][nt][e] = 0.0;
#endif
          }
#pragma unroll
      for (int kt = 0; kt < 2; ++kt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (8 * kt >= NX) continue;
#pragma unroll
          for (int nt = 0; nt < ZT; ++nt) {
            const double xb = x[nt][kt][e];  // X[8nt + g][2t + e + 8kt]
#pragma unroll
            for (int mt = 0; mt < ZT; ++mt) dmma884(c[mt][nt][0], c[mt][nt][1], fa[mt][kt][e], xb);
          }
        }
      double* Ub = wkq[q] + WM::X2;
      __syncwarp();  // U overwrites Vs (same region X): every lane's Vs fragment loads are done
#pragma unroll
      for (int mt = 0; mt < ZT; ++mt)
#pragma unroll
        for (int nt = 0; nt < ZT; ++nt) {
          const int r = 8 * mt + g, col = 8 * nt + 2 * t;
          Ub[col * WM::ULD + r] = c[mt][nt][0];
          Ub[(col + 1) * WM::ULD + r] = c[mt][nt][1];
        }
    }
    __syncwarp();
    // (3) b_j = [q + Aᵀg; r + Bᵀg]_j  (g from (2), per instance)
    const int jc = (j < NZ) ? j : 0;
    {
      double gk[NX];
      ST::bcast(wk + WK::gb, gk);
      double b0 = qjf(), b1 = 0.0;
      const bool rot = (j & 4) != 0;
#pragma unroll
      for (int k = 0; k < NX; k += 2) {
        const int kr = (k + 2) % NX;
        const double2 f2 = *reinterpret_cast<const double2*>(F + jc * NX + (rot ? kr : k));
        b0 = fma(f2.x, rot ? gk[kr] : gk[k], b0);
        b1 = fma(f2.y, rot ? gk[kr + 1] : gk[k + 1], b1);
      }
      bj = b0 + b1;
    }
    // (6) Gauss-Jordan on the u-block (SIMT, lane j owns column j)
#pragma unroll
    for (int s = 0; s < NZ; s += 2) {
      const double2 u2 = *reinterpret_cast<const double2*>(wk + WM::X2 + jc * WM::ULD + s);
      U[s] = (j < NZ) ? u2.x : 0.0;
      U[s + 1] = (j < NZ) ? u2.y : 0.0;
    }
#if !defined(RR_NO_PTAB) && defined(RR_P_SIMT)
    // U = FᵀWF + P: lane j adds column j of P (packed Q / M / R of its own instance's stage)
#pragma unroll
    for (int s = 0; s < NZ; ++s) U[s] += Pat(s);
#endif
    // b is distributed: lane j updates its own entry b_j with the pivot-column entry of row j
    // (own U[p] by symmetry, or lane p's published row for already processed pivots) and the
    // published b_p
    bool gbad = false;
#ifndef RR_AB_SKIP_GJ  // A/B probe only: cost of the u-block elimination (wrong results)
#pragma unroll
    for (int p = NX; p < NZ; ++p) {
      double* pb = wk + WK::pub + (p & 1) * WK::NZP;
      if (j < NZ) pb[j] = U[p];
      if (j == p) {
#pragma unroll
        for (int qq = NX; qq < p; ++qq) wk[WK::pq + (qq - NX)] = U[qq];
        wk[WM::BP + (p & 1)] = bj;
      }
      __syncwarp();
      double col[NZ];
#pragma unroll
      for (int s = 0; s < NZ; s += 2) {  // published row p (= column p) as 128-bit broadcasts
        const double2 v2 = *reinterpret_cast<const double2*>(pb + s);
        col[s] = v2.x;
        col[s + 1] = v2.y;
      }
      if (!FAC) {  // rows of already processed pivots: lane p's own column (GJ is not symmetric there)
#pragma unroll
        for (int s = NX; s < p; ++s) col[s] = wk[WK::pq + (s - NX)];
      }
      const double cj = (!FAC && j >= NX && j < p) ? wk[WK::pq + (j - NX)] : U[p];  // pivot-column entry of row j
      const double piv = col[p];
      gbad |= !(piv > 0.0);
      const double ip = rcp_nr(piv);
      const double rp = U[p] * ip;
      const double bp = wk[WM::BP + (p & 1)] * ip;
      if (FAC && j == p) {  // symmetric sweep: pivot column scaled, pivot -> −1/piv
#pragma unroll
        for (int s = 0; s < NZ; ++s) U[s] = (s == p) ? -ip : U[s] * ip;
      } else {
#pragma unroll
        for (int s = 0; s < NZ; ++s) {
          if (s == p) continue;
          U[s] = fma(-col[s], rp, U[s]);
        }
        U[p] = rp;
      }
      bj = (j == p) ? bp : fma(-cj, bp, bj);
      __syncwarp();
    }
#endif
    if (gbad && st == 0) st = mk_status(RR_ST_G_NOT_PD, stage);
    // lanes j < NX: U = [V_i; −K_i] column j, bj = (v_i)_j;  lanes NX + u: bj = −(k_i)_u
    if (j < NZ) wk[WK::vb + j] = bj;
    __syncwarp();
    if constexpr (FAC) {  // factor record i (and S_{i+1}⁻¹ into record i+1); no closed loop
      __syncwarp();
      prefetch();
      constexpr int SN = NX * (NX + 1) / 2;
      constexpr int RECD = (NX * (NX + 1) + NX * NU + NU * (NU + 1) / 2 + 1) & ~1;
      constexpr int REC = sizeof(RT) == 4 ? ((RECD + 3) & ~3) : RECD;  // FP32 records: 16-byte multiple
      // FP64 records: staged in X in the record layout [V_i | S_{i+1}⁻¹ | K_i | G_i⁻¹] and written by three
      // TMA bulk stores (V, K, G⁻¹ -> record i; S_{i+1}⁻¹ -> record i+1's S slot); FP32: direct stores
      constexpr bool STAGE = sizeof(RT) == 8 && (SN % 2) == 0 && ((RECD - 2 * SN) % 2) == 0;
      RT* const grec = grp ? recq[1] : recq[0];
      RT* rec = grec;
      RT* recS = grec != nullptr ? grec + REC : nullptr;  // record i+1 (its S slot at + SN)
      if constexpr (STAGE) {
        rec = grec != nullptr ? reinterpret_cast<RT*>(wk + WM::X) : nullptr;
        recS = rec;
      }
      if (rec != nullptr) {
        if (j < NX) {
          // row j (= column j) of the symmetric V_i and S_{i+1}⁻¹ along packed columns: entries (j, c),
          // c <= j, at c(2n − c − 1)/2 + j (consecutive lanes, consecutive addresses)
#pragma unroll
          for (int c = 0; c < NX; ++c)
            if (c <= j) {
              const int pc = c * (2 * NX - c - 1) / 2 + j;
              rec[pc] = (RT)U[c];
              recS[SN + pc] = (RT)wk[WK::Si + c * NX + j];
            }
#pragma unroll
          for (int u = 0; u < NU; ++u) rec[2 * SN + j * NU + u] = (RT)(-U[NX + u]);
        } else if (j < NZ) {
          const int w = j - NX;
          RT* Gp = rec + 2 * SN + NX * NU + w * (2 * NU - w - 1) / 2;
#pragma unroll
          for (int u = 0; u < NU; ++u)
            if (u >= w) Gp[u] = (RT)(-U[NX + u]);
        }
      }
      if constexpr (STAGE) {
        static_assert(RECD <= WM::XSZ, "factor record staging needs X");
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (recq[q] == nullptr) continue;
            const double* xs = wkq[q] + WM::X;
            double* gr = reinterpret_cast<double*>(recq[q]);
            bulk_s2g(gr, xs, 8u * SN);                                     // V_i
            bulk_s2g(gr + 2 * SN, xs + 2 * SN, 8u * (RECD - 2 * SN));       // K_i | G_i⁻¹ (| pad)
            bulk_s2g(gr + REC + SN, xs + SN, 8u * SN);                       // S_{i+1}⁻¹ -> record i+1
          }
          bulk_commit();
        }
      }
#pragma unroll
      for (int r = 0; r < NX; ++r) Vc[r] = (j < NX) ? U[r] : 0.0;
      __syncwarp();
      return;
    }
    {  // record: S_{i+1}⁻¹, e, K, k, V, v (no closed-loop products)
      __syncwarp();
      prefetch();
#ifndef RR_REC_STG
      // staged in this instance's X2 (U is in registers since the elimination) and written to HBM
      // by one TMA bulk store per instance: the scattered 8-byte global stores of the packed columns
      // cost L1 wavefronts on the LSU pipe the kernel is bound by
      double* rec = (grp ? recq[1] : recq[0]) != nullptr ? wk + WM::X2 : nullptr;
#else
      auto* rec = grp ? recq[1] : recq[0];
#endif
      if (rec != nullptr) {
        if (j < NX) {
#ifndef RR_REC_STG
          // row j of the (symmetric) S⁻¹ and V_i: entries (j, c), c <= j, at packed index pidx(j, c) =
          // c(2n − c − 1)/2 + j -- for each c consecutive lanes write consecutive doubles (conflict-free)
#pragma unroll
          for (int c = 0; c < NX; ++c)
            if (c <= j) {
              const int pc = c * (2 * NX - c - 1) / 2 + j;
              rec[RC::S + pc] = wk[WK::Si + c * NX + j];
              rec[RC::V + pc] = U[c];
            }
          if constexpr (NU % 2 == 0 && (RC::K % 2) == 0) {  // column j of K (m × n col-major) as 16-byte pairs
#pragma unroll
            for (int u = 0; u < NU; u += 2)
              *reinterpret_cast<double2*>(rec + RC::K + j * NU + u) = make_double2(-U[NX + u], -U[NX + u + 1]);
          } else {
#pragma unroll
            for (int u = 0; u < NU; ++u) rec[RC::K + j * NU + u] = -U[NX + u];
          }
#else
          auto* Sp = rec + RC::S + j * (2 * NX - j - 1) / 2;
          auto* Vp = rec + RC::V + j * (2 * NX - j - 1) / 2;
#pragma unroll
          for (int r = 0; r < NX; ++r)
            if (r >= j) {
              Sp[r] = wk[WK::Si + r * NX + j];
              Vp[r] = U[r];
            }
#pragma unroll
          for (int u = 0; u < NU; ++u) rec[RC::K + j * NU + u] = -U[NX + u];
#endif
          rec[RC::v + j] = bj;
          rec[RC::e + j] = wk[WM::E + j];
        } else if (j < NZ) {
          rec[RC::k + (j - NX)] = -bj;
        }
      }
#ifndef RR_REC_STG
      static_assert(RC::SIZE <= 16 * WM::ULD && (RC::SIZE % 2) == 0, "record staging needs X2 and 16-byte size");
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
#pragma unroll
        for (int q = 0; q < 2; ++q)
          if (recq[q] != nullptr) bulk_s2g(recq[q], wkq[q] + WM::X2, 8u * RC::SIZE);
        bulk_commit();
      }
#endif
#pragma unroll
      for (int r = 0; r < NX; ++r) Vc[r] = (j < NX) ? U[r] : 0.0;
      __syncwarp();
      if (j < NX) wk[WK::vs + j] = bj;
      __syncwarp();
      return;
    }
  }
};

}  // namespace rrk
