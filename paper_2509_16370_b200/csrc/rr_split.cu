// rr_split.cu -- rr_factor / rr_solve: the factorization / solve split of the regularized Riccati
// recursion (the paper's "KKT system factorization callback" and "KKT system solve callback",
// P:660-667), one lane group per instance (sm_100a).
//
// Method (arXiv 2509.16370, P:n = PAPER.md line n):
//   rr_factor: the matrix half of Eq.(RR), i = N-1..0, V_N = Q_N:
//       S_{i+1}⁻¹ = (I + δV_{i+1})⁻¹, W_i = S⁻¹V_{i+1}, G_i = BᵀWB + R, H_i = BᵀWA + Mᵀ,
//       K_i = −G⁻¹H, V_i = AᵀWA + Q + KᵀH;  finally S_0⁻¹ (for x_0).
//     It writes the factor record of every stage (layout in include/rr.h):
//       record i = [ V_i (packed) | S_i⁻¹ = (I+δV_i)⁻¹ (packed) | K_i (m×n) | G_i⁻¹ (packed) ].
//   rr_solve: the vector half of Eq.(RR) for a right-hand side (q, r, c, q_N, c_0):
//       g_i = v_{i+1} + W_i(c_{i+1} − δv_{i+1}) = S_{i+1}⁻¹(v_{i+1} + V_{i+1}c_{i+1})  (S⁻¹ = I − δW)
//       h_i = r + Bᵀg, k_i = −G⁻¹h, v_i = q + Aᵀg + Kᵀh
//     then the forward sweep x_0 = S_0⁻¹(c_0 − δv_0), u_i = K_i x_i + k_i,
//     x_{i+1} = S_{i+1}⁻¹(A x + B u + c_{i+1} − δv_{i+1}) and the duals
//     y_i = V_i x_i + v_i.
//
// B200 organisation (kernels K2/K3): lane j of the group owns column j of the
// (n+m)-wide stage matrices (rr_stage.cuh).  rr_factor: S⁻¹ by the symmetric sweep operator,
// products as register FMA chains, then the symmetric sweep operator on the u-block of
// U = FᵀWF + P, which leaves [V_i; G⁻¹H] in the x-columns and −G⁻¹ in the u-columns (so G⁻¹
// comes for free; same exact result as a Cholesky of G, reading R9).  rr_solve: mat-vecs only
// (HBM-bound); stage data and factor records stream through shared memory with cp.async, three
// record buffers so that record i+1 (V_{i+1}, S_{i+1}⁻¹) stays resident while record i−1 loads.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "rr_common.cuh"
#include "rr_split.cuh"

#include <type_traits>
#include "rr_fused.cuh"
#include "rr_stage.cuh"

namespace rrk {

__host__ __device__ constexpr int symn(int n) { return n * (n + 1) / 2; }

// packed-lower symmetric element (r, c) of an n×n matrix, either triangle
__device__ __forceinline__ int sidx(int n, int r, int c) { return r >= c ? pidx(n, r, c) : pidx(n, c, r); }

// ------------------------------------------------------------------------------------------
// rr_factor kernel
template <int NX, int NU, bool EXACT>
struct FacLayout {
  static constexpr int NZ = NX + NU;
  static constexpr int MSTG = NX * NX + 2 * NX * NU + symn(NX) + symn(NU);  // A, B, Q, M, R
  static constexpr int MSTG_PAD = (MSTG + 1) & ~1;
  static constexpr int PADF = EXACT ? 0 : NX * NZ;
  static constexpr int SLOT = 2 * MSTG_PAD + Work<NX, NU>::PAD + PADF;
  static constexpr int SLOT_PAD = (SLOT + 1) & ~1;
};

template <int NX, int NU, int LG, int WARPS, int MINB, bool EXACT>
__global__ void __launch_bounds__(WARPS * 32, MINB) rr_factor_kernel(const SplitArgs a) {
  using LY = FacLayout<NX, NU, EXACT>;
  using ST = Stage<NX, NU, LG>;
  using WK = Work<NX, NU>;
  constexpr int NZ = LY::NZ;
  constexpr int IPW = 32 / LG;
  const int n = EXACT ? NX : a.nx;
  const int m = EXACT ? NU : a.nu;
  const int N = a.N;
  const int sn = symn(n), sm = symn(m);
  const int oA = 0, oB = n * n, oQ = oB + n * m, oM = oQ + sn, oR = oM + n * m;
  const int REC = frec_doubles(n, m);
  const int rS = sn, rK = 2 * sn, rG = 2 * sn + n * m;

  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / LG, j = lane % LG, gbase = grp * LG;
  double* slot = smem + (warp * IPW + grp) * group_stride(LY::SLOT_PAD, LG);
  double* stg0 = slot;
  double* stg1 = slot + LY::MSTG_PAD;
  double* wk = slot + 2 * LY::MSTG_PAD;
  double* Fp = wk + WK::PAD;

  int64_t inst = ((int64_t)blockIdx.x * WARPS + warp) * IPW + grp;
  const bool valid = inst < a.batch;
  if (!valid) inst = a.batch - 1;
  const double delta = a.p.delta[inst];
  const int64_t sN = (int64_t)N;
  double* rec = a.fr + inst * (sN + 1) * REC;
  int32_t st = 0;

  const int64_t instP = (a.shared & RR_FLAG_SHARED_COST) ? 0 : inst;
  auto issue_stage = [&](int i, double* dst) {
    const int64_t sD = dyn_blk(a.shared, inst, sN, i), sP = cost_blk(a.shared, inst, sN, i);
    copy_async(dst + oA, a.p.A + sD * n * n, n * n, j, LG);
    copy_async(dst + oB, a.p.B + sD * n * m, n * m, j, LG);
    copy_async(dst + oQ, a.p.Q + sP * sn, sn, j, LG);
    copy_async(dst + oM, a.p.M + sP * n * m, n * m, j, LG);
    copy_async(dst + oR, a.p.R + sP * sm, sm, j, LG);
  };
  // P = [[Q M]; [Mᵀ R]] (padded u-diagonal = 1 keeps the padded G block = I)
  auto Pat = [&](const double* sb, int s, int t) -> double {
    if (s < NX && t < NX) return (s < n && t < n) ? sb[oQ + sidx(n, s, t)] : 0.0;
    if (s < NX) {
      const int u = t - NX;
      return (s < n && u < m) ? sb[oM + s + u * n] : 0.0;
    }
    if (t < NX) {
      const int u = s - NX;
      return (t < n && u < m) ? sb[oM + t + u * n] : 0.0;
    }
    const int u = s - NX, w = t - NX;
    if (u < m && w < m) return sb[oR + sidx(m, u, w)];
    return u == w ? 1.0 : 0.0;
  };
  // packed symmetric S⁻¹ (wk[Si], symmetric NX×NX) -> record slot
  auto write_sinv = [&](double* dst) {
    if (valid && j < n)
      for (int r = j; r < n; ++r) dst[pidx(n, r, j)] = wk[WK::Si + r * NX + j];
  };

  // V_N = Q_N (carried as column j in Vc; record N holds V_N and S_N⁻¹)
  double Vc[NX];
  {
    const double* QN = a.p.QN + instP * sn;
#pragma unroll
    for (int r = 0; r < NX; ++r) Vc[r] = (j < n && r < n) ? QN[sidx(n, r, j)] : 0.0;
    if (valid && j < n) {
      for (int r = j; r < n; ++r) rec[sN * REC + pidx(n, r, j)] = QN[pidx(n, r, j)];
      if (a.f.V != nullptr)
        for (int r = j; r < n; ++r) a.f.V[(inst * (sN + 1) + N) * sn + pidx(n, r, j)] = QN[pidx(n, r, j)];
    }
  }
  if (N > 0) issue_stage(N - 1, stg0);
  cp_async_commit();
  __syncwarp();

  for (int i = N - 1; i >= 0; --i) {
    const double* sb = ((N - 1 - i) & 1) ? stg1 : stg0;
    double* nb = ((N - 1 - i) & 1) ? stg0 : stg1;
    if (i > 0) issue_stage(i - 1, nb);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    const double* F = sb + oA;  // [A B] column-major, n × (n+m)
    if (!EXACT) {
      for (int e = j; e < NX * NZ; e += LG) {
        const int k = e % NX, s = e / NX;
        double val = 0.0;
        if (k < n) {
          if (s < NX) val = (s < n) ? sb[oA + k + s * n] : 0.0;
          else val = (s - NX < m) ? sb[oB + k + (s - NX) * n] : 0.0;
        }
        Fp[e] = val;
      }
      __syncwarp();
      F = Fp;
    }
    double* rc = rec + (int64_t)i * REC;

    // (1) S_{i+1}⁻¹ (symmetric sweep; wk[Si]) -> record i+1
    ST::invS(Vc, delta, j, wk, i, st);
    write_sinv(rec + (int64_t)(i + 1) * REC + rS);
    // (2) W = S⁻¹ V_{i+1} (column j)
    {
      double X[NX];
#pragma unroll
      for (int r = 0; r < NX; ++r) X[r] = Vc[r];
      ST::mulSinv(X, wk);
      if (j < NX) ST::store_col(wk + WK::Wb + j * NX, X);
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
    double U[NZ];
#pragma unroll
    for (int s = 0; s < NZ; ++s) {
      const double* Fs = F + s * NX;
      double a0 = (j < NZ) ? Pat(sb, s, j) : 0.0, a1 = 0.0;
#pragma unroll
      for (int k = 0; k < NX; k += 2) {
        const double2 f2 = *reinterpret_cast<const double2*>(Fs + k);
        a0 = fma(f2.x, T[k], a0);
        a1 = fma(f2.y, T[k + 1], a1);
      }
      U[s] = a0 + a1;
    }
    // (4) symmetric sweep operator on the u-block pivots p = NX..NZ-1.  Column p = row p
    // (the swept matrix stays symmetric), so every lane publishes its own element p.
    //   pivot lane:  Ã_sp = A_sp / A_pp (s ≠ p),  Ã_pp = −1 / A_pp
    //   other lanes: Ã_sc = A_sc − A_sp A_pc / A_pp (s ≠ p),  Ã_pc = A_pc / A_pp
    // Result: x-columns [V_i ; G⁻¹H] = [V_i ; −K_i], u-columns [HᵀG⁻¹ ; −G⁻¹].
#pragma unroll
    for (int p = NX; p < NZ; ++p) {
      double* pb = wk + WK::pub + (p & 1) * WK::NZP;
      if (j < NZ) pb[j] = U[p];
      __syncwarp();
      double col[NZ];
#pragma unroll
      for (int s = 0; s < NZ; ++s) col[s] = pb[s];
      const double piv = col[p];
      if (!(piv > 0.0) && st == 0) st = mk_status(RR_ST_G_NOT_PD, i);
      const double ip = rcp_nr(piv);
      const bool pl = (j == p);
      const double sc = pl ? ip : 1.0;
      const double f = pl ? 0.0 : U[p] * ip;
      const double up = pl ? -ip : U[p] * ip;
#pragma unroll
      for (int s = 0; s < NZ; ++s) U[s] = (s == p) ? up : fma(-col[s], f, U[s] * sc);
    }
    // (5) record i: V_i, K_i, G_i⁻¹ (+ optional user copies)
    if (valid) {
      if (j < n) {
#pragma unroll
        for (int r = 0; r < NX; ++r)
          if (r >= j && r < n) {
            rc[pidx(n, r, j)] = U[r];
            if (a.f.V != nullptr) a.f.V[(inst * (sN + 1) + i) * sn + pidx(n, r, j)] = U[r];
          }
#pragma unroll
        for (int u = 0; u < NU; ++u)
          if (u < m) {
            rc[rK + j * m + u] = -U[NX + u];
            if (a.f.K != nullptr) a.f.K[(inst * sN + i) * m * n + j * m + u] = -U[NX + u];
          }
      } else if (j >= NX && j - NX < m) {
        const int w = j - NX;
#pragma unroll
        for (int u = 0; u < NU; ++u)
          if (u < m && u >= w) rc[rG + pidx(m, u, w)] = -U[NX + u];
      }
    }
#pragma unroll
    for (int r = 0; r < NX; ++r) Vc[r] = (j < NX) ? U[r] : 0.0;
    __syncwarp();
  }
  // S_0⁻¹ = (I + δV_0)⁻¹ (for x_0) -> record 0
  ST::invS(Vc, delta, j, wk, 0, st);
  write_sinv(rec + rS);

  int32_t status = st;
#pragma unroll
  for (int off = LG / 2; off > 0; off >>= 1) {
    const int32_t o = __shfl_xor_sync(RR_FULL_MASK, status, off);
    status = o > status ? o : status;
  }
  (void)gbase;
  if (valid && status != 0) {  // a failed instance's factor is NaN: rr_solve reports it non-finite
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    __syncwarp();
    for (int64_t e = j; e < (sN + 1) * REC; e += LG) rec[e] = nan;
  }
  if (valid && j == 0) a.status[inst] = status;
}

// ------------------------------------------------------------------------------------------
// rr_solve kernel
template <int NX, int NU>
struct SolLayout {
  static constexpr int NZ = NX + NU;
  static constexpr int VSTG = NX * NX + NX * NU + 2 * NX + NU;  // A, B, c, q, r
  static constexpr int VSTG_PAD = (VSTG + 1) & ~1;
  static constexpr int REC_PAD = (2 * symn(NX) + NX * NU + symn(NU) + 1) & ~1;
  static constexpr int NXP = (NX + 1) & ~1;
  static constexpr int NUP = (NU + 1) & ~1;
  // 2 stage buffers | 3 record buffers | vs (v_{i+1}) | w/z | g | h/u | x (2 buffers)
  static constexpr int oS = 0;
  static constexpr int oR = 2 * VSTG_PAD;
  static constexpr int ovs = oR + 3 * REC_PAD;
  static constexpr int ow = ovs + NXP;
  static constexpr int og = ow + NXP;
  static constexpr int oh = og + NXP;
  static constexpr int ox = oh + NUP;
  static constexpr int SLOT = ox + 2 * NXP;
  static constexpr int SLOT_PAD = (SLOT + 1) & ~1;
};

// F32: the factor records are FP32 (RR_FLAG_FACTOR_FP32): loaded as floats, used in FP64 arithmetic.
template <int NX, int NU, int LG, int WARPS, int MINB, bool EXACT, bool F32 = false>
__global__ void __launch_bounds__(WARPS * 32, MINB) rr_solve_kernel(const SplitArgs a) {
  using LY = SolLayout<NX, NU>;
  using RT = typename std::conditional<F32, float, double>::type;
  constexpr int IPW = 32 / LG;
  static_assert(NX + NU <= LG, "lane group narrower than n+m");
  const int n = EXACT ? NX : a.nx;
  const int m = EXACT ? NU : a.nu;
  const int N = a.N;
  const int sn = symn(n), sm = symn(m);
  const int oA = 0, oB = n * n, oc = oB + n * m, oq = oc + n, orr = oq + n;
  const int REC = F32 ? frec_floats(n, m) : frec_doubles(n, m);  // record stride in elements
  const int rS = sn, rK = 2 * sn, rG = 2 * sn + n * m;
  (void)sm;

  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / LG, j = lane % LG, gbase = grp * LG;
  double* slot = smem + (warp * IPW + grp) * group_stride(LY::SLOT_PAD, LG);
  auto sbuf = [&](int i) { return slot + LY::oS + (i & 1) * LY::VSTG_PAD; };
  auto rbuf = [&](int i) { return reinterpret_cast<RT*>(slot + LY::oR + (i % 3) * LY::REC_PAD); };
  double* vs = slot + LY::ovs;
  double* wb = slot + LY::ow;
  double* gb = slot + LY::og;
  double* hb = slot + LY::oh;
  auto xb = [&](int i) { return slot + LY::ox + (i & 1) * LY::NXP; };

  int64_t inst = ((int64_t)blockIdx.x * WARPS + warp) * IPW + grp;
  const bool valid = inst < a.batch;
  if (!valid) inst = a.batch - 1;
  const double delta = a.p.delta[inst];
  const int64_t sN = (int64_t)N;
  const RT* rec = reinterpret_cast<const RT*>(a.frc) + inst * (sN + 1) * REC;
  double* kv = a.ws + inst * sN * (n + m);  // per stage: v_i (n) | k_i (m)
  const int ui = j - NX;                     // control row of this lane (0 <= ui < m)
  const bool xl = j < n, ul = ui >= 0 && ui < m;
  const bool acc = a.accumulate;             // RR_FLAG_ACCUMULATE: sol += solution (refinement)

  auto issue_stage = [&](int i) {
    const int64_t s = inst * sN + i, sD = dyn_blk(a.shared, inst, sN, i);
    double* dst = sbuf(i);
    copy_async(dst + oA, a.p.A + sD * n * n, n * n, j, LG);
    copy_async(dst + oB, a.p.B + sD * n * m, n * m, j, LG);
    copy_async(dst + oc, a.p.c + s * n, n, j, LG);
    copy_async(dst + oq, a.p.q + s * n, n, j, LG);
    copy_async(dst + orr, a.p.r + s * m, m, j, LG);
  };
  auto issue_rec = [&](int i) {
    copy_async(reinterpret_cast<double*>(rbuf(i)), reinterpret_cast<const double*>(rec + (int64_t)i * REC),
               REC * (int)sizeof(RT) / 8, j, LG);
  };

  // ---------------- backward vector sweep ----------------
  if (xl) vs[j] = a.p.qN[inst * n + j];
  issue_rec(N);
  if (N > 0) {
    issue_stage(N - 1);
    issue_rec(N - 1);
  }
  cp_async_commit();
  for (int i = N - 1; i >= 0; --i) {
    if (i > 0) {
      issue_stage(i - 1);
      issue_rec(i - 1);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    const double* S = sbuf(i);
    const RT* R1 = rbuf(i + 1);  // V_{i+1}, S_{i+1}⁻¹
    const RT* R0 = rbuf(i);        // K_i, G_i⁻¹
    // w = v_{i+1} + V_{i+1} c_{i+1}
    if (xl) {
      double w0 = vs[j], w1 = 0.0;
#pragma unroll
      for (int k = 0; k < NX; k += 2) {
        if (k < n) w0 = fma(R1[sidx(n, j, k)], S[oc + k], w0);
        if (k + 1 < n) w1 = fma(R1[sidx(n, j, k + 1)], S[oc + k + 1], w1);
      }
      wb[j] = w0 + w1;
    }
    __syncwarp();
    // g = S_{i+1}⁻¹ w
    if (xl) {
      double g0 = 0.0, g1 = 0.0;
#pragma unroll
      for (int k = 0; k < NX; k += 2) {
        if (k < n) g0 = fma(R1[rS + sidx(n, j, k)], wb[k], g0);
        if (k + 1 < n) g1 = fma(R1[rS + sidx(n, j, k + 1)], wb[k + 1], g1);
      }
      gb[j] = g0 + g1;
    }
    __syncwarp();
    // h = r + Bᵀ g
    if (ul) {
      double h0 = S[orr + ui], h1 = 0.0;
#pragma unroll
      for (int k = 0; k < NX; k += 2) {
        if (k < n) h0 = fma(S[oB + k + ui * n], gb[k], h0);
        if (k + 1 < n) h1 = fma(S[oB + k + 1 + ui * n], gb[k + 1], h1);
      }
      hb[ui] = h0 + h1;
    }
    __syncwarp();
    // k = −G⁻¹ h ;  v_i = q + Aᵀ g + Kᵀ h
    double out = 0.0;
    if (ul) {
#pragma unroll
      for (int w = 0; w < NU; ++w)
        if (w < m) out = fma(-R0[rG + sidx(m, ui, w)], hb[w], out);
    } else if (xl) {
      double v0 = S[oq + j], v1 = 0.0;
#pragma unroll
      for (int k = 0; k < NX; k += 2) {
        if (k < n) v0 = fma(S[oA + k + j * n], gb[k], v0);
        if (k + 1 < n) v1 = fma(S[oA + k + 1 + j * n], gb[k + 1], v1);
      }
#pragma unroll
      for (int u = 0; u < NU; ++u)
        if (u < m) v0 = fma(R0[rK + j * m + u], hb[u], v0);
      out = v0 + v1;
    }
    __syncwarp();  // all reads of vs, gb, hb of this stage done
    if (xl) {
      vs[j] = out;
      if (valid) {
        kv[(int64_t)i * (n + m) + j] = out;
        if (a.f.v != nullptr) a.f.v[(inst * (sN + 1) + i) * n + j] = out;
      }
    } else if (ul && valid) {
      kv[(int64_t)i * (n + m) + n + ui] = out;
      if (a.f.k != nullptr) a.f.k[(inst * sN + i) * m + ui] = out;
    }
    __syncwarp();
  }
  if (N == 0) {
    cp_async_wait<0>();
    __syncwarp();
  }
  if (valid && xl && a.f.v != nullptr) a.f.v[(inst * (sN + 1) + N) * n + j] = a.p.qN[inst * n + j];

  // ---------------- forward sweep ----------------
  bool bad = false;
  double* xo = a.s.x + inst * (sN + 1) * n;
  double* uo = a.s.u + inst * sN * m;
  double* yo = a.s.y + inst * (sN + 1) * n;
  // x_0 = S_0⁻¹ (c_0 − δ v_0)   (record 0 is resident in rbuf[0])
  if (xl) wb[j] = a.p.c0[inst * n + j] - delta * vs[j];
  __syncwarp();
  if (xl) {
    double x0 = 0.0, x1 = 0.0;
#pragma unroll
    for (int k = 0; k < NX; k += 2) {
      if (k < n) x0 = fma(rbuf(0)[rS + sidx(n, j, k)], wb[k], x0);
      if (k + 1 < n) x1 = fma(rbuf(0)[rS + sidx(n, j, k + 1)], wb[k + 1], x1);
    }
    const double xv = x0 + x1;
    xb(0)[j] = xv;
    if (valid) xo[j] = acc ? xo[j] + xv : xv;
    bad |= !isfinite(xv);
  }
  __syncwarp();
  // records 0, 1 and stage 0 are resident from the backward sweep (buffers i % 3, i & 1)
  for (int i = 0; i < N; ++i) {
    if (i + 2 <= N) issue_rec(i + 2);
    if (i + 1 < N) issue_stage(i + 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    const double* S = sbuf(i);
    const RT* R0 = rbuf(i);        // V_i, K_i
    const RT* R1 = rbuf(i + 1);  // S_{i+1}⁻¹
    const double* xc = xb(i);
    double* xn = xb(i + 1);
    // y_i = V_i x_i + v_i ;  u_i = K_i x_i + k_i
    if (xl) {
      double y0 = kv[(int64_t)i * (n + m) + j], y1 = 0.0;
#pragma unroll
      for (int k = 0; k < NX; k += 2) {
        if (k < n) y0 = fma(R0[sidx(n, j, k)], xc[k], y0);
        if (k + 1 < n) y1 = fma(R0[sidx(n, j, k + 1)], xc[k + 1], y1);
      }
      const double yv = y0 + y1;
      if (valid) yo[(int64_t)i * n + j] = acc ? yo[(int64_t)i * n + j] + yv : yv;
      bad |= !isfinite(yv);
    } else if (ul) {
      double u0 = kv[(int64_t)i * (n + m) + n + ui], u1 = 0.0;
#pragma unroll
      for (int k = 0; k < NX; k += 2) {
        if (k < n) u0 = fma(R0[rK + k * m + ui], xc[k], u0);
        if (k + 1 < n) u1 = fma(R0[rK + (k + 1) * m + ui], xc[k + 1], u1);
      }
      const double uv = u0 + u1;
      hb[ui] = uv;
      if (valid) uo[(int64_t)i * m + ui] = acc ? uo[(int64_t)i * m + ui] + uv : uv;
      bad |= !isfinite(uv);
    }
    __syncwarp();
    // z = A x_i + B u_i + c_{i+1} − δ v_{i+1}
    if (xl) {
      const double vn = (i + 1 < N) ? kv[(int64_t)(i + 1) * (n + m) + j] : a.p.qN[inst * n + j];
      double z0 = fma(-delta, vn, S[oc + j]), z1 = 0.0;
#pragma unroll
      for (int k = 0; k < NX; k += 2) {
        if (k < n) z0 = fma(S[oA + j + k * n], xc[k], z0);
        if (k + 1 < n) z1 = fma(S[oA + j + (k + 1) * n], xc[k + 1], z1);
      }
#pragma unroll
      for (int u = 0; u < NU; ++u)
        if (u < m) z0 = fma(S[oB + j + u * n], hb[u], z0);
      wb[j] = z0 + z1;
    }
    __syncwarp();
    // x_{i+1} = S_{i+1}⁻¹ z
    if (xl) {
      double x0 = 0.0, x1 = 0.0;
#pragma unroll
      for (int k = 0; k < NX; k += 2) {
        if (k < n) x0 = fma(R1[rS + sidx(n, j, k)], wb[k], x0);
        if (k + 1 < n) x1 = fma(R1[rS + sidx(n, j, k + 1)], wb[k + 1], x1);
      }
      const double xv = x0 + x1;
      xn[j] = xv;
      if (valid) xo[(int64_t)(i + 1) * n + j] = acc ? xo[(int64_t)(i + 1) * n + j] + xv : xv;
      bad |= !isfinite(xv);
    }
    __syncwarp();
  }
  // y_N = V_N x_N + v_N (record N holds V_N = Q_N)
  if (xl) {
    const RT* RN = rbuf(N);
    const double* xc = xb(N);
    double y0 = a.p.qN[inst * n + j], y1 = 0.0;
#pragma unroll
    for (int k = 0; k < NX; k += 2) {
      if (k < n) y0 = fma(RN[sidx(n, j, k)], xc[k], y0);
      if (k + 1 < n) y1 = fma(RN[sidx(n, j, k + 1)], xc[k + 1], y1);
    }
    const double yv = y0 + y1;
    if (valid) yo[sN * n + j] = acc ? yo[sN * n + j] + yv : yv;
    bad |= !isfinite(yv);
  }
  const unsigned anybad = __ballot_sync(RR_FULL_MASK, bad);
  const unsigned gmask = (LG == 32) ? 0xffffffffu : (((1u << LG) - 1u) << gbase);
  const int32_t status = (anybad & gmask) ? RR_ST_NONFINITE : 0;
  if (valid && status != 0) {
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
// rr_residual kernel: r = K [x; y] + [s; c] of the §1.4 system, block by block
// (the paper's residual callback):
//   rq_i = Q_i x_i + M_i u_i + q_i − y_i + A_iᵀ y_{i+1}     rr_i = M_iᵀ x_i + R_i u_i + r_i + B_iᵀ y_{i+1}
//   rqN  = Q_N x_N + q_N − y_N                              rc0  = −x_0 − δ y_0 + c_0
//   rc_i = A_i x_i + B_i u_i − x_{i+1} − δ y_{i+1} + c_{i+1}
// Written into the right-hand-side slots (q, r, c, q_N, c_0) so rr_solve can refine with it.
template <int NX, int NU>
struct ResLayout {
  static constexpr int STG = NX * NX + 2 * NX * NU + symn(NX) + symn(NU) + 2 * NX + NU;
  // stage buffer: stage data | x_i | x_{i+1} | u_i | y_i | y_{i+1}
  static constexpr int BUF = ((STG + 1) & ~1) + 4 * ((NX + 1) & ~1) + ((NU + 1) & ~1);
  static constexpr int SLOT_PAD = 2 * BUF;
};

template <int NX, int NU, int LG, int WARPS, int MINB, bool EXACT>
__global__ void __launch_bounds__(WARPS * 32, MINB) rr_residual_kernel(const ResArgs a) {
  using LY = ResLayout<NX, NU>;
  constexpr int IPW = 32 / LG;
  static_assert(NX + NU <= LG, "lane group narrower than n+m");
  const int n = EXACT ? NX : a.nx;
  const int m = EXACT ? NU : a.nu;
  const int N = a.N;
  const int sn = symn(n), sm = symn(m);
  const int oA = 0, oB = n * n, oQ = oB + n * m, oM = oQ + sn, oR = oM + n * m, oq = oR + sm, orr = oq + n,
            oc = orr + m, STGP = (oc + n + 1) & ~1;
  const int ox0 = STGP, ox1 = ox0 + ((n + 1) & ~1), ou = ox1 + ((n + 1) & ~1), oy0 = ou + ((m + 1) & ~1),
            oy1 = oy0 + ((n + 1) & ~1);

  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / LG, j = lane % LG, gbase = grp * LG;
  double* slot = smem + (warp * IPW + grp) * group_stride(LY::SLOT_PAD, LG);
  auto buf = [&](int i) { return slot + (i & 1) * LY::BUF; };

  int64_t inst = ((int64_t)blockIdx.x * WARPS + warp) * IPW + grp;
  const bool valid = inst < a.batch;
  if (!valid) inst = a.batch - 1;
  const double delta = a.p.delta[inst];
  const int64_t sN = (int64_t)N;
  const double* xg = a.s.x + inst * (sN + 1) * n;
  const double* ug = a.s.u + inst * sN * m;
  const double* yg = a.s.y + inst * (sN + 1) * n;
  const int ui = j - NX;
  const bool xl = j < n, ul = ui >= 0 && ui < m;

  const int64_t instP = (a.shared & RR_FLAG_SHARED_COST) ? 0 : inst;
  auto issue = [&](int i) {
    const int64_t s = inst * sN + i, sD = dyn_blk(a.shared, inst, sN, i), sP = cost_blk(a.shared, inst, sN, i);
    double* d = buf(i);
    copy_async(d + oA, a.p.A + sD * n * n, n * n, j, LG);
    copy_async(d + oB, a.p.B + sD * n * m, n * m, j, LG);
    copy_async(d + oQ, a.p.Q + sP * sn, sn, j, LG);
    copy_async(d + oM, a.p.M + sP * n * m, n * m, j, LG);
    copy_async(d + oR, a.p.R + sP * sm, sm, j, LG);
    copy_async(d + oq, a.p.q + s * n, n, j, LG);
    copy_async(d + orr, a.p.r + s * m, m, j, LG);
    copy_async(d + oc, a.p.c + s * n, n, j, LG);
    copy_async(d + ox0, xg + (int64_t)i * n, n, j, LG);
    copy_async(d + ox1, xg + (int64_t)(i + 1) * n, n, j, LG);
    copy_async(d + ou, ug + (int64_t)i * m, m, j, LG);
    copy_async(d + oy0, yg + (int64_t)i * n, n, j, LG);
    copy_async(d + oy1, yg + (int64_t)(i + 1) * n, n, j, LG);
  };
  double nst = 0.0, npr = 0.0;  // running max |stationarity|, |primal| of this lane
  bool bad = false;
  auto upd = [&](double& nm, double r) {
    bad |= !isfinite(r);
    nm = fmax(nm, fabs(r));
  };
  if (N > 0) issue(0);
  cp_async_commit();
  for (int i = 0; i < N; ++i) {
    if (i + 1 < N) issue(i + 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    const double* S = buf(i);
    const int64_t s = inst * sN + i;
    if (xl) {
      double a0 = S[oq + j] - S[oy0 + j], a1 = 0.0;  // stationarity row x_i[j]
      double p0 = S[oc + j] - S[ox1 + j] - delta * S[oy1 + j], p1 = 0.0;  // primal row i+1, entry j
#pragma unroll
      for (int k = 0; k < NX; ++k)
        if (k < n) {
          a0 = fma(S[oQ + sidx(n, j, k)], S[ox0 + k], a0);
          a1 = fma(S[oA + k + j * n], S[oy1 + k], a1);
          p0 = fma(S[oA + j + k * n], S[ox0 + k], p0);
        }
#pragma unroll
      for (int u = 0; u < NU; ++u)
        if (u < m) {
          a1 = fma(S[oM + j + u * n], S[ou + u], a1);
          p1 = fma(S[oB + j + u * n], S[ou + u], p1);
        }
      const double rq = a0 + a1, rc = p0 + p1;
      upd(nst, rq);
      upd(npr, rc);
      if (valid) {
        if (a.r.q) a.r.q[s * n + j] = rq;
        if (a.r.c) a.r.c[s * n + j] = rc;
      }
    } else if (ul) {
      double a0 = S[orr + ui], a1 = 0.0;
#pragma unroll
      for (int k = 0; k < NX; ++k)
        if (k < n) {
          a0 = fma(S[oM + k + ui * n], S[ox0 + k], a0);
          a1 = fma(S[oB + k + ui * n], S[oy1 + k], a1);
        }
#pragma unroll
      for (int w = 0; w < NU; ++w)
        if (w < m) a0 = fma(S[oR + sidx(m, ui, w)], S[ou + w], a0);
      const double rr = a0 + a1;
      upd(nst, rr);
      if (valid && a.r.r) a.r.r[s * m + ui] = rr;
    }
    __syncwarp();  // buffer i is refilled by issue(i + 2)
  }
  // terminal stationarity and the initial-state row
  if (xl) {
    const double* QN = a.p.QN + instP * sn;
    const double* xN = xg + sN * n;
    double a0 = a.p.qN[inst * n + j] - yg[sN * n + j];
    for (int k = 0; k < n; ++k) a0 = fma(QN[sidx(n, j, k)], xN[k], a0);
    const double r0 = -xg[j] - delta * yg[j] + a.p.c0[inst * n + j];
    upd(nst, a0);
    upd(npr, r0);
    if (valid) {
      if (a.r.qN) a.r.qN[inst * n + j] = a0;
      if (a.r.c0) a.r.c0[inst * n + j] = r0;
    }
  }
#pragma unroll
  for (int off = LG / 2; off > 0; off >>= 1) {
    nst = fmax(nst, __shfl_xor_sync(RR_FULL_MASK, nst, off));
    npr = fmax(npr, __shfl_xor_sync(RR_FULL_MASK, npr, off));
  }
  const unsigned anybad = __ballot_sync(RR_FULL_MASK, bad);
  const unsigned gmask = (LG == 32) ? 0xffffffffu : (((1u << LG) - 1u) << gbase);
  if (valid && j == 0 && a.norms != nullptr) {
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    a.norms[2 * inst] = (anybad & gmask) ? nan : nst;
    a.norms[2 * inst + 1] = (anybad & gmask) ? nan : npr;
  }
}

// ------------------------------------------------------------------------------------------
template <int NX, int NU, int LG, int WARPS, int MINB, bool EXACT, int MINB_F = MINB>
struct SplitCfg {
  static constexpr int IPB = WARPS * (32 / LG);
  static size_t fac_smem() { return sizeof(double) * (size_t)IPB * group_stride(FacLayout<NX, NU, EXACT>::SLOT_PAD, LG); }
  static size_t sol_smem() { return sizeof(double) * (size_t)IPB * group_stride(SolLayout<NX, NU>::SLOT_PAD, LG); }
  static size_t res_smem() { return sizeof(double) * (size_t)IPB * group_stride(ResLayout<NX, NU>::SLOT_PAD, LG); }
  static cudaError_t residual(const ResArgs& a, cudaStream_t s) {
    auto k = rr_residual_kernel<NX, NU, LG, WARPS, MINB, EXACT>;
    const size_t sm = res_smem();
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    k<<<(unsigned)((a.batch + IPB - 1) / IPB), WARPS * 32, sm, s>>>(a);
    return cudaGetLastError();
  }
  static cudaError_t factor(const SplitArgs& a, cudaStream_t s) {
    auto k = rr_factor_kernel<NX, NU, LG, WARPS, MINB_F, EXACT>;
    const size_t sm = fac_smem();
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    k<<<(unsigned)((a.batch + IPB - 1) / IPB), WARPS * 32, sm, s>>>(a);
    return cudaGetLastError();
  }
  static cudaError_t solve(const SplitArgs& a, cudaStream_t s) {
    auto k = a.f32 ? rr_solve_kernel<NX, NU, LG, WARPS, MINB, EXACT, true> : rr_solve_kernel<NX, NU, LG, WARPS, MINB, EXACT>;
    const size_t sm = sol_smem();
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    k<<<(unsigned)((a.batch + IPB - 1) / IPB), WARPS * 32, sm, s>>>(a);
    return cudaGetLastError();
  }
};

template <typename F>
static bool dispatch_split(int nx, int nu, F&& f) {
  if (nx == 12 && nu == 4) return f(SplitCfg<12, 4, 16, 4, 4, true, 3>{});
  if (nx == 4 && nu == 1) return f(SplitCfg<4, 1, 8, 4, 4, true>{});
  if (nx == 2 && nu == 1) return f(SplitCfg<2, 1, 4, 4, 4, true>{});
  if (nx <= 2 && nu <= 2) return f(SplitCfg<2, 2, 4, 4, 1, false>{});
  if (nx <= 4 && nu <= 4) return f(SplitCfg<4, 4, 8, 4, 1, false>{});
  if (nx <= 8 && nu <= 8) return f(SplitCfg<8, 8, 16, 4, 1, false>{});
  if (nx <= 16 && nu <= 16) return f(SplitCfg<16, 16, 32, 4, 1, false>{});
  return false;
}

bool split_supported(int nx, int nu) {
  return dispatch_split(nx, nu, [](auto) { return true; });
}

cudaError_t factor_launch(const SplitArgs& a, cudaStream_t s, bool* supported) {
  cudaError_t err = cudaSuccess;
  // 12x4: the DMMA stage kernel in factor-only mode (RR_B200_FACTOR=simt selects the SIMT kernel)
  const char* fv = getenv("RR_B200_FACTOR");
  if (a.nx == 12 && a.nu == 4 && a.tma16 && !(fv && strcmp(fv, "simt") == 0)) {
    FusedArgs f{};
    f.nx = a.nx;
    f.nu = a.nu;
    f.N = a.N;
    f.batch = a.batch;
    f.p = a.p;
    f.f = a.f;
    f.ws = nullptr;
    f.status = a.status;
    if (a.f32) f.frec32 = reinterpret_cast<float*>(a.fr);  // FP32 records (RR_FLAG_FACTOR_FP32)
    else f.frec = a.fr;
    f.shared = a.shared;
    err = factor_mma_launch(f, s, supported);
    if (*supported) return err;
  }
  if (a.f32) {  // FP32 records are written by the 12x4 DMMA factor kernel only
    *supported = false;
    return cudaSuccess;
  }
  *supported = dispatch_split(a.nx, a.nu, [&](auto cfg) {
    err = decltype(cfg)::factor(a, s);
    return true;
  });
  return err;
}

cudaError_t solve_launch(const SplitArgs& a, cudaStream_t s, bool* supported) {
  cudaError_t err = cudaSuccess;
  *supported = dispatch_split(a.nx, a.nu, [&](auto cfg) {
    err = decltype(cfg)::solve(a, s);
    return true;
  });
  return err;
}

}  // namespace rrk

namespace rrk {
cudaError_t residual_launch(const ResArgs& a, cudaStream_t s, bool* supported) {
  cudaError_t err = cudaSuccess;
  *supported = dispatch_split(a.nx, a.nu, [&](auto cfg) {
    err = decltype(cfg)::residual(a, s);
    return true;
  });
  return err;
}
}  // namespace rrk
