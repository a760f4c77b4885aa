// ipm.cu -- fused batched regularized-IPM step (rows a1-a8), one lane group per instance (sm_100a).
//
// Method (arXiv 2509.16370, P:n = PAPER.md line n), per instance (see include/rr.h, ipm_step):
//   pass 1 (backward): per stage, condense the inequality duals (Σ = (S/Z + I/η)⁻¹,
//     r_z = g + μ/z) and stage-equality duals (η C_eᵀC_e) into the stage's LQR blocks, then one
//     backward step of Eq.(RR) with δ = 1/η (rr_stage.cuh);
//   pass 2 (forward): Δx_{i+1} = Φ Δx_i + φ, Δu, Δy, expand Δz, Δλ, Δs
//     (P:224-227), accumulate D = ∇𝒜·(Δx, Δs), the merit at the
//     iterate and the coefficients of its polynomial part in α, α_max, α_d;
//   pass 3: Armijo backtracking on 𝒜 (reading R12); trial points of the built-in model;
//   pass 4: in-place iterate update.
// Lane roles: lane j < NZ owns column j of the stage matrices (as in rr_stage.cuh); lane e < NG
// owns inequality e, lane e < NC owns stage equality e for the expansion; the line-search pass
// distributes stages over lanes.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ipm.cuh"
#include "ipm_model.cuh"
#include "rr_common.cuh"
#include "rr_stage.cuh"

namespace rrk {

template <int NX, int NU, int NG, int NC>
struct IpmBuf {  // padded per-stage IPM data in shared memory (doubles, even offsets)
  static constexpr int NZ = NX + NU;
  static constexpr int E2 = 2;
  static constexpr int F = 0;                         // [A B] col-major NX × NZ
  static constexpr int P = F + ((NX * NZ + 1) & ~1);  // P full NZ × NZ col-major
  static constexpr int gf = P + ((NZ * NZ + 1) & ~1); // ∇f (NZ)
  static constexpr int cv = gf + ((NZ + 1) & ~1);     // dres (NX)
  static constexpr int G = cv + ((NX + 1) & ~1);      // G col-major NG × NZ
  static constexpr int gv = G + ((NG * NZ + 1) & ~1); // g (NG)
  static constexpr int s = gv + ((NG + 1) & ~1);
  static constexpr int z = s + ((NG + 1) & ~1);
  static constexpr int sig = z + ((NG + 1) & ~1);     // Σ_e
  static constexpr int rz = sig + ((NG + 1) & ~1);    // r_z,e
  static constexpr int Ce = rz + ((NG + 1) & ~1);     // C_e col-major NC × NZ
  static constexpr int ce = Ce + ((NC * NZ + 1) & ~1);
  static constexpr int lam = ce + ((NC + 1) & ~1);
  static constexpr int yi = lam + ((NC + 1) & ~1);    // y_i
  static constexpr int yn = yi + NX;                  // y_{i+1}
  static constexpr int xb = yn + ((NX + 1) & ~1);     // x̄_i
  static constexpr int ub = xb + ((NX + 1) & ~1);     // ū_i
  static constexpr int du = ub + ((NU + 1) & ~1);     // Δu_i exchange
  static constexpr int SIZE = du + ((NU + 1) & ~1);
  static constexpr int PAD = (SIZE + 1) & ~1;
};

// x[e] += α d[e] for e < cnt over the LG lanes of a group (lane j), four independent loads in flight
// per lane before the dependent stores (x and d may not alias, but the compiler cannot know that).
template <int LG>
__device__ __forceinline__ void axpy_lanes(double* x, const double* d, double alpha, int64_t cnt, int j) {
#ifndef RR_AXPY_U
#define RR_AXPY_U 8
#endif
  constexpr int U = RR_AXPY_U;
  int64_t e = j;
  for (; e + (U - 1) * LG < cnt; e += U * LG) {
    double xv[U], dv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      xv[u] = x[e + u * LG];
      dv[u] = d[e + u * LG];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) x[e + u * LG] = fma(alpha, dv[u], xv[u]);
  }
  for (; e < cnt; e += LG) x[e] = fma(alpha, d[e], x[e]);
}

// EXACT: the dimensions are the template's (n = NX, m = NU, n_g = NG, n_c = NC; terminal counts stay
// runtime), so the compiler folds the padding guards and loop bounds.
template <int NX, int NU, int NG, int NC, int LG, int WARPS, bool EXACT = false>
__global__ void __launch_bounds__(WARPS * 32, EXACT ? 4 : 1) ipm_step_kernel(const IpmArgs a) {
  using ST = Stage<NX, NU, LG>;
  using WK = Work<NX, NU>;
  using RC = Rec<NX, NU>;
  using IB = IpmBuf<NX, NU, NG, NC>;
  constexpr int NZ = NX + NU;
  constexpr int IPW = 32 / LG;
  constexpr int SLOT = group_stride(2 * IB::PAD + WK::PAD + 2 * RC::PAD + NX, LG);
  static_assert(NG <= LG && NC <= LG, "constraint count per stage exceeds the lane group");

  const int n = EXACT ? NX : a.d.nx, m = EXACT ? NU : a.d.nu, N = a.d.N, w = n + m;
  const int ngd = EXACT ? NG : a.d.ng, ncd = EXACT ? NC : a.d.nc;
  const int sn = n * (n + 1) / 2, sm = m * (m + 1) / 2;

  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / LG, j = lane % LG, gbase = grp * LG;
  double* slot = smem + (warp * IPW + grp) * SLOT;
  double* wk = slot + 2 * IB::PAD;  // Riccati work area (two padded IPM stage buffers before it)
  double* rbuf = wk + WK::PAD;    // one forward record
  double* xs = rbuf + 2 * RC::PAD;

  int64_t inst = ((int64_t)blockIdx.x * WARPS + warp) * IPW + grp;
  bool valid;
  if (a.list != nullptr) {  // ipm_solve: only the instances on the device-built active list
    const int64_t cnt = *a.count;
    if ((int64_t)blockIdx.x * WARPS * IPW >= cnt) return;  // whole CTA past the list (uniform exit)
    valid = inst < cnt;
    inst = a.list[valid ? inst : 0];
  } else {
    valid = inst < a.d.batch;
    if (!valid) inst = a.d.batch - 1;
  }
  const int64_t sN = N;
  const double mu = a.it.mu[inst], eta = a.it.eta[inst];
  const double delta = 1.0 / eta;  // P:387-394 (reading R15)
  double* rec0 = a.ws + inst * sN * RC::PAD;
  int32_t st = 0;
  int nonpos_stage = 0x7fffffff;

  // double-buffered stage data: sbuf[0], sbuf[1]; `sb` points at the current one
  double* sbuf0 = slot;
  double* sbuf1 = slot + IB::PAD;
  double* sb = sbuf0;
  bool pk = false;  // sb holds a stage loaded by the exact path: P packed (Q | M | R) in the P slot
  // ---- issue the loads of stage i (i == N: terminal) into the padded shared layout `dst` ----
  // Real elements travel by cp.async (8-byte LDGSTS, asynchronous); padding is stored directly.
  // finish_stage() completes Σ, r_z and the positivity check once the copies have landed.
  // the padded layout equals the global one when the dims are the template dims: contiguous copies
  const bool exact = (n == NX && m == NU && ngd == NG && ncd == NC);
  auto issue_stage_data = [&](int i, double* dst) {
    const bool term = (i == N);
    const int ww = term ? n : w;
    const int ng = term ? a.d.ngN : ngd;
    const int nc = term ? a.d.ncN : ncd;
    const int64_t si = inst * sN + i;
    auto put = [&](int off, const double* src, bool ok, double pad) {
      if (ok) cp_async8(dst + off, src);
      else dst[off] = pad;
    };
    if constexpr (EXACT && NX == 4 && NU == 1 && NG == 4 && NC == 0 && LG == 8) {
      if (!term && a.aligned16) {
        // C4 copy plan: the stage's 41 16-byte chunks in 6 LDGSTS.128 rounds over the 8 lanes (lanes of
        // one round serve different arrays) + one LDGSTS.64 round for the odd-sized ∇f, ū, R -- instead
        // of 14 runtime-checked copy loops (their branches and address arithmetic were ~1/3 of the
        // kernel's instructions).  Destinations: the IpmBuf offsets (P slot packed Q | M | R).
        static_assert(IB::F == 0 && IB::P == 20 && IB::gf == 46 && IB::cv == 52 && IB::G == 56 && IB::gv == 76 &&
                          IB::s == 80 && IB::z == 84 && IB::yi == 96 && IB::xb == 104 && IB::ub == 108,
                      "C4 copy plan assumes the 4x1 (n_g 4) IpmBuf layout");
        const int64_t sy = inst * (sN + 1) + i;
        cp_async16(dst + IB::F + 2 * j, a.d_.A + si * 16 + 2 * j);    // A: 8 chunks
        cp_async16(dst + IB::G + 2 * j, a.d_.Gj + si * 20 + 2 * j);   // G: chunks 0..7
        {
          const double* src;
          int d;
          if (j < 2) { src = a.d_.Gj + si * 20 + 16 + 2 * j; d = IB::G + 16 + 2 * j; }         // G 8..9
          else if (j < 4) { src = a.d_.B + si * 4 + 2 * (j - 2); d = IB::F + 16 + 2 * (j - 2); }  // B
          else if (j < 6) { src = a.d_.M + si * 4 + 2 * (j - 4); d = IB::P + 10 + 2 * (j - 4); }  // M
          else { src = a.d_.dres + si * 4 + 2 * (j - 6); d = IB::cv + 2 * (j - 6); }            // dres
          cp_async16(dst + d, src);
        }
        if (j < 7) {
          const double* src = (j < 5) ? a.d_.Q + si * 10 + 2 * j : a.d_.gv + si * 4 + 2 * (j - 5);  // Q | g
          cp_async16(dst + ((j < 5) ? IB::P + 2 * j : IB::gv + 2 * (j - 5)), src);
        }
        {
          const double* src;
          int d;
          if (j < 4) { src = a.it.y + sy * 4 + 2 * j; d = IB::yi + 2 * j; }            // y_i | y_{i+1}
          else if (j < 6) { src = a.it.x + sy * 4 + 2 * (j - 4); d = IB::xb + 2 * (j - 4); }  // x̄_i
          else { src = a.it.s + si * 4 + 2 * (j - 6); d = IB::s + 2 * (j - 6); }        // s
          cp_async16(dst + d, src);
        }
        if (j < 2) cp_async16(dst + IB::z + 2 * j, a.it.z + si * 4 + 2 * j);            // z
        if (j < 7) {
          const double* src = (j < 5) ? a.d_.gradf + si * 5 + j : ((j == 5) ? a.it.u + si : a.d_.R + si);
          cp_async8(dst + ((j < 5) ? IB::gf + j : ((j == 5) ? IB::ub : IB::P + 14)), src);
        }
        return;
      }
    }
    if (exact && !term) {
      copy_async(dst + IB::F, a.d_.A + si * NX * NX, NX * NX, j, LG);       // F = [A | B], ld NX
      copy_async(dst + IB::F + NX * NX, a.d_.B + si * NX * NU, NX * NU, j, LG);
      {  // P packed as Q | M | R in the P slot (read through Pjs): contiguous copies instead of a
         // per-element gather into the unpacked layout (fewer LDGSTS, fewer bank conflicts)
        constexpr int SQ = NX * (NX + 1) / 2, SR = NU * (NU + 1) / 2;
        copy_async(dst + IB::P, a.d_.Q + si * SQ, SQ, j, LG);
        copy_async(dst + IB::P + SQ, a.d_.M + si * (NX * NU), NX * NU, j, LG);
        copy_async(dst + IB::P + SQ + NX * NU, a.d_.R + si * SR, SR, j, LG);
      }
      copy_async(dst + IB::gf, a.d_.gradf + si * NZ, NZ, j, LG);
      copy_async(dst + IB::cv, a.d_.dres + si * NX, NX, j, LG);
      copy_async(dst + IB::yi, a.it.y + (inst * (sN + 1) + i) * NX, 2 * NX, j, LG);  // y_i | y_{i+1}
      copy_async(dst + IB::xb, a.it.x + (inst * (sN + 1) + i) * NX, NX, j, LG);
      copy_async(dst + IB::ub, a.it.u + si * NU, NU, j, LG);
      if (NG > 0) {
        copy_async(dst + IB::G, a.d_.Gj + si * NG * NZ, NG * NZ, j, LG);
        copy_async(dst + IB::gv, a.d_.gv + si * NG, NG, j, LG);
        copy_async(dst + IB::s, a.it.s + si * NG, NG, j, LG);
        copy_async(dst + IB::z, a.it.z + si * NG, NG, j, LG);
      }
      if (NC > 0) {
        copy_async(dst + IB::Ce, a.d_.Ce + si * NC * NZ, NC * NZ, j, LG);
        copy_async(dst + IB::ce, a.d_.ce + si * NC, NC, j, LG);
        copy_async(dst + IB::lam, a.it.lam + si * NC, NC, j, LG);
      }
      return;
    }
    for (int e = j; e < NX * NZ; e += LG) {  // F = [A B]
      const int k = e % NX, c = e / NX;
      const bool okA = !term && k < n && c < n;
      const bool okB = !term && k < n && c >= NX && c - NX < m;
      const double* src = okA ? a.d_.A + si * n * n + k + c * n : (okB ? a.d_.B + si * n * m + k + (c - NX) * n : nullptr);
      put(IB::F + e, src, okA || okB, 0.0);
    }
    for (int e = j; e < NZ * NZ; e += LG) {  // P (padded u-diagonal = 1)
      const int r = e % NZ, c = e / NZ;
      const bool rx = r < NX, cx = c < NX;
      const int rr = rx ? r : r - NX, cc = cx ? c : c - NX;
      const double* src = nullptr;
      double pad = 0.0;
      if (term) {
        if (rx && cx && r < n && c < n) src = a.d_.QN + inst * sn + (r >= c ? pidx(n, r, c) : pidx(n, c, r));
        else if (!rx && !cx && rr == cc) pad = 1.0;
      } else if (rx && cx) {
        if (r < n && c < n) src = a.d_.Q + si * sn + (r >= c ? pidx(n, r, c) : pidx(n, c, r));
      } else if (rx && !cx) {
        if (r < n && cc < m) src = a.d_.M + si * n * m + r + cc * n;
      } else if (!rx && cx) {
        if (c < n && rr < m) src = a.d_.M + si * n * m + c + rr * n;
      } else {
        if (rr < m && cc < m) src = a.d_.R + si * sm + (rr >= cc ? pidx(m, rr, cc) : pidx(m, cc, rr));
        else if (rr == cc) pad = 1.0;
      }
      put(IB::P + e, src, src != nullptr, pad);
    }
    for (int e = j; e < NZ; e += LG) {  // ∇f in the padded (x | u) layout
      const double* src = nullptr;
      if (e < NX) {
        if (e < n) src = term ? a.d_.gradfN + inst * n + e : a.d_.gradf + si * w + e;
      } else if (!term && e - NX < m) {
        src = a.d_.gradf + si * w + n + (e - NX);
      }
      put(IB::gf + e, src, src != nullptr, 0.0);
    }
    for (int e = j; e < NX; e += LG) {
      put(IB::cv + e, a.d_.dres + si * n + e, !term && e < n, 0.0);
      put(IB::yi + e, a.it.y + (inst * (sN + 1) + i) * n + e, e < n, 0.0);
      put(IB::yn + e, a.it.y + (inst * (sN + 1) + i + 1) * n + e, !term && e < n, 0.0);
      put(IB::xb + e, a.it.x + (inst * (sN + 1) + i) * n + e, e < n, 0.0);
    }
    for (int e = j; e < NU; e += LG) put(IB::ub + e, a.it.u + si * m + e, !term && e < m, 0.0);
    const double* Gsrc = term ? a.d_.GjN + inst * (int64_t)ng * n : a.d_.Gj + si * (int64_t)ng * ww;
    for (int e = j; e < NG * NZ; e += LG) {
      const int q = e % NG, c = e / NG;
      const double* src = nullptr;
      if (q < ng) {
        if (c < NX) { if (c < n) src = Gsrc + q + (int64_t)c * ng; }
        else if (!term && c - NX < m) src = Gsrc + q + (int64_t)(n + c - NX) * ng;
      }
      put(IB::G + e, src, src != nullptr, 0.0);
    }
    for (int e = j; e < NG; e += LG) {
      const bool ok = e < ng;
      put(IB::gv + e, term ? a.d_.gvN + inst * ng + e : a.d_.gv + si * ng + e, ok, 0.0);
      put(IB::s + e, term ? a.it.sN + inst * ng + e : a.it.s + si * ng + e, ok, 1.0);
      put(IB::z + e, term ? a.it.zN + inst * ng + e : a.it.z + si * ng + e, ok, 1.0);
    }
    const double* Csrc = term ? a.d_.CeN + inst * (int64_t)nc * n : a.d_.Ce + si * (int64_t)nc * ww;
    constexpr int NCD = NC > 0 ? NC : 1;  // (no iterations when NC == 0)
    for (int e = j; e < NC * NZ; e += LG) {
      const int q = e % NCD, c = e / NCD;
      const double* src = nullptr;
      if (q < nc) {
        if (c < NX) { if (c < n) src = Csrc + q + (int64_t)c * nc; }
        else if (!term && c - NX < m) src = Csrc + q + (int64_t)(n + c - NX) * nc;
      }
      put(IB::Ce + e, src, src != nullptr, 0.0);
    }
    for (int e = j; e < NC; e += LG) {
      const bool ok = e < nc;
      put(IB::ce + e, term ? a.d_.ceN + inst * nc + e : a.d_.ce + si * nc + e, ok, 0.0);
      put(IB::lam + e, term ? a.it.lamN + inst * nc + e : a.it.lam + si * nc + e, ok, 0.0);
    }
  };
  // after the copies of stage i landed in sb: Σ = (s/z + 1/η)⁻¹, r_z = g + μ/z
  auto finish_stage = [&](int i) {
    const int ng = (i == N) ? a.d.ngN : ngd;
    for (int e = j; e < NG; e += LG) {
      const double sv = sb[IB::s + e], zv = sb[IB::z + e], gvv = sb[IB::gv + e];
      if (e < ng && (!(sv > 0.0) || !(zv > 0.0))) nonpos_stage = min(nonpos_stage, i);
      // Σ = (s/z + 1/η)⁻¹ = zη / (sη + z); reciprocals by Newton-refined rcp (≤ 1 ulp) for the divides
      sb[IB::sig + e] = (e < ng) ? zv * eta * rcp_nr(fma(sv, eta, zv)) : 0.0;
      sb[IB::rz + e] = (e < ng) ? fma(mu, rcp_nr(zv), gvv) : 0.0;
    }
    __syncwarp();
  };
  auto load_stage_now = [&](int i) {  // synchronous variant (terminal stage)
    issue_stage_data(i, sb);
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
    finish_stage(i);
  };

  // lane j's own column of Σ^{1/2}-weighted G and η-weighted C_e, cached in registers once per stage
  // (the column-major G / C_e reads at stride NG / NC would otherwise repeat for every column s)
  constexpr int NGR = NG > 0 ? NG : 1, NCR = NC > 0 ? NC : 1;
  double gsj[NGR], cej[NCR];
  auto cache_cols = [&]() {
    const int jc = j < NZ ? j : 0;
#pragma unroll
    for (int e = 0; e < NG; ++e) gsj[e] = sb[IB::sig + e] * sb[IB::G + e + jc * NG];
#pragma unroll
    for (int e = 0; e < NC; ++e) cej[e] = eta * sb[IB::Ce + e + jc * NC];
  };
  // P[s][j] of the current stage: packed Q | M | R (exact path, stages < N) or unpacked NZ × NZ
  auto Pjs = [&](int s_) -> double {
    if (pk) {
      constexpr int MO = NX * (NX + 1) / 2, RO = MO + NX * NU;
      const int jj = j < NZ ? j : 0;
      int off;
      if (s_ < NX) off = (jj < NX) ? ((s_ >= jj) ? pidx(NX, s_, jj) : pidx(NX, jj, s_)) : MO + s_ + (jj - NX) * NX;
      else if (jj < NX) off = MO + jj + (s_ - NX) * NX;
      else off = RO + ((s_ >= jj) ? pidx(NU, s_ - NX, jj - NX) : pidx(NU, jj - NX, s_ - NX));
      return sb[IB::P + off];
    }
    return sb[IB::P + j * NZ + s_];
  };
  // condensed P̃ column j: P + GᵀΣG + η C_eᵀC_e
  auto Pt = [&](int s) -> double {
    if (j >= NZ) return 0.0;
    double v = Pjs(s);
#pragma unroll
    for (int e = 0; e < NG; ++e) v = fma(sb[IB::G + e + s * NG], gsj[e], v);
#pragma unroll
    for (int e = 0; e < NC; ++e) v = fma(sb[IB::Ce + e + s * NC], cej[e], v);
    return v;
  };
  // condensed gradient s̃_j = ∇ₓℒ + GᵀΣ r_z + η C_eᵀ c_e, ∇ₓℒ = ∇f + Cᵀy + Gᵀz + C_eᵀλ
  auto qt = [&]() -> double {
    if (j >= NZ) return 0.0;
    double v = sb[IB::gf + j];
    if (j < NX) v -= sb[IB::yi + j];
#pragma unroll
    for (int r = 0; r < NX; ++r) v = fma(sb[IB::F + r + j * NX], sb[IB::yn + r], v);
#pragma unroll
    for (int e = 0; e < NG; ++e)
      v = fma(sb[IB::G + e + j * NG], sb[IB::z + e], fma(gsj[e], sb[IB::rz + e], v));
#pragma unroll
    for (int e = 0; e < NC; ++e) v = fma(sb[IB::Ce + e + j * NC], sb[IB::lam + e], fma(cej[e], sb[IB::ce + e], v));
    return v;
  };

  // ================= pass 1: backward (condense + Eq.(RR)) =================
  double Vc[NX];
  load_stage_now(N);
  cache_cols();
  {
    // terminal: V_N = Q̃_N (condensed), v_N = q̃_N
#pragma unroll
    for (int r = 0; r < NX; ++r) Vc[r] = (j < NX) ? Pt(r) : 0.0;
    const double qj = qt();
    __syncwarp();
    if (j < NX) wk[WK::vs + j] = qj;
    __syncwarp();
  }
  __syncwarp();
  if (N > 0) issue_stage_data(N - 1, sbuf1);
  cp_async_commit();
  for (int i = N - 1; i >= 0; --i) {
    sb = ((N - 1 - i) & 1) ? sbuf0 : sbuf1;
    pk = exact;
    if (i > 0) issue_stage_data(i - 1, ((N - 1 - i) & 1) ? sbuf1 : sbuf0);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    finish_stage(i);
    cache_cols();
    auto Pcol = [&](int s) -> double { return Pt(s); };
    const double qj = qt();
    double U[NZ], b[NZ];
    ST::backward(sb + IB::F, sb + IB::cv, Pcol, qj, delta, j, wk, Vc, U, b, rec0 + (int64_t)i * RC::PAD, i, st);
  }

  // ================= pass 2: forward + expand + merit/D accumulation =================
  // Δx_0 = (I + δV_0)⁻¹(c_0 − δ v_0), c_0 = s_0 − x̄_0
  ST::invS(Vc, delta, j, wk, 0, st);
  double xr[NX];
  double c0v[NX];
#pragma unroll
  for (int r = 0; r < NX; ++r) {
    c0v[r] = (r < n) ? (a.d_.s0[inst * n + r] - a.it.x[inst * (sN + 1) * n + r]) : 0.0;
    xr[r] = c0v[r] - delta * wk[WK::vs + r];
  }
  ST::mulSinv(xr, wk);
  __syncwarp();
  // per-lane partial sums
  double sD = 0.0, sK0 = 0.0, sK1 = 0.0, sK2 = 0.0;
  LogAcc sLog;  // Σ log s as a renormalised running product (one log at the end)
  double sDyn0 = 0.0;  // nonlinear-model dynamics terms of 𝒜 at α = 0 (trial points recompute them)
  double amax = 1.0, admax = 1.0;
  const double tau = a.prm.tau;
  const int model = a.d.model;
  bool bad = false;
  // row 0 (initial state): c_0(α) = c_0 − αΔx_0 (linear for every model)
  if (j < n) {
    double x0 = 0.0, c0 = 0.0;
#pragma unroll
    for (int r = 0; r < NX; ++r) {
      x0 = (r == j) ? xr[r] : x0;
      c0 = (r == j) ? c0v[r] : c0;
    }
    const double y0 = a.it.y[inst * (sN + 1) * n + j];
    const double cd = -x0;
    sD += (y0 + eta * c0) * cd;
    sK0 += y0 * c0 + 0.5 * eta * c0 * c0;
    sK1 += y0 * cd + eta * c0 * cd;
    sK2 += 0.5 * eta * cd * cd;
    if (valid) a.r.dx[inst * (sN + 1) * n + j] = x0;
  }
  const int ui = j - NX;
  auto expand_stage = [&](int i, const double (&dz_full)[NZ]) {
    // inequality e on lane e; equality e on lane e
    const bool term = (i == N);
    const int ng = term ? a.d.ngN : ngd;
    const int nc = term ? a.d.ncN : ncd;
    const int64_t si = inst * sN + i;
    if (j < ng) {
      double gd = 0.0;
#pragma unroll
      for (int c = 0; c < NZ; ++c) gd = fma(sb[IB::G + j + c * NG], dz_full[c], gd);
      const double s = sb[IB::s + j], z = sb[IB::z + j], g = sb[IB::gv + j];
      const double dzv = sb[IB::sig + j] * (gd + sb[IB::rz + j]);
      const double iz = rcp_nr(z);
      const double dsv = fma(-(s * iz), dzv, fma(mu, iz, -s));
      // fraction to the boundary with Newton-refined reciprocals (the IEEE division is a ~40-instruction
      // subroutine on the dependent chain of every stage)
      if (dsv < 0.0) amax = fmin(amax, tau * s * rcp_nr(-dsv));
      if (dzv < 0.0) admax = fmin(admax, tau * z * rcp_nr(-dzv));
      const double gs = g + s, bq = gd + dsv;
      sD += (z + eta * gs) * bq + (-mu * rcp_nr(s)) * dsv;
      sK0 += z * gs + 0.5 * eta * gs * gs;
      sK1 += z * bq + eta * gs * bq;
      sK2 += 0.5 * eta * bq * bq;
      sLog.add(s);
      if (valid) {
        if (term) {
          a.r.dsN[inst * ng + j] = dsv;
          a.r.dzN[inst * ng + j] = dzv;
        } else {
          a.r.ds[si * ng + j] = dsv;
          a.r.dz[si * ng + j] = dzv;
        }
      }
      bad |= !isfinite(dsv) || !isfinite(dzv);
    }
    if (j < nc) {
      double cd = 0.0;
#pragma unroll
      for (int c = 0; c < NZ; ++c) cd = fma(sb[IB::Ce + j + c * NC], dz_full[c], cd);
      const double ce = sb[IB::ce + j], lam = sb[IB::lam + j];
      const double dl = eta * (cd + ce);
      sD += (lam + eta * ce) * cd;
      sK0 += lam * ce + 0.5 * eta * ce * ce;
      sK1 += lam * cd + eta * ce * cd;
      sK2 += 0.5 * eta * cd * cd;
      if (valid) {
        if (term) a.r.dlamN[inst * nc + j] = dl;
        else a.r.dlam[si * nc + j] = dl;
      }
      bad |= !isfinite(dl);
    }
    // cost: ∇fᵀΔ and ½ΔᵀPΔ (lane j < NZ owns entry j)
    if (j < NZ) {
      double pd = 0.0;
#pragma unroll
      for (int c = 0; c < NZ; ++c) pd = fma(Pjs(c), dz_full[c], pd);
      double dj = 0.0;
#pragma unroll
      for (int c = 0; c < NZ; ++c) dj = (c == j) ? dz_full[c] : dj;
      const double gd = sb[IB::gf + j] * dj;
      sD += gd;
      sK1 += gd;
      sK2 += 0.5 * dj * pd;
    }
  };

  // pipelined loads: stage i+1 data and record i+1 land while stage i computes
  __syncwarp();
  if (N > 0) {
    issue_stage_data(0, sbuf0);
    copy_async(rbuf, rec0, RC::PAD, j, LG);  // PAD (even): 16-byte copies
  } else {
    issue_stage_data(N, sbuf0);
  }
  cp_async_commit();
  for (int i = 0; i < N; ++i) {
    sb = (i & 1) ? sbuf1 : sbuf0;
    pk = exact;
    const double* rc = (i & 1) ? rbuf + RC::PAD : rbuf;
    if (i + 1 < N) {
      issue_stage_data(i + 1, (i & 1) ? sbuf0 : sbuf1);
      copy_async((i & 1) ? rbuf : rbuf + RC::PAD, rec0 + (int64_t)(i + 1) * RC::PAD, RC::PAD, j, LG);
    } else {
      issue_stage_data(N, (i & 1) ? sbuf0 : sbuf1);  // terminal data for after the loop
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    finish_stage(i);
    double a0 = 0.0, a1 = 0.0, c0 = 0.0, c1 = 0.0;
    if (j < NX) {
      a0 = rc[RC::phi + j];
      c0 = rc[RC::v + j];
#pragma unroll
      for (int k = 0; k < NX; ++k) {
        a0 = fma(rc[RC::PHI + k * NX + j], xr[k], a0);
        const int ik = k >= j ? pidx(NX, k, j) : pidx(NX, j, k);
        c1 = fma(rc[RC::V + ik], xr[k], c1);
      }
    } else if (ui < NU) {
      a0 = rc[RC::k + ui];
#pragma unroll
      for (int k = 0; k < NX; ++k) a1 = fma(rc[RC::K + k * NU + ui], xr[k], a1);
    }
    const double acc1 = a0 + a1, acc2 = c0 + c1;  // x_{i+1}[j] | u_i[ui];  y_i[j]
    if (j < NX) xs[j] = acc1;
    if (ui >= 0 && ui < NU) sb[IB::du + ui] = acc1;
    __syncwarp();
    double dz_full[NZ];
#pragma unroll
    for (int c = 0; c < NX; ++c) dz_full[c] = xr[c];
#pragma unroll
    for (int u = 0; u < NU; ++u) dz_full[NX + u] = sb[IB::du + u];
    double xn[NX];
    ST::bcast(xs, xn);
    if (valid) {
      if (j < n) {
        a.r.dy[(inst * (sN + 1) + i) * n + j] = acc2;
        a.r.dx[(inst * (sN + 1) + i + 1) * n + j] = acc1;
      }
      if (ui >= 0 && ui < m) a.r.du[(inst * sN + i) * m + ui] = acc1;
    }
    bad |= ((j < n) && !(isfinite(acc1) && isfinite(acc2))) || ((ui >= 0 && ui < m) && !isfinite(acc1));
    expand_stage(i, dz_full);
    // dynamics row i+1: (CΔ)_r = (FΔ)_r − Δx_{i+1,r};  c_{i+1} at the iterate
    if (j < n) {
      double fd = 0.0;
#pragma unroll
      for (int c = 0; c < NZ; ++c) fd = fma(sb[IB::F + j + c * NX], dz_full[c], fd);
      double xnj = 0.0;
#pragma unroll
      for (int r = 0; r < NX; ++r) xnj = (r == j) ? xn[r] : xnj;
      const double cd = fd - xnj;
      const double yn = sb[IB::yn + j];
      const double dres = sb[IB::cv + j];
      sD += (yn + eta * dres) * cd;
      if (model == IPM_MODEL_LQ) {
        sK0 += yn * dres + 0.5 * eta * dres * dres;
        sK1 += yn * cd + eta * dres * cd;
        sK2 += 0.5 * eta * cd * cd;
      }
    }
#pragma unroll
    for (int r = 0; r < NX; ++r) xr[r] = xn[r];
    __syncwarp();
  }
  // terminal stage: y_N = Ṽ_N x_N + ṽ_N with the condensed terminal blocks; expansions on x_N
  cp_async_wait<0>();
  __syncwarp();
  sb = (N & 1) ? sbuf1 : sbuf0;
  pk = false;
  finish_stage(N);
  cache_cols();
  {
    double dz_full[NZ];
#pragma unroll
    for (int c = 0; c < NZ; ++c) dz_full[c] = (c < NX) ? xr[c] : 0.0;
    // ṽ_N, Ṽ_N recomputed from the condensed terminal data
    const double qj = qt();
    double yj = qj;
#pragma unroll
    for (int r = 0; r < NX; ++r) yj = fma(Pt(r), xr[r], yj);  // Ṽ_N symmetric: row j = column j
    if (valid && j < n) a.r.dy[(inst * (sN + 1) + N) * n + j] = yj;
    bad |= (j < n) && !isfinite(yj);
    expand_stage(N, dz_full);
  }
  // ---- reduce the partial sums over the lane group ----
  // group-masked collectives: pass 3 below runs a data-dependent number of backtracks per instance,
  // so the lane groups of a warp diverge there and must never wait on each other
  const unsigned gmask = (LG == 32) ? 0xffffffffu : (((1u << LG) - 1u) << gbase);
  auto gsum = [&](double v) {
#pragma unroll
    for (int off = LG / 2; off > 0; off >>= 1) v += __shfl_xor_sync(gmask, v, off);
    return v;
  };
  auto gmin = [&](double v) {
#pragma unroll
    for (int off = LG / 2; off > 0; off >>= 1) v = fmin(v, __shfl_xor_sync(gmask, v, off));
    return v;
  };
  const double D = gsum(sD);
  const double K0 = gsum(sK0) + a.d_.fval[inst];
  const double K1 = gsum(sK1), K2 = gsum(sK2);
  const double Abase = K0 - mu * gsum(sLog.value());
  amax = gmin(amax);
  admax = gmin(admax);
  int32_t status = st;
  int np = nonpos_stage;
#pragma unroll
  for (int off = LG / 2; off > 0; off >>= 1) {
    status = max(status, __shfl_xor_sync(gmask, status, off));
    np = min(np, __shfl_xor_sync(gmask, np, off));
  }
  if (status == 0 && (__ballot_sync(gmask, bad) & gmask)) status = RR_ST_NONFINITE;
  if (np != 0x7fffffff) status = mk_status(RR_ST_NONPOS_SLACK, np);
  // dynamics terms of 𝒜 at α = 0 through the built-in model (as the oracle's merit evaluates them),
  // stages distributed over the lanes: inside the first trial of the line search (sharing its loads
  // of x̄, ū, y) when there is one, else in a pass of their own
  const bool fuse0 = model != IPM_MODEL_LQ && status == 0 && !a.direction_only;
  double A0 = Abase;
  if (model != IPM_MODEL_LQ && !fuse0) {
    for (int i = j; i < N; i += LG) {
      const double* xb = a.it.x + (inst * (sN + 1) + i) * n;
      const double* ub = a.it.u + (inst * sN + i) * m;
      const double* yb = a.it.y + (inst * (sN + 1) + i + 1) * n;
      double xa[NX], ua[NU], xnm[NX];
#pragma unroll
      for (int r = 0; r < NX; ++r) xa[r] = (r < n) ? xb[r] : 0.0;
#pragma unroll
      for (int r = 0; r < NU; ++r) ua[r] = (r < m) ? ub[r] : 0.0;
      model_step<NX, NU>(model, a.d_.model_params, xa, ua, xnm);
#pragma unroll
      for (int r = 0; r < NX; ++r) {
        if (r < n) {
          const double cr = xnm[r] - xb[n + r];
          sDyn0 += yb[r] * cr + 0.5 * eta * cr * cr;
        }
      }
    }
    A0 = Abase + gsum(sDyn0);
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
      for (int i = j; i <= N; i += LG) {  // stages distributed over the lanes
        const bool term = (i == N);
        const int ng = term ? a.d.ngN : ngd;
        const double* sp = term ? a.it.sN + inst * ng : a.it.s + (inst * sN + i) * ng;
        const double* dsp = term ? a.r.dsN + inst * ng : a.r.ds + (inst * sN + i) * ng;
        if (ng == NG) {  // all loads of the stage issued before the first use
          double sv[NG], dv[NG];
#pragma unroll
          for (int e = 0; e < NG; ++e) {
            sv[e] = sp[e];
            dv[e] = dsp[e];
          }
#pragma unroll
          for (int e = 0; e < NG; ++e) {
            const double sa = fma(alpha, dv[e], sv[e]);
            pos &= sa > 0.0;
            sl.add(sa);
          }
        } else {
          for (int e = 0; e < ng; ++e) {
            const double sa = fma(alpha, dsp[e], sp[e]);
            pos &= sa > 0.0;
            sl.add(sa);
          }
        }
        if (model != IPM_MODEL_LQ && !term) {
          double xa[NX], ua[NU], xnm[NX];
          const double* xb = a.it.x + (inst * (sN + 1) + i) * n;
          const double* dxb = a.r.dx + (inst * (sN + 1) + i) * n;
          const double* ub = a.it.u + (inst * sN + i) * m;
          const double* dub = a.r.du + (inst * sN + i) * m;
#pragma unroll
          for (int r = 0; r < NX; ++r) xa[r] = (r < n) ? xb[r] + alpha * dxb[r] : 0.0;
#pragma unroll
          for (int r = 0; r < NU; ++r) ua[r] = (r < m) ? ub[r] + alpha * dub[r] : 0.0;
          model_step<NX, NU>(model, a.d_.model_params, xa, ua, xnm);
          const double* yb = a.it.y + (inst * (sN + 1) + i + 1) * n;
#pragma unroll
          for (int r = 0; r < NX; ++r) {
            if (r < n) {
              const double cr = xnm[r] - (xb[n + r] + alpha * dxb[n + r]);
              sdyn += yb[r] * cr + 0.5 * eta * cr * cr;
            }
          }
          if (fuse0 && nb == 0) {  // the α = 0 terms on the same loads
#pragma unroll
            for (int r = 0; r < NX; ++r) xa[r] = (r < n) ? xb[r] : 0.0;
#pragma unroll
            for (int r = 0; r < NU; ++r) ua[r] = (r < m) ? ub[r] : 0.0;
            model_step<NX, NU>(model, a.d_.model_params, xa, ua, xnm);
#pragma unroll
            for (int r = 0; r < NX; ++r) {
              if (r < n) {
                const double cr = xnm[r] - xb[n + r];
                sDyn0 += yb[r] * cr + 0.5 * eta * cr * cr;
              }
            }
          }
        }
      }
      if (fuse0 && nb == 0) A0 = Abase + gsum(sDyn0);
      const double slog = gsum(sl.value());
      sdyn = gsum(sdyn);
      const bool allpos = __ballot_sync(gmask, !pos) == 0;
      const double At = K0 + alpha * (K1 + alpha * K2) - mu * slog + sdyn;
      if (allpos && At <= A0 + a.prm.armijo_c * alpha * D) {
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
  auto axpy_group = [&](double* x, const double* d, double al, int64_t cnt, int jj) { axpy_lanes<LG>(x, d, al, cnt, jj); };
  if (valid && accepted) {
    const int64_t nx1 = (sN + 1) * n;
    axpy_group(a.it.x + inst * nx1, a.r.dx + inst * nx1, alpha, nx1, j);
    axpy_group(a.it.y + inst * nx1, a.r.dy + inst * nx1, alpha, nx1, j);
    axpy_group(a.it.u + inst * sN * m, a.r.du + inst * sN * m, alpha, sN * m, j);
    const int64_t ngt = sN * ngd, nct = sN * ncd;
    axpy_group(a.it.s + inst * ngt, a.r.ds + inst * ngt, alpha, ngt, j);
    axpy_group(a.it.z + inst * ngt, a.r.dz + inst * ngt, admax, ngt, j);
    axpy_group(a.it.sN + inst * a.d.ngN, a.r.dsN + inst * a.d.ngN, alpha, a.d.ngN, j);
    axpy_group(a.it.zN + inst * a.d.ngN, a.r.dzN + inst * a.d.ngN, admax, a.d.ngN, j);
    axpy_group(a.it.lam + inst * nct, a.r.dlam + inst * nct, alpha, nct, j);
    axpy_group(a.it.lamN + inst * a.d.ncN, a.r.dlamN + inst * a.d.ncN, alpha, a.d.ncN, j);
  }
  if (valid && j == 0) {
    a.status[inst] = status;
    const bool ok = (status == 0);
    const bool searched = ok || status == RR_ST_LS_FAILED;  // direction, D and 𝒜(0) are defined
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    if (a.r.alpha_p) a.r.alpha_p[inst] = ok ? alpha : 0.0;
    if (a.r.alpha_d) a.r.alpha_d[inst] = ok ? admax : 0.0;
    if (a.r.D) a.r.D[inst] = searched ? D : nan;
    if (a.r.merit0) a.r.merit0[inst] = searched ? A0 : nan;
    if (a.r.merit_acc) a.r.merit_acc[inst] = ok ? Aacc : nan;
    if (a.r.n_backtracks) a.r.n_backtracks[inst] = searched ? nb : 0;
  }
  if (valid && (status & 0xff) == RR_ST_NONPOS_SLACK) {  // direction undefined: NaN-fill
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    const int64_t nx1 = (sN + 1) * n;
    for (int64_t e = j; e < nx1; e += LG) {
      a.r.dx[inst * nx1 + e] = nan;
      a.r.dy[inst * nx1 + e] = nan;
    }
    for (int64_t e = j; e < sN * m; e += LG) a.r.du[inst * sN * m + e] = nan;
    const int64_t ngt = sN * ngd, nct = sN * ncd;
    for (int64_t e = j; e < ngt; e += LG) {
      a.r.ds[inst * ngt + e] = nan;
      a.r.dz[inst * ngt + e] = nan;
    }
    for (int e = j; e < a.d.ngN; e += LG) {
      a.r.dsN[inst * a.d.ngN + e] = nan;
      a.r.dzN[inst * a.d.ngN + e] = nan;
    }
    for (int64_t e = j; e < nct; e += LG) a.r.dlam[inst * nct + e] = nan;
    for (int e = j; e < a.d.ncN; e += LG) a.r.dlamN[inst * a.d.ncN + e] = nan;
  }
}

// ------------------------------------------------------------------------------------------
template <int NX, int NU, int NG, int NC, int LG, bool EXACT = false>
struct IpmCfg {
  static constexpr int WARPS = 4;
  static constexpr int IPB = WARPS * (32 / LG);
  static constexpr int SLOT =
      group_stride(2 * IpmBuf<NX, NU, NG, NC>::PAD + Work<NX, NU>::PAD + 2 * Rec<NX, NU>::PAD + NX, LG);
  static size_t smem_bytes() { return sizeof(double) * (size_t)IPB * SLOT; }
  static int64_t ws_doubles(int64_t batch, int N) { return batch * (int64_t)N * Rec<NX, NU>::PAD; }
  static cudaError_t launch(const IpmArgs& a, cudaStream_t s) {
    auto k = ipm_step_kernel<NX, NU, NG, NC, LG, WARPS, EXACT>;
    const size_t sm = smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    const int64_t blocks = (a.d.batch + IPB - 1) / IPB;
    k<<<(unsigned)blocks, WARPS * 32, sm, s>>>(a);
    return cudaGetLastError();
  }
};

template <typename F>
static bool dispatch_ipm(const ipm_dims& d, F&& f) {
  const int ngm = d.ng > d.ngN ? d.ng : d.ngN;
  const int ncm = d.nc > d.ncN ? d.nc : d.ncN;
  if (d.model == IPM_MODEL_CARTPOLE && (d.nx != 4 || d.nu != 1)) return false;
  if (d.model == IPM_MODEL_QUADROTOR && (d.nx != 12 || d.nu != 4)) return false;
  if (d.nx == 4 && d.nu == 1 && d.ng == 4 && d.nc == 0 && d.ngN <= 4 && d.ncN == 0)
    return f(IpmCfg<4, 1, 4, 0, 8, true>{});  // C4 (cart-pole) shape
  if (d.nx <= 4 && d.nu <= 1 && ngm <= 4 && ncm == 0) return f(IpmCfg<4, 1, 4, 0, 8>{});
  if (d.nx <= 4 && d.nu <= 4 && ngm <= 8 && ncm <= 4) return f(IpmCfg<4, 4, 8, 4, 8>{});
  if (d.nx <= 8 && d.nu <= 8 && ngm <= 16 && ncm <= 8) return f(IpmCfg<8, 8, 16, 8, 16>{});
  if (d.nx <= 12 && d.nu <= 4 && ngm <= 16 && ncm <= 8) return f(IpmCfg<12, 4, 16, 8, 16>{});
  return false;
}

int64_t ipm_ws_bytes(const ipm_dims& d) {
  int64_t out = -1;
  dispatch_ipm(d, [&](auto cfg) {
    out = 8 * decltype(cfg)::ws_doubles(d.batch, d.N) + 256;
    return true;
  });
  return out;
}

bool ipm_supported(const ipm_dims& d) {
  return dispatch_ipm(d, [](auto) { return true; });
}

cudaError_t ipm_launch(const IpmArgs& a0, cudaStream_t s, bool* supported) {
  cudaError_t err = cudaSuccess;
  IpmArgs a = a0;  // the C4 copy plan needs 16-byte aligned bases of the 16-byte-copied arrays
  const void* ops[] = {a.d_.A, a.d_.B, a.d_.Q, a.d_.M, a.d_.dres, a.it.y, a.it.x, a.d_.Gj, a.d_.gv, a.it.s, a.it.z};
  a.aligned16 = 1;
  for (const void* p : ops)
    if (p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u) != 0) a.aligned16 = 0;
  if (ipm_c4t_applies(a)) {  // C4 shape: one thread per instance (ipm_c4t.cu)
    *supported = true;
    return ipm_c4t_launch(a, s);
  }
  *supported = dispatch_ipm(a.d, [&](auto cfg) {
    err = decltype(cfg)::launch(a, s);
    return true;
  });
  return err;
}

}  // namespace rrk
