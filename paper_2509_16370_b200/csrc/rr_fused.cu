// rr_fused.cu -- fused regularized-Riccati factor + solve, one lane group per instance (sm_100a).
//
// Method (arXiv 2509.16370, P:n = PAPER.md line n):
//   backward sweep i = N-1..0 of Eq.(RR), forward sweep,
//   dual recovery y_i = V_i x_i + v_i.
//
// B200 design (kernel K1):
//   * One lane group of LG lanes (32/LG instances per warp) owns one instance; lane j owns
//     COLUMN j of the stage's (n+m)-wide matrices (rr_stage.cuh), so the dense contractions are
//     register-resident FMA chains fed by broadcast shared-memory reads.
//   * The stage inputs (A, B, Q, M, R, q, r, c) of stage i-1 stream into a double-buffered
//     per-instance shared-memory slot with cp.async while stage i computes.
//   * S = I + δV_{i+1} is factored by a shuffle-broadcast Cholesky; W = S⁻¹V, Φ_i = S⁻¹(A + B K_i)
//     and φ_i = S⁻¹(B k_i + c_{i+1} - δ v_{i+1}) are column-parallel triangular solves.
//   * G⁻¹H, G⁻¹h and V_i = AᵀWA + Q - HᵀG⁻¹H, v_i come out of ONE Gauss-Jordan elimination of the
//     u-block (P:606-611 identities; G SPD so no pivoting is needed, reading R9).
//   * The forward sweep is x_{i+1} = Φ_i x_i + φ_i, u_i = K_i x_i + k_i, y_i = V_i x_i + v_i from
//     one per-stage record (no re-read of A, B, c, no second Cholesky).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include <atomic>
#include <type_traits>

#include "rr_common.cuh"
#include "rr_fused.cuh"
#include "rr_stage.cuh"
#include "rr_stage_mma.cuh"
#include "rr_cta.cuh"

namespace rrk {

template <int NX, int NU, bool EXACT>
struct FusedLayout {
  static constexpr int NZ = NX + NU;
  static constexpr int STG = NX * NX + 2 * NX * NU + NX * (NX + 1) / 2 + NU * (NU + 1) / 2 + 2 * NX + NU;
  static constexpr int STG_PAD = (STG + 1) & ~1;
  static constexpr int PADF = EXACT ? 0 : (NX * NZ + NX);  // padded F and c for the generic kernels
  // per-instance shared slot (doubles): 2 stage buffers | work area | padded F, c  (backward);
  // reused as 2 record buffers in the forward sweep
  static constexpr int SLOT_B = 2 * STG_PAD + Work<NX, NU>::PAD + PADF;
  static constexpr int SLOT_F = 2 * Rec<NX, NU>::PAD + NX;
  static constexpr int SLOT = SLOT_B > SLOT_F ? SLOT_B : SLOT_F;
  static constexpr int SLOT_PAD = (SLOT + 1) & ~1;
};

template <int NX, int NU, int LG, int WARPS, int MINB, bool EXACT>
__global__ void __launch_bounds__(WARPS * 32, MINB) rr_fused_kernel(const FusedArgs a) {
  using LY = FusedLayout<NX, NU, EXACT>;
  using ST = Stage<NX, NU, LG>;
  using WK = Work<NX, NU>;
  using RC = Rec<NX, NU>;
  constexpr int NZ = LY::NZ;
  constexpr int IPW = 32 / LG;
  static_assert(32 % LG == 0, "lane group must divide the warp");

  const int n = EXACT ? NX : a.nx;
  const int m = EXACT ? NU : a.nu;
  const int N = a.N;
  const int sn = n * (n + 1) / 2, sm = m * (m + 1) / 2;
  const int oA = 0, oB = oA + n * n, oQ = oB + n * m, oM = oQ + sn, oR = oM + n * m, oq = oR + sm,
            orr = oq + n, oc = orr + m;

  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / LG, j = lane % LG, gbase = grp * LG;
  double* slot = smem + (warp * IPW + grp) * group_stride(LY::SLOT_PAD, LG);
  double* stg0 = slot;
  double* stg1 = slot + LY::STG_PAD;
  double* wk = slot + 2 * LY::STG_PAD;
  double* Fp = wk + WK::PAD;  // generic kernels only: padded F (NX × NZ) and c (NX)
  double* cp = Fp + NX * NZ;

  int64_t inst = ((int64_t)blockIdx.x * WARPS + warp) * IPW + grp;
  const bool valid = inst < a.batch;
  if (!valid) inst = a.batch - 1;
  const double delta = a.p.delta[inst];
  const int64_t sN = (int64_t)N;
  double* rec0 = a.ws + inst * sN * RC::PAD;
  int32_t st = 0;

  // batch-shared operands (include/rr.h RR_FLAG_SHARED_*): instance index 0 for them
  const int64_t instP = (a.shared & RR_FLAG_SHARED_COST) ? 0 : inst;
  auto issue_stage = [&](int i, double* dst) {
    const int64_t s = inst * sN + i, sD = dyn_blk(a.shared, inst, sN, i), sP = cost_blk(a.shared, inst, sN, i);
    copy_async(dst + oA, a.p.A + sD * n * n, n * n, j, LG);
    copy_async(dst + oB, a.p.B + sD * n * m, n * m, j, LG);
    copy_async(dst + oQ, a.p.Q + sP * sn, sn, j, LG);
    copy_async(dst + oM, a.p.M + sP * n * m, n * m, j, LG);
    copy_async(dst + oR, a.p.R + sP * sm, sm, j, LG);
    copy_async(dst + oq, a.p.q + s * n, n, j, LG);
    copy_async(dst + orr, a.p.r + s * m, m, j, LG);
    copy_async(dst + oc, a.p.c + s * n, n, j, LG);
  };

  // P = [[Q M]; [Mᵀ R]] column j, padded (padded u-diagonal = 1 keeps G_pad = I)
  auto Pat = [&](const double* sb, int s, int t) -> double {
    if (s < NX && t < NX) {
      if (s >= n || t >= n) return 0.0;
      return s >= t ? sb[oQ + pidx(n, s, t)] : sb[oQ + pidx(n, t, s)];
    }
    if (s < NX) {
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

  // ---- carried state: Vc = column j of V_N = Q_N; v_N = q_N ----
  double Vc[NX];
  {
    const double* QN = a.p.QN + instP * sn;
#pragma unroll
    for (int r = 0; r < NX; ++r) {
      double val = 0.0;
      if (j < n && r < n) val = r >= j ? QN[pidx(n, r, j)] : QN[pidx(n, j, r)];
      Vc[r] = val;
    }
    if (j < NX) wk[WK::vs + j] = (j < n) ? a.p.qN[inst * n + j] : 0.0;
    if (valid && a.f.V != nullptr && j < n) {
      double* Vo = a.f.V + (inst * (sN + 1) + N) * sn;
      for (int r = j; r < n; ++r) Vo[pidx(n, r, j)] = QN[pidx(n, r, j)];
    }
    if (valid && a.f.v != nullptr && j < n) a.f.v[(inst * (sN + 1) + N) * n + j] = a.p.qN[inst * n + j];
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
    const double* F = sb + oA;
    const double* cv = sb + oc;
    if (!EXACT) {  // scatter into the padded NX × NZ layout
      for (int e = j; e < NX * NZ; e += LG) {
        const int k = e % NX, s = e / NX;
        double val = 0.0;
        if (k < n) {
          if (s < NX) val = (s < n) ? sb[oA + k + s * n] : 0.0;
          else val = (s - NX < m) ? sb[oB + k + (s - NX) * n] : 0.0;
        }
        Fp[e] = val;
      }
      for (int e = j; e < NX; e += LG) cp[e] = (e < n) ? sb[oc + e] : 0.0;
      __syncwarp();
      F = Fp;
      cv = cp;
    }
    auto Pcol = [&](int s) -> double { return (j < NZ) ? Pat(sb, s, j) : 0.0; };
    const double qj = (j < NX) ? ((j < n) ? sb[oq + j] : 0.0) : ((j < NZ && j - NX < m) ? sb[orr + j - NX] : 0.0);

    double U[NZ], b[NZ];
    ST::backward(F, cv, Pcol, qj, delta, j, wk, Vc, U, b, rec0 + (int64_t)i * RC::PAD, i, st);

    if (valid) {  // optional factor outputs (policy of Eq.(RR))
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
      if (j == 0 && a.f.v != nullptr) {
        double* vo = a.f.v + (inst * (sN + 1) + i) * n;
#pragma unroll
        for (int r = 0; r < NX; ++r)
          if (r < n) vo[r] = b[r];
      }
      if (j == 0 && a.f.k != nullptr) {
        double* ko = a.f.k + (inst * sN + i) * m;
#pragma unroll
        for (int u = 0; u < NU; ++u)
          if (u < m) ko[u] = -b[NX + u];
      }
    }
  }

  // ---- x_0 = (I + δV_0)⁻¹ (c_0 - δ v_0) ----
  ST::invS(Vc, delta, j, wk, 0, st);
  double xr[NX];  // x_i replicated in every lane of the group
#pragma unroll
  for (int r = 0; r < NX; ++r) xr[r] = (r < n) ? (a.p.c0[inst * n + r] - delta * wk[WK::vs + r]) : 0.0;
  ST::mulSinv(xr, wk);

  // ---- status of the backward sweep, combined over the group (first failure in sweep order) ----
  int32_t status = st;
#pragma unroll
  for (int off = LG / 2; off > 0; off >>= 1) {
    const int32_t o = __shfl_xor_sync(RR_FULL_MASK, status, off);
    status = o > status ? o : status;
  }

  // ---- forward sweep: y_i = V_i x_i + v_i, u_i = K_i x_i + k_i, x_{i+1} = Φ_i x_i + φ_i ----
  bool bad = false;
  double* xo = a.s.x + inst * (sN + 1) * n;
  double* uo = a.s.u + inst * sN * m;
  double* yo = a.s.y + inst * (sN + 1) * n;
  const int ui = j - NX;  // control row owned by this lane (if 0 <= ui < NU)
  __syncwarp();            // the work area (x_0 solve) is free from here on: slot -> record buffers
  double* rbuf0 = slot;
  double* rbuf1 = slot + RC::PAD;
  double* xs = slot + 2 * RC::PAD;  // x_{i+1} exchange
  auto issue_rec = [&](int i, double* dst) { copy_async(dst, rec0 + (int64_t)i * RC::PAD, RC::SIZE, j, LG); };
  if (N > 0) issue_rec(0, rbuf0);
  cp_async_commit();
  {
    double xj = 0.0;
#pragma unroll
    for (int r = 0; r < NX; ++r) xj = (r == j) ? xr[r] : xj;
    if (valid && j < n) xo[j] = xj;
    bad |= (j < n) && !isfinite(xj);
  }
  for (int i = 0; i < N; ++i) {
    const double* rc = (i & 1) ? rbuf1 : rbuf0;
    if (i + 1 < N) issue_rec(i + 1, (i & 1) ? rbuf0 : rbuf1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    double a0 = 0.0, a1 = 0.0, c0 = 0.0, c1 = 0.0;
    if (j < NX) {
      a0 = rc[RC::phi + j];
      c0 = rc[RC::v + j];
#pragma unroll
      for (int k = 0; k < NX; k += 2) {
        a0 = fma(rc[RC::PHI + k * NX + j], xr[k], a0);
        a1 = fma(rc[RC::PHI + (k + 1) * NX + j], xr[k + 1], a1);
        const int i0 = k >= j ? pidx(NX, k, j) : pidx(NX, j, k);
        const int i1 = k + 1 >= j ? pidx(NX, k + 1, j) : pidx(NX, j, k + 1);
        c0 = fma(rc[RC::V + i0], xr[k], c0);
        c1 = fma(rc[RC::V + i1], xr[k + 1], c1);
      }
    } else if (ui < NU) {
      a0 = rc[RC::k + ui];
#pragma unroll
      for (int k = 0; k < NX; k += 2) {
        a0 = fma(rc[RC::K + k * NU + ui], xr[k], a0);
        a1 = fma(rc[RC::K + (k + 1) * NU + ui], xr[k + 1], a1);
      }
    }
    const double acc1 = a0 + a1, acc2 = c0 + c1;
    // lanes < NX: acc1 = x_{i+1}[j], acc2 = y_i[j];  lanes NX..: acc1 = u_i[ui]
    if (valid) {
      if (j < n) {
        yo[(int64_t)i * n + j] = acc2;
        xo[(int64_t)(i + 1) * n + j] = acc1;
      }
      if (ui >= 0 && ui < m) uo[(int64_t)i * m + ui] = acc1;
    }
    bad |= ((j < n) && !(isfinite(acc1) && isfinite(acc2))) || ((ui >= 0 && ui < m) && !isfinite(acc1));
    if (j < NX) xs[j] = acc1;
    __syncwarp();
    ST::bcast(xs, xr);
    __syncwarp();  // buffer rc is refilled next iteration
  }
  // y_N = Q_N x_N + q_N
  {
    const double* QN = a.p.QN + instP * sn;
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
template <int NX, int NU, int LG, int WARPS, int MINB, bool EXACT>
struct FusedCfg {
  static constexpr int IPB = WARPS * (32 / LG);  // instances per block
  static size_t smem_bytes() { return sizeof(double) * (size_t)IPB * group_stride(FusedLayout<NX, NU, EXACT>::SLOT_PAD, LG); }
  static int64_t ws_doubles(int64_t batch, int N) { return batch * (int64_t)N * Rec<NX, NU>::PAD; }
  static cudaError_t launch(const FusedArgs& a, cudaStream_t s) {
    auto k = rr_fused_kernel<NX, NU, LG, WARPS, MINB, EXACT>;
    const size_t sm = smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    const int64_t blocks = (a.batch + IPB - 1) / IPB;
    k<<<(unsigned)blocks, WARPS * 32, sm, s>>>(a);
    return cudaGetLastError();
  }
};


// ------------------------------------------------------------------------------------------
// K1-MMA: same method, stage contractions on DMMA (rr_stage_mma.cuh); exact shapes with
// NX % 4 == 0, NX + NU <= 16; two instances per warp (lane groups of 16).
template <int NX, int NU>
struct MmaLayout {
  static constexpr int STG = NX * NX + 2 * NX * NU + NX * (NX + 1) / 2 + NU * (NU + 1) / 2 + 2 * NX + NU;
  static constexpr int STG_PAD = (STG + 1) & ~1;
  static constexpr int SLOT_B = STG_PAD + WorkM<NX, NU>::PAD;  // single stage buffer (prefetched mid-stage)
  static constexpr int SLOT_F = 2 * RecM<NX, NU>::PAD + 2 * (((NX * NX + NX * NU) + 1) & ~1) + ((NU + 1) & ~1) + 2 * NX;
  static constexpr int BAR = ((SLOT_B > SLOT_F ? SLOT_B : SLOT_F) + 1) & ~1;  // 2 mbarriers (TMA completion)
  static constexpr int SLOT = BAR + 2;
  // slot stride ≡ 8 (mod 16) doubles: the two instances of a warp (half-warps) reading the same
  // offset of their own slots (SIMT broadcasts, per-lane columns) fall in different banks
  static constexpr int SLOT_PAD = ((SLOT + 1) & ~1) + ((8 - (((SLOT + 1) & ~1) % 16) + 16) % 16);
  // TMA bulk copies need 16-byte sizes/offsets for every operand block of a stage
  // P-gather table: per lane, the stage-buffer offset of each P_i element of its U C-fragments
  // (ZT × ZT tiles × 2 values), -1 outside NZ; stage independent, built once per CTA
  static constexpr int ZT = (NX + NU + 7) / 8;
  static constexpr int PTAB = ZT * ZT * 2;
  static constexpr bool BULK = (NX * NX) % 2 == 0 && (NX * NU) % 2 == 0 && (NX * (NX + 1) / 2) % 2 == 0 &&
                               (NU * (NU + 1) / 2) % 2 == 0 && NX % 2 == 0 && NU % 2 == 0 &&
                               RecM<NX, NU>::SIZE % 2 == 0;
};

// FAC = true: rr_factor (the matrix half only): stage loads of A, B, Q, M, R, factor records
// [V_i | S_i⁻¹ | K_i | G_i⁻¹] to a.frec (rr_split.cuh layout), no forward sweep.
// F32 (with FAC): the factor records are written in FP32 (RR_FLAG_FACTOR_FP32, a.frec32).
template <int NX, int NU, int WARPS, int MINB, bool FAC = false, bool F32 = false>
__global__ void __launch_bounds__(WARPS * 32, MINB) rr_fused_mma_kernel(const FusedArgs a) {
  using LY = MmaLayout<NX, NU>;
  using SM = StageMMA<NX, NU>;
  using ST = Stage<NX, NU, 16>;
  using WK = Work<NX, NU>;
  using RC = RecM<NX, NU>;
  constexpr int NZ = NX + NU;
  constexpr int n = NX, m = NU;
  constexpr int sn = n * (n + 1) / 2, sm = m * (m + 1) / 2;
  constexpr int oA = 0, oB = oA + n * n, oQ = oB + n * m, oM = oQ + sn, oR = oM + n * m, oq = oR + sm,
                orr = oq + n, oc = orr + m;
  const int N = a.N;

  extern __shared__ __align__(16) double smem[];
  // warp index through a shuffle from lane 0: provably warp-uniform, so the TMA issue below
  // (addresses from blockIdx, warp, stage) runs on uniform registers without a per-lane loop
  const int warp = __shfl_sync(RR_FULL_MASK, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int grp = lane >> 4, j = lane & 15, gbase = grp * 16;
  double* slotq[2] = {smem + (warp * 2 + 0) * LY::SLOT_PAD, smem + (warp * 2 + 1) * LY::SLOT_PAD};
  double* slot = grp ? slotq[1] : slotq[0];
  double* wkq[2] = {slotq[0] + LY::STG_PAD, slotq[1] + LY::STG_PAD};
#ifndef RR_NO_PTAB
  // P-gather offsets of this lane's U C-fragment positions (k = (mt·ZT + nt)·2 + e: row 8mt + g,
  // column 8nt + 2t + e of P = [[Q M]; [Mᵀ R]] in the stage buffer), two 16-bit offsets per register
  static_assert((NX + NU) % 8 == 0 && LY::STG < 65536, "register P-gather offsets need full 8-wide tiles");
  uint32_t ptw[LY::PTAB / 2];
  {
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int k2 = 0; k2 < LY::PTAB / 2; ++k2) {
      uint32_t o2[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = 2 * k2 + h;
        const int e = k & 1, nt = (k >> 1) % LY::ZT, mt = (k >> 1) / LY::ZT;
        const int s_ = 8 * mt + g, c = 8 * nt + 2 * t + e;
        int off;
        if (s_ < NX && c < NX) off = oQ + (s_ >= c ? pidx(n, s_, c) : pidx(n, c, s_));
        else if (s_ < NX) off = oM + s_ + (c - NX) * n;
        else if (c < NX) off = oM + c + (s_ - NX) * n;
        else off = oR + (s_ >= c ? pidx(m, s_ - NX, c - NX) : pidx(m, c - NX, s_ - NX));
        o2[h] = (uint32_t)off;
      }
      ptw[k2] = o2[0] | (o2[1] << 16);
    }
  }
#endif
  double* wk = grp ? wkq[1] : wkq[0];
  const int64_t sN = (int64_t)N;

  // stage inputs: TMA bulk copies for BOTH instances of the warp issued by lane 0, completion on
  // each instance's bar[0] (records in the forward sweep: bar[0] / bar[1] by buffer)
  uint64_t* bar = reinterpret_cast<uint64_t*>(slot + LY::BAR);
  uint64_t* barq[2] = {reinterpret_cast<uint64_t*>(slotq[0] + LY::BAR),
                       reinterpret_cast<uint64_t*>(slotq[1] + LY::BAR)};
  if (j == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncwarp();
  uint32_t ph0 = 0, ph1 = 0;
  constexpr uint32_t STG_BYTES = 8u * (n * n + 2 * n * m + sn + sm + (FAC ? 0 : 2 * n + m));
  using RT = typename std::conditional<F32, float, double>::type;  // factor record element type
  constexpr int FRECD = (NX * (NX + 1) + NX * NU + NU * (NU + 1) / 2 + 1) & ~1;  // factor record doubles
  constexpr int FREC = F32 ? ((FRECD + 3) & ~3) : FRECD;  // record stride in elements (16-byte multiple)
  RT* const frecb = F32 ? reinterpret_cast<RT*>(a.frec32) : reinterpret_cast<RT*>(a.frec);

  // Persistent warps (DESIGN.md §5 "phase staggering"): warp w of CTA b solves the instance pairs
  // p0 + k·stride, k = 0, 1, ...  The backward sweep is compute / shared-memory bound and the forward
  // sweep is HBM bound; run in lockstep (every warp backward, then every warp forward) the two never
  // overlap.  Each CTA therefore runs the forward sweep of pair k − d after the backward sweep of
  // pair k, with a per-CTA delay d = (b / #SMs) mod a.defer_mod: the CTAs sharing an SM are then in
  // their forward sweeps at different times and the forward's HBM traffic hides under the other
  // CTAs' backward sweeps.  x_0 and the backward status go through the output arrays in between.
  const int64_t npairs = (a.batch + 1) / 2;
  const int64_t stride = (int64_t)gridDim.x * WARPS;
  const int64_t p0 = (int64_t)blockIdx.x * WARPS + warp;
  const int64_t K = p0 < npairs ? (npairs - 1 - p0) / stride + 1 : 0;
  const int defer = (FAC || a.defer_mod <= 1) ? 0 : (int)((blockIdx.x / (a.nsm > 0 ? a.nsm : 1)) % a.defer_mod);

  auto pair_insts = [&](int64_t pair, int64_t (&instq)[2], bool (&validq)[2]) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      instq[q] = 2 * pair + q;
      validq[q] = instq[q] < a.batch;
      if (!validq[q]) instq[q] = a.batch - 1;
    }
  };

  // ---------------- backward sweep of one pair (+ x_0 and the backward status) ----------------
  auto backward_pair = [&](int64_t pair) {
    int64_t instq[2];
    bool validq[2];
    pair_insts(pair, instq, validq);
    const int64_t inst = grp ? instq[1] : instq[0];
    const bool valid = grp ? validq[1] : validq[0];
    const int64_t instP = (a.shared & RR_FLAG_SHARED_COST) ? 0 : inst;  // batch-shared Q, M, R, Q_N
    const double delta = a.p.delta[inst];
    double* rec0q[2] = {validq[0] ? a.ws + instq[0] * sN * RC::PAD : nullptr,
                        validq[1] ? a.ws + instq[1] * sN * RC::PAD : nullptr};
    int32_t st = 0;
    // generic-proxy writes of the previous pair's phase to this slot before the TMA refills it
    fence_proxy_async();
    __syncwarp();
    if constexpr (FAC) {  // no right-hand side: q, r, c slots of the stage buffers stay zero
      for (int e = j; e < 2 * n + m; e += 16) slot[oq + e] = 0.0;
    }
    auto issue_stage = [&](int i, double* dst) {
      const int64_t s = inst * sN + i;
      if constexpr (LY::BULK) {
        if (lane == 0) {
          fence_proxy_async();
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int64_t sq = instq[q] * sN + i;
            const int64_t sD = dyn_blk(a.shared, instq[q], sN, i);
            const int64_t sP = cost_blk(a.shared, instq[q], sN, i);
            double* d = slotq[q];
            uint64_t* bq = barq[q];
            mbar_arrive_expect_tx(bq, STG_BYTES);
            bulk_g2s(d + oA, a.p.A + sD * n * n, 8 * n * n, bq);
            bulk_g2s(d + oB, a.p.B + sD * n * m, 8 * n * m, bq);
            bulk_g2s(d + oQ, a.p.Q + sP * sn, 8 * sn, bq);
            bulk_g2s(d + oM, a.p.M + sP * n * m, 8 * n * m, bq);
            bulk_g2s(d + oR, a.p.R + sP * sm, 8 * sm, bq);
            if constexpr (!FAC) {
              bulk_g2s(d + oq, a.p.q + sq * n, 8 * n, bq);
              bulk_g2s(d + orr, a.p.r + sq * m, 8 * m, bq);
              bulk_g2s(d + oc, a.p.c + sq * n, 8 * n, bq);
            }
          }
        }
        (void)s;
        (void)dst;
      } else {
        const int64_t sD = dyn_blk(a.shared, inst, sN, i);
        const int64_t sP = cost_blk(a.shared, inst, sN, i);
        copy_async(dst + oA, a.p.A + sD * n * n, n * n, j, 16);
        copy_async(dst + oB, a.p.B + sD * n * m, n * m, j, 16);
        copy_async(dst + oQ, a.p.Q + sP * sn, sn, j, 16);
        copy_async(dst + oM, a.p.M + sP * n * m, n * m, j, 16);
        copy_async(dst + oR, a.p.R + sP * sm, sm, j, 16);
        copy_async(dst + oq, a.p.q + s * n, n, j, 16);
        copy_async(dst + orr, a.p.r + s * m, m, j, 16);
        copy_async(dst + oc, a.p.c + s * n, n, j, 16);
        cp_async_commit();
      }
    };
    auto wait_stage = [&]() {
      if constexpr (LY::BULK) {
        mbar_wait_parity(&bar[0], ph0);
        ph0 ^= 1u;
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
    };
    // P = [[Q M]; [Mᵀ R]] of the stage buffer sb (exact shape: no padding inside NZ)
    auto Pat = [&](const double* sb, int s, int t) -> double {
      if (s < NX && t < NX) return s >= t ? sb[oQ + pidx(n, s, t)] : sb[oQ + pidx(n, t, s)];
      if (s < NX) return sb[oM + s + (t - NX) * n];
      if (t < NX) return sb[oM + t + (s - NX) * n];
      const int u = s - NX, w = t - NX;
      return u >= w ? sb[oR + pidx(m, u, w)] : sb[oR + pidx(m, w, u)];
    };

    double Vc[NX];
    {
      const double* QN = a.p.QN + instP * sn;
#pragma unroll
      for (int r = 0; r < NX; ++r) Vc[r] = (j < n) ? (r >= j ? QN[pidx(n, r, j)] : QN[pidx(n, j, r)]) : 0.0;
      if (j < NX) wk[WK::vs + j] = FAC ? 0.0 : a.p.qN[inst * n + j];
      if (FAC && valid && j < n)  // record N: V_N = Q_N
        for (int r = j; r < n; ++r) frecb[inst * (sN + 1) * FREC + sN * FREC + pidx(n, r, j)] = (RT)QN[pidx(n, r, j)];
      if (valid && a.f.V != nullptr && j < n) {
        double* Vo = a.f.V + (inst * (sN + 1) + N) * sn;
        for (int r = j; r < n; ++r) Vo[pidx(n, r, j)] = QN[pidx(n, r, j)];
      }
      if (!FAC && valid && a.f.v != nullptr && j < n) a.f.v[(inst * (sN + 1) + N) * n + j] = a.p.qN[inst * n + j];
    }
    __syncwarp();  // (FAC) zeroed rhs slots visible before the first stage
    if (N > 0) issue_stage(N - 1, slot);
    __syncwarp();

    for (int i = N - 1; i >= 0; --i) {
      const double* sbq[2] = {slotq[0], slotq[1]};
      const double* Fq[2] = {sbq[0] + oA, sbq[1] + oA};
      const double* cvq[2] = {sbq[0] + oc, sbq[1] + oc};
      const double* sb = grp ? sbq[1] : sbq[0];
      auto qjf = [&]() -> double { return (j < NX) ? sb[oq + j] : sb[orr + j - NX]; };
#if defined(RR_NO_PTAB)
      auto P2 = [&](int q, int s, int t) -> double { return Pat(sbq[q], s, t); };
#elif defined(RR_P_SIMT)
      auto P2 = [&](int s) -> double { return Pat(sb, s, j); };  // column j of this lane's P
#else
      auto P2 = [&](int q, int k) -> double {
        return sbq[q][(int)((ptw[k >> 1] >> (16 * (k & 1))) & 0xffffu)];  // offsets in registers
      };
      (void)Pat;
#endif
      auto wait_inputs = [&]() { wait_stage(); };
      auto prefetch = [&]() {
        if (i > 0) issue_stage(i - 1, slot);
      };
      RT* recq[2];
      if constexpr (FAC) {
#pragma unroll
        for (int q = 0; q < 2; ++q) recq[q] = validq[q] ? frecb + (instq[q] * (sN + 1) + i) * FREC : nullptr;
      } else {
#pragma unroll
        for (int q = 0; q < 2; ++q) recq[q] = rec0q[q] ? reinterpret_cast<RT*>(rec0q[q] + (int64_t)i * RC::PAD) : nullptr;
      }
      double U[NZ], bj;
      SM::template backward<FAC, RT>(wkq, Fq, cvq, P2, qjf, wait_inputs, prefetch, delta, grp, j, lane, Vc, U, bj,
                                 recq, i, st);
      if (valid) {
        if (a.f.V != nullptr && j < n) {
          double* Vo = a.f.V + (inst * (sN + 1) + i) * sn;
#pragma unroll
          for (int r = 0; r < NX; ++r)
            if (r >= j) Vo[pidx(n, r, j)] = U[r];
        }
        if (a.f.K != nullptr && j < n) {
          double* Ko = a.f.K + (inst * sN + i) * m * n;
#pragma unroll
          for (int u = 0; u < NU; ++u) Ko[j * m + u] = -U[NX + u];
        }
        if (!FAC && j < NX && a.f.v != nullptr) a.f.v[(inst * (sN + 1) + i) * n + j] = bj;
        if (!FAC && j >= NX && j < NX + NU && a.f.k != nullptr) a.f.k[(inst * sN + i) * m + (j - NX)] = -bj;
      }
    }
    if constexpr (FAC) {  // S_0⁻¹ -> record 0; status; NaN-fill a failed instance's records
      if (lane == 0) bulk_wait0();  // the staged record bulk stores are complete (NaN-fill may overwrite them)
      __syncwarp();
      ST::invS(Vc, delta, j, wk, 0, st);
      RT* rec = frecb + inst * (sN + 1) * FREC;
      if (valid && j < n)
        for (int r = j; r < n; ++r) rec[sn + pidx(n, r, j)] = (RT)wk[WK::Si + r * NX + j];
      int32_t status = st;
#pragma unroll
      for (int off = 8; off > 0; off >>= 1) {
        const int32_t o = __shfl_xor_sync(RR_FULL_MASK, status, off);
        status = o > status ? o : status;
      }
      __syncwarp();
      if (valid && status != 0) {
        const double nan = __longlong_as_double(0x7ff8000000000000LL);
        for (int64_t e = j; e < (sN + 1) * FREC; e += 16) rec[e] = (RT)nan;
      }
      if (valid && j == 0) a.status[inst] = status;
      return;
    }
    // x_0 = (I + δV_0)⁻¹ (c_0 − δ v_0) -> x output row 0; backward status -> status (provisional)
    ST::invS(Vc, delta, j, wk, 0, st);
    double xr[NX];
#pragma unroll
    for (int r = 0; r < NX; ++r) xr[r] = a.p.c0[inst * n + r] - delta * wk[WK::vs + r];
    ST::mulSinv(xr, wk);
    int32_t status = st;
#pragma unroll
    for (int off = 8; off > 0; off >>= 1) {
      const int32_t o = __shfl_xor_sync(RR_FULL_MASK, status, off);
      status = o > status ? o : status;
    }
    double xj = 0.0;
#pragma unroll
    for (int r = 0; r < NX; ++r) xj = (r == j) ? xr[r] : xj;
    if (valid && j < n) a.s.x[inst * (sN + 1) * n + j] = xj;
    if (valid && j == 0) a.status[inst] = status;
    __syncwarp();  // x_0 / status visible to the group's forward sweep (same warp)
  };

  // ------- forward sweep of one pair: u = K x + k, y = V x + v, x⁺ = S_{i+1}⁻¹ (A x + B u + e) -------
  // (P:496-509); record i and A_i, B_i streamed by TMA into double buffers (one stage ahead)
  auto forward_pair = [&](int64_t pair) {
    if constexpr (!FAC) {
      int64_t instq[2];
      bool validq[2];
      pair_insts(pair, instq, validq);
      const int64_t inst = grp ? instq[1] : instq[0];
      const bool valid = grp ? validq[1] : validq[0];
      const int64_t instP = (a.shared & RR_FLAG_SHARED_COST) ? 0 : inst;
      double* xo = a.s.x + inst * (sN + 1) * n;
      double* uo = a.s.u + inst * sN * m;
      double* yo = a.s.y + inst * (sN + 1) * n;
      int32_t status = a.status[inst];
      double xr[NX], xj = 0.0;
#pragma unroll
      for (int r = 0; r < NX; ++r) {
        xr[r] = xo[r];
        xj = (r == j) ? xr[r] : xj;
      }
      bool bad = (j < n) && !isfinite(xj);
      const int ui = j - NX;
      constexpr int ABP = ((n * n + n * m) + 1) & ~1;
      // record offsets of row j of V_i (packed symmetric) or of K_i (lanes NX..), two per register
      uint32_t yofs[NX / 2];
#pragma unroll
      for (int k = 0; k < NX; k += 2) {
        uint32_t o[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int kk = k + h;
          o[h] = (j < NX) ? (uint32_t)(RC::V + (kk >= j ? pidx(NX, kk, j) : pidx(NX, j, kk)))
                          : (uint32_t)(RC::K + kk * NU + (ui < NU ? ui : 0));
        }
        yofs[k >> 1] = o[0] | (o[1] << 16);
      }
      const int ybase = (j < NX) ? RC::v + j : RC::k + (ui < NU ? ui : 0);
      auto rbuf = [&](double* sl, int b) { return sl + b * RC::PAD; };
      auto abuf = [&](double* sl, int b) { return sl + 2 * RC::PAD + b * ABP; };
      double* xch = slot + 2 * RC::PAD + 2 * ABP;  // exchange: u (NU, padded to even) | z (NX) | x (NX)
      double* uch = xch;
      double* zch = xch + ((NU + 1) & ~1);
      double* xsh = zch + NX;
      // records: the backward's TMA bulk stores must be complete before the TMA loads read them (lane 0
      // issued both); generic shared-memory writes of this slot ordered before the TMA refills
      if (lane == 0) bulk_wait0();
      asm volatile("fence.proxy.async;\n" ::: "memory");
      __syncwarp();
      auto issue_fwd = [&](int i, int b) {
        if (lane == 0) {
          fence_proxy_async();
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int64_t sD = dyn_blk(a.shared, instq[q], sN, i);
            mbar_arrive_expect_tx(&barq[q][b], 8u * (RC::SIZE + n * n + n * m));
            bulk_g2s(rbuf(slotq[q], b), a.ws + (instq[q] * sN + i) * RC::PAD, 8u * RC::SIZE, &barq[q][b]);
            bulk_g2s(abuf(slotq[q], b), a.p.A + sD * n * n, 8u * n * n, &barq[q][b]);
            bulk_g2s(abuf(slotq[q], b) + n * n, a.p.B + sD * n * m, 8u * n * m, &barq[q][b]);
          }
        }
      };
      auto wait_fwd = [&](int b) {
        if (b == 0) {
          mbar_wait_parity(&bar[0], ph0);
          ph0 ^= 1u;
        } else {
          mbar_wait_parity(&bar[1], ph1);
          ph1 ^= 1u;
        }
        __syncwarp();
      };
      if (N > 0) issue_fwd(0, 0);
#ifdef RR_AB_SKIP_FWD  // A/B probe only: cost of the forward sweep (wrong results)
      for (int i = 0; i < 0; ++i) {
#else
      for (int i = 0; i < N; ++i) {
#endif
        const int b = i & 1;
        const double* rc = rbuf(slot, b);
        const double* ab = abuf(slot, b);
        if (i + 1 < N) issue_fwd(i + 1, b ^ 1);
        wait_fwd(b);
        // y_i = V_i x_i + v_i (lanes < NX);  u_i = K_i x_i + k_i (lanes NX..): one code path for
        // all lanes through the per-lane record offsets yofs (no divergent V / K branches)
        double a0 = (j < NZ) ? rc[ybase] : 0.0, a1 = 0.0;
#pragma unroll
        for (int k = 0; k < NX; k += 2) {
          const uint32_t o2 = yofs[k >> 1];
          a0 = fma(rc[o2 & 0xffffu], xr[k], a0);
          a1 = fma(rc[o2 >> 16], xr[k + 1], a1);
        }
        const double yu = a0 + a1;
        if (valid) {
          if (j < n) yo[(int64_t)i * n + j] = yu;
          if (ui >= 0 && ui < m) uo[(int64_t)i * m + ui] = yu;
        }
        bad |= (j < NZ) && !isfinite(yu);
        if (ui >= 0 && ui < NU) uch[ui] = yu;
        __syncwarp();
        // z = A x + B u + e  (A, B column-major: row j)
        if (j < NX) {
          double z0 = rc[RC::e + j], z1 = 0.0;
#pragma unroll
          for (int k = 0; k < NX; k += 2) {
            z0 = fma(ab[j + k * n], xr[k], z0);
            z1 = fma(ab[j + (k + 1) * n], xr[k + 1], z1);
          }
#pragma unroll
          for (int u = 0; u < NU; ++u) z0 = fma(ab[n * n + j + u * n], uch[u], z0);
          zch[j] = z0 + z1;
        }
        __syncwarp();
        // x_{i+1} = S_{i+1}⁻¹ z
        double zr[NX];
        ST::bcast(zch, zr);
        if (j < NX) {
          double x0 = 0.0, x1 = 0.0;
#pragma unroll
          for (int k = 0; k < NX; k += 2) {
            const int i0 = k >= j ? pidx(NX, k, j) : pidx(NX, j, k);
            const int i1 = k + 1 >= j ? pidx(NX, k + 1, j) : pidx(NX, j, k + 1);
            x0 = fma(rc[RC::S + i0], zr[k], x0);
            x1 = fma(rc[RC::S + i1], zr[k + 1], x1);
          }
          const double xv = x0 + x1;
          if (valid && j < n) xo[(int64_t)(i + 1) * n + j] = xv;
          bad |= !isfinite(xv);
          xsh[j] = xv;
        }
        __syncwarp();
        ST::bcast(xsh, xr);
        __syncwarp();
      }
      {
        const double* QN = a.p.QN + instP * sn;
        if (j < n) {
          double acc = a.p.qN[inst * n + j];
#pragma unroll
          for (int k = 0; k < NX; ++k) acc = fma(k >= j ? QN[pidx(n, k, j)] : QN[pidx(n, j, k)], xr[k], acc);
          if (valid) yo[sN * n + j] = acc;
          bad |= !isfinite(acc);
        }
      }
      const unsigned anybad = __ballot_sync(RR_FULL_MASK, bad);
      const unsigned gmask = 0xffffu << gbase;
      if (status == 0 && (anybad & gmask)) status = RR_ST_NONFINITE;
      if (valid && status != 0) {
        const double nan = __longlong_as_double(0x7ff8000000000000LL);
        for (int64_t e = j; e < (sN + 1) * n; e += 16) {
          xo[e] = nan;
          yo[e] = nan;
        }
        for (int64_t e = j; e < sN * m; e += 16) uo[e] = nan;
      }
      if (valid && j == 0) a.status[inst] = status;
      __syncwarp();
    }
  };

  for (int64_t k = 0; k < K + defer; ++k) {
    if (k < K) backward_pair(p0 + k * stride);
    if (k >= defer && k - defer < K) forward_pair(p0 + (k - defer) * stride);
  }
}

template <int NX, int NU, int WARPS, int MINB, bool FAC = false, bool F32 = false>
struct MmaCfg {
  static constexpr int IPB = WARPS * 2;
  static size_t smem_bytes() {
    return sizeof(double) * (size_t)IPB * MmaLayout<NX, NU>::SLOT_PAD;
  }
  static int64_t ws_doubles(int64_t batch, int N) { return batch * (int64_t)N * RecM<NX, NU>::PAD; }
  static cudaError_t launch(const FusedArgs& a0, cudaStream_t s) {
    auto k = rr_fused_mma_kernel<NX, NU, WARPS, MINB, FAC, F32>;
    const size_t sm = smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    // persistent grid: every resident CTA slot once (the warps loop over instance pairs)
    // (SM count and occupancy are per device and kernel: queried once per device and cached -- the
    // values are immutable, so a racing first call at worst queries twice)
    int dev = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    constexpr int MAXDEV = 64;
    static std::atomic<int> cache[MAXDEV];  // (nsm << 8) | occ, 0 = not yet queried
    int nsm = 0, occ = 0;
    const int cv = (dev >= 0 && dev < MAXDEV) ? cache[dev].load(std::memory_order_relaxed) : 0;
    if (cv != 0) {
      nsm = cv >> 8;
      occ = cv & 0xff;
    } else {
      if ((e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
      if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, WARPS * 32, sm)) != cudaSuccess) return e;
      if (dev >= 0 && dev < MAXDEV && occ > 0 && occ < 256) cache[dev].store((nsm << 8) | occ, std::memory_order_relaxed);
    }
    FusedArgs a = a0;
    a.nsm = nsm;
    a.defer_mod = 1;  // measured: staggering by occ (3) is 1-2% slower on C2 (profiles/r02_stagger_ab.txt)
    if (const char* v = getenv("RR_DEFER_MOD")) a.defer_mod = atoi(v);  // A/B knob (1 = no staggering)
    const int64_t need = ((a.batch + 1) / 2 + WARPS - 1) / WARPS;
    int64_t blocks = (int64_t)nsm * (occ > 0 ? occ : 1);
    if (const char* v = getenv("RR_PERSIST")) {  // A/B knob: 0 = one CTA per 2*WARPS instances
      if (atoi(v) == 0) blocks = need;
    }
    if (blocks > need) blocks = need;
    if (blocks < 1) blocks = 1;
    k<<<(unsigned)blocks, WARPS * 32, sm, s>>>(a);
    return cudaGetLastError();
  }
};

// Shape dispatch: exact specialisations for the BASELINE configs, padded fallbacks otherwise.
// RR_B200_VARIANT (environment, read per call; tuning knob for the 12x4 kernel): 0 = default
// (DMMA stage kernel rr_stage_mma.cuh, TMA stage loads, 3 CTAs/SM), 1/2 = SIMT stage kernel with
// 3 / 2 CTAs/SM, 3/4 = DMMA kernel with 2-warp CTAs / 2 CTAs/SM.
static int variant() {
  const char* v = getenv("RR_B200_VARIANT");
  return v ? atoi(v) : 0;
}

template <typename F>
static bool dispatch_fused(int nx, int nu, F&& f) {
  if (nx == 12 && nu == 4) {
    const int v = variant();
    if (v == 1) return f(FusedCfg<12, 4, 16, 4, 3, true>{});
    if (v == 2) return f(FusedCfg<12, 4, 16, 4, 2, true>{});
    if (v == 3) return f(MmaCfg<12, 4, 2, 6>{});
    if (v == 4) return f(MmaCfg<12, 4, 4, 2>{});
    if (v == 5) return f(MmaCfg<12, 4, 4, 3>{});  // A/B: 3 CTAs per SM (168 registers)
    return f(MmaCfg<12, 4, 4, 4>{});              // 4 CTAs (16 warps) per SM: 128 registers, 55.5 KB
  }
  if (nx == 4 && nu == 1) return f(FusedCfg<4, 1, 8, 4, 4, true>{});
  if (nx == 2 && nu == 1) return f(FusedCfg<2, 1, 4, 4, 4, true>{});
  if (nx <= 2 && nu <= 2) return f(FusedCfg<2, 2, 4, 4, 1, false>{});
  if (nx <= 4 && nu <= 4) return f(FusedCfg<4, 4, 8, 4, 1, false>{});
  if (nx <= 8 && nu <= 8) return f(FusedCfg<8, 8, 16, 4, 1, false>{});
  if (nx <= 16 && nu <= 16) return f(FusedCfg<16, 16, 32, 4, 1, false>{});
  return false;
}

int64_t fused_workspace_bytes(int nx, int nu, int N, int64_t batch) {
  int64_t out = -1;
  const bool small = dispatch_fused(nx, nu, [&](auto cfg) {
    out = 8 * decltype(cfg)::ws_doubles(batch, N) + 256;
    return true;
  });
  if (!small) out = cta_workspace_bytes(nx, nu, N, batch);  // large stages: CTA per instance
  if (nx == 12 && nu == 4) {  // room for the LDGSTS fallback taken when operands are not 16-byte aligned
    const int64_t simt = 8 * FusedCfg<12, 4, 16, 4, 3, true>::ws_doubles(batch, N) + 256;
    if (simt > out) out = simt;
  }
  return out;
}

cudaError_t fused_launch(const FusedArgs& a, cudaStream_t s, bool* supported) {
  cudaError_t err = cudaSuccess;
  if (a.nx == 12 && a.nu == 4 && !a.tma16) {  // operands not 16-byte aligned: no TMA bulk copies
    *supported = true;
    return FusedCfg<12, 4, 16, 4, 3, true>::launch(a, s);
  }
  *supported = dispatch_fused(a.nx, a.nu, [&](auto cfg) {
    err = decltype(cfg)::launch(a, s);
    return true;
  });
  if (!*supported) err = cta_launch(a, s, supported);
  return err;
}

}  // namespace rrk

namespace rrk {
// rr_factor for the 12x4 shape on the DMMA stage kernel (factor-only mode).
cudaError_t factor_mma_launch(const FusedArgs& a, cudaStream_t s, bool* supported) {
  *supported = (a.nx == 12 && a.nu == 4);
  if (!*supported) return cudaSuccess;
  // 3 CTAs per SM: at 4 (128 registers) the factor-only kernel spills, 11.40 vs 10.99 ms on C2
  const char* v = getenv("RR_B200_FAC_CTAS");  // A/B knob: 4 = 4 CTAs per SM
  if (v && atoi(v) == 4) {
    if (a.frec32 != nullptr) return MmaCfg<12, 4, 4, 4, true, true>::launch(a, s);
    return MmaCfg<12, 4, 4, 4, true>::launch(a, s);
  }
  if (a.frec32 != nullptr) return MmaCfg<12, 4, 4, 3, true, true>::launch(a, s);  // FP32 records
  return MmaCfg<12, 4, 4, 3, true>::launch(a, s);
}
}  // namespace rrk
