// rr_cta.cu -- fused regularized-Riccati factor + solve for LARGE stages (C3: n_x = 64, n_u = 32):
// one CTA per instance, all stage matrices resident in shared memory, every dense contraction on
// the FP64 tensor-core path (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4), pivots on the SIMT path.
//
// Method (arXiv 2509.16370, P:n = PAPER.md line n), per stage i = N-1..0 (Eq.(RR)):
//   S⁻¹ = (I + δV_{i+1})⁻¹                      symmetric sweep (SPD, eigenvalues >= 1)
//   [W | W e] = S⁻¹ [V | V e], e = c_{i+1} − δ v_{i+1}          (W_i; g_i = v + W e)
//   [T | g] = [W F | g],  F = [A B]
//   [U | b] = Fᵀ [T | g] + [P | (q; r)]          U = [[AᵀWA+Q, Hᵀ]; [H, G]], b = [q+Aᵀg; r+Bᵀg]
//   G⁻¹ by a symmetric sweep; K̃ = G⁻¹ [H | h]                    (−K_i, −k_i)
//   [V_i | v_i] = [AᵀWA+Q | q+Aᵀg] − Hᵀ K̃                        (P:623-624 with P:606-611)
//   [Φ_i | φ_i] = S⁻¹ ([A | c_{i+1} − δ v_{i+1}] − B K̃)  -> record for the forward sweep
// forward: x_{i+1} = Φ_i x_i + φ_i, u_i = K_i x_i + k_i, y_i = V_i x_i + v_i.
// Shared-memory plan (doubles) for one instance: stage input (cp.async) | S⁻¹ | V/W/U | T/K̃/M |
// vectors -- about 230 KB, one CTA per SM; the next stage's input streams in during the last
// contraction of the current stage.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rr_common.cuh"
#include "rr_cta.cuh"
#include "rr_stage_mma.cuh"

namespace rrk {

template <int NX, int NU>
struct CtaLayout {
  static constexpr int NZ = NX + NU;
  static constexpr int SN = NX * (NX + 1) / 2, SMU = NU * (NU + 1) / 2;
  // stage input in the global operand order: A | B (= F, col-major ld NX) | Q | M | R | q | r | c
  static constexpr int oA = 0, oB = NX * NX, oQ = oB + NX * NU, oM = oQ + SN, oR = oM + NX * NU, oq = oR + SMU,
                       orr = oq + NX, oc = orr + NU;
  static constexpr int IN = ((oc + NX + 1) & ~1);
  static constexpr int SI = IN;                                   // S⁻¹, NX × NX (ld NX)
  static constexpr int VW = SI + NX * NX;                         // [V | Ve] / [W | We] (ld NX, NX+1 cols)
  // U parts (after W is consumed): Uxx | bx (ld NX, NX+1 cols), Uux | bu (ld NU, NX+1 cols), Uuu (ld NU)
  static constexpr int Uxx = VW;
  static constexpr int Uux = Uxx + NX * (NX + 1);
  static constexpr int Uuu = Uux + NU * (NX + 1);
  static constexpr int VWU_END = Uuu + NU * NU;
  static constexpr int TT = ((VWU_END + 1) & ~1);                 // [T | g] (ld NX, NZ+1 cols); later K̃, M
  static constexpr int Kt = TT;                                   // K̃ = G⁻¹[Uux | bu] (ld NU, NX+1 cols)
  static constexpr int MM = Kt + ((NU * (NX + 1) + 1) & ~1);      // M (ld NX, NX+1 cols)
  static constexpr int T_END = TT + (NX * (NZ + 1) > (MM - TT) + NX * (NX + 1) ? NX * (NZ + 1) : (MM - TT) + NX * (NX + 1));
  static constexpr int VEC = ((T_END + 1) & ~1);
  static constexpr int vs = VEC;         // v_{i+1} (NX)
  static constexpr int pr = vs + NX;     // pivot column buffer / g / x_{i+1} (2 × NX)
  static constexpr int xs = pr + 2 * NX;  // x (NX)
  static constexpr int TOTAL = xs + NX;
  static constexpr int red = TT;          // forward-pass partial sums (4 × (2NX+NU)), TT is dead then
  static_assert(4 * (2 * NX + NU) <= T_END - TT, "partial-sum buffer does not fit the T region");
  // forward record (global, per stage): Φ̃ (ld NX, NX+1 cols) | K (ld NU, NX cols) | k | V (ld NX) | v
  static constexpr int rPHI = 0, rK = NX * (NX + 1), rk = rK + NU * NX, rV = rk + NU, rv = rV + NX * NX;
  static constexpr int REC = ((rv + NX + 1) & ~1);
};

// Shared-memory index of element (r, c) of a column-major matrix with leading dimension LD.
// For LD % 16 == 0 the row index is XOR-swizzled inside 16-element groups (bits 2-3 flipped by a
// function of the column) so that the DMMA fragment loads (A, Aᵀ, B patterns), the C-fragment
// stores and 16-byte column copies are bank-conflict free per half-warp; otherwise plain.
template <int LD>
__device__ __forceinline__ int swz(int r, int c) {
  if constexpr (LD % 16 == 0) return c * LD + (r ^ (((c ^ (c >> 2)) & 3) << 2));
  else return c * LD + r;
}

// C (rows < Mlim, cols < Nlim) = sign * op(A) · B + Cinit, all column-major in shared memory.
// op(A) = A (M×K, ld lda) or Aᵀ (A stored K×M, ld lda).  M, N multiples of 8 (padded tiles are
// computed and masked on store); K multiple of 4.  Warps take 16×16 super-tiles round-robin.
// Cinit(r, c) is a functor (returns 0 for a plain product).  Store(r, c, v) writes the result.
template <int M, int N, int K, bool TRANS_A, typename LoadA, typename LoadB, typename Init, typename Store>
__device__ __forceinline__ void cta_gemm(LoadA&& la, LoadB&& lb, Init&& init, Store&& store, int warp, int nwarps,
                                         int lane) {
  constexpr int MT = (M + 15) / 16, NT = (N + 15) / 16, KT = K / 4;
  static_assert(K % 4 == 0, "K must be a multiple of 4");
  const int g = lane >> 2, t = lane & 3;
  for (int tile = warp; tile < MT * NT; tile += nwarps) {
    const int m0 = (tile % MT) * 16, n0 = (tile / MT) * 16;
    double c[2][2][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = m0 + 8 * a + g, col = n0 + 8 * b + 2 * t + e;
          c[a][b][e] = (r < M && col < N) ? init(r, col) : 0.0;
        }
#pragma unroll 4
    for (int kt = 0; kt < KT; ++kt) {
      double av[2], bv[2];
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const int r = m0 + 8 * a + g;
        av[a] = (r < M) ? la(r, 4 * kt + t) : 0.0;
      }
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int col = n0 + 8 * b + g;
        bv[b] = (col < N) ? lb(4 * kt + t, col) : 0.0;
      }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) dmma884(c[a][b][0], c[a][b][1], av[a], bv[b]);
    }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = m0 + 8 * a + g, col = n0 + 8 * b + 2 * t + e;
          if (r < M && col < N) store(r, col, c[a][b][e]);
        }
  }
}

// Lower-tile GEMM for a SYMMETRIC M×M result: C = op(A)·B + init over the 16×16 super-tiles
// (R, C) with R >= C only (masked to M); store(r, c, v, mirror) is told whether the tile is
// off-diagonal, so the caller can write the transposed entry.  Halves the DMMA work of W, U, V_i.
template <int M, int K, typename LoadA, typename LoadB, typename Init, typename Store>
__device__ __forceinline__ void cta_gemm_lower(LoadA&& la, LoadB&& lb, Init&& init, Store&& store, int warp,
                                               int nwarps, int lane) {
  constexpr int MT = (M + 15) / 16, NTL = MT * (MT + 1) / 2, KT = K / 4;
  static_assert(K % 4 == 0, "K must be a multiple of 4");
  const int g = lane >> 2, t = lane & 3;
  for (int tile = warp; tile < NTL; tile += nwarps) {
    int R = 0, rem = tile;
    while (rem > R) {
      rem -= R + 1;
      ++R;
    }
    const int C = rem, m0 = 16 * R, n0 = 16 * C;
    const bool mir = R != C;
    double c[2][2][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = m0 + 8 * a + g, col = n0 + 8 * b + 2 * t + e;
          c[a][b][e] = (r < M && col < M) ? init(r, col) : 0.0;
        }
#pragma unroll 4
    for (int kt = 0; kt < KT; ++kt) {
      double av[2], bv[2];
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const int r = m0 + 8 * a + g;
        av[a] = (r < M) ? la(r, 4 * kt + t) : 0.0;
      }
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int col = n0 + 8 * b + g;
        bv[b] = (col < M) ? lb(4 * kt + t, col) : 0.0;
      }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) dmma884(c[a][b][0], c[a][b][1], av[a], bv[b]);
    }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = m0 + 8 * a + g, col = n0 + 8 * b + 2 * t + e;
          if (r < M && col < M) store(r, col, c[a][b][e], mir);
        }
  }
}

// y = init + A x for an M×K matrix on the SIMT pipe: PARTS adjacent threads per row (power of
// two), partial sums combined by shuffles.  All NTHREADS threads must call it (uniform loop).
template <int M, int K, int NTHREADS, typename LoadA, typename LoadX, typename Init, typename Out>
__device__ __forceinline__ void cta_matvec(LoadA&& la, LoadX&& x, Init&& init, Out&& out, int tid) {
  constexpr int P0 = NTHREADS / M;
  constexpr int PARTS = P0 >= 8 ? 8 : (P0 >= 4 ? 4 : (P0 >= 2 ? 2 : 1));
  for (int base = 0; base < M * PARTS; base += NTHREADS) {
    const int task = base + tid, row = task / PARTS, part = task % PARTS;
    double acc = 0.0;
    if (row < M)
      for (int k = part; k < K; k += PARTS) acc = fma(la(row, k), x(k), acc);
#pragma unroll
    for (int off = PARTS / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(RR_FULL_MASK, acc, off);
    if (row < M && part == 0) out(row, init(row) + acc);
  }
}

// In-place symmetric sweep of the n×n SPD matrix A (ld lda) in shared memory: A <- −A⁻¹.
// Pivot p: Ã_pp = −1/A_pp, Ã_rp = A_rp/A_pp, Ã_pc = A_pc/A_pp, Ã_rc = A_rc − A_rp A_pc/A_pp.
// Returns (in *fail) whether a pivot was not > 0 (block-uniform).
template <int n>
__device__ __forceinline__ void cta_sweep(double* A, int lda, double* colbuf, int tid, int nthreads, bool* fail) {
  bool bad = false;
  for (int p = 0; p < n; ++p) {
    for (int r = tid; r < n; r += nthreads) colbuf[r] = A[swz<n>(r, p)];  // column p (= row p)
    __syncthreads();
    const double d = colbuf[p];
    bad |= !(d > 0.0);
    const double id = rcp_nr(d);
    for (int e = tid; e < n * n; e += nthreads) {
      const int r = e % n, c = e / n;
      const double arc = A[swz<n>(r, c)];
      double v;
      if (r == p && c == p) v = -id;
      else if (r == p) v = colbuf[c] * id;           // row p = column p (symmetric)
      else if (c == p) v = colbuf[r] * id;
      else v = fma(-colbuf[r] * id, colbuf[c], arc);
      A[swz<n>(r, c)] = v;
    }
    __syncthreads();
  }
  *fail = bad;
}

// Register-blocked version of cta_sweep for n % 16 == 0 with 256 threads: thread (rb, cb) of a
// 16 × 16 grid owns the BR × BR block (BR = n/16) in registers; per pivot the column (= row, by
// symmetry) is published through a double-buffered shared vector, one barrier per pivot.
template <int n>
__device__ __forceinline__ void cta_sweep_reg(double* A, int /*lda == n*/, double* colbuf2, int tid, bool* fail) {
  constexpr int BR = n / 16;
  static_assert(n % 16 == 0, "register sweep needs n % 16 == 0");
  const int rb = tid & 15, cb = tid >> 4;  // 256 threads
  double a[BR][BR];
#pragma unroll
  for (int i = 0; i < BR; ++i)
#pragma unroll
    for (int k = 0; k < BR; ++k) a[i][k] = A[swz<n>(rb * BR + i, cb * BR + k)];
  bool bad = false;
  for (int p = 0; p < n; ++p) {
    double* cb_ = colbuf2 + (p & 1) * n;
    const int pb = p / BR, pi = p - pb * BR;
    if (cb == pb) {
#pragma unroll
      for (int k = 0; k < BR; ++k)
        if (k == pi) {
#pragma unroll
          for (int i = 0; i < BR; ++i) cb_[rb * BR + i] = a[i][k];
        }
    }
    __syncthreads();
    const double d = cb_[p];
    bad |= !(d > 0.0);
    const double id = rcp_nr(d);
    double cr[BR], cc[BR];
#pragma unroll
    for (int i = 0; i < BR; ++i) {
      cr[i] = cb_[rb * BR + i] * id;
      cc[i] = cb_[cb * BR + i];
    }
#pragma unroll
    for (int i = 0; i < BR; ++i)
#pragma unroll
      for (int k = 0; k < BR; ++k) a[i][k] = fma(-cr[i], cc[k], a[i][k]);
    if (rb == pb) {  // row p: Ã_pc = A_pc / d
#pragma unroll
      for (int i = 0; i < BR; ++i)
        if (i == pi) {
#pragma unroll
          for (int k = 0; k < BR; ++k) a[i][k] = cc[k] * id;
        }
    }
    if (cb == pb) {  // column p: Ã_rp = A_rp / d, Ã_pp = −1/d
#pragma unroll
      for (int k = 0; k < BR; ++k)
        if (k == pi) {
#pragma unroll
          for (int i = 0; i < BR; ++i) a[i][k] = (rb == pb && i == pi) ? -id : cr[i];
        }
    }
  }
#pragma unroll
  for (int i = 0; i < BR; ++i)
#pragma unroll
    for (int k = 0; k < BR; ++k) A[swz<n>(rb * BR + i, cb * BR + k)] = a[i][k];
  __syncthreads();
  *fail = bad;
}

// One 16×16 output tile at (r0, c0) of  C = op_A · B + init  (K multiple of 4) on one warp.
template <int K, typename LoadA, typename LoadB, typename Init, typename Store>
__device__ __forceinline__ void warp_tile16(int r0, int c0, LoadA&& la, LoadB&& lb, Init&& init, Store&& store,
                                            int lane) {
  const int g = lane >> 2, t = lane & 3;
  double c[2][2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) c[a][b][e] = init(r0 + 8 * a + g, c0 + 8 * b + 2 * t + e);
#pragma unroll
  for (int kt = 0; kt < K / 4; ++kt) {
    double av[2], bv[2];
#pragma unroll
    for (int a = 0; a < 2; ++a) av[a] = la(r0 + 8 * a + g, 4 * kt + t);
#pragma unroll
    for (int b = 0; b < 2; ++b) bv[b] = lb(4 * kt + t, c0 + 8 * b + g);
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) dmma884(c[a][b][0], c[a][b][1], av[a], bv[b]);
  }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) store(r0 + 8 * a + g, c0 + 8 * b + 2 * t + e, c[a][b][e]);
}

// Symmetric sweep of a 16×16 diagonal block held in one warp's registers: lane l owns column
// c = l & 15, rows 8h .. 8h+7 (h = l >> 4).  Pivots 0..15 in order (the scalar sweep of the
// block); pivot column / row entries travel by shuffles (row k = column k by symmetry).
__device__ __forceinline__ void warp_sweep16(double (&a)[8], int lane, bool* bad) {
  const int c = lane & 15, h = lane >> 4;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const double d = __shfl_sync(RR_FULL_MASK, a[k & 7], k + 16 * (k >> 3));
    const double rowk = __shfl_sync(RR_FULL_MASK, a[k & 7], c + 16 * (k >> 3));  // A[k][c]
    double colk[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) colk[i] = __shfl_sync(RR_FULL_MASK, a[i], k + 16 * h);  // A[8h+i][k]
    *bad |= !(d > 0.0);
    const double id = rcp_nr(d);
    const double rs = rowk * id;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = 8 * h + i;
      const double upd = fma(-colk[i], rs, a[i]);
      a[i] = (r == k) ? ((c == k) ? -id : rs) : ((c == k) ? colk[i] * id : upd);
    }
  }
}

// Block (16-pivot) symmetric sweep of the n×n SPD matrix A (n % 16 == 0, swizzled ld n):
// A <- −A⁻¹.  Sweeping the pivots of block p at once is the block form of the sweep operator:
//   Z = A_pp⁻¹:  A_pp <- −Z,  A_rp <- A_rp Z,  A_pc <- Z A_pc,  A_rc <- A_rc − A_rp Z A_pc,
// identical (up to rounding) to the 16 scalar sweeps of block p.  Per block: warp 0 sweeps A_pp in
// registers; Y = A_{:,p} Z (DMMA, into `Y`, n × 16); the trailing update A_RC −= Y_R A_pC over the
// lower tiles R >= C (mirrored to C, R) on DMMA; then column / row block p <- Y / Yᵀ (overlapped
// with the next block's diagonal sweep).  3 barriers per block instead of 2 per pivot.
// (A lookahead variant -- warp 0 updating and sweeping tile (p+1, p+1) during the trailing update --
// measured slower on C3: the dependency chain tile -> sweep -> Y tile is the same length.)
template <int n, int NTHREADS>
__device__ __forceinline__ void cta_sweep_blk(double* A, double* Y, int tid, bool* fail) {
  constexpr int NB = n / 16;
  constexpr int NW = NTHREADS / 32;
  static_assert(n % 16 == 0, "block sweep needs n % 16 == 0");
  const int lane = tid & 31, warp = tid >> 5;
  bool bad = false;
  auto S = [](int r, int c) { return swz<n>(r, c); };
  for (int p = 0; p < NB; ++p) {
    const int p0 = 16 * p;
    if (warp == 0) {
      double a[8];
      const int c = lane & 15, h = lane >> 4;
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = A[S(p0 + 8 * h + i, p0 + c)];
      warp_sweep16(a, lane, &bad);
#pragma unroll
      for (int i = 0; i < 8; ++i) A[S(p0 + 8 * h + i, p0 + c)] = a[i];  // −Z
    } else if (p > 0) {
      // previous block q = p − 1: column block q <- Y, row block q <- Yᵀ (rows outside block q)
      const int q0 = p0 - 16;
      for (int e = tid - 32; e < n * 16; e += NTHREADS - 32) {
        const int r = e % n, cc = e / n;
        if (r >= q0 && r < q0 + 16) continue;
        const double v = Y[S(r, cc)];
        A[S(r, q0 + cc)] = v;
        A[S(q0 + cc, r)] = v;
      }
    }
    __syncthreads();
    // Y_R = A_{R,p} Z = −A_{R,p} A'_pp for the row tiles R != p
    for (int R = warp; R < NB; R += NW) {
      if (R == p) continue;
      warp_tile16<16>(
          16 * R, 0, [&](int r, int k) { return A[S(r, p0 + k)]; }, [&](int k, int c) { return -A[S(p0 + k, p0 + c)]; },
          [&](int, int) { return 0.0; }, [&](int r, int c, double v) { Y[S(r, c)] = v; }, lane);
    }
    __syncthreads();
    // trailing update of the lower tiles R >= C (R, C != p), mirrored: A_RC −= Y_R A_pC
    constexpr int NO = NB - 1, NT = NO * (NO + 1) / 2;
    for (int tt = warp; tt < NT; tt += NW) {
      int R = 0, C = 0, cnt = tt;  // tt-th pair (R >= C) of the blocks other than p
      for (int cc = 0; cc < NO; ++cc) {
        if (cnt < NO - cc) {
          C = cc;
          R = cc + cnt;
          break;
        }
        cnt -= NO - cc;
      }
      R += (R >= p);
      C += (C >= p);
      const int r0 = 16 * R, c0 = 16 * C;
      warp_tile16<16>(
          r0, c0, [&](int r, int k) { return -Y[S(r, k)]; }, [&](int k, int c) { return A[S(p0 + k, c)]; },
          [&](int r, int c) { return A[S(r, c)]; },
          [&](int r, int c, double v) {
            A[S(r, c)] = v;
            if (R != C) A[S(c, r)] = v;
          },
          lane);
    }
    __syncthreads();
  }
  {  // last block's row / column
    const int q0 = n - 16;
    for (int e = tid; e < n * 16; e += NTHREADS) {
      const int r = e % n, cc = e / n;
      if (r >= q0) continue;
      const double v = Y[S(r, cc)];
      A[S(r, q0 + cc)] = v;
      A[S(q0 + cc, r)] = v;
    }
  }
  __syncthreads();
  *fail = bad;
}

template <int n, int NTHREADS>
__device__ __forceinline__ void cta_sweep_any(double* A, int lda, double* colbuf2, double* ytmp, int tid, bool* fail) {
  if constexpr (n % 16 == 0 && n >= 32) cta_sweep_blk<n, NTHREADS>(A, ytmp, tid, fail);
  else if constexpr (n % 16 == 0 && NTHREADS == 256) cta_sweep_reg<n>(A, lda, colbuf2, tid, fail);
  else cta_sweep<n>(A, lda, colbuf2, tid, NTHREADS, fail);
}

template <int NX, int NU, int NTHREADS>
__global__ void __launch_bounds__(NTHREADS, 1) rr_cta_kernel(const FusedArgs a) {
  using L = CtaLayout<NX, NU>;
  constexpr int NZ = NX + NU;
  constexpr int n = NX, m = NU;
  constexpr int NW = NTHREADS / 32;
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t inst = blockIdx.x;
  const int N = a.N;
  const int64_t sN = N;
  const double delta = a.p.delta[inst];
  double* rec0 = a.ws + inst * sN * L::REC;
  int32_t st = 0;

  auto X = [](int r, int c) { return swz<NX>(r, c); };  // ld NX matrices (F, S⁻¹, V/W/Uxx, T, M)
  auto Y = [](int r, int c) { return swz<NU>(r, c); };  // ld NU matrices (Uux, Uuu, K̃)
  auto issue_stage = [&](int i) {
    const int64_t s = inst * sN + i;
    // F = [A B]: 16-byte chunks (rows r, r+1) to their swizzled column positions
    const double* gA = a.p.A + s * n * n;
    const double* gB = a.p.B + s * n * m;
    for (int e = 2 * tid; e < n * NZ; e += 2 * NTHREADS) {
      const int r = e % n, c = e / n;
      const double* src = c < NX ? gA + r + c * n : gB + r + (c - NX) * n;
      cp_async16(sm + L::oA + X(r, c), src);
    }
    copy_async(sm + L::oQ, a.p.Q + s * L::SN, L::SN, tid, NTHREADS);
    copy_async(sm + L::oM, a.p.M + s * n * m, n * m, tid, NTHREADS);
    copy_async(sm + L::oR, a.p.R + s * L::SMU, L::SMU, tid, NTHREADS);
    copy_async(sm + L::oq, a.p.q + s * n, n, tid, NTHREADS);
    copy_async(sm + L::orr, a.p.r + s * m, m, tid, NTHREADS);
    copy_async(sm + L::oc, a.p.c + s * n, n, tid, NTHREADS);
    cp_async_commit();
  };
  // V_N = Q_N -> [V | ·] region (ld NX), v_N = q_N
  {
    const double* QN = a.p.QN + inst * L::SN;
    for (int e = tid; e < n * n; e += NTHREADS) {
      const int r = e % n, c = e / n;
      sm[L::VW + X(r, c)] = r >= c ? QN[pidx(n, r, c)] : QN[pidx(n, c, r)];
    }
    for (int r = tid; r < n; r += NTHREADS) sm[L::vs + r] = a.p.qN[inst * n + r];
    if (a.f.V != nullptr)
      for (int e = tid; e < L::SN; e += NTHREADS) a.f.V[(inst * (sN + 1) + N) * L::SN + e] = QN[e];
    if (a.f.v != nullptr)
      for (int r = tid; r < n; r += NTHREADS) a.f.v[(inst * (sN + 1) + N) * n + r] = a.p.qN[inst * n + r];
  }
  if (N > 0) issue_stage(N - 1);
  __syncthreads();

  auto Pat = [&](int s, int t) -> double {  // P = [[Q M]; [Mᵀ R]] from the stage input (plain layout)
    if (s < NX && t < NX) return s >= t ? sm[L::oQ + pidx(n, s, t)] : sm[L::oQ + pidx(n, t, s)];
    if (s < NX) return sm[L::oM + s + (t - NX) * n];
    if (t < NX) return sm[L::oM + t + (s - NX) * n];
    const int u = s - NX, w = t - NX;
    return u >= w ? sm[L::oR + pidx(m, u, w)] : sm[L::oR + pidx(m, w, u)];
  };

  for (int i = N - 1; i >= 0; --i) {
    cp_async_wait<0>();
    __syncthreads();
    double* rec = rec0 + (int64_t)i * L::REC;
    // S = I + δV -> SI; column NX of [V | ·] = V e with e = c_{i+1} − δ v_{i+1}
    for (int e = tid; e < n * n; e += NTHREADS) {
      const int r = e % n, c = e / n;
      sm[L::SI + X(r, c)] = delta * sm[L::VW + X(r, c)] + (r == c ? 1.0 : 0.0);
    }
    {  // V e with 4 threads per row (NTHREADS >= 4 n)
      static_assert(NTHREADS >= 4 * NX, "V e matvec layout");
      const int r = tid >> 2, part = tid & 3;
      double acc = 0.0;
      if (r < n)
        for (int k = part; k < n; k += 4) acc = fma(sm[L::VW + X(r, k)], sm[L::oc + k] - delta * sm[L::vs + k], acc);
      acc += __shfl_xor_sync(RR_FULL_MASK, acc, 1);
      acc += __shfl_xor_sync(RR_FULL_MASK, acc, 2);
      if (r < n && part == 0) sm[L::VW + X(r, NX)] = acc;
    }
    __syncthreads();
    bool fail = false;
    cta_sweep_any<NX, NTHREADS>(sm + L::SI, n, sm + L::pr, sm + L::TT, tid, &fail);  // SI = −S⁻¹
    if (fail && st == 0) st = mk_status(RR_ST_S_NOT_PD, i);
    // W = S⁻¹ V (symmetric: S⁻¹ and V commute) -> TT region temporarily (same ld / swizzle), lower
    // tiles mirrored; g = v_{i+1} + S⁻¹ (V e) on the SIMT pipe in the same phase
    cta_gemm_lower<NX, NX>(
        [&](int r, int k) { return -sm[L::SI + X(r, k)]; }, [&](int k, int c) { return sm[L::VW + X(k, c)]; },
        [&](int, int) { return 0.0; },
        [&](int r, int c, double v, bool mir) {
          sm[L::TT + X(r, c)] = v;
          if (mir) sm[L::TT + X(c, r)] = v;
        },
        warp, NW, lane);
    cta_matvec<NX, NX, NTHREADS>(
        [&](int r, int k) { return -sm[L::SI + X(r, k)]; }, [&](int k) { return sm[L::VW + X(k, NX)]; },
        [&](int r) { return sm[L::vs + r]; }, [&](int r, double v) { sm[L::pr + r] = v; }, tid);
    __syncthreads();
    for (int e = tid; e < n * n; e += NTHREADS) sm[L::VW + e] = sm[L::TT + e];  // same layout: flat copy of W
    __syncthreads();
    // T = W F (F = [A B] = stage input columns, ld NX);  b = (q; r) + Fᵀ g  (SIMT, same phase)
    cta_gemm<NX, NZ, NX, false>(
        [&](int r, int k) { return sm[L::VW + X(r, k)]; }, [&](int k, int c) { return sm[L::oA + X(k, c)]; },
        [&](int, int) { return 0.0; }, [&](int r, int c, double v) { sm[L::TT + X(r, c)] = v; }, warp, NW, lane);
    cta_matvec<NZ, NX, NTHREADS>(
        [&](int r, int k) { return sm[L::oA + X(k, r)]; }, [&](int k) { return sm[L::pr + k]; },
        [&](int r) { return r < NX ? sm[L::oq + r] : sm[L::orr + r - NX]; },
        [&](int r, double v) {
          if (r < NX) sm[L::Uxx + X(r, NX)] = v;  // b_x (column NX of the V/W region: W uses 0..NX-1)
          else sm[L::Uux + Y(r - NX, NX)] = v;    // b_u
        },
        tid);
    __syncthreads();
    // U = Fᵀ T + P (symmetric): lower tiles only.  Rows x -> Uxx (lower part suffices: V_i below
    // reads only its own lower tiles), rows u -> Uux = H and Uuu = G (mirrored: the sweep needs all)
    cta_gemm_lower<NZ, NX>(
        [&](int r, int k) { return sm[L::oA + X(k, r)]; }, [&](int k, int c) { return sm[L::TT + X(k, c)]; },
        [&](int r, int c) { return Pat(r, c); },
        [&](int r, int c, double v, bool mir) {
          if (r < NX) {
            if (c < NX) sm[L::Uxx + X(r, c)] = v;  // (r < NX, c >= NX: the Hᵀ entry, stored as H)
          } else {
            const int u = r - NX;
            if (c < NX) {
              sm[L::Uux + Y(u, c)] = v;
            } else {
              sm[L::Uuu + Y(u, c - NX)] = v;
              if (mir) sm[L::Uuu + Y(c - NX, u)] = v;
            }
          }
        },
        warp, NW, lane);
    __syncthreads();
    // G⁻¹ (sweep in place: Uuu = −G⁻¹), K̃ = G⁻¹ H,  k̃ = G⁻¹ h  (= −K_i, −k_i)
    cta_sweep_any<NU, NTHREADS>(sm + L::Uuu, m, sm + L::pr, sm + L::TT, tid, &fail);
    if (fail && st == 0) st = mk_status(RR_ST_G_NOT_PD, i);
    cta_gemm<NU, NX, NU, false>(
        [&](int r, int k) { return -sm[L::Uuu + Y(r, k)]; }, [&](int k, int c) { return sm[L::Uux + Y(k, c)]; },
        [&](int, int) { return 0.0; }, [&](int r, int c, double v) { sm[L::Kt + Y(r, c)] = v; }, warp, NW, lane);
    cta_matvec<NU, NU, NTHREADS>(
        [&](int r, int k) { return -sm[L::Uuu + Y(r, k)]; }, [&](int k) { return sm[L::Uux + Y(k, NX)]; },
        [&](int) { return 0.0; }, [&](int r, double v) { sm[L::Kt + Y(r, NX)] = v; }, tid);
    __syncthreads();
    // V_i = Uxx − Hᵀ K̃ (symmetric: lower tiles, mirrored, in place), v_i = b_x − Hᵀ k̃,
    // M = A − B K̃,  m = c − δ v_{i+1} − B k̃   (M | m: [A | c − δv] − B [K̃ | k̃])
    cta_gemm_lower<NX, NU>(
        [&](int r, int k) { return -sm[L::Uux + Y(k, r)]; }, [&](int k, int c) { return sm[L::Kt + Y(k, c)]; },
        [&](int r, int c) { return sm[L::Uxx + X(r, c)]; },
        [&](int r, int c, double v, bool mir) {
          sm[L::Uxx + X(r, c)] = v;
          if (mir) sm[L::Uxx + X(c, r)] = v;
        },
        warp, NW, lane);
    cta_gemm<NX, NX, NU, false>(
        [&](int r, int k) { return -sm[L::oA + X(r, NX + k)]; }, [&](int k, int c) { return sm[L::Kt + Y(k, c)]; },
        [&](int r, int c) { return sm[L::oA + X(r, c)]; }, [&](int r, int c, double v) { sm[L::MM + X(r, c)] = v; },
        warp, NW, lane);
    cta_matvec<NX, NU, NTHREADS>(
        [&](int r, int k) { return -sm[L::Uux + Y(k, r)]; }, [&](int k) { return sm[L::Kt + Y(k, NX)]; },
        [&](int r) { return sm[L::Uxx + X(r, NX)]; }, [&](int r, double v) { sm[L::Uxx + X(r, NX)] = v; }, tid);
    cta_matvec<NX, NU, NTHREADS>(
        [&](int r, int k) { return -sm[L::oA + X(r, NX + k)]; }, [&](int k) { return sm[L::Kt + Y(k, NX)]; },
        [&](int r) { return sm[L::oc + r] - delta * sm[L::vs + r]; }, [&](int r, double v) { sm[L::MM + X(r, NX)] = v; },
        tid);
    __syncthreads();
    // record K = −K̃[:, :NX] (ld NU), k = −K̃[:, NX], V_i (ld NX), v_i; optional factor outputs
    for (int e = tid; e < m * n; e += NTHREADS) rec[L::rK + e] = -sm[L::Kt + Y(e % m, e / m)];
    for (int u = tid; u < m; u += NTHREADS) rec[L::rk + u] = -sm[L::Kt + Y(u, NX)];
    for (int e = tid; e < n * n; e += NTHREADS) rec[L::rV + e] = sm[L::Uxx + X(e % n, e / n)];
    for (int r = tid; r < n; r += NTHREADS) rec[L::rv + r] = sm[L::Uxx + X(r, NX)];
    if (a.f.K != nullptr)
      for (int e = tid; e < m * n; e += NTHREADS) a.f.K[(inst * sN + i) * m * n + e] = -sm[L::Kt + Y(e % m, e / m)];
    if (a.f.k != nullptr)
      for (int u = tid; u < m; u += NTHREADS) a.f.k[(inst * sN + i) * m + u] = -sm[L::Kt + Y(u, NX)];
    if (a.f.V != nullptr)
      for (int e = tid; e < L::SN; e += NTHREADS) {
        int c = 0, off = e;
        while (off >= n - c) { off -= n - c; ++c; }
        a.f.V[(inst * (sN + 1) + i) * L::SN + e] = sm[L::Uxx + X(c + off, c)];
      }
    if (a.f.v != nullptr)
      for (int r = tid; r < n; r += NTHREADS) a.f.v[(inst * (sN + 1) + i) * n + r] = sm[L::Uxx + X(r, NX)];
    __syncthreads();
    // stage input is dead: stream the next stage in while [Φ | φ] = S⁻¹ [M | m] is formed
    if (i > 0) issue_stage(i - 1);
    cta_gemm<NX, NX, NX, false>(
        [&](int r, int k) { return -sm[L::SI + X(r, k)]; }, [&](int k, int c) { return sm[L::MM + X(k, c)]; },
        [&](int, int) { return 0.0; }, [&](int r, int c, double v) { rec[L::rPHI + r + c * n] = v; }, warp, NW, lane);
    cta_matvec<NX, NX, NTHREADS>(
        [&](int r, int k) { return -sm[L::SI + X(r, k)]; }, [&](int k) { return sm[L::MM + X(k, NX)]; },
        [&](int) { return 0.0; }, [&](int r, double v) { rec[L::rPHI + r + NX * n] = v; }, tid);
    // carry: V_i -> VW region (already in place: Uxx == VW, same layout), v_i -> vs
    for (int r = tid; r < n; r += NTHREADS) sm[L::vs + r] = sm[L::Uxx + X(r, NX)];
    __syncthreads();
  }

  // x_0 = (I + δV_0)⁻¹ (c_0 − δ v_0)
  for (int e = tid; e < n * n; e += NTHREADS) {
    const int r = e % n, c = e / n;
    sm[L::SI + X(r, c)] = delta * sm[L::VW + X(r, c)] + (r == c ? 1.0 : 0.0);
  }
  __syncthreads();
  {
    bool fail = false;
    cta_sweep_any<NX, NTHREADS>(sm + L::SI, n, sm + L::pr, sm + L::TT, tid, &fail);
    if (fail && st == 0) st = mk_status(RR_ST_S_NOT_PD, 0);
  }
  for (int r = tid; r < n; r += NTHREADS) {
    double acc = 0.0;
    for (int k = 0; k < n; ++k) acc = fma(-sm[L::SI + X(r, k)], a.p.c0[inst * n + k] - delta * sm[L::vs + k], acc);
    sm[L::xs + r] = acc;
  }
  __syncthreads();
  // block-wide status: any thread's failure (same value on all threads of a block in practice)
  __shared__ int sst;
  if (tid == 0) sst = 0;
  __syncthreads();
  if (st != 0) atomicMax(&sst, st);
  __syncthreads();
  int32_t status = sst;

  double* xo = a.s.x + inst * (sN + 1) * n;
  double* uo = a.s.u + inst * sN * m;
  double* yo = a.s.y + inst * (sN + 1) * n;
  for (int r = tid; r < n; r += NTHREADS) xo[r] = sm[L::xs + r];
  bool bad = false;
  // forward: thread (row, part): row = tid % NZ-ish split; 4 partial sums per output row
  constexpr int PARTS = NTHREADS / 64 > 4 ? 4 : NTHREADS / 64;
  for (int i = 0; i < N; ++i) {
    const double* rec = rec0 + (int64_t)i * L::REC;
    for (int task = tid; task < PARTS * (2 * NX + NU); task += NTHREADS) {
      const int part = task / (2 * NX + NU), row = task % (2 * NX + NU);
      const int k0 = part * (NX / PARTS), k1 = k0 + NX / PARTS;
      double acc = 0.0;
      if (row < NX) {  // x_{i+1} row
        for (int k = k0; k < k1; ++k) acc = fma(rec[L::rPHI + row + k * n], sm[L::xs + k], acc);
      } else if (row < 2 * NX) {  // y_i row
        const int rr = row - NX;
        for (int k = k0; k < k1; ++k) acc = fma(rec[L::rV + rr + k * n], sm[L::xs + k], acc);
      } else {  // u_i row
        const int u = row - 2 * NX;
        for (int k = k0; k < k1; ++k) acc = fma(rec[L::rK + u + k * m], sm[L::xs + k], acc);
      }
      sm[L::red + part * (2 * NX + NU) + row] = acc;
    }
    __syncthreads();
    for (int row = tid; row < 2 * NX + NU; row += NTHREADS) {
      double acc = 0.0;
      for (int p = 0; p < PARTS; ++p) acc += sm[L::red + p * (2 * NX + NU) + row];
      if (row < NX) {
        acc += rec[L::rPHI + row + NX * n];
        xo[(int64_t)(i + 1) * n + row] = acc;
        sm[L::pr + row] = acc;
      } else if (row < 2 * NX) {
        acc += rec[L::rv + row - NX];
        yo[(int64_t)i * n + row - NX] = acc;
      } else {
        acc += rec[L::rk + row - 2 * NX];
        uo[(int64_t)i * m + row - 2 * NX] = acc;
      }
      bad |= !isfinite(acc);
    }
    __syncthreads();
    for (int r = tid; r < n; r += NTHREADS) sm[L::xs + r] = sm[L::pr + r];
    __syncthreads();
  }
  {  // y_N = Q_N x_N + q_N
    const double* QN = a.p.QN + inst * L::SN;
    for (int r = tid; r < n; r += NTHREADS) {
      double acc = a.p.qN[inst * n + r];
      for (int k = 0; k < n; ++k) acc = fma(k >= r ? QN[pidx(n, k, r)] : QN[pidx(n, r, k)], sm[L::xs + k], acc);
      yo[sN * n + r] = acc;
      bad |= !isfinite(acc);
    }
  }
  if (__syncthreads_or(bad) && status == 0) status = RR_ST_NONFINITE;
  if (status != 0) {
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    for (int64_t e = tid; e < (sN + 1) * n; e += NTHREADS) {
      xo[e] = nan;
      yo[e] = nan;
    }
    for (int64_t e = tid; e < sN * m; e += NTHREADS) uo[e] = nan;
  }
  if (tid == 0) a.status[inst] = status;
}

template <int NX, int NU, int NT_ = 256>
struct CtaCfg {
  static constexpr int NTHREADS = NT_;
  static size_t smem_bytes() { return sizeof(double) * (size_t)CtaLayout<NX, NU>::TOTAL; }
  static int64_t ws_doubles(int64_t batch, int N) { return batch * (int64_t)N * CtaLayout<NX, NU>::REC; }
  static cudaError_t launch(const FusedArgs& a, cudaStream_t s) {
    auto k = rr_cta_kernel<NX, NU, NTHREADS>;
    const size_t smb = smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb);
    if (e != cudaSuccess) return e;
    k<<<(unsigned)a.batch, NTHREADS, smb, s>>>(a);
    return cudaGetLastError();
  }
};

template <typename F>
static bool dispatch_cta(int nx, int nu, F&& f) {
  if (nx == 64 && nu == 32) return f(CtaCfg<64, 32, 512>{});
  if (nx == 32 && nu == 16) return f(CtaCfg<32, 16>{});
  if (nx == 24 && nu == 8) return f(CtaCfg<24, 8>{});
  return false;
}

int64_t cta_workspace_bytes(int nx, int nu, int N, int64_t batch) {
  int64_t out = -1;
  dispatch_cta(nx, nu, [&](auto cfg) {
    out = 8 * decltype(cfg)::ws_doubles(batch, N) + 256;
    return true;
  });
  return out;
}

cudaError_t cta_launch(const FusedArgs& a, cudaStream_t s, bool* supported) {
  cudaError_t err = cudaSuccess;
  *supported = dispatch_cta(a.nx, a.nu, [&](auto cfg) {
    err = decltype(cfg)::launch(a, s);
    return true;
  });
  return err;
}

}  // namespace rrk
