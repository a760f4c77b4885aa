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
//   record for the forward sweep: K_i, k_i, V_i, v_i, S_{i+1}⁻¹ (packed), e_i
// forward: u_i = K_i x_i + k_i, y_i = V_i x_i + v_i,
//   x_{i+1} = S_{i+1}⁻¹ (A_i x_i + B_i u_i + e_i) with A_i, B_i re-read by TMA (no Φ products).
// Shared-memory plan (doubles) for one instance: stage input (cp.async) | S⁻¹ | V/W/U | T/K̃/M |
// vectors -- about 230 KB, one CTA per SM; the next stage's input streams in during the last
// contraction of the current stage.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "rr_common.cuh"
#include "rr_cta.cuh"
#include "rr_stage_mma.cuh"

namespace rrk {

// Phase timestamps of one stage of CTA 0 (tools/cta_phase_probe.cu builds with RR_CTA_PROFILE);
// compiled out otherwise.
#ifdef RR_CTA_PROFILE
#define RR_CTA_PROFILE_FWD RR_CTA_PROFILE
__device__ long long g_cta_prof[32];
#define RR_PROF(i, slot)                                                           \
  do {                                                                             \
    if (blockIdx.x == 0 && threadIdx.x == 0 && (i) == RR_CTA_PROFILE) g_cta_prof[slot] = clock64(); \
  } while (0)
#else
#define RR_PROF(i, slot) \
  do {                   \
  } while (0)
#endif

template <int NX, int NU>
struct CtaLayout {
  static constexpr int NZ = NX + NU;
  static constexpr int SN = NX * (NX + 1) / 2, SMU = NU * (NU + 1) / 2;
  // stage input in the global operand order: A | B (= F, col-major ld NX) | Q | M | R | q | r | c
  static constexpr int oA = 0, oB = NX * NX, oQ = oB + NX * NU, oM = oQ + SN, oR = oM + NX * NU, oq = oR + SMU,
                       orr = oq + NX, oc = orr + NU;
  static constexpr int IN = ((oc + NX + 1) & ~1);
  // SI: S = I + δV -> −S⁻¹ (ld NX); once T is formed: K̃ (ld NU, NX cols)
  static constexpr int SI = IN;
  static constexpr int Kt = SI;
  static constexpr int SI_SZ = NX * NX;
  // R1: V_{i+1} (ld NX) + S-sweep scratch | T = S⁻¹(V F) (ld NX, NZ cols) | T_A + H = Uux (ld NU, NX
  // cols, over T_B) | V_i
  static constexpr int R1 = SI + ((SI_SZ + 1) & ~1);
  static constexpr int YS = R1 + NX * NX;  // S-sweep scratch (NX × 16) behind V
  static constexpr int Uux = R1 + NX * NX;
  static constexpr int R1_SZ = (NX * NZ > NX * NX + NX * 16) ? NX * NZ : NX * NX + NX * 16;
  // R2: V F (ld NX, NZ cols) | Uxx (ld NX) + G = Uuu (ld NU, over (V F)_B)
  static constexpr int R2 = R1 + ((R1_SZ + 1) & ~1);
  static constexpr int Uxx = R2, Uuu = R2 + NX * NX;
  static constexpr int R2_SZ = NX * NZ;
  static_assert(NU <= NX && NU * NX <= SI_SZ, "C3 layout assumes n_u <= n_x");
  static constexpr int VEC = R2 + ((R2_SZ + 1) & ~1);
  static constexpr int vs = VEC;       // v_{i+1}, then v_i (NX)
  static constexpr int ve = vs + NX;   // V e (NX)
  static constexpr int ee = ve + NX;   // e = c_{i+1} − δ v_{i+1} (NX)
  static constexpr int gg = ee + NX;   // g = v_{i+1} + S⁻¹ V e (NX)
  static constexpr int bb = gg + NX;   // b = (q; r) + Fᵀ g (NZ)
  static constexpr int kt = bb + NZ;   // k̃ = G⁻¹ b_u (NU)
  static constexpr int gpb = kt + NU;  // G-sweep pivot buffer (2 NU)
  static constexpr int xs = gpb + 2 * NU;  // forward: x_i (NX)
  static constexpr int us = xs + NX;   // forward: u_i (NU)
  static constexpr int ws = us + NU;   // forward: z = A x + e (NX)
  static constexpr int pr2 = ws + NX;  // forward: w = z + B u (NX)
  static constexpr int TOTAL = pr2 + NX;
  // forward record (global, per stage i): K_i (ld NU, NX cols) | k_i | V_i (packed 'L') | v_i |
  // e_i = c_{i+1} − δ v_{i+1} | S⁻¹_{i+1} = (I + δV_{i+1})⁻¹ (packed 'L')
  static constexpr int rK = 0, rk = rK + NU * NX, rV = rk + NU, rv = rV + SN, re = rv + NX, rS = re + NX;
  static constexpr int REC = ((rS + SN + 1) & ~1);
  // forward sweep: two TMA-filled stage buffers [record | A_i | B_i] over the dead backward regions
  static constexpr int FA = REC, FB = FA + NX * NX;
  static constexpr int FBUF = ((FB + NX * NU + 1) & ~1);
  static constexpr int zs = ws;  // forward: z = A x + e, then w = z + B u (reuses ws)
  static_assert(2 * FBUF <= VEC, "forward stage buffers overlap the vectors");
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

// Symmetric sweep of an n×n block held in one warp's registers (n = 16 or 32).  The 32 lanes form
// a 4 × 8 grid of row groups × column groups: lane l = 8·rg + cg owns rows R·rg .. R·rg+R−1 and
// columns C·cg .. C·cg+C−1 (R = n/4, C = n/8), a[i][j] = A[R·rg+i][C·cg+j].  Pivots 0..n−1 in order;
// per pivot the diagonal entry, the pivot column at the lane's R rows and the pivot row at its C
// columns travel by R + C + 1 shuffles (row k = column k by symmetry).  The 4 × 8 grid needs 30 %
// fewer shuffles than a column-per-lane layout (measured 1772 vs 2316 cycles for n = 16).
template <int n>
__device__ __forceinline__ void warp_sweep_reg(double (&a)[n / 4][n / 8], int lane, bool* bad) {
  constexpr int R = n / 4, C = n / 8;
  const int rg = lane >> 3, cg = lane & 7;
  // outer loop over the 4 pivot row groups kept rolled (code size: the unrolled body covers R
  // pivots, whose register positions ki = kk, kj = kk % C are compile-time)
#pragma unroll 1
  for (int kr = 0; kr < 4; ++kr) {
#pragma unroll
    for (int kk = 0; kk < R; ++kk) {
      const int k = kr * R + kk, ki = kk, kj = kk % C, kc = k / C;
      const double d = __shfl_sync(RR_FULL_MASK, a[ki][kj], kr * 8 + kc);
      double colk[R], rowk[C];
#pragma unroll
      for (int i = 0; i < R; ++i) colk[i] = __shfl_sync(RR_FULL_MASK, a[i][kj], rg * 8 + kc);  // A[R·rg+i][k]
#pragma unroll
      for (int j = 0; j < C; ++j) rowk[j] = __shfl_sync(RR_FULL_MASK, a[ki][j], kr * 8 + cg);  // A[k][C·cg+j]
      *bad |= !(d > 0.0);
      const double id = rcp_nr(d);
#pragma unroll
      for (int j = 0; j < C; ++j) {
        const int c = C * cg + j;
        const double rs = rowk[j] * id;
#pragma unroll
        for (int i = 0; i < R; ++i) {
          const int r = R * rg + i;
          const double upd = fma(-colk[i], rs, a[i][j]);
          a[i][j] = (r == k) ? ((c == k) ? -id : rs) : ((c == k) ? colk[i] * id : upd);
        }
      }
    }
  }
}

// A (n×n at (q0, q0) of a swizzled ld-LD matrix in shared memory) <- its sweep, on one warp.
template <int n, int LD>
__device__ __forceinline__ void warp_sweep_smem(double* A, int q0, int lane, bool* bad) {
  constexpr int R = n / 4, C = n / 8;
  const int rg = lane >> 3, cg = lane & 7;
  double a[R][C];
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < C; ++j) a[i][j] = A[swz<LD>(q0 + R * rg + i, q0 + C * cg + j)];
  warp_sweep_reg<n>(a, lane, bad);
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < C; ++j) A[swz<LD>(q0 + R * rg + i, q0 + C * cg + j)] = a[i][j];
}

// Block (16-pivot) symmetric sweep of the n×n SPD matrix A (n % 16 == 0, swizzled ld n):
// A <- −A⁻¹.  Sweeping the pivots of block p at once is the block form of the sweep operator:
//   Z = A_pp⁻¹:  A_pp <- −Z,  A_rp <- A_rp Z,  A_pc <- Z A_pc,  A_rc <- A_rc − A_rp Z A_pc,
// identical (up to rounding) to the 16 scalar sweeps of block p.  Per block: warp 0 sweeps A_pp in
// registers; Y = A_{:,p} Z (DMMA, into `Y`, n × 16); the trailing update A_RC −= Y_R A_pC over the
// lower tiles R >= C (mirrored to C, R) on DMMA; then column / row block p <- Y / Yᵀ (overlapped
// with the next block's diagonal sweep).  3 barriers per block instead of 2 per pivot.  While warp 0
// sweeps, the other warps also run side(p, NB, slot, nslots): caller work independent of A.
// (A lookahead variant -- warp 0 updating and sweeping tile (p+1, p+1) during the trailing update --
// measured slower on C3: the dependency chain tile -> sweep -> Y tile is the same length.)
template <int n, int NTHREADS, typename Side>
__device__ __forceinline__ void cta_sweep_blk(double* A, double* Y, int tid, bool* fail, Side&& side,
                                              int prof = -1) {
  constexpr int NB = n / 16;
  constexpr int NW = NTHREADS / 32;
  static_assert(n % 16 == 0, "block sweep needs n % 16 == 0");
  const int lane = tid & 31, warp = tid >> 5;
  bool bad = false;
  auto S = [](int r, int c) { return swz<n>(r, c); };
  for (int p = 0; p < NB; ++p) {
    const int p0 = 16 * p;
#ifdef RR_CTA_PROFILE
    if (prof >= 0 && tid == 32) g_cta_prof[prof + 3 * p] = clock64();
#endif
    if (warp == 0) {
      warp_sweep_smem<16, n>(A, p0, lane, &bad);  // A_pp <- −Z
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
    if (warp != 0) side(p, NB, warp - 1, NW - 1);  // independent work of the caller, hidden behind warp 0
    __syncthreads();
#ifdef RR_CTA_PROFILE
    if (prof >= 0 && tid == 32) g_cta_prof[prof + 3 * p + 1] = clock64();
#endif
    // Y_R = A_{R,p} Z = −A_{R,p} A'_pp for the row tiles R != p
    for (int R = warp; R < NB; R += NW) {
      if (R == p) continue;
      warp_tile16<16>(
          16 * R, 0, [&](int r, int k) { return A[S(r, p0 + k)]; }, [&](int k, int c) { return -A[S(p0 + k, p0 + c)]; },
          [&](int, int) { return 0.0; }, [&](int r, int c, double v) { Y[S(r, c)] = v; }, lane);
    }
    __syncthreads();
#ifdef RR_CTA_PROFILE
    if (prof >= 0 && tid == 32) g_cta_prof[prof + 3 * p + 2] = clock64();
#endif
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

// Cooperative symmetric sweep A <- −A⁻¹ of an n×n SPD matrix (swizzled ld n, n % 32 == 0) by the
// first NWS warps: warp w owns columns CW·w .. CW·w+CW−1 (CW = n / NWS), lane l rows l + 32q, all in
// registers.  Per pivot k the column k (= row k, by symmetry) is read from a double-buffered shared
// vector pb; its owner publishes the updated column k+1 before the one named barrier per pivot.
// The other warps (NWS..) are free for independent work meanwhile (run by the caller).
// Measured (tools/cta_phase_probe): n = 32 on 4 warps 8.9 K cycles (vs 14 K for the 16-block sweep);
// n = 64 on 8 warps 38 K (vs 21 K for the block sweep: the per-pivot chain LDS -> rcp -> update ->
// STS -> barrier dominates), so only n = 32 takes this path.
template <int n, int NWS>
__device__ __forceinline__ void coop_sweep(double* A, double* pb, int tid, bool* bad) {
  constexpr int CW = n / NWS, RQ = n / 32;
  static_assert(n % 32 == 0 && n % NWS == 0, "coop sweep layout");
  const int lane = tid & 31, w = tid >> 5;
  auto bar = [] { asm volatile("bar.sync 1, %0;\n" ::"n"(NWS * 32) : "memory"); };
  double a[RQ][CW];
#pragma unroll
  for (int q = 0; q < RQ; ++q)
#pragma unroll
    for (int j = 0; j < CW; ++j) a[q][j] = A[swz<n>(lane + 32 * q, CW * w + j)];
  if (w == 0)
#pragma unroll
    for (int q = 0; q < RQ; ++q) pb[lane + 32 * q] = a[q][0];
  bar();
#pragma unroll 1
  for (int kb = 0; kb < NWS; ++kb) {
#pragma unroll
    for (int kj = 0; kj < CW; ++kj) {
      const int k = kb * CW + kj;
      const double* buf = pb + (k & 1) * n;
      const double d = buf[k];
      double colk[RQ], rowk[CW];
#pragma unroll
      for (int q = 0; q < RQ; ++q) colk[q] = buf[lane + 32 * q];
#pragma unroll
      for (int j = 0; j < CW; ++j) rowk[j] = buf[CW * w + j];
      *bad |= !(d > 0.0);
      const double id = rcp_nr(d);
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        const int c = CW * w + j;
        const double rs = rowk[j] * id;
#pragma unroll
        for (int q = 0; q < RQ; ++q) {
          const int r = lane + 32 * q;
          const double upd = fma(-colk[q], rs, a[q][j]);
          a[q][j] = (r == k) ? ((c == k) ? -id : rs) : ((c == k) ? colk[q] * id : upd);
        }
      }
      if (k + 1 < n && w == (k + 1) / CW) {  // publish column k+1 (register index (kj+1) % CW)
        double* nb = pb + ((k + 1) & 1) * n;
#pragma unroll
        for (int q = 0; q < RQ; ++q) nb[lane + 32 * q] = a[q][(kj + 1) % CW];
      }
      bar();
    }
  }
#pragma unroll
  for (int q = 0; q < RQ; ++q)
#pragma unroll
    for (int j = 0; j < CW; ++j) A[swz<n>(lane + 32 * q, CW * w + j)] = a[q][j];
}

// A <- −A⁻¹ by the block sweep when n is a multiple of 16 (>= 32), else the register / scalar
// sweep; side(p, nphases, slot, nslots) is run by warps 1.. alongside (blocked) or before it.
template <int n, int NTHREADS, typename Side>
__device__ __forceinline__ void cta_sweep_any(double* A, int lda, double* scratch, int tid, bool* fail, Side&& side,
                                              int prof = -1) {
  const int warp = tid >> 5;
  constexpr int NW = NTHREADS / 32;
  if constexpr (n == 32 && n / 8 <= NW / 2) {
    // cooperative register sweep on n/8 warps (8 columns each); the remaining warps run `side`
    constexpr int NWS = n / 8;
    bool bad = false;
    if (warp < NWS) coop_sweep<n, NWS>(A, scratch, tid, &bad);
    else side(0, 1, warp - NWS, NW - NWS);
    __syncthreads();
    *fail = bad;
    (void)prof;
  } else if constexpr (n % 16 == 0 && n >= 32) {
    cta_sweep_blk<n, NTHREADS>(A, scratch, tid, fail, side, prof);
  } else {
    side(0, 1, warp, NW);
    __syncthreads();
    if constexpr (n % 16 == 0 && NTHREADS == 256) cta_sweep_reg<n>(A, lda, scratch, tid, fail);
    else cta_sweep<n>(A, lda, scratch, tid, NTHREADS, fail);
  }
}

// One 16×16 super-tile at (m0, n0) of C = op_A · B + init (K multiple of 4) on one warp, masked to M × N.
template <int M, int N, int K, int UNR = 4, typename LoadA, typename LoadB, typename Init, typename Store>
__device__ __forceinline__ void warp_tile_at(int m0, int n0, LoadA&& la, LoadB&& lb, Init&& init, Store&& store,
                                             int lane) {
  const int g = lane >> 2, t = lane & 3;
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
#pragma unroll UNR
  for (int kt = 0; kt < K / 4; ++kt) {
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

// Tile index tt (column-major tile order) of an M×N result.
template <int M, int N, int K, int UNR = 4, typename LoadA, typename LoadB, typename Init, typename Store>
__device__ __forceinline__ void warp_tile_mn(int tt, LoadA&& la, LoadB&& lb, Init&& init, Store&& store, int lane) {
  constexpr int MT = (M + 15) / 16;
  warp_tile_at<M, N, K, UNR>((tt % MT) * 16, (tt / MT) * 16, la, lb, init, store, lane);
}

// (R, C) of the t-th lower tile (R >= C) in row-major lower order.
__device__ __forceinline__ void lower_tile(int t, int& R, int& C) {
  R = 0;
  while (t > R) {
    t -= R + 1;
    ++R;
  }
  C = t;
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

  auto X = [](int r, int c) { return swz<NX>(r, c); };  // ld NX matrices (F, S⁻¹, V, T, Uxx)
  auto Y = [](int r, int c) { return swz<NU>(r, c); };  // ld NU matrices (Uux = H, Uuu = G, K̃)
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
  // V_N = Q_N -> R1 (ld NX), v_N = q_N
  {
    const double* QN = a.p.QN + inst * L::SN;
    for (int e = tid; e < n * n; e += NTHREADS) {
      const int r = e % n, c = e / n;
      sm[L::R1 + X(r, c)] = r >= c ? QN[pidx(n, r, c)] : QN[pidx(n, c, r)];
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
  constexpr int NT_VF = ((NX + 15) / 16) * ((NZ + 15) / 16);  // tiles of V F
  auto no_side = [](int, int, int, int) {};

  for (int i = N - 1; i >= 0; --i) {
    cp_async_wait<0>();
    __syncthreads();
    RR_PROF(i, 0);
    double* rec = rec0 + (int64_t)i * L::REC;
    // S = I + δV_{i+1} -> SI;  e = c_{i+1} − δ v_{i+1};  V e
    for (int e = tid; e < n * n; e += NTHREADS) {
      const int r = e % n, c = e / n;
      sm[L::SI + X(r, c)] = delta * sm[L::R1 + X(r, c)] + (r == c ? 1.0 : 0.0);
    }
    for (int r = tid; r < n; r += NTHREADS) {
      const double ev = sm[L::oc + r] - delta * sm[L::vs + r];
      sm[L::ee + r] = ev;
      rec[L::re + r] = ev;
    }
    __syncthreads();
    cta_matvec<NX, NX, NTHREADS>(
        [&](int r, int k) { return sm[L::R1 + X(r, k)]; }, [&](int k) { return sm[L::ee + k]; },
        [&](int) { return 0.0; }, [&](int r, double v) { sm[L::ve + r] = v; }, tid);
    // S⁻¹ by the block sweep (SI = −S⁻¹, scratch behind V in R1); meanwhile the idle warps form
    // V F -> R2 (independent of S⁻¹):  T = W F = S⁻¹ (V F) below needs no W
    RR_PROF(i, 1);
    bool fail = false;
    cta_sweep_any<NX, NTHREADS>(
        sm + L::SI, n, sm + L::YS, tid, &fail,
        [&](int p, int nph, int slot, int nslots) {
          const int t0 = p * NT_VF / nph, t1 = (p + 1) * NT_VF / nph;
          for (int tt = t0 + slot; tt < t1; tt += nslots)
            warp_tile_mn<NX, NZ, NX>(
                tt, [&](int r, int k) { return sm[L::R1 + X(r, k)]; },
                [&](int k, int c) { return sm[L::oA + X(k, c)]; }, [&](int, int) { return 0.0; },
                [&](int r, int c, double v) { sm[L::R2 + X(r, c)] = v; }, lane);
        },
#ifdef RR_CTA_PROFILE
        (blockIdx.x == 0 && i == RR_CTA_PROFILE) ? 12 : -1
#else
        -1
#endif
    );
    if (fail && st == 0) st = mk_status(RR_ST_S_NOT_PD, i);
    RR_PROF(i, 2);
    // T = S⁻¹ (V F) -> R1 (V is dead), U = Fᵀ T + P, scheduled so that G = Uuu is ready first and
    // the rest of U runs beside the G⁻¹ sweep:
    //   P1: the T tiles holding B columns (T_B) + the first T_A tiles;  g = v_{i+1} + S⁻¹ V e;  record S⁻¹
    //   P2: G = Bᵀ T_B + R (lower tiles) + the remaining T_A tiles;  b = (q; r) + Fᵀ g
    //   P3: G⁻¹ sweep  ‖  H = Uux = Bᵀ T_A + Mᵀ and Uxx = Aᵀ T_A + Q (lower tiles) on the other warps
    constexpr int MT_T = (NX + 15) / 16, NT_T = MT_T * ((NZ + 15) / 16), CTB = NX / 16;
    constexpr int NB_T = MT_T * (((NZ + 15) / 16) - CTB);  // T tiles holding B columns (first in order)
    static_assert(NB_T <= NW, "T_B tiles must fit one round");
    auto t_tile = [&](int o) {  // o-th T tile in the order: B-column tiles first
      const int tt = (o + MT_T * CTB) % NT_T;
      warp_tile_mn<NX, NZ, NX>(
          tt, [&](int r, int k) { return -sm[L::SI + X(r, k)]; }, [&](int k, int c) { return sm[L::R2 + X(k, c)]; },
          [&](int, int) { return 0.0; }, [&](int r, int c, double v) { sm[L::R1 + X(r, c)] = v; }, lane);
    };
    constexpr int P1T = NT_T < NW ? NT_T : NW;
    for (int o = warp; o < P1T; o += NW) t_tile(o);
    cta_matvec<NX, NX, NTHREADS>(
        [&](int r, int k) { return -sm[L::SI + X(r, k)]; }, [&](int k) { return sm[L::ve + k]; },
        [&](int r) { return sm[L::vs + r]; }, [&](int r, double v) { sm[L::gg + r] = v; }, tid);
    for (int e = tid; e < n * n; e += NTHREADS) {
      const int r = e % n, c = e / n;
      if (r >= c) rec[L::rS + pidx(n, r, c)] = -sm[L::SI + X(r, c)];
    }
    __syncthreads();
    RR_PROF(i, 3);
    {
      constexpr int MTU = (NU + 15) / 16, NGT = MTU * (MTU + 1) / 2;  // lower tiles of G
      for (int task = warp; task < NGT + (NT_T - P1T); task += NW) {
        if (task < NGT) {
          int R, C;
          lower_tile(task, R, C);
          const bool mir = R != C;
          warp_tile_at<NU, NU, NX>(
              16 * R, 16 * C, [&](int r, int k) { return sm[L::oA + X(k, NX + r)]; },
              [&](int k, int c) { return sm[L::R1 + X(k, NX + c)]; }, [&](int r, int c) { return Pat(NX + r, NX + c); },
              [&](int r, int c, double v) {
                sm[L::Uuu + Y(r, c)] = v;
                if (mir) sm[L::Uuu + Y(c, r)] = v;
              },
              lane);
        } else {
          t_tile(P1T + task - NGT);
        }
      }
    }
    cta_matvec<NZ, NX, NTHREADS>(
        [&](int r, int k) { return sm[L::oA + X(k, r)]; }, [&](int k) { return sm[L::gg + k]; },
        [&](int r) { return r < NX ? sm[L::oq + r] : sm[L::orr + r - NX]; }, [&](int r, double v) { sm[L::bb + r] = v; },
        tid);
    __syncthreads();
    RR_PROF(i, 4);
    // P3: G⁻¹ (sweep in place: Uuu = −G⁻¹)  ‖  H and Uxx
    cta_sweep_any<NU, NTHREADS>(sm + L::Uuu, m, sm + L::gpb, tid, &fail, [&](int, int, int slot, int nslots) {
      constexpr int MTX = (NX + 15) / 16, MTU = (NU + 15) / 16;
      constexpr int NH = MTU * MTX, NXX = MTX * (MTX + 1) / 2;
      for (int task = slot; task < NH + NXX; task += nslots) {
        if (task < NH) {  // H = Uux (u, c) = Σ_k F[k][NX+u] T[k][c] + M[c][u]
          warp_tile_mn<NU, NX, NX>(
              task, [&](int r, int k) { return sm[L::oA + X(k, NX + r)]; },
              [&](int k, int c) { return sm[L::R1 + X(k, c)]; }, [&](int r, int c) { return Pat(NX + r, c); },
              [&](int r, int c, double v) { sm[L::Uux + Y(r, c)] = v; }, lane);
        } else {  // Uxx lower tiles (the lower part is all V_i below reads)
          int R, C;
          lower_tile(task - NH, R, C);
          warp_tile_at<NX, NX, NX>(
              16 * R, 16 * C, [&](int r, int k) { return sm[L::oA + X(k, r)]; },
              [&](int k, int c) { return sm[L::R1 + X(k, c)]; }, [&](int r, int c) { return Pat(r, c); },
              [&](int r, int c, double v) { sm[L::Uxx + X(r, c)] = v; }, lane);
        }
      }
    });
    if (fail && st == 0) st = mk_status(RR_ST_G_NOT_PD, i);
    RR_PROF(i, 5);
    // the stage input is dead: stream the next stage in behind the rest of this one
    if (i > 0) issue_stage(i - 1);
    // K̃ = G⁻¹ H, k̃ = G⁻¹ b_u (= −K_i, −k_i) -> SI region (S⁻¹ is dead)
    cta_gemm<NU, NX, NU, false>(
        [&](int r, int k) { return -sm[L::Uuu + Y(r, k)]; }, [&](int k, int c) { return sm[L::Uux + Y(k, c)]; },
        [&](int, int) { return 0.0; }, [&](int r, int c, double v) { sm[L::Kt + Y(r, c)] = v; }, warp, NW, lane);
    cta_matvec<NU, NU, NTHREADS>(
        [&](int r, int k) { return -sm[L::Uuu + Y(r, k)]; }, [&](int k) { return sm[L::bb + NX + k]; },
        [&](int) { return 0.0; }, [&](int r, double v) { sm[L::kt + r] = v; }, tid);
    __syncthreads();
    RR_PROF(i, 6);
    // V_i = Uxx − Hᵀ K̃ -> R1 (symmetric: lower tiles, mirrored);  v_i = b_x − Hᵀ k̃ -> vs
    cta_gemm_lower<NX, NU>(
        [&](int r, int k) { return -sm[L::Uux + Y(k, r)]; }, [&](int k, int c) { return sm[L::Kt + Y(k, c)]; },
        [&](int r, int c) { return sm[L::Uxx + X(r, c)]; },
        [&](int r, int c, double v, bool mir) {
          sm[L::R1 + X(r, c)] = v;
          if (mir) sm[L::R1 + X(c, r)] = v;
        },
        warp, NW, lane);
    cta_matvec<NX, NU, NTHREADS>(
        [&](int r, int k) { return -sm[L::Uux + Y(k, r)]; }, [&](int k) { return sm[L::kt + k]; },
        [&](int r) { return sm[L::bb + r]; }, [&](int r, double v) { sm[L::vs + r] = v; }, tid);
    __syncthreads();
    RR_PROF(i, 7);
    // record K = −K̃ (ld NU), k = −k̃, V_i (ld NX), v_i; optional factor outputs
    for (int e = tid; e < m * n; e += NTHREADS) rec[L::rK + e] = -sm[L::Kt + Y(e % m, e / m)];
    for (int u = tid; u < m; u += NTHREADS) rec[L::rk + u] = -sm[L::kt + u];
    {
      double* fV = a.f.V != nullptr ? a.f.V + (inst * (sN + 1) + i) * L::SN : nullptr;
      for (int e = tid; e < n * n; e += NTHREADS) {
        const int r = e % n, c = e / n;
        if (r >= c) {
          const double v = sm[L::R1 + X(r, c)];
          rec[L::rV + pidx(n, r, c)] = v;
          if (fV != nullptr) fV[pidx(n, r, c)] = v;
        }
      }
    }
    for (int r = tid; r < n; r += NTHREADS) rec[L::rv + r] = sm[L::vs + r];
    if (a.f.K != nullptr)
      for (int e = tid; e < m * n; e += NTHREADS) a.f.K[(inst * sN + i) * m * n + e] = -sm[L::Kt + Y(e % m, e / m)];
    if (a.f.k != nullptr)
      for (int u = tid; u < m; u += NTHREADS) a.f.k[(inst * sN + i) * m + u] = -sm[L::kt + u];
    if (a.f.v != nullptr)
      for (int r = tid; r < n; r += NTHREADS) a.f.v[(inst * (sN + 1) + i) * n + r] = sm[L::vs + r];
    // (the next iteration's leading barrier orders these reads before R1 / vs are rewritten)
  }
  cp_async_wait<0>();
  __syncthreads();
  RR_PROF(RR_CTA_PROFILE_FWD, 8);

  // x_0 = (I + δV_0)⁻¹ (c_0 − δ v_0)
  for (int e = tid; e < n * n; e += NTHREADS) {
    const int r = e % n, c = e / n;
    sm[L::SI + X(r, c)] = delta * sm[L::R1 + X(r, c)] + (r == c ? 1.0 : 0.0);
  }
  for (int r = tid; r < n; r += NTHREADS) sm[L::ee + r] = a.p.c0[inst * n + r] - delta * sm[L::vs + r];
  __syncthreads();
  {
    bool fail = false;
    cta_sweep_any<NX, NTHREADS>(sm + L::SI, n, sm + L::YS, tid, &fail, no_side);
    if (fail && st == 0) st = mk_status(RR_ST_S_NOT_PD, 0);
  }
  cta_matvec<NX, NX, NTHREADS>(
      [&](int r, int k) { return -sm[L::SI + X(r, k)]; }, [&](int k) { return sm[L::ee + k]; }, [&](int) { return 0.0; },
      [&](int r, double v) { sm[L::xs + r] = v; }, tid);
  __syncthreads();
  // block-wide status: any thread's failure
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
  RR_PROF(RR_CTA_PROFILE_FWD, 9);
  // forward: u_i = K_i x_i + k_i,  y_i = V_i x_i + v_i,
  //   x_{i+1} = (I + δV_{i+1})⁻¹ (A_i x_i + B_i u_i + c_{i+1} − δ v_{i+1}).
  // Stage data (record | A_i | B_i) streams into two shared buffers by TMA bulk copies, one stage ahead.
  __shared__ __align__(8) uint64_t fbar[2];
  auto issue_fwd = [&](int i) {  // one thread
    double* dst = sm + (i & 1) * L::FBUF;
    const int64_t s = inst * sN + i;
    constexpr uint32_t brec = 8u * L::REC, bA = 8u * NX * NX, bB = 8u * NX * NU;
    fence_proxy_async();  // order the CTA's earlier generic accesses of the buffer (after a barrier) before the TMA writes
    mbar_arrive_expect_tx(&fbar[i & 1], brec + bA + bB);
    bulk_g2s(dst, rec0 + (int64_t)i * L::REC, brec, &fbar[i & 1]);
    bulk_g2s(dst + L::FA, a.p.A + s * n * n, bA, &fbar[i & 1]);
    bulk_g2s(dst + L::FB, a.p.B + s * n * m, bB, &fbar[i & 1]);
  };
  if (tid == 0) {
    mbar_init(&fbar[0], 1);
    mbar_init(&fbar[1], 1);
  }
  __syncthreads();
  if (tid == 0 && N > 0) issue_fwd(0);
  for (int i = 0; i < N; ++i) {
    const double* fb = sm + (i & 1) * L::FBUF;
    mbar_wait_parity(&fbar[i & 1], (i >> 1) & 1);
    if (tid == 0 && i + 1 < N) issue_fwd(i + 1);  // its buffer was last read by stage i−1 (barriers since)
    // [u_i; y_i; z] = [K_i; V_i; A_i] x_i + [k_i; v_i; e_i]
    cta_matvec<NU + 2 * NX, NX, NTHREADS>(
        [&](int r, int k) {
          if (r < NU) return fb[L::rK + r + k * m];
          if (r < NU + NX) {
            const int rr = r - NU;
            return fb[L::rV + (rr >= k ? pidx(n, rr, k) : pidx(n, k, rr))];
          }
          return fb[L::FA + (r - NU - NX) + k * n];
        },
        [&](int k) { return sm[L::xs + k]; },
        [&](int r) { return r < NU ? fb[L::rk + r] : (r < NU + NX ? fb[L::rv + r - NU] : fb[L::re + r - NU - NX]); },
        [&](int r, double v) {
          if (r < NU) {
            sm[L::us + r] = v;
            uo[(int64_t)i * m + r] = v;
            bad |= !isfinite(v);
          } else if (r < NU + NX) {
            yo[(int64_t)i * n + r - NU] = v;
            bad |= !isfinite(v);
          } else {
            sm[L::zs + r - NU - NX] = v;
          }
        },
        tid);
    __syncthreads();
    // w = z + B_i u_i
    cta_matvec<NX, NU, NTHREADS>(
        [&](int r, int k) { return fb[L::FB + r + k * n]; }, [&](int k) { return sm[L::us + k]; },
        [&](int r) { return sm[L::zs + r]; }, [&](int r, double v) { sm[L::pr2 + r] = v; }, tid);
    __syncthreads();
    // x_{i+1} = S⁻¹_{i+1} w
    cta_matvec<NX, NX, NTHREADS>(
        [&](int r, int k) { return fb[L::rS + (r >= k ? pidx(n, r, k) : pidx(n, k, r))]; },
        [&](int k) { return sm[L::pr2 + k]; }, [&](int) { return 0.0; },
        [&](int r, double v) {
          sm[L::xs + r] = v;
          xo[(int64_t)(i + 1) * n + r] = v;
          bad |= !isfinite(v);
        },
        tid);
    __syncthreads();
  }
  {  // y_N = Q_N x_N + q_N
    const double* QN = a.p.QN + inst * L::SN;
    cta_matvec<NX, NX, NTHREADS>(
        [&](int r, int k) { return k >= r ? QN[pidx(n, k, r)] : QN[pidx(n, r, k)]; }, [&](int k) { return sm[L::xs + k]; },
        [&](int r) { return a.p.qN[inst * n + r]; },
        [&](int r, double v) {
          yo[sN * n + r] = v;
          bad |= !isfinite(v);
        },
        tid);
  }
  if (__syncthreads_or(bad) && status == 0) status = RR_ST_NONFINITE;
  RR_PROF(RR_CTA_PROFILE_FWD, 10);
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

// ==========================================================================================
// K4b -- the C3 shape at TWO instances per SM (two CTAs of 8 warps, ~108 KB of shared memory each).
// K4 above keeps one instance per SM (all stage matrices resident, ~224 KB), so its serial pivot
// chains (the S⁻¹ diagonal-block sweeps on one warp, the G⁻¹ sweep on four) leave the tensor pipe
// idle for about half of every stage (tools/cta_phase_probe).  K4b halves the footprint so that a
// second instance's contractions run on the SM while the first one sweeps:
//   * only B_i is staged in shared memory (cp.async, one stage ahead); A_i, Q_i, M_i, R_i, q, r, c
//     are read from L2, pulled there one stage ahead by bulk L2 prefetches (cp.async.bulk.prefetch);
//   * W = S⁻¹V (symmetric: W = V(I + δV)⁻¹) is formed explicitly, in place over V; T = W F is
//     formed at once (T_A = W A over the dead S⁻¹, T_B = W B beside B), so that G = Bᵀ T_B + R and
//     H = Uux = Bᵀ T_A + Mᵀ come from shared memory and only Uxx = Aᵀ T_A + Q runs beside the G⁻¹
//     sweep (A from L2);
//   * V_i = Uxx − Hᵀ K̃ is formed in registers and stored over the dead G, H (V's home region);
//   * the forward sweep stages its per-stage record [K k V v e S⁻¹] by TMA bulk copies into two
//     shared buffers (one stage ahead) and reads A_i, B_i from L2 (prefetched two stages ahead).
// Same record layout, status semantics and outputs as K4 (Eq.(RR); forward P:496-509,
// P:640-644; duals P:627-650).
template <int NX, int NU>
struct Cta2Layout {
  using K4 = CtaLayout<NX, NU>;
  static constexpr int NZ = NX + NU;
  static constexpr int SN = K4::SN, SMU = K4::SMU, REC = K4::REC;
  // backward: three NX×NX regions
  static constexpr int RV = 0;             // V_{i+1} -> W (in place) -> G (ld NU) | H (ld NU) -> V_i
  static constexpr int RS = RV + NX * NX;  // S -> −S⁻¹ -> T_A (ld NX) -> K̃ (ld NU)
  static constexpr int RB = RS + NX * NX;  // B (ld NX) | T_B (ld NX) = S-sweep scratch;  Uxx (ld NX) over both
  static constexpr int Gs = RV, Hs = RV + NU * NU, TA = RS, Kt = RS, Bs = RB, TB = RB + NX * NU, YS = TB,
                       Ux = RB;
  static_assert(NU * NU + NU * NX <= NX * NX && 2 * NX * NU <= NX * NX && NX * 16 <= NX * NU,
                "K4b layout assumes n_u = n_x / 2");
  // forward: two record buffers over the dead backward regions
  static constexpr int FR0 = 0, FR1 = REC;
  static constexpr int VEC0 = RB + NX * NX > 2 * REC ? RB + NX * NX : 2 * REC;
  static constexpr int VEC = (VEC0 + 1) & ~1;
  static constexpr int vs = VEC, ve = vs + NX, ee = ve + NX, gg = ee + NX, bb = gg + NX, kt = bb + NZ,
                       gpb = kt + NU, xs = gpb + 2 * NU, us = xs + NX, zs = us + NU, pr2 = zs + NX;
  static constexpr int TOTAL = pr2 + NX;
};

__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

// One 16×16 tile of C = op_A · B + init on one warp (K multiple of 4) where one operand lives in L2
// (GA: op_A, else B): all of that operand's fragments (2 per k-step) are loaded before the first DMMA,
// so a tile waits for one L2 round trip instead of one per unrolled batch; the init values (global
// too) are loaded up front and added after the contraction.  No masking (M, N multiples of 16).
template <int K, bool GA, typename LoadA, typename LoadB, typename Init, typename Store>
__device__ __forceinline__ void warp_tile_l2(int m0, int n0, LoadA&& la, LoadB&& lb, Init&& init, Store&& store,
                                             int lane) {
  const int g = lane >> 2, t = lane & 3;
  double pre[K / 4][2], ini[2][2][2], c[2][2][2];
#pragma unroll
  for (int kt = 0; kt < K / 4; ++kt)
#pragma unroll
    for (int x = 0; x < 2; ++x)
      pre[kt][x] = GA ? la(m0 + 8 * x + g, 4 * kt + t) : lb(4 * kt + t, n0 + 8 * x + g);
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 2; ++y)
#pragma unroll
      for (int z = 0; z < 2; ++z) {
        ini[x][y][z] = init(m0 + 8 * x + g, n0 + 8 * y + 2 * t + z);
        c[x][y][z] = 0.0;
      }
#pragma unroll
  for (int kt = 0; kt < K / 4; ++kt) {
    double o[2];
#pragma unroll
    for (int x = 0; x < 2; ++x) o[x] = GA ? lb(4 * kt + t, n0 + 8 * x + g) : la(m0 + 8 * x + g, 4 * kt + t);
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) {
        if (GA) dmma884(c[x][y][0], c[x][y][1], pre[kt][x], o[y]);
        else dmma884(c[x][y][0], c[x][y][1], o[x], pre[kt][y]);
      }
  }
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 2; ++y)
#pragma unroll
      for (int z = 0; z < 2; ++z) store(m0 + 8 * x + g, n0 + 8 * y + 2 * t + z, c[x][y][z] + ini[x][y][z]);
}

template <int NX, int NU, int NTHREADS>
__global__ void __launch_bounds__(NTHREADS, 2) rr_cta2_kernel(const FusedArgs a) {
  using L = Cta2Layout<NX, NU>;
  using RL = CtaLayout<NX, NU>;  // record layout
  constexpr int NZ = NX + NU;
  constexpr int n = NX, m = NU;
  constexpr int NW = NTHREADS / 32;
  static_assert(NW == 8, "K4b is written for 8 warps (4 sweep + 4 side warps in the G⁻¹ phase)");
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t inst = blockIdx.x;
  const int N = a.N;
  const int64_t sN = N;
  const double delta = a.p.delta[inst];
  double* rec0 = a.ws + inst * sN * L::REC;
  int32_t st = 0;

  auto X = [](int r, int c) { return swz<NX>(r, c); };
  auto Y = [](int r, int c) { return swz<NU>(r, c); };
  // B_i -> Bs (16-byte chunks, rows r, r+1, to their swizzled positions)
  auto issue_B = [&](int i) {
    const double* gB = a.p.B + (inst * sN + i) * n * m;
    for (int e = 2 * tid; e < n * m; e += 2 * NTHREADS) {
      const int r = e % n, c = e / n;
      cp_async16(sm + L::Bs + X(r, c), gB + r + c * n);
    }
    cp_async_commit();
  };
  auto prefetch_stage = [&](int i) {  // backward stage i's operands into L2 (one thread per array)
    const int64_t s = inst * sN + i;
    if (tid == 0) bulk_prefetch_l2(a.p.A + s * n * n, 8u * n * n);
    else if (tid == 32) bulk_prefetch_l2(a.p.Q + s * L::SN, 8u * L::SN);
    else if (tid == 64) bulk_prefetch_l2(a.p.M + s * n * m, 8u * n * m);
    else if (tid == 96) bulk_prefetch_l2(a.p.R + s * L::SMU, 8u * L::SMU);
    else if (tid == 128) bulk_prefetch_l2(a.p.q + s * n, 8u * n);
    else if (tid == 160) bulk_prefetch_l2(a.p.r + s * m, 8u * m);
    else if (tid == 192) bulk_prefetch_l2(a.p.c + s * n, 8u * n);
    else if (tid == 224) bulk_prefetch_l2(a.p.B + s * n * m, 8u * n * m);
  };

  // V_N = Q_N -> RV (ld NX), v_N = q_N
  {
    const double* QN = a.p.QN + inst * L::SN;
    for (int e = tid; e < n * n; e += NTHREADS) {
      const int r = e % n, c = e / n;
      const double v = r >= c ? QN[pidx(n, r, c)] : QN[pidx(n, c, r)];
      sm[L::RV + X(r, c)] = v;
      sm[L::RS + X(r, c)] = delta * v + (r == c ? 1.0 : 0.0);  // S = I + δV_N for the first stage
    }
    for (int r = tid; r < n; r += NTHREADS) sm[L::vs + r] = a.p.qN[inst * n + r];
    if (a.f.V != nullptr)
      for (int e = tid; e < L::SN; e += NTHREADS) a.f.V[(inst * (sN + 1) + N) * L::SN + e] = QN[e];
    if (a.f.v != nullptr)
      for (int r = tid; r < n; r += NTHREADS) a.f.v[(inst * (sN + 1) + N) * n + r] = a.p.qN[inst * n + r];
  }
  if (N > 0) {
    issue_B(N - 1);
    prefetch_stage(N - 1);
  }
  auto no_side = [](int, int, int, int) {};
  static_assert(NX <= NTHREADS, "one thread per row of c");
  double c_next = (tid < n && N > 0) ? a.p.c[(inst * sN + N - 1) * n + tid] : 0.0;  // c_{i+1}, a stage ahead

  for (int i = N - 1; i >= 0; --i) {
    const int64_t s = inst * sN + i;
    const double* gA = a.p.A + s * n * n;
    const double* gQ = a.p.Q + s * L::SN;
    const double* gM = a.p.M + s * n * m;
    const double* gR = a.p.R + s * L::SMU;
    double* rec = rec0 + (int64_t)i * L::REC;
    RR_PROF(i, 0);
    if (i > 0) prefetch_stage(i - 1);
    const double c_cur = c_next;
    if (i > 0 && tid < n) c_next = a.p.c[(s - 1) * n + tid];
    // (1) e = c_{i+1} − δ v_{i+1};  V e  (S = I + δV_{i+1} is in RS: formed with V_{i+1} by stage i+1)
    if (tid < n) {
      const double ev = c_cur - delta * sm[L::vs + tid];
      sm[L::ee + tid] = ev;
      rec[RL::re + tid] = ev;
    }
    __syncthreads();
    cta_matvec<NX, NX, NTHREADS>(
        [&](int r, int k) { return sm[L::RV + X(r, k)]; }, [&](int k) { return sm[L::ee + k]; },
        [&](int) { return 0.0; }, [&](int r, double v) { sm[L::ve + r] = v; }, tid);
    RR_PROF(i, 1);
    // (2) RS <- −S⁻¹ (block sweep; scratch in the T_B slot)
    bool fail = false;
    cta_sweep_blk<NX, NTHREADS>(sm + L::RS, sm + L::YS, tid, &fail, no_side
#ifdef RR_CTA_PROFILE
                                ,
                                (blockIdx.x == 0 && i == RR_CTA_PROFILE) ? 12 : -1
#endif
    );
    if (fail && st == 0) st = mk_status(RR_ST_S_NOT_PD, i);
    RR_PROF(i, 2);
    // (3) W = S⁻¹ V in place over V (symmetric: W = V(I + δV)⁻¹; the 10 lower 16×16 tiles in
    //     registers, mirrored on the store after one barrier);  g = v_{i+1} + S⁻¹ V e;  record S⁻¹
    cp_async_wait<0>();  // B_i (made visible by the barriers below)
    {
      constexpr int MT = NX / 16, NTL = MT * (MT + 1) / 2, TPW = (NTL + NW - 1) / NW;
      const int g = lane >> 2, t = lane & 3;
      double c[TPW][2][2][2];
#pragma unroll
      for (int q = 0; q < TPW; ++q) {
        const int tile = warp + q * NW;
#pragma unroll
        for (int x = 0; x < 8; ++x) (&c[q][0][0][0])[x] = 0.0;
        if (tile < NTL) {
          int R, C;
          lower_tile(tile, R, C);
          const int r0 = 16 * R, c0 = 16 * C;
#pragma unroll 8
          for (int kk = 0; kk < NX / 4; ++kk) {
            double av[2], bv[2];
#pragma unroll
            for (int x = 0; x < 2; ++x) av[x] = -sm[L::RS + X(r0 + 8 * x + g, 4 * kk + t)];
#pragma unroll
            for (int y = 0; y < 2; ++y) bv[y] = sm[L::RV + X(4 * kk + t, c0 + 8 * y + g)];
#pragma unroll
            for (int x = 0; x < 2; ++x)
#pragma unroll
              for (int y = 0; y < 2; ++y) dmma884(c[q][x][y][0], c[q][x][y][1], av[x], bv[y]);
          }
        }
      }
      cta_matvec<NX, NX, NTHREADS>(
          [&](int r, int k) { return -sm[L::RS + X(r, k)]; }, [&](int k) { return sm[L::ve + k]; },
          [&](int r) { return sm[L::vs + r]; }, [&](int r, double v) { sm[L::gg + r] = v; }, tid);
      for (int e = tid; e < n * n; e += NTHREADS) {
        const int r = e % n, cc = e / n;
        if (r >= cc) rec[RL::rS + pidx(n, r, cc)] = -sm[L::RS + X(r, cc)];
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < TPW; ++q) {
        const int tile = warp + q * NW;
        if (tile < NTL) {
          int R, C;
          lower_tile(tile, R, C);
          const int r0 = 16 * R, c0 = 16 * C;
#pragma unroll
          for (int x = 0; x < 2; ++x)
#pragma unroll
            for (int y = 0; y < 2; ++y)
#pragma unroll
              for (int z = 0; z < 2; ++z) {
                const int r = r0 + 8 * x + g, cc = c0 + 8 * y + 2 * t + z;
                sm[L::RV + X(r, cc)] = c[q][x][y][z];
                if (R != C) sm[L::RV + X(cc, r)] = c[q][x][y][z];
              }
        }
      }
    }
    __syncthreads();
    RR_PROF(i, 3);
    // (4) T = W F:  T_B = W B -> TB (B in shared memory),  T_A = W A -> TA over the dead S⁻¹ (A in L2)
    {
      constexpr int NTB = (NX / 16) * (NU / 16), NTA = (NX / 16) * (NX / 16);
      for (int tt = warp; tt < NTB + NTA; tt += NW) {
        if (tt < NTB)
          warp_tile_mn<NX, NU, NX>(
              tt, [&](int r, int k) { return sm[L::RV + X(r, k)]; }, [&](int k, int cc) { return sm[L::Bs + X(k, cc)]; },
              [&](int, int) { return 0.0; }, [&](int r, int cc, double v) { sm[L::TB + X(r, cc)] = v; }, lane);
        else
          warp_tile_l2<NX, false>(
              ((tt - NTB) % (NX / 16)) * 16, ((tt - NTB) / (NX / 16)) * 16, [&](int r, int k) { return sm[L::RV + X(r, k)]; },
              [&](int k, int cc) { return gA[k + cc * n]; }, [&](int, int) { return 0.0; },
              [&](int r, int cc, double v) { sm[L::TA + X(r, cc)] = v; }, lane);
      }
    }
    __syncthreads();
    RR_PROF(i, 4);
    // (5) G = Bᵀ T_B + R (lower tiles, mirrored) -> Gs;  H = Bᵀ T_A + Mᵀ -> Hs (both over the dead W);
    //     b = (q; r) + Fᵀ g
    {
      constexpr int MTU = NU / 16, NGT = MTU * (MTU + 1) / 2, NH = MTU * (NX / 16);
      for (int task = warp; task < NGT + NH; task += NW) {
        if (task < NGT) {
          int R, C;
          lower_tile(task, R, C);
          const bool mir = R != C;
          warp_tile_l2<NX, true>(  // (both operands in shared memory; R, the init, from L2)
              16 * R, 16 * C, [&](int r, int k) { return sm[L::Bs + X(k, r)]; },
              [&](int k, int cc) { return sm[L::TB + X(k, cc)]; },
              [&](int r, int cc) { return r >= cc ? gR[pidx(m, r, cc)] : gR[pidx(m, cc, r)]; },
              [&](int r, int cc, double v) {
                sm[L::Gs + Y(r, cc)] = v;
                if (mir) sm[L::Gs + Y(cc, r)] = v;
              },
              lane);
        } else {
          warp_tile_l2<NX, true>(
              ((task - NGT) % MTU) * 16, ((task - NGT) / MTU) * 16, [&](int r, int k) { return sm[L::Bs + X(k, r)]; },
              [&](int k, int cc) { return sm[L::TA + X(k, cc)]; }, [&](int r, int cc) { return gM[cc + r * n]; },
              [&](int r, int cc, double v) { sm[L::Hs + Y(r, cc)] = v; }, lane);
        }
      }
      cta_matvec<NZ, NX, NTHREADS>(
          [&](int r, int k) { return r < NX ? gA[k + r * n] : sm[L::Bs + X(k, r - NX)]; },
          [&](int k) { return sm[L::gg + k]; },
          [&](int r) { return r < NX ? a.p.q[s * n + r] : a.p.r[s * m + r - NX]; },
          [&](int r, double v) { sm[L::bb + r] = v; }, tid);
    }
    __syncthreads();
    RR_PROF(i, 5);
    // (6) G⁻¹ (coop sweep on warps 0-3, Gs <- −G⁻¹)  ‖  warps 4-7: Uxx = Aᵀ T_A + Q (lower tiles) -> Ux
    //     over the dead B / T_B (A from L2)
    cta_sweep_any<NU, NTHREADS>(sm + L::Gs, m, sm + L::gpb, tid, &fail, [&](int, int, int slot, int nslots) {
      constexpr int MTX = NX / 16, NXX = MTX * (MTX + 1) / 2;
      for (int tt = slot; tt < NXX; tt += nslots) {
        int R, C;
        lower_tile(tt, R, C);
        warp_tile_l2<NX, true>(
            16 * R, 16 * C, [&](int r, int k) { return gA[k + r * n]; }, [&](int k, int cc) { return sm[L::TA + X(k, cc)]; },
            [&](int r, int cc) { return r >= cc ? gQ[pidx(n, r, cc)] : gQ[pidx(n, cc, r)]; },
            [&](int r, int cc, double v) { sm[L::Ux + X(r, cc)] = v; }, lane);
      }
    });
    if (fail && st == 0) st = mk_status(RR_ST_G_NOT_PD, i);
    RR_PROF(i, 6);
    // (7) K̃ = G⁻¹ H -> Kt over the dead T_A;  k̃ = G⁻¹ b_u
    cta_gemm<NU, NX, NU, false>(
        [&](int r, int k) { return -sm[L::Gs + Y(r, k)]; }, [&](int k, int cc) { return sm[L::Hs + Y(k, cc)]; },
        [&](int, int) { return 0.0; },
        [&](int r, int cc, double v) {
          sm[L::Kt + Y(r, cc)] = v;
          rec[RL::rK + r + cc * m] = -v;  // K_i = −K̃ (ld NU)
          if (a.f.K != nullptr) a.f.K[(inst * sN + i) * m * n + r + cc * m] = -v;
        },
        warp, NW, lane);
    cta_matvec<NU, NU, NTHREADS>(
        [&](int r, int k) { return -sm[L::Gs + Y(r, k)]; }, [&](int k) { return sm[L::bb + NX + k]; },
        [&](int) { return 0.0; }, [&](int r, double v) { sm[L::kt + r] = v; }, tid);
    __syncthreads();
    RR_PROF(i, 7);
    // (8) V_i = Uxx − Hᵀ K̃ (lower tiles in registers), v_i = b_x − Hᵀ k̃;  then V_i (mirrored) -> RV
    //     over the dead G, H
    {
      constexpr int MT = NX / 16, NTL = MT * (MT + 1) / 2, TPW = (NTL + NW - 1) / NW;
      const int g = lane >> 2, t = lane & 3;
      double c[TPW][2][2][2];
#pragma unroll
      for (int q = 0; q < TPW; ++q) {
        const int tile = warp + q * NW;
        if (tile < NTL) {
          int R, C;
          lower_tile(tile, R, C);
          const int r0 = 16 * R, c0 = 16 * C;
#pragma unroll
          for (int x = 0; x < 2; ++x)
#pragma unroll
            for (int y = 0; y < 2; ++y)
#pragma unroll
              for (int z = 0; z < 2; ++z) c[q][x][y][z] = sm[L::Ux + X(r0 + 8 * x + g, c0 + 8 * y + 2 * t + z)];
#pragma unroll
          for (int kk = 0; kk < NU / 4; ++kk) {
            double av[2], bv[2];
#pragma unroll
            for (int x = 0; x < 2; ++x) av[x] = -sm[L::Hs + Y(4 * kk + t, r0 + 8 * x + g)];
#pragma unroll
            for (int y = 0; y < 2; ++y) bv[y] = sm[L::Kt + Y(4 * kk + t, c0 + 8 * y + g)];
#pragma unroll
            for (int x = 0; x < 2; ++x)
#pragma unroll
              for (int y = 0; y < 2; ++y) dmma884(c[q][x][y][0], c[q][x][y][1], av[x], bv[y]);
          }
        }
      }
      cta_matvec<NX, NU, NTHREADS>(
          [&](int r, int k) { return -sm[L::Hs + Y(k, r)]; }, [&](int k) { return sm[L::kt + k]; },
          [&](int r) { return sm[L::bb + r]; }, [&](int r, double v) { sm[L::vs + r] = v; }, tid);
      __syncthreads();
#pragma unroll
      for (int q = 0; q < TPW; ++q) {
        const int tile = warp + q * NW;
        if (tile < NTL) {
          int R, C;
          lower_tile(tile, R, C);
          const int r0 = 16 * R, c0 = 16 * C;
          double* fV = a.f.V != nullptr ? a.f.V + (inst * (sN + 1) + i) * L::SN : nullptr;
#pragma unroll
          for (int x = 0; x < 2; ++x)
#pragma unroll
            for (int y = 0; y < 2; ++y)
#pragma unroll
              for (int z = 0; z < 2; ++z) {
                const int r = r0 + 8 * x + g, cc = c0 + 8 * y + 2 * t + z;
                const double v = c[q][x][y][z], sv = delta * v + (r == cc ? 1.0 : 0.0);
                sm[L::RV + X(r, cc)] = v;  // V_i, and S = I + δV_i for stage i − 1 (RS: K̃ is dead)
                sm[L::RS + X(r, cc)] = sv;
                if (R != C) {
                  sm[L::RV + X(cc, r)] = v;
                  sm[L::RS + X(cc, r)] = sv;
                }
                if (r >= cc) {
                  rec[RL::rV + pidx(n, r, cc)] = v;
                  if (fV != nullptr) fV[pidx(n, r, cc)] = v;
                }
              }
        }
      }
    }
    __syncthreads();
    RR_PROF(i, 8);
    // (9) B_{i−1} streams into Bs (Uxx is dead);  record k = −k̃, v_i (K_i, V_i were written from registers)
    if (i > 0) issue_B(i - 1);
    for (int u = tid; u < m; u += NTHREADS) rec[RL::rk + u] = -sm[L::kt + u];
    for (int r = tid; r < n; r += NTHREADS) rec[RL::rv + r] = sm[L::vs + r];
    if (a.f.k != nullptr)
      for (int u = tid; u < m; u += NTHREADS) a.f.k[(inst * sN + i) * m + u] = -sm[L::kt + u];
    if (a.f.v != nullptr)
      for (int r = tid; r < n; r += NTHREADS) a.f.v[(inst * (sN + 1) + i) * n + r] = sm[L::vs + r];
  }
  cp_async_wait<0>();
  __syncthreads();
  RR_PROF(RR_CTA_PROFILE_FWD, 9);

  // x_0 = (I + δV_0)⁻¹ (c_0 − δ v_0)  (S = I + δV_0 was formed by stage 0)
  for (int r = tid; r < n; r += NTHREADS) sm[L::ee + r] = a.p.c0[inst * n + r] - delta * sm[L::vs + r];
  // records 0 and 1, A, B of the first forward stages into L2 while x_0 is solved
  auto prefetch_fwd = [&](int i) {
    const int64_t s = inst * sN + i;
    if (tid == 0) bulk_prefetch_l2(rec0 + (int64_t)i * L::REC, 8u * L::REC);
    else if (tid == 32) bulk_prefetch_l2(a.p.A + s * n * n, 8u * n * n);
    else if (tid == 64) bulk_prefetch_l2(a.p.B + s * n * m, 8u * n * m);
  };
  for (int i = 0; i < N && i < 2; ++i) prefetch_fwd(i);
  __syncthreads();
  {
    bool fail = false;
    cta_sweep_blk<NX, NTHREADS>(sm + L::RS, sm + L::YS, tid, &fail, no_side);
    if (fail && st == 0) st = mk_status(RR_ST_S_NOT_PD, 0);
  }
  cta_matvec<NX, NX, NTHREADS>(
      [&](int r, int k) { return -sm[L::RS + X(r, k)]; }, [&](int k) { return sm[L::ee + k]; }, [&](int) { return 0.0; },
      [&](int r, double v) { sm[L::xs + r] = v; }, tid);
  __shared__ int sst;
  __shared__ __align__(8) uint64_t fbar[2];
  if (tid == 0) {
    sst = 0;
    mbar_init(&fbar[0], 1);
    mbar_init(&fbar[1], 1);
  }
  __syncthreads();
  if (st != 0) atomicMax(&sst, st);
  __syncthreads();  // also: RS / RV (the record buffers' area) no longer read
  int32_t status = sst;

  double* xo = a.s.x + inst * (sN + 1) * n;
  double* uo = a.s.u + inst * sN * m;
  double* yo = a.s.y + inst * (sN + 1) * n;
  for (int r = tid; r < n; r += NTHREADS) xo[r] = sm[L::xs + r];
  bool bad = false;
  // forward: record i by TMA into buffer i & 1 one stage ahead; A_i, B_i from L2
  //   u_i = K_i x_i + k_i,  y_i = V_i x_i + v_i,  z = A_i x_i + e_i,  x_{i+1} = S⁻¹_{i+1} (z + B_i u_i)
  auto issue_fwd = [&](int i) {  // one thread
    fence_proxy_async();  // the CTA's earlier generic accesses of the buffer (after a barrier) before the TMA write
    mbar_arrive_expect_tx(&fbar[i & 1], 8u * L::REC);
    bulk_g2s(sm + ((i & 1) ? L::FR1 : L::FR0), rec0 + (int64_t)i * L::REC, 8u * L::REC, &fbar[i & 1]);
  };
  if (tid == 0 && N > 0) issue_fwd(0);
  RR_PROF(RR_CTA_PROFILE_FWD, 10);
  // A_i x and B_i u on registers: thread (row = tid / 4, part = tid % 4) holds A_i[row][part + 4j] and
  // B_i[row][part + 4j] (the cta_matvec mapping for 64 rows), loaded from L2 one stage ahead
  static_assert(NTHREADS == 4 * NX && NX % 4 == 0 && NU % 4 == 0, "forward register mapping");
  const int frow = tid >> 2, fpart = tid & 3;
  double pa[NX / 4], pb[NU / 4];
  auto load_AB = [&](int i, double (&qa)[NX / 4], double (&qb)[NU / 4]) {
    const double* gA = a.p.A + (inst * sN + i) * n * n + frow;
    const double* gB = a.p.B + (inst * sN + i) * n * m + frow;
#pragma unroll
    for (int jj = 0; jj < NX / 4; ++jj) qa[jj] = gA[(fpart + 4 * jj) * n];
#pragma unroll
    for (int jj = 0; jj < NU / 4; ++jj) qb[jj] = gB[(fpart + 4 * jj) * n];
  };
  auto reduce4 = [](double v) {
    v += __shfl_xor_sync(RR_FULL_MASK, v, 2);
    return v + __shfl_xor_sync(RR_FULL_MASK, v, 1);
  };
  if (N > 0) load_AB(0, pa, pb);
  for (int i = 0; i < N; ++i) {
    const double* rc = sm + ((i & 1) ? L::FR1 : L::FR0);
    double na[NX / 4], nb[NU / 4];
    if (i + 1 < N) load_AB(i + 1, na, nb);  // lands during this stage
    if (i + 2 < N) prefetch_fwd(i + 2);
    mbar_wait_parity(&fbar[i & 1], (i >> 1) & 1);
    if (tid == 0 && i + 1 < N) issue_fwd(i + 1);  // its buffer was last read by stage i−1 (barriers since)
    {  // z = A_i x_i + e_i
      double acc = 0.0;
#pragma unroll
      for (int jj = 0; jj < NX / 4; ++jj) acc = fma(pa[jj], sm[L::xs + fpart + 4 * jj], acc);
      acc = reduce4(acc);
      if (fpart == 0) sm[L::zs + frow] = rc[RL::re + frow] + acc;
    }
    cta_matvec<NU, NX, NTHREADS>(
        [&](int r, int k) { return rc[RL::rK + r + k * m]; }, [&](int k) { return sm[L::xs + k]; },
        [&](int r) { return rc[RL::rk + r]; },
        [&](int r, double v) {
          sm[L::us + r] = v;
          uo[(int64_t)i * m + r] = v;
          bad |= !isfinite(v);
        },
        tid);
    cta_matvec<NX, NX, NTHREADS>(
        [&](int r, int k) { return rc[RL::rV + (r >= k ? pidx(n, r, k) : pidx(n, k, r))]; },
        [&](int k) { return sm[L::xs + k]; }, [&](int r) { return rc[RL::rv + r]; },
        [&](int r, double v) {
          yo[(int64_t)i * n + r] = v;
          bad |= !isfinite(v);
        },
        tid);
    __syncthreads();
    {  // w = z + B_i u_i
      double acc = 0.0;
#pragma unroll
      for (int jj = 0; jj < NU / 4; ++jj) acc = fma(pb[jj], sm[L::us + fpart + 4 * jj], acc);
      acc = reduce4(acc);
      if (fpart == 0) sm[L::pr2 + frow] = sm[L::zs + frow] + acc;
    }
    __syncthreads();
    cta_matvec<NX, NX, NTHREADS>(
        [&](int r, int k) { return rc[RL::rS + (r >= k ? pidx(n, r, k) : pidx(n, k, r))]; },
        [&](int k) { return sm[L::pr2 + k]; }, [&](int) { return 0.0; },
        [&](int r, double v) {
          sm[L::xs + r] = v;
          xo[(int64_t)(i + 1) * n + r] = v;
          bad |= !isfinite(v);
        },
        tid);
    __syncthreads();
#pragma unroll
    for (int jj = 0; jj < NX / 4; ++jj) pa[jj] = na[jj];
#pragma unroll
    for (int jj = 0; jj < NU / 4; ++jj) pb[jj] = nb[jj];
  }
  {  // y_N = Q_N x_N + q_N
    const double* QN = a.p.QN + inst * L::SN;
    cta_matvec<NX, NX, NTHREADS>(
        [&](int r, int k) { return k >= r ? QN[pidx(n, k, r)] : QN[pidx(n, r, k)]; }, [&](int k) { return sm[L::xs + k]; },
        [&](int r) { return a.p.qN[inst * n + r]; },
        [&](int r, double v) {
          yo[sN * n + r] = v;
          bad |= !isfinite(v);
        },
        tid);
  }
  if (__syncthreads_or(bad) && status == 0) status = RR_ST_NONFINITE;
  RR_PROF(RR_CTA_PROFILE_FWD, 11);
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

template <int NX, int NU>
struct Cta2Cfg {
  static constexpr int NTHREADS = 256;
  static size_t smem_bytes() { return sizeof(double) * (size_t)Cta2Layout<NX, NU>::TOTAL; }
  static int64_t ws_doubles(int64_t batch, int N) { return batch * (int64_t)N * CtaLayout<NX, NU>::REC; }
  static cudaError_t launch(const FusedArgs& a, cudaStream_t s) {
    auto k = rr_cta2_kernel<NX, NU, NTHREADS>;
    const size_t smb = smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb);
    if (e != cudaSuccess) return e;
    k<<<(unsigned)a.batch, NTHREADS, smb, s>>>(a);
    return cudaGetLastError();
  }
};

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
  if (nx == 64 && nu == 32) {
    // K4b (two instances per SM) by default; RR_B200_CTA=1 selects K4 (one instance per SM, 16 warps)
    const char* v = getenv("RR_B200_CTA");
    if (v == nullptr || v[0] != '1') return f(Cta2Cfg<64, 32>{});
    return f(CtaCfg<64, 32, 512>{});
  }
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
