// rr_pit.cu -- parallel-in-time regularized LQR solve (the paper's future work,
// "derive an efficient parallel version of the regularized LQR algorithm").
//
// Method.  For δ > 0 the regularized system [P Cᵀ; C −δI][z; y] = −[s; c] is equivalent
// to (δP + CᵀC) z = −(δs + Cᵀc) with y = (Cz + c)/δ (reading R2).  That is the minimum of
//     δ(½zᵀPz + sᵀz) + ½‖c_0 − x_0‖² + ½ Σ_i ‖A_i x_i + B_i u_i + c_{i+1} − x_{i+1}‖²,
// a sum of stage terms that couple (x_i, u_i, x_{i+1}) only.  Eliminating u_i inside its stage
// (Schur complement on G'_i = δR_i + B_iᵀB_i, SPD) leaves a block-tridiagonal SPD system in the
// states x_0..x_N, which block cyclic reduction solves in ⌈log2(N+1)⌉ levels instead of N
// sequential stages:
//   level with stride s: every index k ≡ s (mod 2s) is eliminated (Y1 = D_k⁻¹ C_{k−s},
//   Y2 = D_k⁻¹ C_kᵀ, yb = D_k⁻¹ b_k), every remaining index j gathers the two Schur updates
//   D_j −= C_jᵀY1_{j+s} + C_{j−s}Y2_{j−s}, b_j −= C_jᵀyb_{j+s} + C_{j−s}yb_{j−s}, C_j ← −C_{j+s}Y1_{j+s};
//   then x_0 = D_0⁻¹b_0 and, level by level in reverse, x_k = yb_k − Y1_k x_{k−s} − Y2_k x_{k+s}.
// Finally u_i = −G'⁻¹(Hᵤₓx_i − B_iᵀx_{i+1} + l_u) and y_0 = (c_0 − x_0)/δ,
// y_{i+1} = (A_i x_i + B_i u_i + c_{i+1} − x_{i+1})/δ (the dual identity of P:627-650).
// The same unique solution as the recursion (DESIGN.md §9 f3); y inherits a cancellation error of
// order ε·|x|/δ, so the path is meant for δ >= ~1e-6.
//
// B200 organisation: every step is a map over (instance, index) with one warp per item (n, m <= 16:
// lane j owns column j, n×n blocks staged in the warp's shared-memory tile), so a batch-1 problem
// with N = 4096 exposes 2048-way parallelism at the first level.  Up to 2,048 items per step, all steps
// run in ONE cooperative launch (pit_fused_kernel: persistent warps, a grid-wide barrier between
// steps) instead of ~3 launches per level and refinement pass; wider problems (and RR_PIT_STEPS=1,
// for A/B) launch one kernel per step.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <cooperative_groups.h>
#include <stdlib.h>

#include "rr_common.cuh"
#include "rr_pit.cuh"

namespace rrk {

namespace {

constexpr int NM = 16;          // max n, m
constexpr int TILE = NM * NM;   // one matrix tile in shared memory
constexpr int WPB = 4;          // warps per block

__device__ __forceinline__ int pk(int n, int r, int c) { return r >= c ? pidx(n, r, c) : pidx(n, c, r); }

struct PitWs {  // per-instance views
  double *D, *C, *b, *Y1, *Y2, *yb;  // [(N+1)][n*n] / [(N+1)][n]
  double *Gi, *Hux, *lu;             // [N][m*m], [N][m*n], [N][m]
  double* Di;                        // [(N+1)][n*n] D_k⁻¹ of the eliminated / root indices (re-solves)
};

// doubles of the per-instance region
__host__ __device__ __forceinline__ int64_t pit_per(int N, int n, int m) {
  return (int64_t)(N + 1) * (5 * n * n + 2 * n) + (int64_t)N * (m * m + m * n + m);
}

__device__ __forceinline__ PitWs views(double* ws, int64_t inst, int N, int n, int m) {
  double* base = ws + inst * pit_per(N, n, m);
  PitWs v;
  v.D = base;
  v.C = v.D + (int64_t)(N + 1) * n * n;
  v.Y1 = v.C + (int64_t)(N + 1) * n * n;
  v.Y2 = v.Y1 + (int64_t)(N + 1) * n * n;
  v.b = v.Y2 + (int64_t)(N + 1) * n * n;
  v.yb = v.b + (int64_t)(N + 1) * n;
  v.Gi = v.yb + (int64_t)(N + 1) * n;
  v.Hux = v.Gi + (int64_t)N * m * m;
  v.lu = v.Hux + (int64_t)N * m * n;
  v.Di = v.lu + (int64_t)N * m;
  return v;
}

// In-place inverse of the SPD k×k matrix T (column-major, ld NM, shared) by the symmetric sweep
// operator, lane j owning column j; flags a non-positive pivot.
__device__ void warp_inv_spd(double* T, int k, int lane, bool& bad) {
  double a[NM];
#pragma unroll
  for (int r = 0; r < NM; ++r) a[r] = (lane < k && r < k) ? T[lane * NM + r] : 0.0;
  __syncwarp();
  for (int p = 0; p < k; ++p) {
    const double ap = __shfl_sync(RR_FULL_MASK, a[p], p);  // pivot
    double col[NM];
#pragma unroll
    for (int r = 0; r < NM; ++r) col[r] = __shfl_sync(RR_FULL_MASK, a[p], r);  // column p = row p
    bad |= !(ap > 0.0);
    const double ip = 1.0 / ap;
    if (lane == p) {
#pragma unroll
      for (int r = 0; r < NM; ++r) a[r] = (r == p) ? -ip : a[r] * ip;
    } else {
      const double f = a[p] * ip;
#pragma unroll
      for (int r = 0; r < NM; ++r) a[r] = (r == p) ? f : fma(-col[r], f, a[r]);
    }
  }
  if (lane < k)
#pragma unroll
    for (int r = 0; r < NM; ++r)
      if (r < k) T[lane * NM + r] = -a[r];
  __syncwarp();
}

// Out (r×q, ld NM) = X (r×p, ld NM) · Y (p×q, ld NM); lane j < q computes column j.  trX: X is given
// transposed (X = Zᵀ with Z p×r stored).  All operands in shared memory; Out may not alias.
__device__ void warp_mm(const double* X, bool trX, const double* Y, double* Out, int r, int p, int q, int lane,
                        double alpha = 1.0, const double* Add = nullptr) {
  if (lane < q) {
    double acc[NM];
#pragma unroll
    for (int i = 0; i < NM; ++i) acc[i] = (Add != nullptr && i < r) ? Add[lane * NM + i] : 0.0;
    for (int k = 0; k < p; ++k) {
      const double y = alpha * Y[lane * NM + k];
#pragma unroll
      for (int i = 0; i < NM; ++i)
        if (i < r) acc[i] = fma(trX ? X[i * NM + k] : X[k * NM + i], y, acc[i]);
    }
#pragma unroll
    for (int i = 0; i < NM; ++i)
      if (i < r) Out[lane * NM + i] = acc[i];
  }
  __syncwarp();
}

__device__ void load_tile(double* T, const double* g, int rows, int cols, int lane) {  // g col-major rows×cols
  for (int e = lane; e < rows * cols; e += 32) T[(e / rows) * NM + e % rows] = g[e];
  __syncwarp();
}
__device__ void store_tile(double* g, const double* T, int rows, int cols, int lane) {
  for (int e = lane; e < rows * cols; e += 32) g[e] = T[(e / rows) * NM + e % rows];
  __syncwarp();
}

// δ of the reduction solve: max(δ, delta_floor) (PitArgs); the residual kernel keeps the caller's δ
__device__ __forceinline__ double pit_delta(const PitArgs& a, int64_t inst) {
  return fmax(a.p.delta[inst], a.delta_floor);
}

// ---- 1. stage assembly: warp per (instance, stage) ----
__device__ void pit_assemble_item(const PitArgs& a, int64_t item, double* T, int lane) {  // T: 8 tiles
  const int n = a.nx, m = a.nu, N = a.N;
  const int64_t inst = item / N;
  const int i = (int)(item % N);
  double *tA = T, *tB = T + TILE, *tG = T + 2 * TILE, *tHxu = T + 3 * TILE, *tW1 = T + 4 * TILE, *tW2 = T + 5 * TILE,
         *tE = T + 6 * TILE, *tv = T + 7 * TILE;
  const double d = pit_delta(a, inst);
  const int64_t sD = dyn_blk(a.shared, inst, N, i);
  const int64_t sP = cost_blk(a.shared, inst, N, i);
  const int64_t s = inst * N + i;
  const int sn = n * (n + 1) / 2, smm = m * (m + 1) / 2;
  load_tile(tA, a.p.A + sD * n * n, n, n, lane);
  load_tile(tB, a.p.B + sD * n * m, n, m, lane);
  // G' = δR + BᵀB ; Hxu = δM + AᵀB ; E_xx = δQ + AᵀA (assembled below)
  warp_mm(tB, true, tB, tG, m, n, m, lane);
  if (lane < m)
    for (int r = 0; r < m; ++r) tG[lane * NM + r] += d * a.p.R[sP * smm + pk(m, r, lane)];
  __syncwarp();
  warp_mm(tA, true, tB, tHxu, n, n, m, lane);
  if (lane < m)
    for (int r = 0; r < n; ++r) tHxu[lane * NM + r] += d * a.p.M[sP * n * m + r + lane * n];
  __syncwarp();
  bool bad = false;
  warp_inv_spd(tG, m, lane, bad);  // G'⁻¹
  PitWs v = views(a.ws, inst, N, n, m);
  // vectors: c = c_{i+1}, l_u = δr + Bᵀc, l_x = δq + Aᵀc
  double* c = tv;
  double* lu = tv + NM;
  double* lx = tv + 2 * NM;
  double* t1 = tv + 3 * NM;
  if (lane < n) c[lane] = a.p.c[s * n + lane];
  __syncwarp();
  if (lane < m) {
    double acc = d * a.p.r[s * m + lane];
    for (int k = 0; k < n; ++k) acc = fma(tB[lane * NM + k], c[k], acc);
    lu[lane] = acc;
  }
  if (lane < n) {
    double acc = d * a.p.q[s * n + lane];
    for (int k = 0; k < n; ++k) acc = fma(tA[lane * NM + k], c[k], acc);
    lx[lane] = acc;
  }
  __syncwarp();
  // W1 = G'⁻¹ Hux (m×n) with Hux = Hxuᵀ ; W2 = G'⁻¹ Bᵀ (m×n) ; t1 = G'⁻¹ l_u (m)
  // W1 = G'⁻¹ Hux with Hux(k, j) = Hxu(j, k) = tHxu[k*NM + j];  W2 = G'⁻¹ Bᵀ
  if (lane < n) {
    double acc[NM];
#pragma unroll
    for (int r = 0; r < NM; ++r) acc[r] = 0.0;
    for (int k = 0; k < m; ++k) {
      const double hk = tHxu[k * NM + lane];  // Hux(k, lane)
#pragma unroll
      for (int r = 0; r < NM; ++r)
        if (r < m) acc[r] = fma(tG[k * NM + r], hk, acc[r]);
    }
#pragma unroll
    for (int r = 0; r < NM; ++r)
      if (r < m) tW1[lane * NM + r] = acc[r];
#pragma unroll
    for (int r = 0; r < NM; ++r) acc[r] = 0.0;
    for (int k = 0; k < m; ++k) {
      const double bk = tB[k * NM + lane];
#pragma unroll
      for (int r = 0; r < NM; ++r)
        if (r < m) acc[r] = fma(tG[k * NM + r], bk, acc[r]);
    }
#pragma unroll
    for (int r = 0; r < NM; ++r)
      if (r < m) tW2[lane * NM + r] = acc[r];
  }
  if (lane < m) {
    double acc = 0.0;
    for (int k = 0; k < m; ++k) acc = fma(tG[k * NM + lane], lu[k], acc);
    t1[lane] = acc;
  }
  __syncwarp();
  // E_xx = δQ + AᵀA − Hxu W1  -> contribution to D_i
  warp_mm(tA, true, tA, tE, n, n, n, lane);
  if (lane < n)
    for (int r = 0; r < n; ++r) {
      double acc = tE[lane * NM + r] + d * a.p.Q[sP * sn + pk(n, r, lane)];
      for (int k = 0; k < m; ++k) acc = fma(-tHxu[k * NM + r], tW1[lane * NM + k], acc);
      tE[lane * NM + r] = acc;
    }
  __syncwarp();
  store_tile(v.Y1 + (int64_t)i * n * n, tE, n, n, lane);  // stage part "Dx" parked in Y1 (assembly only)
  // E_x'x = −A + B W1 (row block x_{i+1}, column block x_i) -> coupling C_i = H_{i+1,i}
  if (lane < n)
    for (int r = 0; r < n; ++r) {
      double acc = -tA[lane * NM + r];
      for (int k = 0; k < m; ++k) acc = fma(tB[k * NM + r], tW1[lane * NM + k], acc);
      tE[lane * NM + r] = acc;
    }
  __syncwarp();
  store_tile(v.C + (int64_t)i * n * n, tE, n, n, lane);
  // E_x'x' = I − B W2 -> contribution to D_{i+1}, parked in Y2
  if (lane < n)
    for (int r = 0; r < n; ++r) {
      double acc = (r == lane) ? 1.0 : 0.0;
      for (int k = 0; k < m; ++k) acc = fma(-tB[k * NM + r], tW2[lane * NM + k], acc);
      tE[lane * NM + r] = acc;
    }
  __syncwarp();
  store_tile(v.Y2 + (int64_t)i * n * n, tE, n, n, lane);
  // linear parts: e_x = l_x − Hxu t1 (to b_i, parked in yb), e_x' = −c + B t1 (to b_{i+1}, parked in b)
  if (lane < n) {
    double ex = lx[lane], ey = -c[lane];
    for (int k = 0; k < m; ++k) {
      ex = fma(-tHxu[k * NM + lane], t1[k], ex);
      ey = fma(tB[k * NM + lane], t1[k], ey);
    }
    v.yb[(int64_t)i * n + lane] = ex;
    v.b[(int64_t)(i + 1) * n + lane] = ey;
  }
  // recovery data: G'⁻¹, Hux = Hxuᵀ, l_u
  for (int e = lane; e < m * m; e += 32) v.Gi[(int64_t)i * m * m + e] = tG[(e / m) * NM + e % m];
  for (int e = lane; e < m * n; e += 32) {
    const int r = e % m, col = e / m;  // Hux (m×n) column-major: (r, col) = Hxu(col, r)
    v.Hux[(int64_t)i * m * n + e] = tHxu[r * NM + col];
  }
  if (lane < m) v.lu[(int64_t)i * m + lane] = lu[lane];
  if (bad && lane == 0) atomicMax(a.status + inst, (int32_t)mk_status(RR_ST_G_NOT_PD, i));
}

// ---- 2. block-tridiagonal system: D_k, b_k (warp per (instance, k)) ----
__device__ void pit_diag_item(const PitArgs& a, int64_t item, int lane) {
  const int n = a.nx, m = a.nu, N = a.N;
  const int64_t inst = item / (N + 1);
  const int k = (int)(item % (N + 1));
  PitWs v = views(a.ws, inst, N, n, m);
  const double d = pit_delta(a, inst);
  const int sn = n * (n + 1) / 2;
  const int64_t iP = (a.shared & RR_FLAG_SHARED_COST) ? 0 : inst;
  // D_k = [k < N] E_xx,k + [k > 0] E_x'x',k−1 + [k == 0] I + [k == N] δQ_N ; the linear term g_k likewise
  // (E parts parked in Y1 / Y2, e_x in yb, e_x' in b by the assembly); b_k = −g_k
  for (int e = lane; e < n * n; e += 32) {
    const int r = e % n, col = e / n;
    double val = 0.0;
    if (k < N) val += v.Y1[(int64_t)k * n * n + e];
    if (k > 0) val += v.Y2[(int64_t)(k - 1) * n * n + e];
    if (k == 0 && r == col) val += 1.0;
    if (k == N) val += d * a.p.QN[iP * sn + pk(n, r, col)];
    v.D[(int64_t)k * n * n + e] = val;
  }
  if (lane < n) {
    double g = 0.0;
    if (k < N) g += v.yb[(int64_t)k * n + lane];
    if (k > 0) g += v.b[(int64_t)k * n + lane];
    if (k == 0) g -= a.p.c0[inst * n + lane];
    if (k == N) g += d * a.p.qN[inst * n + lane];
    v.b[(int64_t)k * n + lane] = -g;
  }
}
// (the two reads of b[k] / write of b[k] above touch only this item's own entries; yb / Y1 / Y2 of
//  index k are overwritten later only by the elimination of index k itself)

// ---- 3a. cyclic reduction, elimination of the indices k ≡ s (mod 2s) ----
__device__ void pit_elim_item(const PitArgs& a, int s, int64_t item, double* T, int lane) {  // T: 4 tiles
  const int n = a.nx, m = a.nu, N = a.N;
  const int64_t per = (int64_t)((N - s) / (2 * s) + 1);  // eliminated indices per instance
  const int64_t inst = item / per;
  const int k = s + 2 * s * (int)(item % per);
  PitWs v = views(a.ws, inst, N, n, m);
  double *tD = T, *tC = T + TILE, *tY = T + 2 * TILE, *tb = T + 3 * TILE;
  load_tile(tD, v.D + (int64_t)k * n * n, n, n, lane);
  bool bad = false;
  warp_inv_spd(tD, n, lane, bad);
  store_tile(v.Di + (int64_t)k * n * n, tD, n, n, lane);
  // Y1 = D_k⁻¹ C_{k−s}  (C_{k−s} = H_{k, k−s})
  load_tile(tC, v.C + (int64_t)(k - s) * n * n, n, n, lane);
  warp_mm(tD, false, tC, tY, n, n, n, lane);
  store_tile(v.Y1 + (int64_t)k * n * n, tY, n, n, lane);
  // Y2 = D_k⁻¹ C_kᵀ (C_k = H_{k+s, k}); zero when k + s > N
  if (k + s <= N) {
    load_tile(tC, v.C + (int64_t)k * n * n, n, n, lane);
    if (lane < n) {
      double acc[NM];
#pragma unroll
      for (int r = 0; r < NM; ++r) acc[r] = 0.0;
      for (int q = 0; q < n; ++q) {
        const double cq = tC[q * NM + lane];  // C_kᵀ(q, lane) = C_k(lane, q)
#pragma unroll
        for (int r = 0; r < NM; ++r)
          if (r < n) acc[r] = fma(tD[q * NM + r], cq, acc[r]);
      }
#pragma unroll
      for (int r = 0; r < NM; ++r)
        if (r < n) tY[lane * NM + r] = acc[r];
    }
    __syncwarp();
    store_tile(v.Y2 + (int64_t)k * n * n, tY, n, n, lane);
  } else {
    for (int e = lane; e < n * n; e += 32) v.Y2[(int64_t)k * n * n + e] = 0.0;
  }
  // yb = D_k⁻¹ b_k
  if (lane < n) tb[lane] = v.b[(int64_t)k * n + lane];
  __syncwarp();
  if (lane < n) {
    double acc = 0.0;
    for (int q = 0; q < n; ++q) acc = fma(tD[q * NM + lane], tb[q], acc);
    v.yb[(int64_t)k * n + lane] = acc;
  }
  if (bad && lane == 0) atomicMax(a.status + inst, (int32_t)mk_status(RR_ST_S_NOT_PD, k));
}

// ---- 3b. cyclic reduction, Schur updates of the remaining indices j ≡ 0 (mod 2s) ----
__device__ void pit_update_item(const PitArgs& a, int s, int64_t item, double* T, int lane) {  // T: 4 tiles
  const int n = a.nx, m = a.nu, N = a.N;
  const int64_t per = (int64_t)(N / (2 * s) + 1);
  const int64_t inst = item / per;
  const int j = 2 * s * (int)(item % per);
  PitWs v = views(a.ws, inst, N, n, m);
  double *tD = T, *tC = T + TILE, *tY = T + 2 * TILE, *tb = T + 3 * TILE;
  load_tile(tD, v.D + (int64_t)j * n * n, n, n, lane);
  if (lane < n) tb[lane] = v.b[(int64_t)j * n + lane];
  __syncwarp();
  if (j + s <= N) {  // right neighbour k = j + s: D_j −= C_jᵀ Y1_k, b_j −= C_jᵀ yb_k, C_j ← −C_k Y1_k
    const int k = j + s;
    load_tile(tC, v.C + (int64_t)j * n * n, n, n, lane);
    load_tile(tY, v.Y1 + (int64_t)k * n * n, n, n, lane);
    warp_mm(tC, true, tY, tD, n, n, n, lane, -1.0, tD);
    if (lane < n) {
      double acc = tb[lane];
      for (int q = 0; q < n; ++q) acc = fma(-tC[lane * NM + q], v.yb[(int64_t)k * n + q], acc);
      tb[lane] = acc;
    }
    __syncwarp();
    if (k + s <= N) {  // new coupling H_{j+2s, j} = −C_k Y1_k
      load_tile(tC, v.C + (int64_t)k * n * n, n, n, lane);
      if (lane < n) {
        double acc[NM];
#pragma unroll
        for (int r = 0; r < NM; ++r) acc[r] = 0.0;
        for (int q = 0; q < n; ++q) {
          const double yq = tY[lane * NM + q];
#pragma unroll
          for (int r = 0; r < NM; ++r)
            if (r < n) acc[r] = fma(-tC[q * NM + r], yq, acc[r]);
        }
#pragma unroll
        for (int r = 0; r < NM; ++r)
          if (r < n) v.C[(int64_t)j * n * n + lane * n + r] = acc[r];
      }
      __syncwarp();
    }
  }
  if (j - s >= 0) {  // left neighbour k = j − s: D_j −= C_{j−s} Y2_k, b_j −= C_{j−s} yb_k
    const int k = j - s;
    load_tile(tC, v.C + (int64_t)(j - s) * n * n, n, n, lane);
    load_tile(tY, v.Y2 + (int64_t)k * n * n, n, n, lane);
    warp_mm(tC, false, tY, tD, n, n, n, lane, -1.0, tD);
    if (lane < n) {
      double acc = tb[lane];
      for (int q = 0; q < n; ++q) acc = fma(-tC[q * NM + lane], v.yb[(int64_t)k * n + q], acc);
      tb[lane] = acc;
    }
    __syncwarp();
  }
  store_tile(v.D + (int64_t)j * n * n, tD, n, n, lane);
  if (lane < n) v.b[(int64_t)j * n + lane] = tb[lane];
}

// ---- 3c. root x_0 = D_0⁻¹ b_0, then back-substitution per level ----
__device__ void pit_root_item(const PitArgs& a, int64_t inst, double* T, int lane) {  // T: 1 tile
  const int n = a.nx, m = a.nu, N = a.N;
  PitWs v = views(a.ws, inst, N, n, m);
  load_tile(T, v.D, n, n, lane);
  bool bad = false;
  warp_inv_spd(T, n, lane, bad);
  store_tile(v.Di, T, n, n, lane);
  if (lane < n) {
    double acc = 0.0;
    for (int q = 0; q < n; ++q) acc = fma(T[q * NM + lane], v.b[q], acc);
    a.s.x[inst * (int64_t)(N + 1) * n + lane] = acc;
  }
  if (bad && lane == 0) atomicMax(a.status + inst, (int32_t)mk_status(RR_ST_S_NOT_PD, 0));
}

__device__ void pit_backsub_item(const PitArgs& a, int s, int64_t item, int lane) {
  const int n = a.nx, m = a.nu, N = a.N;
  const int64_t per = (int64_t)((N - s) / (2 * s) + 1);
  const int64_t inst = item / per;
  const int k = s + 2 * s * (int)(item % per);
  PitWs v = views(a.ws, inst, N, n, m);
  double* x = a.s.x + inst * (int64_t)(N + 1) * n;
  if (lane < n) {
    double acc = v.yb[(int64_t)k * n + lane];
    const double* Y1 = v.Y1 + (int64_t)k * n * n;
    for (int q = 0; q < n; ++q) acc = fma(-Y1[q * n + lane], x[(int64_t)(k - s) * n + q], acc);
    if (k + s <= N) {
      const double* Y2 = v.Y2 + (int64_t)k * n * n;
      for (int q = 0; q < n; ++q) acc = fma(-Y2[q * n + lane], x[(int64_t)(k + s) * n + q], acc);
    }
    x[(int64_t)k * n + lane] = acc;
  }
}

// ---- 4. controls and duals: warp per (instance, stage) ----
__device__ void pit_recover_item(const PitArgs& a, int64_t item, int lane) {
  const int n = a.nx, m = a.nu, N = a.N;
  const int64_t inst = item / (N + 1);
  const int i = (int)(item % (N + 1));
  const double d = pit_delta(a, inst);
  const double* x = a.s.x + inst * (int64_t)(N + 1) * n;
  double* y = a.s.y + inst * (int64_t)(N + 1) * n;
  if (i == 0) {  // y_0 = (c_0 − x_0)/δ
    const double y0 = (lane < n) ? (a.p.c0[inst * n + lane] - x[lane]) / d : 0.0;
    if (lane < n) y[lane] = y0;
    if (__any_sync(RR_FULL_MASK, !isfinite(y0)) && lane == 0) atomicMax(a.status + inst, (int32_t)RR_ST_NONFINITE);
    return;
  }
  const int st = i - 1;  // stage producing x_i: u_{st}, y_i
  PitWs v = views(a.ws, inst, N, n, m);
  const int64_t s = inst * N + st;
  const int64_t sD = dyn_blk(a.shared, inst, N, st);
  const double* B = a.p.B + sD * n * m;
  const double* A = a.p.A + sD * n * n;
  const double* xi = x + (int64_t)st * n;
  const double* x1 = x + (int64_t)i * n;
  // t = Hux x_i − Bᵀx_{i+1} + l_u (lanes < m), u = −G'⁻¹ t
  double t = 0.0;
  if (lane < m) {
    t = v.lu[(int64_t)st * m + lane];
    const double* H = v.Hux + (int64_t)st * m * n;
    for (int q = 0; q < n; ++q) t = fma(H[lane + q * m], xi[q], t);
    for (int q = 0; q < n; ++q) t = fma(-B[q + lane * n], x1[q], t);
  }
  double u = 0.0;
  const double* G = v.Gi + (int64_t)st * m * m;
  for (int q = 0; q < m; ++q) {
    const double tq = __shfl_sync(RR_FULL_MASK, t, q);
    if (lane < m) u = fma(-G[lane + q * m], tq, u);
  }
  if (lane < m) a.s.u[s * m + lane] = u;
  bool bad = (lane < m) && !isfinite(u);
  // y_{i} = (A x_{i−1} + B u_{i−1} + c_i − x_i)/δ
  double r = 0.0;
  if (lane < n) {
    r = a.p.c[s * n + lane] - x1[lane];
    for (int q = 0; q < n; ++q) r = fma(A[lane + q * n], xi[q], r);
  }
  for (int q = 0; q < m; ++q) {
    const double uq = __shfl_sync(RR_FULL_MASK, u, q);
    if (lane < n) r = fma(B[lane + q * n], uq, r);
  }
  if (lane < n) y[(int64_t)i * n + lane] = r / d;
  bad |= (lane < n) && !(isfinite(r / d) && isfinite(x1[lane]));
  if (__any_sync(RR_FULL_MASK, bad) && lane == 0) atomicMax(a.status + inst, (int32_t)RR_ST_NONFINITE);
}

// ---- refinement (re-solve with the stored reduction for a new right-hand side) ----
// rhs assembly: l_u = δr + Bᵀc, l_x = δq + Aᵀc, t1 = G'⁻¹l_u, e_x = l_x − Hxu t1 (-> yb_i),
// e_x' = −c + B t1 (-> b_{i+1}), l_u kept for the recovery of u
__device__ void pit_rhs_assemble_item(const PitArgs& a, int64_t item, int lane) {
  const int n = a.nx, m = a.nu, N = a.N;
  const int64_t inst = item / N;
  const int i = (int)(item % N);
  PitWs v = views(a.ws, inst, N, n, m);
  const double d = pit_delta(a, inst);
  const int64_t s = inst * N + i;
  const int64_t sD = dyn_blk(a.shared, inst, N, i);
  const double* A = a.p.A + sD * n * n;
  const double* B = a.p.B + sD * n * m;
  const double* c = a.p.c + s * n;
  double lu = 0.0;
  if (lane < m) {
    lu = d * a.p.r[s * m + lane];
    for (int k = 0; k < n; ++k) lu = fma(B[k + lane * n], c[k], lu);
    v.lu[(int64_t)i * m + lane] = lu;
  }
  double t1 = 0.0;
  const double* G = v.Gi + (int64_t)i * m * m;
  for (int q = 0; q < m; ++q) {
    const double lq = __shfl_sync(RR_FULL_MASK, lu, q);
    if (lane < m) t1 = fma(G[lane + q * m], lq, t1);
  }
  const double* H = v.Hux + (int64_t)i * m * n;  // Hux (m×n): Hxu(j, q) = Hux(q, j)
  double ex = 0.0, ey = 0.0;
  if (lane < n) {
    ex = d * a.p.q[s * n + lane];
    for (int k = 0; k < n; ++k) ex = fma(A[k + lane * n], c[k], ex);
    ey = -c[lane];
  }
  for (int q = 0; q < m; ++q) {
    const double tq = __shfl_sync(RR_FULL_MASK, t1, q);
    if (lane < n) {
      ex = fma(-H[q + lane * m], tq, ex);
      ey = fma(B[lane + q * n], tq, ey);
    }
  }
  if (lane < n) {
    v.yb[(int64_t)i * n + lane] = ex;
    v.b[(int64_t)(i + 1) * n + lane] = ey;
  }
}

__device__ void pit_rhs_diag_item(const PitArgs& a, int64_t item, int lane) {
  const int n = a.nx, m = a.nu, N = a.N;
  const int64_t inst = item / (N + 1);
  const int k = (int)(item % (N + 1));
  PitWs v = views(a.ws, inst, N, n, m);
  if (lane < n) {
    double g = 0.0;
    if (k < N) g += v.yb[(int64_t)k * n + lane];
    if (k > 0) g += v.b[(int64_t)k * n + lane];
    if (k == 0) g -= a.p.c0[inst * n + lane];
    if (k == N) g += pit_delta(a, inst) * a.p.qN[inst * n + lane];
    v.b[(int64_t)k * n + lane] = -g;
  }
}

__device__ void pit_rhs_elim_item(const PitArgs& a, int s, int64_t item, int lane) {  // yb_k = D_k⁻¹ b_k
  const int n = a.nx, m = a.nu, N = a.N;
  const int64_t per = (int64_t)((N - s) / (2 * s) + 1);
  const int64_t inst = item / per;
  const int k = s + 2 * s * (int)(item % per);
  PitWs v = views(a.ws, inst, N, n, m);
  if (lane < n) {
    const double* Di = v.Di + (int64_t)k * n * n;
    double acc = 0.0;
    for (int q = 0; q < n; ++q) acc = fma(Di[lane + q * n], v.b[(int64_t)k * n + q], acc);
    v.yb[(int64_t)k * n + lane] = acc;
  }
}

__device__ void pit_rhs_update_item(const PitArgs& a, int s, int64_t item, int lane) {
  // b_j −= C_jᵀ yb_{j+s} + C_{j−s} yb_{j−s} = Y1_{j+s}ᵀ b_{j+s} + Y2_{j−s}ᵀ b_{j−s}
  const int n = a.nx, m = a.nu, N = a.N;
  const int64_t per = (int64_t)(N / (2 * s) + 1);
  const int64_t inst = item / per;
  const int j = 2 * s * (int)(item % per);
  PitWs v = views(a.ws, inst, N, n, m);
  if (lane < n) {
    double acc = v.b[(int64_t)j * n + lane];
    if (j + s <= N) {
      const double* Y1 = v.Y1 + (int64_t)(j + s) * n * n;
      for (int q = 0; q < n; ++q) acc = fma(-Y1[q + lane * n], v.b[(int64_t)(j + s) * n + q], acc);
    }
    if (j - s >= 0) {
      const double* Y2 = v.Y2 + (int64_t)(j - s) * n * n;
      for (int q = 0; q < n; ++q) acc = fma(-Y2[q + lane * n], v.b[(int64_t)(j - s) * n + q], acc);
    }
    v.b[(int64_t)j * n + lane] = acc;
  }
}

__device__ void pit_rhs_root_item(const PitArgs& a, int64_t inst, int lane) {
  const int n = a.nx, m = a.nu, N = a.N;
  PitWs v = views(a.ws, inst, N, n, m);
  if (lane < n) {
    double acc = 0.0;
    for (int q = 0; q < n; ++q) acc = fma(v.Di[lane + q * n], v.b[q], acc);
    a.s.x[inst * (int64_t)(N + 1) * n + lane] = acc;
  }
}

// KKT residual r = K[x; y] + [s; c] (as rr_residual), one warp per (instance, stage i):
// rows x_i, u_i, primal row i+1 (item i < N); rows x_N and primal row 0 (item N) -- stage-parallel,
// unlike rr_residual's lane group walking the horizon, so a single long instance is not serialised
__device__ void pit_residual_item(const PitArgs& a, const rr_residual_buf& rb, int64_t item, int lane) {
  const int n = a.nx, m = a.nu, N = a.N;
  const int64_t inst = item / (N + 1);
  const int i = (int)(item % (N + 1));
  const double d = a.p.delta[inst];
  const double* x = a.s.x + inst * (int64_t)(N + 1) * n;
  const double* y = a.s.y + inst * (int64_t)(N + 1) * n;
  const int sn = n * (n + 1) / 2, smm = m * (m + 1) / 2;
  if (i == N) {
    const int64_t iP = (a.shared & RR_FLAG_SHARED_COST) ? 0 : inst;
    if (lane < n) {
      double g = a.p.qN[inst * n + lane] - y[(int64_t)N * n + lane];
      for (int k = 0; k < n; ++k) g = fma(a.p.QN[iP * sn + pk(n, lane, k)], x[(int64_t)N * n + k], g);
      rb.qN[inst * n + lane] = g;
      rb.c0[inst * n + lane] = a.p.c0[inst * n + lane] - x[lane] - d * y[lane];
    }
    return;
  }
  const int64_t s = inst * N + i;
  const int64_t sD = dyn_blk(a.shared, inst, N, i);
  const int64_t sP = cost_blk(a.shared, inst, N, i);
  const double *A = a.p.A + sD * n * n, *B = a.p.B + sD * n * m;
  const double *Q = a.p.Q + sP * sn, *M = a.p.M + sP * n * m, *R = a.p.R + sP * smm;
  const double* xi = x + (int64_t)i * n;
  const double* x1 = xi + n;
  const double* yi = y + (int64_t)i * n;
  const double* y1 = yi + n;
  const double* u = a.s.u + s * m;
  if (lane < n) {  // stationarity x_i and primal row i+1, entry `lane`
    double g = a.p.q[s * n + lane] - yi[lane], pr = a.p.c[s * n + lane] - x1[lane] - d * y1[lane];
    for (int k = 0; k < n; ++k) {
      g = fma(Q[pk(n, lane, k)], xi[k], g);
      g = fma(A[k + lane * n], y1[k], g);
      pr = fma(A[lane + k * n], xi[k], pr);
    }
    for (int k = 0; k < m; ++k) {
      g = fma(M[lane + k * n], u[k], g);
      pr = fma(B[lane + k * n], u[k], pr);
    }
    rb.q[s * n + lane] = g;
    rb.c[s * n + lane] = pr;
  } else if (lane - 16 >= 0 && lane - 16 < m) {  // stationarity u_i
    const int w = lane - 16;
    double g = a.p.r[s * m + w];
    for (int k = 0; k < n; ++k) {
      g = fma(M[k + w * n], xi[k], g);
      g = fma(B[k + w * n], y1[k], g);
    }
    for (int k = 0; k < m; ++k) g = fma(R[pk(m, w, k)], u[k], g);
    rb.r[s * m + w] = g;
  }
}

__global__ void pit_axpy_kernel(double* __restrict__ y, const double* __restrict__ x, int64_t cnt) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < cnt) y[t] += x[t];
}

__global__ void pit_status_init(PitArgs a) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b < a.batch) a.status[b] = 0;
}

__global__ void pit_nanfill(PitArgs a) {  // NaN-fill the outputs of failed instances (thread per element)
  const int n = a.nx, m = a.nu;
  const int64_t N = a.N, per = (N + 1) * n * 2 + N * m;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.batch * per) return;
  const int64_t b = t / per, e = t % per;
  if (a.status[b] == 0) return;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  if (e < (N + 1) * n) a.s.x[b * (N + 1) * n + e] = nan;
  else if (e < 2 * (N + 1) * n) a.s.y[b * (N + 1) * n + e - (N + 1) * n] = nan;
  else a.s.u[b * N * m + e - 2 * (N + 1) * n] = nan;
}

// ---- one launch per step (any batch): warp per item ----
#define PIT_ITEM_PROLOGUE(count)                                   \
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;     \
  const int64_t item = (int64_t)blockIdx.x * WPB + warp;          \
  if (item >= (count)) return;
__global__ void __launch_bounds__(WPB * 32) pit_assemble_kernel(PitArgs a) {
  extern __shared__ __align__(16) double sm[];
  PIT_ITEM_PROLOGUE(a.batch * (int64_t)a.N)
  pit_assemble_item(a, item, sm + warp * 8 * TILE, lane);
}
__global__ void __launch_bounds__(WPB * 32) pit_diag_kernel(PitArgs a) {
  PIT_ITEM_PROLOGUE(a.batch * (int64_t)(a.N + 1))
  pit_diag_item(a, item, lane);
}
__global__ void __launch_bounds__(WPB * 32) pit_elim_kernel(PitArgs a, int s) {
  extern __shared__ __align__(16) double sm[];
  PIT_ITEM_PROLOGUE(a.batch * (int64_t)((a.N - s) / (2 * s) + 1))
  pit_elim_item(a, s, item, sm + warp * 4 * TILE, lane);
}
__global__ void __launch_bounds__(WPB * 32) pit_update_kernel(PitArgs a, int s) {
  extern __shared__ __align__(16) double sm[];
  PIT_ITEM_PROLOGUE(a.batch * (int64_t)(a.N / (2 * s) + 1))
  pit_update_item(a, s, item, sm + warp * 4 * TILE, lane);
}
__global__ void __launch_bounds__(WPB * 32) pit_root_kernel(PitArgs a) {
  extern __shared__ __align__(16) double sm[];
  PIT_ITEM_PROLOGUE(a.batch)
  pit_root_item(a, item, sm + warp * 4 * TILE, lane);
}
__global__ void __launch_bounds__(WPB * 32) pit_backsub_kernel(PitArgs a, int s) {
  PIT_ITEM_PROLOGUE(a.batch * (int64_t)((a.N - s) / (2 * s) + 1))
  pit_backsub_item(a, s, item, lane);
}
__global__ void __launch_bounds__(WPB * 32) pit_recover_kernel(PitArgs a) {
  PIT_ITEM_PROLOGUE(a.batch * (int64_t)(a.N + 1))
  pit_recover_item(a, item, lane);
}
__global__ void __launch_bounds__(WPB * 32) pit_rhs_assemble_kernel(PitArgs a) {
  PIT_ITEM_PROLOGUE(a.batch * (int64_t)a.N)
  pit_rhs_assemble_item(a, item, lane);
}
__global__ void __launch_bounds__(WPB * 32) pit_rhs_diag_kernel(PitArgs a) {
  PIT_ITEM_PROLOGUE(a.batch * (int64_t)(a.N + 1))
  pit_rhs_diag_item(a, item, lane);
}
__global__ void __launch_bounds__(WPB * 32) pit_rhs_elim_kernel(PitArgs a, int s) {
  PIT_ITEM_PROLOGUE(a.batch * (int64_t)((a.N - s) / (2 * s) + 1))
  pit_rhs_elim_item(a, s, item, lane);
}
__global__ void __launch_bounds__(WPB * 32) pit_rhs_update_kernel(PitArgs a, int s) {
  PIT_ITEM_PROLOGUE(a.batch * (int64_t)(a.N / (2 * s) + 1))
  pit_rhs_update_item(a, s, item, lane);
}
__global__ void __launch_bounds__(WPB * 32) pit_rhs_root_kernel(PitArgs a) {
  PIT_ITEM_PROLOGUE(a.batch)
  pit_rhs_root_item(a, item, lane);
}
__global__ void __launch_bounds__(WPB * 32) pit_residual_kernel(PitArgs a, rr_residual_buf rb) {
  PIT_ITEM_PROLOGUE(a.batch * (int64_t)(a.N + 1))
  pit_residual_item(a, rb, item, lane);
}
#undef PIT_ITEM_PROLOGUE

// ---- all steps in one cooperative launch: persistent warps, grid-wide barrier between steps ----
__global__ void __launch_bounds__(WPB * 32) pit_fused_kernel(PitArgs a, PitArgs c, rr_residual_buf rb, int levels) {
  extern __shared__ __align__(16) double sm[];
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * WPB + warp, nw = (int64_t)gridDim.x * WPB;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  double* T = sm + warp * 8 * TILE;
  const int64_t b = a.batch;
  const int N = a.N, n = a.nx, m = a.nu;
  auto items = [&](int64_t count, auto&& f) {  // warp-per-item map, then the grid barrier
    for (int64_t it = gw; it < count; it += nw) f(it);
    grid.sync();
  };
  for (int64_t t = gt; t < b; t += nt) a.status[t] = 0;
  grid.sync();
  if (N > 0) items(b * N, [&](int64_t it) { pit_assemble_item(a, it, T, lane); });
  items(b * (N + 1), [&](int64_t it) { pit_diag_item(a, it, lane); });
  for (int st = 1; st <= N; st *= 2) {
    items(b * ((N - st) / (2 * st) + 1), [&](int64_t it) { pit_elim_item(a, st, it, T, lane); });
    items(b * (N / (2 * st) + 1), [&](int64_t it) { pit_update_item(a, st, it, T, lane); });
  }
  items(b, [&](int64_t it) { pit_root_item(a, it, T, lane); });
  for (int l = levels - 1; l >= 0; --l) {
    const int st = 1 << l;
    items(b * ((N - st) / (2 * st) + 1), [&](int64_t it) { pit_backsub_item(a, st, it, lane); });
  }
  items(b * (N + 1), [&](int64_t it) { pit_recover_item(a, it, lane); });
  for (int r = 0; r < a.refine; ++r) {
    items(b * (N + 1), [&](int64_t it) { pit_residual_item(a, rb, it, lane); });
    if (N > 0) items(b * N, [&](int64_t it) { pit_rhs_assemble_item(c, it, lane); });
    items(b * (N + 1), [&](int64_t it) { pit_rhs_diag_item(c, it, lane); });
    for (int st = 1; st <= N; st *= 2) {
      items(b * ((N - st) / (2 * st) + 1), [&](int64_t it) { pit_rhs_elim_item(c, st, it, lane); });
      items(b * (N / (2 * st) + 1), [&](int64_t it) { pit_rhs_update_item(c, st, it, lane); });
    }
    items(b, [&](int64_t it) { pit_rhs_root_item(c, it, lane); });
    for (int l = levels - 1; l >= 0; --l) {
      const int st = 1 << l;
      items(b * ((N - st) / (2 * st) + 1), [&](int64_t it) { pit_backsub_item(c, st, it, lane); });
    }
    items(b * (N + 1), [&](int64_t it) { pit_recover_item(c, it, lane); });
    const int64_t nx1 = b * (N + 1) * n, nu1 = b * (int64_t)N * m;
    for (int64_t t = gt; t < nx1; t += nt) {
      a.s.x[t] += c.s.x[t];
      a.s.y[t] += c.s.y[t];
    }
    for (int64_t t = gt; t < nu1; t += nt) a.s.u[t] += c.s.u[t];
    grid.sync();
  }
  const int64_t per = (int64_t)(N + 1) * n * 2 + (int64_t)N * m;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  for (int64_t t = gt; t < b * per; t += nt) {  // NaN-fill the outputs of failed instances
    const int64_t bi = t / per, e = t % per;
    if (a.status[bi] == 0) continue;
    if (e < (N + 1) * n) a.s.x[bi * (N + 1) * n + e] = nan;
    else if (e < 2 * (N + 1) * n) a.s.y[bi * (N + 1) * n + e - (N + 1) * n] = nan;
    else a.s.u[bi * N * m + e - 2 * (N + 1) * n] = nan;
  }
}

unsigned blocks_for(int64_t items) { return (unsigned)((items + WPB - 1) / WPB); }

}  // namespace

int64_t pit_ws_bytes(int nx, int nu, int N, int64_t batch) {
  if (nx < 1 || nu < 1 || nx > NM || nu > NM || N < 0) return -1;
  // per-instance reduction + batch-wide residual (q, r, c, qN, c0) and correction (x, u, y) buffers
  const int64_t glob = (int64_t)N * (2 * nx + nu) + 2 * nx + (int64_t)(N + 1) * 2 * nx + (int64_t)N * nu;
  return batch * (pit_per(N, nx, nu) + glob) * 8 + 256;
}

// the correction system of the refinement step: right-hand side = the residual, solution → (cx, cu, cy)
static void pit_buffers(const PitArgs& a, rr_residual_buf& rb, PitArgs& c) {
  const int64_t b = a.batch;
  const int N = a.N, n = a.nx, m = a.nu;
  double* glob = a.ws + b * pit_per(N, n, m);
  rb = rr_residual_buf{glob, glob + b * N * n, glob + b * N * (n + m), glob + b * N * (2 * n + m),
                       glob + b * (N * (2 * n + m) + n)};
  double* cx = glob + b * (N * (2 * n + m) + 2 * n);
  double* cu = cx + b * (N + 1) * n;
  double* cy = cu + b * N * m;
  c = a;
  c.p.q = rb.q;
  c.p.r = rb.r;
  c.p.c = rb.c;
  c.p.qN = rb.qN;
  c.p.c0 = rb.c0;
  c.s = rr_solution{cx, cu, cy};
}

// One cooperative launch of every step (default); false if the device cannot run it co-resident.
static bool pit_fused_launch(const PitArgs& a, cudaStream_t s, cudaError_t* err) {
  const char* v = getenv("RR_PIT_STEPS");
  if (v != nullptr && v[0] == '1') return false;
  int dev = 0, coop = 0, nsm = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (!coop || nsm <= 0) return false;
  const size_t smb = sizeof(double) * WPB * 8 * TILE;
  if (cudaFuncSetAttribute(pit_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb) != cudaSuccess)
    return false;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pit_fused_kernel, WPB * 32, smb) != cudaSuccess ||
      per_sm <= 0)
    return false;
  // as many CTAs as the widest step has warps' worth of items, capped by co-residency.  Wide problems
  // keep the per-step launches: measured (bench --workload pit, batch 1) fused vs per-step launches
  // 0.38 vs 0.52 ms at N = 64, 0.53 vs 0.74 ms at N = 512, 1.05 vs 1.07 ms at N = 4096 (0.81 ms when
  // the per-step launches are replayed from a CUDA graph, where the fused kernel stays at 1.06 ms)
  const int64_t widest = a.batch * (int64_t)(a.N + 1);
  if (widest > 2048) return false;
  const int64_t want = (widest + WPB - 1) / WPB;
  const int64_t cap = (int64_t)per_sm * nsm;
  const unsigned grid = (unsigned)(want < cap ? want : cap);
  int levels = 0;
  for (int st = 1; st <= a.N; st *= 2) ++levels;
  rr_residual_buf rb;
  PitArgs c;
  pit_buffers(a, rb, c);
  PitArgs aa = a;
  void* args[] = {&aa, &c, &rb, &levels};
  *err = cudaLaunchCooperativeKernel((const void*)pit_fused_kernel, dim3(grid), dim3(WPB * 32), args, smb, s);
  return true;
}

cudaError_t pit_launch(const PitArgs& a, cudaStream_t s) {
  const int64_t b = a.batch;
  const int N = a.N;
  {
    cudaError_t e = cudaSuccess;
    if (b > 0 && pit_fused_launch(a, s, &e)) return e;
  }
  pit_status_init<<<(unsigned)((b + 255) / 256), 256, 0, s>>>(a);
  const size_t sm8 = sizeof(double) * WPB * 8 * TILE, sm4 = sizeof(double) * WPB * 4 * TILE;
  // per call (the attribute is per device; no global state in the library)
  cudaError_t ea = cudaFuncSetAttribute(pit_assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm8);
  if (ea != cudaSuccess) return ea;
  if (N > 0) pit_assemble_kernel<<<blocks_for(b * N), WPB * 32, sm8, s>>>(a);
  pit_diag_kernel<<<blocks_for(b * (N + 1)), WPB * 32, 0, s>>>(a);
  int levels = 0;
  for (int st = 1; st <= N; st *= 2) {
    pit_elim_kernel<<<blocks_for(b * ((N - st) / (2 * st) + 1)), WPB * 32, sm4, s>>>(a, st);
    pit_update_kernel<<<blocks_for(b * (N / (2 * st) + 1)), WPB * 32, sm4, s>>>(a, st);
    ++levels;
  }
  pit_root_kernel<<<blocks_for(b), WPB * 32, sm4, s>>>(a);
  for (int l = levels - 1; l >= 0; --l) {
    const int st = 1 << l;
    pit_backsub_kernel<<<blocks_for(b * ((N - st) / (2 * st) + 1)), WPB * 32, 0, s>>>(a, st);
  }
  pit_recover_kernel<<<blocks_for(b * (N + 1)), WPB * 32, 0, s>>>(a);
  // iterative refinement in FP64: residual of the caller's system (true δ), re-solve with the stored
  // reduction (δ_s = max(δ, delta_floor)): corrects the 1/δ_s conditioning of the δ-scaled state
  // system and, where the floor binds, the difference between the δ_s and the δ solutions
  const int n = a.nx, m = a.nu;
  rr_residual_buf rb;
  PitArgs c;
  pit_buffers(a, rb, c);
  double *cx = c.s.x, *cu = c.s.u, *cy = c.s.y;
  for (int it = 0; it < a.refine; ++it) {
    pit_residual_kernel<<<blocks_for(b * (N + 1)), WPB * 32, 0, s>>>(a, rb);
    if (N > 0) pit_rhs_assemble_kernel<<<blocks_for(b * N), WPB * 32, 0, s>>>(c);
    pit_rhs_diag_kernel<<<blocks_for(b * (N + 1)), WPB * 32, 0, s>>>(c);
    for (int st = 1; st <= N; st *= 2) {
      pit_rhs_elim_kernel<<<blocks_for(b * ((N - st) / (2 * st) + 1)), WPB * 32, 0, s>>>(c, st);
      pit_rhs_update_kernel<<<blocks_for(b * (N / (2 * st) + 1)), WPB * 32, 0, s>>>(c, st);
    }
    pit_rhs_root_kernel<<<blocks_for(b), WPB * 32, 0, s>>>(c);
    for (int l = levels - 1; l >= 0; --l) {
      const int st = 1 << l;
      pit_backsub_kernel<<<blocks_for(b * ((N - st) / (2 * st) + 1)), WPB * 32, 0, s>>>(c, st);
    }
    pit_recover_kernel<<<blocks_for(b * (N + 1)), WPB * 32, 0, s>>>(c);
    const int64_t nx1 = b * (N + 1) * n, nu1 = b * (int64_t)N * m;
    pit_axpy_kernel<<<(unsigned)((nx1 + 255) / 256), 256, 0, s>>>(a.s.x, cx, nx1);
    if (nu1 > 0) pit_axpy_kernel<<<(unsigned)((nu1 + 255) / 256), 256, 0, s>>>(a.s.u, cu, nu1);
    pit_axpy_kernel<<<(unsigned)((nx1 + 255) / 256), 256, 0, s>>>(a.s.y, cy, nx1);
  }
  const int64_t per = (int64_t)(N + 1) * a.nx * 2 + (int64_t)N * a.nu;
  pit_nanfill<<<(unsigned)((b * per + 255) / 256), 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace rrk
