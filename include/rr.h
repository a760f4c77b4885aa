/*
 * rr.h -- C-ABI of the B200 (sm_100a) batched regularized-Riccati / regularized-IPM library
 *         (paper_2509_16370_b200/librr_b200.so).
 *
 * Method: arXiv 2509.16370.  P:n = line n of the paper text.
 *
 * CONVENTIONS (all entry points)
 *  - Precision: IEEE FP64 throughout.
 *  - Memory: every pointer in the problem / factor / solution / workspace structs is a DEVICE
 *    pointer on the current CUDA device, allocated and owned by the caller.  The library never
 *    allocates on a call path and keeps no global mutable state; size-query functions
 *    give the workspace sizes.  Calls are asynchronous on the caller's stream and do not
 *    synchronise the host.  Calls on distinct streams/devices are independent.
 *  - Layout: one array per operand, instance-major [batch][stage][element] (terminal data
 *    [batch][element]); matrices COLUMN-MAJOR; symmetric matrices (Q, R, Q_N, V) PACKED LOWER
 *    in LAPACK 'L' packed order: element (r, c), r >= c, at c*(2n-c-1)/2 + r.
 *    Alignment: every array must be 8-byte aligned (FP64).  rr_factor_solve / rr_factor stream
    stage operands with TMA bulk copies (cp.async.bulk), which need 16-byte-aligned addresses:
    when all of A, B, Q, M, R, q, r, c are 16-byte aligned (e.g. fresh cudaMalloc / torch
    allocations) the TMA kernels run; otherwise n, m <= 16 shapes run the LDGSTS kernels (8-byte
    copies where needed; same results) and n or m > 16 returns RR_E_INVALID.  Workspaces and
    factor buffers must be 16-byte aligned (RR_E_INVALID otherwise).
 *  - Call-level errors (return value): RR_OK, RR_E_INVALID (bad dims, null required pointer,
 *    workspace too small), RR_E_UNSUPPORTED (shape outside the compiled kernels), RR_E_CUDA
 *    (launch error).  rr_last_error() returns a thread-local message.
 *  - Per-instance errors: int32 status[batch] (device), 0 = OK, else (code | stage << 8) with
 *    code RR_ST_*.  A failed instance's x, u, y are NaN-filled; other instances are unaffected.
 */
#ifndef RR_B200_H
#define RR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t rr_err;
#define RR_OK 0
#define RR_E_INVALID (-1)
#define RR_E_UNSUPPORTED (-2)
#define RR_E_CUDA (-3)

/* per-instance status codes (low byte); stage index in bits 8.. */
#define RR_ST_OK 0
#define RR_ST_G_NOT_PD 1     /* Cholesky/elimination pivot of G_i = BᵀWB + R not > 0 */
#define RR_ST_S_NOT_PD 2     /* pivot of S = I + δV_{i+1} not > 0; stage i       */
#define RR_ST_NONFINITE 3    /* non-finite output without a pivot failure                 */
#define RR_ST_NONPOS_SLACK 4 /* ipm_step: s <= 0 or z <= 0 on entry (P:53-59 needs log s)  */
#define RR_ST_LS_FAILED 5    /* ipm_step: no Armijo point within max_backtracks           */
#define RR_ST_MAXITER 6      /* ipm_solve: not converged within max_iters                */

/* rr_dims.flags: RR_FLAG_ACCUMULATE makes rr_solve ADD its solution to sol (x += Δx, u += Δu,
 * y += Δy) instead of overwriting it -- the update step of iterative refinement with rr_residual.
 * (ipm_step / ipm_solve have their own dims.) */
#define RR_FLAG_ACCUMULATE 1
/* Batch-shared operands (LTI / fleet MPC): with RR_FLAG_SHARED_DYN, A and B are ONE
 * [N][...] array used by every instance (no batch dimension); with RR_FLAG_SHARED_COST, Q, M, R
 * ([N][...]) and Q_N ([sym n]) are shared the same way.  Everything else stays per instance.
 * Accepted by rr_factor_solve (n, m <= 16 kernels), rr_factor, rr_solve, rr_residual and their size
 * queries; rr_factor_solve on the CTA kernels (n or m > 16) returns RR_E_UNSUPPORTED. */
#define RR_FLAG_SHARED_DYN 2
#define RR_FLAG_SHARED_COST 4
/* Stage-invariant operands (LTI MPC, A_i = A for every stage): with
 * RR_FLAG_STAGE_INVARIANT_DYN, A and B hold ONE stage block per instance ([batch][elems]; with
 * RR_FLAG_SHARED_DYN too, one block for everything: [elems]); RR_FLAG_STAGE_INVARIANT_COST does the
 * same for Q, M, R (Q_N is per instance or shared as before).  q, r, c stay per stage.  Accepted
 * wherever RR_FLAG_SHARED_* is (rr_factor_solve for n, m <= 16, rr_factor, rr_solve, rr_residual,
 * rr_factor_solve_pit, the host paths and the size queries). */
#define RR_FLAG_STAGE_INVARIANT_DYN 16
#define RR_FLAG_STAGE_INVARIANT_COST 32
/* FP32 factor record (the paper's low-precision factorization + residual callback,
 * P:664-666): rr_factor stores its records in FP32 (same layout and element offsets, record stride
 * rr_factor_bytes()/(batch*(N+1)*4) = the double count rounded up to a multiple of 4 floats) and
 * rr_solve reads them (arithmetic stays FP64).  The solution then carries the FP32 rounding of the
 * factor (~1e-7 relative times the conditioning); one or two rr_residual + rr_solve(ACCUMULATE)
 * refinement steps restore the FP64 result.  rr_factor_bytes, rr_factor, rr_solve and
 * rr_solve_workspace_bytes accept it; compiled for nx = 12, nu = 4 only (else RR_E_UNSUPPORTED /
 * -1) and the stage operands must be 16-byte aligned. */
#define RR_FLAG_FACTOR_FP32 8

typedef struct {
  int32_t nx;    /* state dimension n   (1 <= nx)            */
  int32_t nu;    /* control dimension m (1 <= nu)            */
  int32_t N;     /* horizon (number of stages, N >= 0)       */
  int32_t flags; /* RR_FLAG_* (0 = all operands per instance)  */
  int64_t batch; /* number of independent instances (>= 0)  */
} rr_dims;

/*
 * Regularized LQR problem (§1.4): the linear system
 *     [P  Cᵀ; C  -δI] [x; y] = -[s; c]
 * with P = blkdiag(P_0..P_{N-1}, Q_N), P_i = [[Q_i, M_i], [M_iᵀ, R_i]] (P_i PSD, R_i PD),
 * C the banded dynamics Jacobian with block rows -x_0 and A_i x_i + B_i u_i - x_{i+1},
 * s = (q_0, r_0, ..., q_N), c = (c_0, ..., c_N) (N+1 blocks, reading R1), δ >= 0.
 */
typedef struct {
  const double* A;     /* [batch][N][n*n]      A_i, column-major                    */
  const double* B;     /* [batch][N][n*m]      B_i, column-major                    */
  const double* Q;     /* [batch][N][n(n+1)/2] Q_i, packed lower                    */
  const double* M;     /* [batch][N][n*m]      M_i, column-major                    */
  const double* R;     /* [batch][N][m(m+1)/2] R_i, packed lower                    */
  const double* q;     /* [batch][N][n]        q_i                                  */
  const double* r;     /* [batch][N][m]        r_i                                  */
  const double* c;     /* [batch][N][n]        c[i] = c_{i+1}, residual of the row producing x_{i+1} */
  const double* QN;    /* [batch][n(n+1)/2]    Q_N, packed lower                    */
  const double* qN;    /* [batch][n]           q_N                                  */
  const double* c0;    /* [batch][n]           c_0 (initial-state row, Jacobian -I) */
  const double* delta; /* [batch]              δ >= 0 (δ = 0: classic LQR)   */
} rr_problem;

/* Policy of Eq.(RR).  Any pointer may be NULL (not written). */
typedef struct {
  double* V; /* [batch][N+1][n(n+1)/2] V_i packed lower, V_N = Q_N */
  double* v; /* [batch][N+1][n]        v_i, v_N = q_N               */
  double* K; /* [batch][N][m*n]        K_i column-major (m×n)       */
  double* k; /* [batch][N][m]          k_i                          */
} rr_factor_buf;

/* Solution: x = (x_0..x_N), u = (u_0..u_{N-1}), y = (y_0..y_N). */
typedef struct {
  double* x; /* [batch][N+1][n] */
  double* u; /* [batch][N][m]   */
  double* y; /* [batch][N+1][n] */
} rr_solution;

/* Bytes of device workspace rr_factor_solve needs for `dims` (>= 0), or -1 if unsupported. */
int64_t rr_workspace_bytes(const rr_dims* dims);

/*
 * rr_factor_solve: the fused hot path, rows a2-a5 of DESIGN.md §1:
 *   backward sweep i = N-1..0 of Eq.(RR):
 *     W_i = (I+δV_{i+1})⁻¹V_{i+1}; G_i = BᵀWB + R; g_i = v_{i+1} + W(c_{i+1} - δv_{i+1});
 *     H_i = BᵀWA + Mᵀ; h_i = r + Bᵀg; K_i = -G⁻¹H; k_i = -G⁻¹h;
 *     V_i = AᵀWA + Q + KᵀH; v_i = q + Aᵀg + Kᵀh           (V_N = Q_N, v_N = q_N)
 *   forward sweep: x_0 = (I+δV_0)⁻¹(c_0 - δv_0); u_i = K_i x_i + k_i;
 *     x_{i+1} = (I+δV_{i+1})⁻¹(A_i x_i + B_i u_i + c_{i+1} - δv_{i+1});
 *   dual recovery: y_i = V_i x_i + v_i.
 * prob, sol, status: required (status may be NULL when batch == 0: the call is then a no-op).  fac: optional (NULL or any NULL member = not written).
 * workspace: device buffer of >= rr_workspace_bytes(dims) bytes, 16-byte aligned (256 recommended);
 * contents are scratch.  Operand alignment selects the kernel (CONVENTIONS above).  Asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream).
 */
rr_err rr_factor_solve(const rr_dims* dims, const rr_problem* prob, const rr_factor_buf* fac,
                       const rr_solution* sol, void* workspace, int64_t workspace_bytes,
                       int32_t* status, void* stream);

/*
 * rr_factor_solve_host: the same computation with HOST buffers (the end-to-end path).
 * prob_host / sol_host / status_host: host pointers (pinned memory makes the copies
 * asynchronous); prob_dev / sol_dev / status_dev: caller-owned device staging buffers of the
 * same shapes (rr_problem's members are written through a cast: they must be writable device
 * memory).  Enqueues on `stream`: H2D copy of every problem operand, rr_factor_solve, D2H copy
 * of x, u, y and status.  The caller synchronises `stream` before reading sol_host.
 */
rr_err rr_factor_solve_host(const rr_dims* dims, const rr_problem* prob_host, const rr_solution* sol_host,
                            int32_t* status_host, const rr_problem* prob_dev, const rr_solution* sol_dev,
                            int32_t* status_dev, void* workspace, int64_t workspace_bytes, void* stream);

/*
 * rr_factor_solve_host_pipelined: rr_factor_solve_host with the copies overlapped with the solve.
 * The batch is cut into `nchunks` contiguous instance ranges; chunk c runs on streams[c % nstreams]:
 * H2D of its slices of every per-instance operand, rr_factor_solve on them, D2H of its x, u, y and
 * status -- so the H2D of one chunk, the solve of another and the D2H of a third proceed together on
 * the two copy engines and the SMs (the whole-batch version serialises them on one stream).
 * Batch-shared operands (RR_FLAG_SHARED_*) are copied once on streams[0] first.  streams[0] is the
 * completion stream: the other streams wait for it on entry and it waits for them on exit, so
 * synchronising streams[0] completes the call.  workspace: >= sum over the chunks of
 * rr_workspace_bytes(chunk dims) rounded up to 256 B each, 256-byte aligned (per-chunk slices: chunks
 * on different streams run concurrently).  Results are bitwise those of rr_factor_solve_host.
 */
rr_err rr_factor_solve_host_pipelined(const rr_dims* dims, const rr_problem* prob_host, const rr_solution* sol_host,
                                      int32_t* status_host, const rr_problem* prob_dev, const rr_solution* sol_dev,
                                      int32_t* status_dev, void* workspace, int64_t workspace_bytes, int32_t nchunks,
                                      void* const* streams, int32_t nstreams);

/* ============================ factorization / solve split (rows a2 | a3-a5) ============================
 * The paper's solver plugs problem-specific "KKT system factorization" and "KKT system solve"
 * callbacks into a shared backend.  rr_factor is the matrix half of Eq.(RR),
 * which depends only on (A, B, Q, M, R, Q_N, δ); rr_solve is the vector half plus the forward sweep
 * and dual recovery for one right-hand side (q, r, c, q_N, c_0).  One rr_factor serves any number of
 * rr_solve calls with different right-hand sides (iterative refinement, corrector steps).
 *
 * FACTOR RECORD (device memory written by rr_factor, read by rr_solve; [batch][N+1][R] doubles,
 * R = rr_factor_record_doubles(n, m) = n(n+1) + nm + m(m+1)/2 rounded up to even).  Record i:
 *     [0, s)            V_i                 packed lower (s = n(n+1)/2; V_N = Q_N)
 *     [s, 2s)           S_i⁻¹ = (I + δV_i)⁻¹  packed lower (the (I+δV)⁻¹ of P:616)
 *     [2s, 2s+nm)       K_i                 m×n column-major   (record N: unused)
 *     [2s+nm, +m(m+1)/2) G_i⁻¹ = (BᵀW_iB + R_i)⁻¹ packed lower (record N: unused)
 * An instance whose factorization failed (status != 0) has its records NaN-filled.
 */
int32_t rr_factor_record_doubles(int32_t n, int32_t m);

/* Bytes of the factor record array for `dims` (batch * (N+1) * R * 8; with RR_FLAG_FACTOR_FP32
 * batch * (N+1) * R32 * 4, R32 = R rounded up to a multiple of 4), or -1 if no kernel covers
 * (nx, nu) (rr_factor / rr_solve are compiled for nx, nu <= 16; FP32 records for 12 x 4). */
int64_t rr_factor_bytes(const rr_dims* dims);

/*
 * rr_factor: backward matrix sweep i = N-1..0 (row a2), V_N = Q_N:
 *     S_{i+1}⁻¹ = (I + δV_{i+1})⁻¹; W_i = S⁻¹V_{i+1}; G_i = BᵀWB + R; H_i = BᵀWA + Mᵀ;
 *     K_i = −G_i⁻¹H_i; V_i = AᵀWA + Q + K_iᵀH_i;   then S_0⁻¹ = (I + δV_0)⁻¹.
 * prob: A, B, Q, M, R, QN, delta are read (q, r, c, qN, c0 ignored, may be NULL).
 * factor: device buffer of >= rr_factor_bytes(dims) bytes, 16-byte aligned (output, layout above).
 * fac: optional (NULL or NULL members): V [batch][N+1][sym n] and K [batch][N][m*n] copies.
 * status: [batch] device int32 (RR_ST_S_NOT_PD / RR_ST_G_NOT_PD | stage << 8, as rr_factor_solve).
 */
rr_err rr_factor(const rr_dims* dims, const rr_problem* prob, void* factor, int64_t factor_bytes,
                 const rr_factor_buf* fac, int32_t* status, void* stream);

/* Bytes of device scratch rr_solve needs (batch * N * (n+m) * 8 + 256), or -1 if unsupported. */
int64_t rr_solve_workspace_bytes(const rr_dims* dims);

/*
 * rr_solve: rows a3-a5 for the right-hand side (q, r, c, q_N, c_0) of prob, given rr_factor's records:
 *   backward vector sweep: g_i = v_{i+1} + W_i(c_{i+1} − δv_{i+1}) (evaluated as
 *     S_{i+1}⁻¹(v_{i+1} + V_{i+1}c_{i+1}), the same quantity since S⁻¹ = I − δW), h_i = r + Bᵀg,
 *     k_i = −G_i⁻¹h_i, v_i = q + Aᵀg + K_iᵀh_i  (v_N = q_N);
 *   forward sweep: x_0 = S_0⁻¹(c_0 − δv_0), u_i = K_i x_i + k_i,
 *     x_{i+1} = S_{i+1}⁻¹(A_i x_i + B_i u_i + c_{i+1} − δv_{i+1});  duals y_i = V_i x_i + v_i.
 * prob: A, B, q, r, c, qN, c0, delta are read (Q, M, R, QN ignored: the factor carries them).
 *   A, B and delta must be the ones the factor was computed with.
 * fac: optional v [batch][N+1][n] and k [batch][N][m] copies (V, K members ignored).
 * status: [batch] device int32, 0 or RR_ST_NONFINITE (e.g. the instance's factor failed: see
 *   rr_factor's status for the reason); outputs of a non-finite instance are NaN-filled.
 * dims->flags: 0 (sol = solution) or RR_FLAG_ACCUMULATE (sol += solution; see rr_residual).
 */
rr_err rr_solve(const rr_dims* dims, const rr_problem* prob, const void* factor, int64_t factor_bytes,
                const rr_factor_buf* fac, const rr_solution* sol, void* workspace, int64_t workspace_bytes,
                int32_t* status, void* stream);

/* ======================== parallel-in-time solve (the paper's future work) ========================
 * rr_factor_solve_pit: the same solution (x, u, y) as rr_factor_solve, computed with O(log N) depth
 * instead of N sequential stages -- for few instances with long horizons (latency).  For δ_s > 0 the
 * regularized system is equivalent to (δ_s P + CᵀC) z = −(δ_s s + Cᵀc), y = (Cz + c)/δ_s:
 * the controls are eliminated stage by stage (Schur complement on δ_s R_i + B_iᵀB_i), the remaining
 * block-tridiagonal SPD system in x_0..x_N is solved by block cyclic reduction (⌈log2(N+1)⌉ levels),
 * then u_i follows per stage and y from the dual identity.  The reduction is built at
 * δ_s = max(δ, 1e-4) and followed by 2 steps of FP64 iterative refinement on the caller's system
 * (residual at the caller's δ, correction with the stored reduction), which converges to the
 * solution at δ for every δ >= 0 -- classic LQR (δ = 0) included -- as long as the contraction
 * δ_s-vs-δ is small (measured 1e-8 -> 1e-12 -> 1e-16 at δ = 0 on C2- and C4-shaped data).
 * nx, nu <= 16; RR_FLAG_SHARED_* accepted.  status: 0, RR_ST_G_NOT_PD | stage << 8,
 * RR_ST_S_NOT_PD | index << 8 (a non-positive pivot of the reduced system), RR_ST_NONFINITE.
 * workspace: >= rr_pit_workspace_bytes(dims) device bytes.
 */
int64_t rr_pit_workspace_bytes(const rr_dims* dims);
rr_err rr_factor_solve_pit(const rr_dims* dims, const rr_problem* prob, const rr_solution* sol, void* workspace,
                           int64_t workspace_bytes, int32_t* status, void* stream);

/* ================================ KKT residual (the paper's third callback) ================================
 * rr_residual: r = K [x; y] + [s; c] for the §1.4 system K [x; y] = −[s; c], i.e. the
 * paper's "KKT system residual computation callback", block by block:
 *   stationarity  x_i: Q_i x_i + M_i u_i + q_i − y_i + A_iᵀ y_{i+1}      (i < N)
 *                 u_i: M_iᵀ x_i + R_i u_i + r_i + B_iᵀ y_{i+1}
 *                 x_N: Q_N x_N + q_N − y_N
 *   primal   row 0:    −x_0 − δ y_0 + c_0
 *            row i+1:  A_i x_i + B_i u_i − x_{i+1} − δ y_{i+1} + c_{i+1}
 * The blocks are written into the right-hand-side slots of an rr_problem (q, r, c, q_N, c_0 layouts),
 * so {A, B, delta, res} is directly the right-hand side of the correction system: rr_solve on it with
 * RR_FLAG_ACCUMULATE performs one step of iterative refinement (x, u, y) += K⁻¹(−r).
 * res: optional (NULL or NULL members: not written).  norms: optional device [batch][2] =
 * (max |stationarity|, max |primal|) per instance (NaN if any residual entry is non-finite).
 * prob: every operand read.  sol: x, u, y read.  Same shape support as rr_factor.
 */
typedef struct {
  double* q;  /* [batch][N][n]  stationarity rows x_i  */
  double* r;  /* [batch][N][m]  stationarity rows u_i  */
  double* c;  /* [batch][N][n]  primal rows i+1        */
  double* qN; /* [batch][n]     stationarity rows x_N  */
  double* c0; /* [batch][n]     primal row 0           */
} rr_residual_buf;

rr_err rr_residual(const rr_dims* dims, const rr_problem* prob, const rr_solution* sol, const rr_residual_buf* res,
                   double* norms, void* stream);

/* ================================ regularized IPM step (rows a1-a8) ================================
 * One iteration of the regularized interior point method of §1.2 on the stagewise OCP of
 * §1.1, per instance, with the Newton system solved stagewise (§1.3):
 *   a1 condense: Σ = (S Z⁻¹ + I/η)⁻¹ (W = Z⁻¹S), r_z = g + μ Z⁻¹e,
 *      P̃_i = P_i + G_iᵀΣG_i + η C_eᵀC_e,  s̃_i = ∇ₓℒ + G_iᵀΣ r_z + η C_eᵀ c_e,
 *      c_0 = s_0 − x̄_0, c_{i+1} = d_i(x̄_i, ū_i) − x̄_{i+1}, δ = 1/η;
 *   a2-a5 regularized Riccati solve of the condensed problem (Δx, Δu, Δy = LQR y; reading R8);
 *   a6 expand: Δz = Σ(GΔ + r_z), Δλ = η(C_eΔ + c_e), Δs = −Z⁻¹SΔz + μZ⁻¹e − s;
 *   a7 merit 𝒜 and D = ∇ₓ𝒜·Δx + ∇ₛ𝒜·Δs (Theorem);
 *   a8 α_max = min(1, min τs/(−Δs)); largest α = α_max βᵏ (k ≤ max_backtracks) with
 *      𝒜(x̄+αΔx, s+αΔs) ≤ 𝒜(x̄, s) + c₁ α D (reading R12); α_d = min(1, min τz/(−Δz));
 *      update x, u, s, y, λ with α, z with α_d (in place).
 * Trial merit values use the built-in model `model` (reading R19): IPM_MODEL_LQ (dynamics,
 * constraints linear: trial values exact from the linearisation), IPM_MODEL_CARTPOLE (n = 4, m = 1;
 * dynamics x⁺ = cartpole(x, u; model_params = [dt, m_c, m_p, l, g]) evaluated at trial points) or
 * IPM_MODEL_QUADROTOR (n = 12, m = 4; x⁺ = x + dt f(x, u) with f the SURVEY §8(d) C5 quadrotor:
 * x = (p, ZYX Euler angles φ θ ψ, world velocity, body rates), u = (thrust, 3 torques),
 * model_params = [dt, mass, J_x, J_y, J_z, g]).  Costs are quadratic with Hessian P for all three,
 * so f(x̄ + αΔ) = f̄ + α∇fᵀΔ + ½α²ΔᵀPΔ exactly.
 */
#define IPM_MODEL_LQ 0
#define IPM_MODEL_CARTPOLE 1
#define IPM_MODEL_QUADROTOR 2

typedef struct {
  int32_t nx, nu, N;
  int32_t ng;    /* inequalities per stage i < N        */
  int32_t ngN;   /* terminal inequalities (on x_N)      */
  int32_t nc;    /* stage equalities per stage i < N    */
  int32_t ncN;   /* terminal equalities                 */
  int32_t model; /* IPM_MODEL_*                         */
  int64_t batch;
} ipm_dims;

/* Problem data evaluated at the current iterate.  Device pointers. Matrices column-major,
 * symmetric packed lower; "w" = n+m (stage i < N) — Jacobian rows are over (x_i, u_i). */
typedef struct {
  const double* s0;           /* [b][n]         fixed initial state                       */
  const double* fval;         /* [b]            f(x̄) (for the merit)                             */
  const double* gradf;        /* [b][N][w]      ∇_{x_i,u_i} f                                    */
  const double* gradfN;       /* [b][n]         ∇_{x_N} f                                        */
  const double *Q, *M, *R;    /* [b][N][sym n], [b][N][n*m], [b][N][sym m]: P_i (PD approx) */
  const double* QN;           /* [b][sym n]                                                       */
  const double *A, *B;        /* [b][N][n*n], [b][N][n*m]: ∂d_i/∂x, ∂d_i/∂u at the iterate      */
  const double* dres;         /* [b][N][n]      d_i(x̄_i, ū_i) − x̄_{i+1}                          */
  const double *ce, *Ce;      /* [b][N][nc], [b][N][nc*w]   stage equalities c_i = 0 and Jacobian */
  const double *ceN, *CeN;    /* [b][ncN], [b][ncN*n]                                             */
  const double *gv, *Gj;      /* [b][N][ng], [b][N][ng*w]   stage inequalities g_i ≤ 0, Jacobian  */
  const double *gvN, *GjN;    /* [b][ngN], [b][ngN*n]                                             */
  const double* model_params; /* [8] shared by the batch (cart-pole: dt, m_c, m_p, l, g;           */
                              /*     quadrotor: dt, mass, J_x, J_y, J_z, g)                       */
} ipm_stage_data;

/* Iterate (updated in place on success). */
typedef struct {
  double *x, *u;        /* [b][N+1][n], [b][N][m]                           */
  double *s, *z;        /* [b][N][ng] slacks / inequality duals (> 0)       */
  double *sN, *zN;      /* [b][ngN]                                         */
  double* y;            /* [b][N+1][n] initial-state + dynamics multipliers */
  double *lam, *lamN;   /* [b][N][nc], [b][ncN] stage-equality multipliers  */
  const double *mu, *eta; /* [b] barrier and penalty parameters (δ = 1/η)   */
} ipm_iterate;

typedef struct {
  double tau;      /* fraction to boundary, e.g. 0.995 */
  double armijo_c; /* c₁, e.g. 1e-4                    */
  double beta;     /* backtracking factor, e.g. 0.5    */
  int32_t max_backtracks; /* e.g. 50                   */
  int32_t pad;
} ipm_params;

/* Outputs (device).  Direction arrays have the iterate's shapes. */
typedef struct {
  double *dx, *du, *ds, *dsN, *dy, *dlam, *dlamN, *dz, *dzN;
  double* alpha_p;       /* [b] accepted primal step (0 on failure)   */
  double* alpha_d;       /* [b] dual step for z                        */
  double* D;             /* [b] directional derivative ∇𝒜·(Δx, Δs)    */
  double* merit0;        /* [b] 𝒜 at the iterate                       */
  double* merit_acc;     /* [b] 𝒜 at the accepted point               */
  int32_t* n_backtracks; /* [b] k of the accepted α = α_max βᵏ         */
} ipm_result;

/* Bytes of device workspace ipm_step needs (-1 if no kernel covers the dims). */
int64_t ipm_workspace_bytes(const ipm_dims* dims);

/* One batched regularized-IPM step (rows a1-a8).  status: [b] (may be NULL when b == 0: no-op) (RR_ST_NONPOS_SLACK: s or z not > 0
 * on entry -> iterate untouched, direction NaN; RR_ST_LS_FAILED: no Armijo point -> iterate
 * untouched, alpha_p = 0; pivot failures as in rr_factor_solve). */
rr_err ipm_step(const ipm_dims* dims, const ipm_stage_data* data, const ipm_iterate* it,
                const ipm_params* params, const ipm_result* res, void* workspace, int64_t workspace_bytes,
                int32_t* status, void* stream);

/* ======================= caller-evaluated line search (user models) =======================
 * For models other than the built-in ones, the step is split in three calls:
 *   ipm_direction: rows a1-a7 of ipm_step (same arguments): the direction (res->dx..dzN), D, 𝒜(0)
 *     (merit0), the fraction-to-boundary caps α_max (alpha_p) and α_d (alpha_d); no line search, the
 *     iterate is not modified.
 *   ipm_merit: 𝒜(α) = f − μΣlog(s+αΔs) + yᵀc + λᵀc_e + zᵀ(g+s+αΔs) + η/2(‖c‖² + ‖c_e‖² + ‖g+s+αΔs‖²)
 *     (reading R14) at the trial point, from the caller's model values there (ipm_trial_values,
 *     layouts of ipm_stage_data: f, d_i(trial) − x_{i+1}(trial), c_e, g); c_0 = s_0 − (x_0 + αΔx_0) and the
 *     trial slacks are formed inside.  alpha, merit: [b] device arrays; NaN if a trial slack is <= 0.
 *   ipm_update: x, u, s, y, λ += α_p Δ; z += α_d Δz (reading R12) for the caller's accepted α_p, α_d
 *     ([b] device arrays; 0 leaves an instance untouched).
 */
typedef struct {
  const double* fval;             /* [b]            f at the trial point               */
  const double* dres;             /* [b][N][n]      d_i(x_i, u_i) − x_{i+1} at the trial */
  const double *ce, *ceN;         /* [b][N][nc], [b][ncN]                              */
  const double *gv, *gvN;         /* [b][N][ng], [b][ngN]                              */
} ipm_trial_values;

rr_err ipm_direction(const ipm_dims* dims, const ipm_stage_data* data, const ipm_iterate* it,
                     const ipm_params* params, const ipm_result* res, void* workspace, int64_t workspace_bytes,
                     int32_t* status, void* stream);
rr_err ipm_merit(const ipm_dims* dims, const ipm_stage_data* data, const ipm_iterate* it, const ipm_result* res,
                 const double* alpha, const ipm_trial_values* trial, double* merit, void* stream);
rr_err ipm_update(const ipm_dims* dims, const ipm_iterate* it, const ipm_result* res, const double* alpha_p,
                  const double* alpha_d, void* stream);

/* ================================ batched IPM solve ================================
 * ipm_solve: repeated ipm_step on every instance until its KKT residual meets the tolerance.  The
 * paper fixes the step but not the outer loop; the loop is SPEC's ipm_solve /
 * update_parameters (reading R21).  At iteration k, for every running instance:
 *   evaluate the problem data at the iterate: costs quadratic with Hessian P and constraints linear
 *     (exact from `data`, the evaluation at the INITIAL iterate, which serves as the model reference);
 *     dynamics linear (IPM_MODEL_LQ) or the cart-pole / quadrotor model with analytic Jacobians;
 *   residuals r_stat = ||∇ₓL||∞ (∇ₓL = ∇f + Cᵀy + C_eᵀλ + Gᵀz), r_feas = max(||c||∞, ||c_e||∞, ||g+s||∞),
 *     r_comp = ||Sz − μe||∞, r_comp0 = ||Sz||∞;
 *   converged (status 0) if max(r_stat, r_feas, r_comp0) <= tol_kkt and μ <= 10 mu_min;
 *   RR_ST_MAXITER if k == max_iters;
 *   μ <- max(mu_min, min(kappa_mu μ, μ^theta_mu)) if max(r_stat, r_feas, r_comp) <= kappa μ;
 *   η <- min(eta_max, kappa_eta η) if k >= 5, r_feas > tol_kkt and r_feas > 0.9 r_feas(k−5);
 *   one ipm_step (rows a1-a8) with (μ, η, δ = 1/η); a failed step ends the instance with its status
 *     (settings->linear_merit: the step's trial merits use the linearised dynamics, reading R22).
 * Converged instances are masked out of later iterations (no host synchronisation: the step
 * kernel runs over a device-built list of running instances).
 * it: the iterate, updated in place (it->mu / it->eta are the initial values and are NOT written:
 * the final μ, η are in the report).  report: any member may be NULL.
 * workspace: >= ipm_solve_workspace_bytes(dims) device bytes, 256-byte aligned.
 */
typedef struct {
  double mu_min;      /* 1e-9  */
  double kappa;       /* 10    barrier-subproblem tolerance factor */
  double kappa_mu;    /* 0.2   */
  double theta_mu;    /* 1.5   */
  double eta_max;     /* 1e8   */
  double kappa_eta;   /* 10    */
  double tol_kkt;     /* 1e-6  */
  int32_t max_iters;  /* 100   */
  int32_t linear_merit; /* 0: each step's trial merits through the model (ipm_step as is); 1: through
                           the linearisation at the iterate, i.e. the step's line search runs with
                           IPM_MODEL_LQ on the re-evaluated Jacobians (SQP-style globalisation of the
                           outer loop; reading R22 -- converges the C4 swing-up)        */
  ipm_params step;    /* line search of each step (tau, armijo_c, beta, max_backtracks) */
} ipm_solve_settings;

typedef struct {
  int32_t* status;  /* [b] 0 converged, RR_ST_MAXITER, RR_ST_LS_FAILED, RR_ST_NONPOS_SLACK, pivot codes */
  int32_t* iters;   /* [b] IPM steps taken                                                          */
  double *mu, *eta; /* [b] final barrier / penalty parameters                                       */
  double *r_stat, *r_feas, *r_comp; /* [b] residuals at the last evaluated iterate (r_comp = ||Sz||∞) */
} ipm_solve_report;

int64_t ipm_solve_workspace_bytes(const ipm_dims* dims);

rr_err ipm_solve(const ipm_dims* dims, const ipm_stage_data* data, const ipm_iterate* it,
                 const ipm_solve_settings* settings, const ipm_solve_report* report, void* workspace,
                 int64_t workspace_bytes, void* stream);

/* Human-readable message of the last call-level error on this host thread. */
const char* rr_last_error(void);

/* Library version string and build target (e.g. "rr_b200 0.1 sm_100a"). */
const char* rr_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RR_B200_H */
