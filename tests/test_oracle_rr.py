"""Pins of the regularized-LQR oracle (T1 dense definition, T2 literal recursion) to things
other than themselves: closed forms, a textbook reformulation, scipy's DARE, invariants of
the paper, and tiny worked examples (DESIGN.md §3 "Pins").  CPU only."""
import ctypes
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg
import torch

import oracle
import synth
from oracle.dense import assemble_reglqr, instance_blocks

HERE = os.path.dirname(os.path.abspath(__file__))


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def scalar_problem(delta, N=0, QN=2.0, qN=1.0, c0=3.0):
    """N = 0, nx = nu = 1 instance of S:132/S:141-151."""
    z = lambda *s: torch.zeros(*s, dtype=torch.float64)
    return synth.RRProblem(1, 1, N, A=z(1, N, 1), B=z(1, N, 1), Q=z(1, N, 1), M=z(1, N, 1),
                           R=torch.ones(1, N, 1, dtype=torch.float64), q=z(1, N, 1), r=z(1, N, 1),
                           c=z(1, N, 1), QN=torch.tensor([[QN]], dtype=torch.float64),
                           qN=torch.tensor([[qN]], dtype=torch.float64),
                           c0=torch.tensor([[c0]], dtype=torch.float64),
                           delta=torch.tensor([delta], dtype=torch.float64))


# ---------------------------------------------------------------- dense_core examples
def test_chol_spec_examples():
    lib = oracle.load_oracle()
    f = lib.orc_chol
    f.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    S = np.array([[4.0, 2.0], [2.0, 3.0]], order="F")
    L = np.zeros((2, 2), order="F")
    assert f(2, S.ctypes.data, L.ctypes.data) == 0
    assert np.allclose(L, [[2, 0], [1, math.sqrt(2)]], atol=1e-15, rtol=0)
    S2 = np.array([[1.0, 2.0], [2.0, 1.0]], order="F")
    assert f(2, S2.ctypes.data, L.ctypes.data) == 1                             # S:53 not PD
    g = lib.orc_chol_solve
    g.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    f(2, S.ctypes.data, L.ctypes.data)
    b = np.array([6.0, 5.0])
    g(2, L.ctypes.data, b.ctypes.data)
    assert np.allclose(b, [1, 1], atol=1e-15)


# ---------------------------------------------------------------- SPEC scalar closed forms
@pytest.mark.parametrize("delta,x0,y0", [(0.0, 3.0, 7.0), (1.0, 2.0 / 3.0, 7.0 / 3.0)])
def test_scalar_closed_forms(delta, x0, y0):
    """x0 = (c0 - δ qN)/(1 + δ QN), y0 = QN x0 + qN, and y0 = (c0 - x0)/δ."""
    p = scalar_problem(delta)
    t2 = oracle.rr_solve_t2(p, want_policy=True)
    assert t2["status"][0] == 0
    assert abs(t2["x"][0, 0, 0] - x0) <= 1e-15 * 3
    assert abs(t2["y"][0, 0, 0] - y0) <= 1e-15 * 7
    assert abs(t2["V"][0, 0, 0] - 2.0) == 0 and abs(t2["v"][0, 0, 0] - 1.0) == 0
    t1 = oracle.rr_solve_dense(p)
    assert abs(t1["x"][0, 0] - x0) <= 1e-15 * 3 and abs(t1["y"][0, 0] - y0) <= 1e-15 * 7
    K, rhs, _ = assemble_reglqr(instance_blocks(p, 0))
    if delta == 1.0:
        # S:391 prints rhs = [-1, 3]; the definition rhs = -[s; c] gives
        # [-1, -3], and only that rhs reproduces S:400's x0 = 2/3, y0 = 7/3 (reading R18).
        assert np.array_equal(K, [[2.0, -1.0], [-1.0, -1.0]]) and np.array_equal(rhs, [-1.0, -3.0])


def test_zero_rhs_zero_solution():
    p = synth.random_stable_lqr(3, 2, 4, 2, seed=5)
    for f in ("q", "r", "c", "qN", "c0"):
        getattr(p, f).zero_()
    t2 = oracle.rr_solve_t2(p)
    assert np.all(t2["x"] == 0) and np.all(t2["u"] == 0) and np.all(t2["y"] == 0)


# ---------------------------------------------------------------- textbook reformulation pin
def condensed_augmented_qp(blk):
    """Independent route (DESIGN.md pin P-TEXTBOOK): the §1.4 system is the optimality condition of
    min ½ zᵀPz + sᵀz + ‖Cz + c‖²/(2δ).  Introduce slack controls w with x_0 = c_0 + w_{-1},
    x_{i+1} = A_i x_i + B_i u_i + c_{i+1} + w_i (so Cz + c = -w), eliminate the states by
    single shooting (x affine in the decisions ξ = (w_{-1}, u_0, w_0, ...)), and minimise the
    resulting unconstrained QP ½ξᵀHξ + gᵀξ with a dense solve.  Then y = (Cz+c)/δ = -w/δ.
    For δ = 0 the w's are absent (classic LQR)."""
    n, m, N, d = blk["n"], blk["m"], blk["N"], blk["delta"]
    use_w = d > 0
    nd = (n if use_w else 0) + N * (m + (n if use_w else 0))
    # x_i = Fx[i] ξ + fx[i];  u_i = Fu[i] ξ
    off = 0
    Fx, fx, Fu, Fw = [], [], [], []
    F0 = np.zeros((n, nd))
    if use_w:
        F0[:, off:off + n] = np.eye(n)
        Fw.append(F0.copy())
        off += n
    Fx.append(F0)
    fx.append(blk["c0"].copy())
    for i in range(N):
        Ui = np.zeros((m, nd)); Ui[:, off:off + m] = np.eye(m); off += m
        Fu.append(Ui)
        Xn = blk["A"][i] @ Fx[i] + blk["B"][i] @ Ui
        xn = blk["A"][i] @ fx[i] + blk["c"][i]
        if use_w:
            Wi = np.zeros((n, nd)); Wi[:, off:off + n] = np.eye(n); off += n
            Fw.append(Wi)
            Xn = Xn + Wi
        Fx.append(Xn)
        fx.append(xn)
    H = np.zeros((nd, nd)); g = np.zeros(nd)
    for i in range(N):
        Z = np.vstack([Fx[i], Fu[i]]); zc = np.concatenate([fx[i], np.zeros(m)])
        Pi = np.block([[blk["Q"][i], blk["M"][i]], [blk["M"][i].T, blk["R"][i]]])
        H += Z.T @ Pi @ Z
        g += Z.T @ (Pi @ zc + np.concatenate([blk["q"][i], blk["r"][i]]))
    H += Fx[N].T @ blk["QN"] @ Fx[N]
    g += Fx[N].T @ (blk["QN"] @ fx[N] + blk["qN"])
    if use_w:
        for Wm in Fw:
            H += Wm.T @ Wm / d
    xi = scipy.linalg.solve(H, -g, assume_a="pos")
    x = np.stack([Fx[i] @ xi + fx[i] for i in range(N + 1)])
    u = np.stack([Fu[i] @ xi for i in range(N)])
    y = np.stack([-(Wm @ xi) / d for Wm in Fw]) if use_w else None
    return x, u, y


@pytest.mark.parametrize("delta", [0.0, 1e-8, 1e-4, 1e-1, 1.0])
def test_t1_t2_match_textbook_reformulation(delta):
    for seed in range(6):
        n, m, N = 1 + seed % 4, 1 + (seed * 3) % 4, 1 + (seed * 5) % 9
        p = synth.random_stable_lqr(n, m, N, 1, seed=100 + seed, delta=delta)
        blk = instance_blocks(p, 0)
        x, u, y = condensed_augmented_qp(blk)
        t1 = oracle.rr_solve_dense(p)
        t2 = oracle.rr_solve_t2(p)
        tol = 1e-8 if delta >= 1e-4 or delta == 0 else 1e-6   # H has 1/δ entries: cond ~ 1/δ
        assert rel(t1["x"], x) < tol and rel(t1["u"], u) < tol
        assert rel(t2["x"][0], x) < tol and rel(t2["u"][0], u) < tol
        if y is not None:
            assert rel(t1["y"], y) < max(tol, 1e-9 / max(delta, 1e-12) * 1e-8)
            assert rel(t2["y"][0], y) < max(tol, 1e-9 / max(delta, 1e-12) * 1e-8)


# ---------------------------------------------------------------- T2 against T1
def test_t2_matches_t1_random_grid():
    """SPEC acceptance 1: 200 random instances, N in 1..10, nx, nu in 1..4,
    δ in {1e-8, 1e-4, 1e-1, 1}, relative ∞-norm error ≤ 1e-8 on x, u, y."""
    rng = np.random.default_rng(7)
    worst = 0.0
    for t in range(200):
        n, m, N = int(rng.integers(1, 5)), int(rng.integers(1, 5)), int(rng.integers(1, 11))
        d = [1e-8, 1e-4, 1e-1, 1.0][t % 4]
        p = synth.random_stable_lqr(n, m, N, 1, seed=1000 + t, delta=d)
        t1 = oracle.rr_solve_dense(p)
        t2 = oracle.rr_solve_t2(p)
        assert t2["status"][0] == 0
        for k in ("x", "u", "y"):
            worst = max(worst, rel(t2[k][0], t1[k]))
    assert worst <= 1e-8, worst


def test_t2_matches_t1_psd_singular_q():
    """P_i only PSD (rank-one Q_i, M_i = 0), R_i PD."""
    for d in (0.0, 1e-4, 1.0):
        p = synth.small_random(4, 2, 6, 3, seed=11, delta=d, psd_q=True)
        t2 = oracle.rr_solve_t2(p)
        for b in range(3):
            t1 = oracle.rr_solve_dense(p, b)
            for k in ("x", "u", "y"):
                assert rel(t2[k][b], t1[k]) < 1e-9


def test_kkt_residual_and_dual_identity():
    """S:164 KKT residual ≤ 1e-8 (1 + ‖[s;c]‖); S:167 / P:627-650: y = (Cx + c)/δ."""
    p = synth.random_stable_lqr(5, 3, 12, 4, seed=3, delta=1e-2)
    t2 = oracle.rr_solve_t2(p)
    for b in range(4):
        blk = instance_blocks(p, b)
        K, rhs, C = assemble_reglqr(blk)
        n, m, N = 5, 3, 12
        z = np.concatenate([np.concatenate([t2["x"][b, i], t2["u"][b, i]]) for i in range(N)] + [t2["x"][b, N]])
        sol = np.concatenate([z, t2["y"][b].ravel()])
        res = K @ sol - rhs
        assert np.max(np.abs(res)) <= 1e-8 * (1 + np.max(np.abs(rhs)))
        cvec = -rhs[len(z):]
        yv = (C @ z + cvec) / blk["delta"]
        assert rel(t2["y"][b].ravel(), yv) < 1e-7


def test_lti_stationary_value_equals_scipy_dare():
    """Textbook pin: the regularized LQR is a classic LQR with input [B I] and input cost
    blkdiag(R, I/δ) (cross term [M 0]); for LTI data and a long horizon V_0 is the DARE solution."""
    n, m, N = 4, 2, 400
    p = synth.random_stable_lqr(n, m, N, 1, seed=21, delta=0.05)
    for f in ("A", "B", "Q", "M", "R"):
        t = getattr(p, f)
        t[:] = t[:, :1].expand_as(t)
    t2 = oracle.rr_solve_t2(p, want_policy=True)
    blk = instance_blocks(p, 0)
    A, B, Q, M, R = blk["A"][0], blk["B"][0], blk["Q"][0], blk["M"][0], blk["R"][0]
    d = 0.05
    Bt = np.hstack([B, np.eye(n)])
    Rt = scipy.linalg.block_diag(R, np.eye(n) / d)
    St = np.hstack([M, np.zeros((n, n))])
    X = scipy.linalg.solve_discrete_are(A, Bt, Q, Rt, s=St)
    V0 = synth.unpack_lower(torch.from_numpy(t2["V"][0, 0]), n).numpy()
    assert rel(V0, X) < 1e-10
    # δ = 0: classic DARE
    p0 = p.with_delta(0.0)
    t20 = oracle.rr_solve_t2(p0, want_policy=True)
    X0 = scipy.linalg.solve_discrete_are(A, B, Q, R, s=M)
    assert rel(synth.unpack_lower(torch.from_numpy(t20["V"][0, 0]), n).numpy(), X0) < 1e-10


def test_delta_zero_recovers_classic_lqr_rollout():
    """S:499 / P:382: at δ = 0, x_0 = c_0 and x_{i+1} = A x + B u + c_{i+1} exactly (≤1e-12)."""
    p = synth.random_stable_lqr(4, 2, 10, 3, seed=8, delta=0.0)
    t2 = oracle.rr_solve_t2(p)
    for b in range(3):
        blk = instance_blocks(p, b)
        x, u = t2["x"][b], t2["u"][b]
        assert np.max(np.abs(x[0] - blk["c0"])) <= 1e-12
        for i in range(10):
            xn = blk["A"][i] @ x[i] + blk["B"][i] @ u[i] + blk["c"][i]
            assert np.max(np.abs(x[i + 1] - xn)) <= 1e-12 * (1 + np.max(np.abs(xn)))


def test_eta_to_infinity_limit_is_classic_riccati_first_order():
    """δ = 1/η → 0 converges to the classic solution, at first order."""
    p = synth.random_stable_lqr(4, 2, 10, 1, seed=9, delta=0.0)
    s0 = oracle.rr_solve_t2(p)
    diffs = []
    for d in (1e-3, 5e-4, 2.5e-4, 1.25e-4):
        s = oracle.rr_solve_t2(p.with_delta(d))
        diffs.append(max(np.max(np.abs(s[k] - s0[k])) for k in ("x", "u")))
    ratios = [diffs[i] / diffs[i + 1] for i in range(3)]
    assert all(abs(r - 2.0) < 0.02 for r in ratios), ratios
    s10 = oracle.rr_solve_t2(p.with_delta(1e-10))
    assert max(np.max(np.abs(s10[k] - s0[k])) for k in ("x", "u", "y")) <= 1e-6


def test_f_relation_naive_recursion():
    """S:165 / P:557-567: the pre-simplification F/f recursion (written here from P:557-564,
    test-only) gives F_i = I + δ V_i and f_i = δ v_i - c_i."""
    n, m, N = 3, 2, 5
    for d in (1e-2, 1e-1, 1.0):
        p = synth.random_stable_lqr(n, m, N, 1, seed=31, delta=d)
        blk = instance_blocks(p, 0)
        t2 = oracle.rr_solve_t2(p, want_policy=True)
        A, B, Q, M, R, q, r, c = (blk[k] for k in ("A", "B", "Q", "M", "R", "q", "r", "c"))
        cs = [blk["c0"]] + list(c)                 # c_0..c_N
        I = np.eye(n)
        F = I + d * blk["QN"]
        f = d * blk["qN"] - cs[N]                  # z_N = δ q_N - c_N
        Fs, fs = {N: F}, {N: f}
        for i in range(N - 1, -1, -1):
            Fi = np.linalg.inv(F)
            IF = I - Fi
            zx = d * q[i] - cs[i] + A[i].T @ cs[i + 1]
            zu = d * r[i] + B[i].T @ cs[i + 1]
            Gm = B[i].T @ IF @ B[i] + d * R[i]
            Hm = B[i].T @ IF @ A[i] + d * M[i].T
            K = -np.linalg.solve(Gm, Hm)
            k = -np.linalg.solve(Gm, zu + B[i].T @ Fi @ f)
            Fn = (I + A[i].T @ IF @ A[i] + d * Q[i]) + (A[i].T @ IF @ B[i] + d * M[i]) @ K
            fn = zx + A[i].T @ Fi @ f + (A[i].T @ IF @ B[i] + d * M[i]) @ k
            F, f = Fn, fn
            Fs[i], fs[i] = F, f
        for i in range(N + 1):
            V = synth.unpack_lower(torch.from_numpy(t2["V"][0, i]), n).numpy()
            assert np.linalg.norm(Fs[i] - (I + d * V)) <= 1e-9 * (1 + np.linalg.norm(Fs[i]))
            assert rel((fs[i] + cs[i]) / d, t2["v"][0, i]) < 1e-8


def test_inverse_identity():
    """P:569-575 / S:504: (I+δV)⁻¹δV = I − (I+δV)⁻¹ for PSD V."""
    rng = np.random.default_rng(0)
    for _ in range(100):
        n = int(rng.integers(1, 8))
        L = rng.uniform(-1, 1, (n, n))
        V = L @ L.T
        d = 10 ** rng.uniform(-8, 0)
        S = np.eye(n) + d * V
        lhs = np.linalg.solve(S, d * V)
        rhs = np.eye(n) - np.linalg.inv(S)
        assert np.linalg.norm(lhs - rhs) <= 1e-12


def test_golden_c1_double_integrator():
    """BASELINE configs[0]: fixture written by tests/golden/make_golden.py (oracle T1 only)."""
    g = json.load(open(os.path.join(HERE, "golden", "c1_double_integrator.json")))
    p = synth.double_integrator_c1()
    t2 = oracle.rr_solve_t2(p)
    for k in ("x", "u", "y"):
        assert rel(t2[k][0], np.array(g[k])) < 1e-11
    t20 = oracle.rr_solve_t2(p.with_delta(0.0))
    assert abs(t20["u"][0, 0, 0] - g["u0_delta0"]) < 1e-11 * abs(g["u0_delta0"])
    # the condensed textbook route agrees as well (independent of T1's assembly)
    x, u, y = condensed_augmented_qp(instance_blocks(p, 0))
    assert rel(x, np.array(g["x"])) < 1e-9 and rel(u, np.array(g["u"])) < 1e-9


def test_status_on_not_pd_g():
    """G_i not PD (R_i negative) → status G_NOT_PD | stage << 8, outputs NaN."""
    p = synth.random_stable_lqr(3, 2, 4, 2, seed=4, delta=1e-3)
    p.R[1, 2] = torch.tensor([-50.0, 0.0, -50.0], dtype=torch.float64)
    t2 = oracle.rr_solve_t2(p)
    assert t2["status"][0] == 0
    assert t2["status"][1] == (1 | (2 << 8))
    assert np.all(np.isnan(t2["x"][1]))


def test_threads_identical():
    p = synth.random_stable_lqr(6, 3, 8, 37, seed=12)
    a = oracle.rr_solve_t2(p, nthreads=1)
    b = oracle.rr_solve_t2(p, nthreads=5)
    for k in ("x", "u", "y"):
        assert np.array_equal(a[k], b[k])


def test_t1_bunch_kaufman_ldlt_equals_lu_and_t2():
    """North star (a): the dense symmetric-indefinite LDLᵀ (Bunch-Kaufman, 1×1 / 2×2 pivots) of the
    full KKT matrix gives the LU solution, and the recursion T2 matches it, δ ∈ {0, 1e-8, 1e-4, 1}."""
    from oracle.dense import ldl_solve
    saw_2x2 = False
    for t, d in enumerate((0.0, 1e-8, 1e-4, 1.0)):
        p = synth.random_stable_lqr(3, 2, 7, 2, seed=40 + t, delta=d)
        for b in range(2):
            lu = oracle.rr_solve_dense(p, b)
            ld = oracle.rr_solve_dense(p, b, method="ldl")
            assert rel(ld["sol"], lu["sol"]) <= 1e-11
            t2 = oracle.rr_solve_t2(p)
            for k in ("x", "u", "y"):
                assert rel(t2[k][b], ld[k]) <= 1e-8, (d, k)
            _, D, _ = scipy.linalg.ldl(ld["K"], lower=True)
            saw_2x2 |= bool(np.any(np.diag(D, -1) != 0.0))
    assert saw_2x2  # the KKT matrix is indefinite: Bunch-Kaufman takes 2×2 pivots
    # a plain symmetric indefinite matrix with a zero diagonal (only 2×2 pivots work)
    K = np.array([[0.0, 2.0, 1.0], [2.0, 0.0, 3.0], [1.0, 3.0, 0.0]])
    rhs = np.array([1.0, -2.0, 0.5])
    assert np.max(np.abs(K @ ldl_solve(K, rhs) - rhs)) <= 1e-14
