"""Pins of the oracle's quadrotor model (IPM_MODEL_QUADROTOR; SURVEY §8(d) C5 dynamics, explicit
Euler x⁺ = x + dt f(x, u)) by physics that any correct implementation satisfies, plus agreement with
the workload generator's copy and the descent Theorem on the quadrotor IPM batch.  CPU only."""
import numpy as np
import torch

from oracle.ipm import ipm_merit_oracle, ipm_step_oracle, quadrotor_step_oracle
from synth.ipm_workloads import quadrotor_ipm, quadrotor_params, quadrotor_step_torch

PRM = quadrotor_params().numpy()
DT, MASS, J, G = PRM[0], PRM[1], PRM[2:5], PRM[5]


def accel(x, u):
    """world acceleration of the oracle's step: (v⁺ − v)/dt."""
    return (quadrotor_step_oracle(PRM, x, u)[6:9] - x[6:9]) / DT


def test_hover_is_an_equilibrium():
    """Level attitude, zero body rates, thrust mg, zero torques: only the position moves (by dt v)."""
    rng = np.random.default_rng(0)
    for _ in range(5):
        x = np.zeros(12)
        x[:3] = rng.uniform(-1, 1, 3)
        x[5] = rng.uniform(-3, 3)  # any yaw
        x[6:9] = rng.uniform(-1, 1, 3)
        xn = quadrotor_step_oracle(PRM, x, np.array([MASS * G, 0, 0, 0]))
        exp = x.copy()
        exp[:3] += DT * x[6:9]
        assert np.max(np.abs(xn - exp)) <= 1e-15


def test_free_fall_and_thrust_magnitude():
    """T = 0: a = (0, 0, −g).  Any attitude: |a + g e₃| = T/m (a rotation preserves length)."""
    rng = np.random.default_rng(1)
    x = np.zeros(12)
    x[3:6] = rng.uniform(-1, 1, 3)
    assert np.max(np.abs(accel(x, np.zeros(4)) - np.array([0, 0, -G]))) <= 1e-14
    for _ in range(10):
        x = rng.uniform(-1, 1, 12)
        T = rng.uniform(0.5, 10)
        a = accel(x, np.array([T, 0.01, -0.02, 0.03]))
        assert abs(np.linalg.norm(a + np.array([0, 0, G])) - T / MASS) <= 1e-12 * T / MASS


def test_pure_roll_and_pure_pitch_thrust_direction():
    """ZYX convention: roll φ tilts thrust to (0, −sin φ, cos φ); pitch θ to (sin θ, 0, cos θ)."""
    T = 7.0
    for ang in (0.3, -0.7):
        x = np.zeros(12); x[3] = ang
        assert np.max(np.abs(accel(x, np.array([T, 0, 0, 0])) - (T / MASS * np.array([0, -np.sin(ang), np.cos(ang)]) - [0, 0, G]))) <= 1e-13
        x = np.zeros(12); x[4] = ang
        assert np.max(np.abs(accel(x, np.array([T, 0, 0, 0])) - (T / MASS * np.array([np.sin(ang), 0, np.cos(ang)]) - [0, 0, G]))) <= 1e-13


def test_euler_rates_and_rigid_body_rotation():
    """Level attitude: angle rates = body rates.  Torque-free: J ω̇ = −ω × Jω, so ωᵀJω̇ = 0 (kinetic
    energy stationary) and a rotation about a principal axis keeps its rate; torque τ alone adds
    dt τ/J to ω."""
    rng = np.random.default_rng(2)
    w = rng.uniform(-2, 2, 3)
    x = np.zeros(12); x[9:12] = w
    xn = quadrotor_step_oracle(PRM, x, np.array([MASS * G, 0, 0, 0]))
    assert np.max(np.abs((xn[3:6] - x[3:6]) / DT - w)) <= 1e-13
    wdot = (xn[9:12] - w) / DT
    assert abs(np.dot(w, J * wdot)) <= 1e-12 * np.dot(w, J * w) / DT
    assert np.max(np.abs(wdot - (-np.cross(w, J * w) / J))) <= 1e-9 * np.max(np.abs(wdot))
    for ax in range(3):
        x = np.zeros(12); x[9 + ax] = 1.5
        assert np.max(np.abs(quadrotor_step_oracle(PRM, x, np.array([0, 0, 0, 0]))[9:12] - x[9:12])) <= 1e-15
    tau = np.array([0.01, -0.02, 0.03])
    xn = quadrotor_step_oracle(PRM, np.zeros(12), np.concatenate([[0.0], tau]))
    assert np.max(np.abs(xn[9:12] - DT * tau / J)) <= 1e-15


def test_generator_copy_agrees_and_jacobians_match_fd():
    """The generator's step (torch) equals the oracle's; its autograd Jacobians A_i, B_i equal central
    finite differences of the ORACLE's model."""
    rng = np.random.default_rng(3)
    for _ in range(20):
        x = rng.uniform(-1, 1, 12)
        u = rng.uniform(-1, 1, 4) + np.array([5.0, 0, 0, 0])
        a = quadrotor_step_oracle(PRM, x, u)
        b = quadrotor_step_torch(torch.from_numpy(PRM), torch.from_numpy(x), torch.from_numpy(u)).numpy()
        assert np.max(np.abs(a - b)) <= 1e-14 * (1 + np.max(np.abs(a)))
    p = quadrotor_ipm(2, N=4, seed=5)
    h = 1e-6
    for b in range(2):
        for i in range(4):
            x, u = p.it["x"][b, i].numpy(), p.it["u"][b, i].numpy()
            A = p.data["A"][b, i].numpy().reshape(12, 12).T
            B = p.data["B"][b, i].numpy().reshape(4, 12).T
            for j in range(12):
                e = np.zeros(12); e[j] = h
                col = (quadrotor_step_oracle(PRM, x + e, u) - quadrotor_step_oracle(PRM, x - e, u)) / (2 * h)
                assert np.max(np.abs(col - A[:, j])) < 1e-6
            for j in range(4):
                e = np.zeros(4); e[j] = h
                col = (quadrotor_step_oracle(PRM, x, u + e) - quadrotor_step_oracle(PRM, x, u - e)) / (2 * h)
                assert np.max(np.abs(col - B[:, j])) < 1e-6


def test_descent_theorem_quadrotor():
    """D < 0, equal to the closed form and to the FD slope of 𝒜 evaluated through the nonlinear
    quadrotor dynamics; the accepted step satisfies Armijo; fraction-to-boundary is exercised."""
    p = quadrotor_ipm(6, N=20)
    res, _ = ipm_step_oracle(p)
    assert np.all(res["status"] == 0)
    assert np.any(res["alpha_p"] < 1.0)
    for b in range(6):
        D = res["D"][b]
        assert D < 0 and abs(D - res["D_closed"][b]) <= 1e-8 * abs(D)
        h = 1e-6
        fd = (ipm_merit_oracle(p, res, b, h) - ipm_merit_oracle(p, res, b, -h)) / (2 * h)
        assert abs(fd - D) <= max(1e-6, 1e-4 * abs(D)), (fd, D)
        assert res["merit_acc"][b] <= res["merit0"][b] + 1e-4 * res["alpha_p"][b] * D


def test_solve_loop_converges_on_quadrotor():
    """The oracle IPM loop (reading R21) with the quadrotor model converges on the hover problems."""
    from oracle.ipm_solve import ipm_solve_oracle
    _, rep = ipm_solve_oracle(quadrotor_ipm(4, N=20))
    assert np.all(rep["status"] == 0) and np.all(rep["iters"] <= 60)
    assert np.all(np.maximum(np.maximum(rep["r_stat"], rep["r_feas"]), rep["r_comp0"]) <= 1e-6)
