"""Pins of the KKT-residual oracle (oracle/residual.py; the paper's residual callback).

* block form == the dense definition K [z; y] - rhs for random (x, u, y);
* SPEC's scalar example (N = 0): at the closed-form solution x0 = 2/3, y0 = 7/3
  (δ = 1) the residual is exactly 0; at (0, 0) it is [s; c] = (q_N, c_0) = (1, 3);
* hand-computed N = 1 scalar case (every block of the formula exercised, integers);
* the residual of the T2 solution is at rounding level, of a perturbed solution it is K e."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle.dense import assemble_reglqr, instance_blocks


def scalar_problem(delta, N=0):
    z = lambda *s: torch.zeros(*s, dtype=torch.float64)
    return synth.RRProblem(1, 1, N, A=z(1, N, 1), B=z(1, N, 1), Q=z(1, N, 1), M=z(1, N, 1),
                           R=torch.ones(1, N, 1, dtype=torch.float64), q=z(1, N, 1), r=z(1, N, 1),
                           c=z(1, N, 1), QN=torch.tensor([[2.0]], dtype=torch.float64),
                           qN=torch.tensor([[1.0]], dtype=torch.float64),
                           c0=torch.tensor([[3.0]], dtype=torch.float64),
                           delta=torch.tensor([delta], dtype=torch.float64))


def test_scalar_spec_example():
    p = scalar_problem(1.0)
    x = np.array([[[2.0 / 3.0]]])
    y = np.array([[[7.0 / 3.0]]])
    r = oracle.residual_blocks(p, x, np.zeros((1, 0, 1)), y)
    assert abs(r["rqN"][0, 0]) < 1e-15 and abs(r["rc0"][0, 0]) < 1e-15
    r0 = oracle.residual_blocks(p, np.zeros((1, 1, 1)), np.zeros((1, 0, 1)), np.zeros((1, 1, 1)))
    assert r0["rqN"][0, 0] == 1.0 and r0["rc0"][0, 0] == 3.0          # [s; c] at zero
    assert np.array_equal(r0["norms"][0], [1.0, 3.0])


def test_hand_computed_n1():
    """n = m = 1, N = 1: A = 2, B = 3, Q = 4, M = 5, R = 6, q = 7, r = 8, c_1 = 9, Q_N = 10,
    q_N = 11, c_0 = 12, δ = 0.5 at x = (1, 2), u = 3, y = (4, 5):
      stat x_0 = 4*1 + 5*3 + 7 - 4 + 2*5 = 32;  stat u_0 = 5*1 + 6*3 + 8 + 3*5 = 46;
      stat x_1 = 10*2 + 11 - 5 = 26;  prim 0 = -1 - 0.5*4 + 12 = 9;
      prim 1 = 2*1 + 3*3 - 2 - 0.5*5 + 9 = 15.5."""
    t = lambda v: torch.tensor([[[float(v)]]], dtype=torch.float64)
    p = synth.RRProblem(1, 1, 1, A=t(2), B=t(3), Q=t(4), M=t(5), R=t(6), q=t(7), r=t(8), c=t(9),
                        QN=torch.tensor([[10.0]], dtype=torch.float64), qN=torch.tensor([[11.0]], dtype=torch.float64),
                        c0=torch.tensor([[12.0]], dtype=torch.float64), delta=torch.tensor([0.5], dtype=torch.float64))
    x = np.array([[[1.0], [2.0]]])
    u = np.array([[[3.0]]])
    y = np.array([[[4.0], [5.0]]])
    r = oracle.residual_blocks(p, x, u, y)
    assert r["rq"][0, 0, 0] == 32 and r["rr"][0, 0, 0] == 46 and r["rqN"][0, 0] == 26
    assert r["rc0"][0, 0] == 9 and r["rc"][0, 0, 0] == 15.5
    st, pr = oracle.residual_dense(p, 0, x[0], u[0], y[0])
    assert np.array_equal(st, [32, 46, 26]) and np.array_equal(pr, [9, 15.5])


@pytest.mark.parametrize("nx,nu,N", [(3, 2, 4), (4, 1, 6), (2, 3, 1), (5, 2, 0)])
def test_blocks_equal_dense_definition(nx, nu, N):
    p = synth.small_random(nx, nu, N, 3, seed=nx + 10 * nu + N, delta=0.3)
    rng = np.random.default_rng(1)
    x, u, y = rng.standard_normal((3, N + 1, nx)), rng.standard_normal((3, N, nu)), rng.standard_normal((3, N + 1, nx))
    r = oracle.residual_blocks(p, x, u, y)
    for b in range(3):
        st, pr = oracle.residual_dense(p, b, x[b], u[b], y[b])
        n, m = nx, nu
        st_b = np.concatenate([np.concatenate([r["rq"][b, i], r["rr"][b, i]]) for i in range(N)] + [r["rqN"][b]])
        pr_b = np.concatenate([r["rc0"][b]] + [r["rc"][b, i] for i in range(N)])
        assert np.allclose(st, st_b, rtol=0, atol=1e-12) and np.allclose(pr, pr_b, rtol=0, atol=1e-12)
        assert abs(r["norms"][b, 0] - np.abs(st).max()) < 1e-12 and abs(r["norms"][b, 1] - np.abs(pr).max()) < 1e-12


def test_solution_residual_small_and_linear_in_perturbation():
    p = synth.random_stable_lqr(4, 2, 8, 2, seed=3, delta=1e-2)
    o = oracle.rr_solve_t2(p)
    r = oracle.residual_blocks(p, o["x"], o["u"], o["y"])
    assert np.max(r["norms"]) < 1e-12
    rng = np.random.default_rng(0)
    ex = rng.standard_normal(o["x"].shape) * 1e-3
    r2 = oracle.residual_blocks(p, o["x"] + ex, o["u"], o["y"])
    blk = instance_blocks(p, 0)
    K, _, _ = assemble_reglqr(blk)
    n, m, N = 4, 2, 8
    e = np.zeros(K.shape[0])
    for i in range(N + 1):
        e[i * (n + m):i * (n + m) + n] = ex[0, i]
    Ke = K @ e
    st_b = np.concatenate([np.concatenate([r2["rq"][0, i], r2["rr"][0, i]]) for i in range(N)] + [r2["rqN"][0]])
    nz = N * (n + m) + n
    assert np.allclose(st_b, Ke[:nz], atol=1e-12)
