"""Pins of the batched IPM-solve oracle (oracle/ipm_solve.py, DESIGN reading R21).

* evaluate() at the reference iterate reproduces the reference data (the model is exact there);
* the cart-pole Jacobians of evaluate() equal central finite differences of the oracle's own C
  cart-pole step (an implementation independent of the generator's autograd);
* SPEC's end-to-end double-integrator OCP: converges, KKT <= 1e-6, controls equal an
  independent solve of the same QP (scipy SLSQP on the condensed problem) to 1e-4, the bound is
  active with z > 0 where u = -1;
* random LQ OCPs (convex) all converge."""
import numpy as np
import pytest
import torch

from oracle.ipm import cartpole_step_oracle
from oracle.ipm_solve import SolveSettings, evaluate, ipm_solve_oracle
from synth.ipm_workloads import cartpole_c4, double_integrator_ocp, random_lq_ocp


@pytest.mark.parametrize("make", [lambda: random_lq_ocp(4, 2, 6, 5, seed=1, ng=2, ngN=1, nc=1, ncN=1),
                                  lambda: cartpole_c4(3, N=12), lambda: double_integrator_ocp(batch=2)])
def test_evaluate_at_reference_is_identity(make):
    b = make()
    d = evaluate(b, b.it["x"].numpy(), b.it["u"].numpy())
    for k, v in b.data.items():
        assert np.allclose(d[k], v.numpy(), rtol=1e-13, atol=1e-13), k


def test_cartpole_jacobians_match_finite_differences():
    b = cartpole_c4(2, N=6)
    rng = np.random.default_rng(0)
    x = b.it["x"].numpy() + 0.3 * rng.standard_normal(b.it["x"].shape)
    u = b.it["u"].numpy() + 0.3 * rng.standard_normal(b.it["u"].shape)
    d = evaluate(b, x, u)
    prm = b.data["model_params"].numpy()
    h = 1e-6
    for bi in range(2):
        for i in range(6):
            A = d["A"][bi, i].reshape(4, 4).T   # column-major -> row-major
            Bm = d["B"][bi, i].reshape(1, 4).T
            for c in range(4):
                e = np.zeros(4)
                e[c] = h
                fd = (cartpole_step_oracle(prm, x[bi, i] + e, u[bi, i]) - cartpole_step_oracle(prm, x[bi, i] - e, u[bi, i])) / (2 * h)
                assert np.allclose(A[:, c], fd, atol=1e-7)
            fd = (cartpole_step_oracle(prm, x[bi, i], u[bi, i] + h) - cartpole_step_oracle(prm, x[bi, i], u[bi, i] - h)) / (2 * h)
            assert np.allclose(Bm[:, 0], fd, atol=1e-7)
            assert np.allclose(d["dres"][bi, i], cartpole_step_oracle(prm, x[bi, i], u[bi, i]) - x[bi, i + 1], atol=1e-14)


def test_double_integrator_end_to_end_matches_independent_qp():
    scipy_opt = pytest.importorskip("scipy.optimize")
    N, h = 20, 0.1
    b = double_integrator_ocp(N=N, h=h, eta=1e4)
    it, rep = ipm_solve_oracle(b, SolveSettings())
    assert rep["status"][0] == 0 and rep["iters"][0] <= 50
    assert max(rep["r_stat"][0], rep["r_feas"][0], rep["r_comp0"][0]) <= 1e-6
    # independent solve: min ½Σ(|x_i|² + 0.1 u_i²) + 5|x_N|², x_{i+1} = A x_i + B u_i, x_0 = (5, 0), |u| <= 1
    A = np.array([[1, h], [0, 1]])
    B = np.array([h * h / 2, h])

    def roll(u):
        xs = [np.array([5.0, 0.0])]
        for k in range(N):
            xs.append(A @ xs[-1] + B * u[k])
        return np.array(xs)

    def cost(u):
        xs = roll(u)
        return 0.5 * (xs[:N] ** 2).sum() + 0.05 * (u ** 2).sum() + 5.0 * (xs[N] ** 2).sum()

    r = scipy_opt.minimize(cost, np.zeros(N), method="SLSQP", bounds=[(-1, 1)] * N,
                           options=dict(ftol=1e-14, maxiter=500))
    assert r.success
    assert np.max(np.abs(it["u"][0, :, 0] - r.x)) < 1e-4
    assert np.allclose(it["x"][0], roll(it["u"][0, :, 0]), atol=1e-5)        # dynamics satisfied
    act = it["u"][0, :, 0] < -1 + 1e-4
    assert act.sum() >= 5 and np.all(it["z"][0, act, 1] > 1e-3)            # lower bound active, dual > 0


def test_random_lq_all_converge():
    b = random_lq_ocp(4, 2, 10, 16, seed=3, ng=2, ngN=1, nc=0, ncN=0, eta=1e4)
    it, rep = ipm_solve_oracle(b, SolveSettings())
    assert np.all(rep["status"] == 0)
    assert np.all(np.maximum(np.maximum(rep["r_stat"], rep["r_feas"]), rep["r_comp0"]) <= 1e-6)


def test_merit_at_values_matches_c_oracle_on_lq():
    """The caller-evaluated merit (numpy, the definition) equals the C oracle's merit for the LQ model,
    whose trial values are exact from the linearisation (evaluate() at the trial point)."""
    from oracle.ipm import ipm_merit_oracle, ipm_step_oracle
    from oracle.ipm_solve import merit_at_values
    b = random_lq_ocp(4, 2, 6, 3, seed=7, ng=2, ngN=1, nc=1, ncN=1)
    res, _ = ipm_step_oracle(b)
    for alpha in (0.0, 0.05, 0.3, 0.9):
        x = b.it["x"].numpy() + alpha * res["dx"]
        u = b.it["u"].numpy() + alpha * res["du"]
        d = evaluate(b, x, u)
        trial = {k: d[k] for k in ("fval", "dres", "ce", "ceN", "gv", "gvN")}
        got = merit_at_values(b, res, np.full(3, alpha), trial)
        for k in range(3):
            ref = ipm_merit_oracle(b, res, k, alpha)
            if np.isnan(ref):  # a trial slack left the positive orthant: both sides NaN
                assert np.isnan(got[k])
            else:
                assert abs(got[k] - ref) <= 1e-10 * max(1.0, abs(ref)), (alpha, k, got[k], ref)


def test_cartpole_swing_up_converges_with_linearised_merit():
    """Reading R22: the C4 swing-up from the C4 iterate converges (status 0, KKT
    residuals <= tol) to the upright goal when the step's trial merits use the linearised
    dynamics; with the nonlinear trial merits the same loop stalls (tiny accepted steps)."""
    from synth.ipm_workloads import cartpole_c4
    b = cartpole_c4(3, N=100)
    it, rep = ipm_solve_oracle(b, SolveSettings(max_iters=300, linear_merit=True), nthreads=3)
    assert np.all(rep["status"] == 0), rep["status"]
    assert np.all(np.maximum(np.maximum(rep["r_stat"], rep["r_feas"]), rep["r_comp0"]) <= 1e-6)
    assert np.all(np.abs(it["x"][:, -1, 1] - np.pi) < 0.05)
    assert np.all(np.abs(it["u"]) <= 3.0 + 1e-6) and np.all(np.abs(it["x"][..., 0]) <= 0.5 + 1e-6)
    it2, rep2 = ipm_solve_oracle(b, SolveSettings(max_iters=40), nthreads=3)
    assert np.all(rep2["status"] == 6)   # MAXITER: the nonlinear-merit loop has not converged
