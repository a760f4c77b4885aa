"""GPU parity of ipm_solve (the batched regularized-IPM loop) against the oracle loop
(oracle/ipm_solve.py) on identical inputs: per-instance status and iteration count bit-exact, final
μ, η and iterate to 1e-9 relative (FP64), the north-star bar, in every case (measured worst case
1.4e-10 on the random LQ with stage equalities, tools/f1_errors.py).  The cart-pole swing-up is
nonconvex and does not converge within the budget; it is compared over its first 1-20 iterations."""
import numpy as np
import pytest
import torch

from oracle.ipm_solve import SolveSettings, ipm_solve_oracle
from synth.ipm_workloads import cartpole_c4, double_integrator_ocp, quadrotor_ipm, random_lq_ocp

pytestmark = pytest.mark.gpu
TOL = 1e-9


def rel(g, o):
    g = np.asarray(g, dtype=np.float64).reshape(len(g), -1)
    o = np.asarray(o, dtype=np.float64).reshape(len(o), -1)
    if g.size == 0:
        return 0.0
    return float(np.max(np.max(np.abs(g - o), axis=1) / np.maximum(np.max(np.abs(o), axis=1), 1e-300)))


def run_both(b, **S):
    import paper_2509_16370_b200 as m
    bg = b.to("cuda")
    rep = m.ipm_solve(bg, **S)
    torch.cuda.synchronize()
    it_o, rep_o = ipm_solve_oracle(b, SolveSettings(**S))
    rep_g = {k: v.cpu().numpy() for k, v in rep.items()}
    it_g = {k: v.cpu().numpy() for k, v in bg.it.items()}
    return it_g, rep_g, it_o, rep_o


def check(it_g, rep_g, it_o, rep_o, keys=("x", "u", "s", "z", "y"), tol=TOL):
    assert np.array_equal(rep_g["status"], rep_o["status"]), (rep_g["status"], rep_o["status"])
    assert np.array_equal(rep_g["iters"], rep_o["iters"]), (rep_g["iters"], rep_o["iters"])
    assert rel(rep_g["mu"], rep_o["mu"]) <= tol and rel(rep_g["eta"], rep_o["eta"]) <= tol
    for k in keys:
        if it_o[k].size:
            assert rel(it_g[k], it_o[k]) <= tol, (k, rel(it_g[k], it_o[k]))


def test_double_integrator_converges_like_oracle():
    it_g, rep_g, it_o, rep_o = run_both(double_integrator_ocp(batch=3))
    check(it_g, rep_g, it_o, rep_o)
    assert np.all(rep_g["status"] == 0) and np.all(rep_g["iters"] <= 50)
    assert np.all(np.maximum(np.maximum(rep_g["r_stat"], rep_g["r_feas"]), rep_g["r_comp"]) <= 1e-6)


@pytest.mark.parametrize("nx,nu,ng,ngN,nc,ncN", [(4, 2, 2, 1, 0, 0), (4, 1, 3, 2, 0, 0), (3, 2, 2, 1, 1, 1),
                                                 (8, 3, 4, 2, 2, 1), (12, 4, 6, 2, 2, 0)])
def test_random_lq_parity(nx, nu, ng, ngN, nc, ncN):
    b = random_lq_ocp(nx, nu, 12, 24, seed=nx * 7 + ng, ng=ng, ngN=ngN, nc=nc, ncN=ncN, eta=1e4)
    it_g, rep_g, it_o, rep_o = run_both(b)
    check(it_g, rep_g, it_o, rep_o, keys=("x", "u", "s", "z", "y", "lam"))
    conv = rep_g["status"] == 0
    assert conv.mean() >= 0.5 or nc > 0   # random stage equalities + inequalities may be infeasible


@pytest.mark.parametrize("iters", [1, 3, 6, 20])
def test_cartpole_first_iterations(iters):
    b = cartpole_c4(16, N=40)
    it_g, rep_g, it_o, rep_o = run_both(b, max_iters=iters)
    check(it_g, rep_g, it_o, rep_o)
    assert np.all(rep_g["status"] == 6)


def test_converged_instances_are_frozen_and_empty_batch():
    """A converged iterate is a fixed point of the loop: solving S:269's scalar problem, then
    re-solving from the converged (x, s, z) with its final μ and η (the data re-generated at that
    iterate: μ and the data are inputs of ipm_solve, include/rr.h) reports status 0 after zero
    steps and leaves every iterate array bitwise unchanged.  An empty batch is a no-op.
    (Instances converging at different iterations inside one batch: the next test.)"""
    import paper_2509_16370_b200 as m
    from synth.ipm_workloads import spec_scalar_ocp
    b = spec_scalar_ocp(batch=3, xbar=3.0, s=2.0, z=0.05, mu=0.1, eta=1e4).to("cuda")
    rep = m.ipm_solve(b)
    torch.cuda.synchronize()
    assert torch.all(rep["status"] == 0) and torch.all(rep["iters"] > 0)
    u, sl, z = (float(b.it[k][0].reshape(-1)[0]) for k in ("u", "s", "z"))
    mu, eta = float(rep["mu"][0]), float(rep["eta"][0])
    b2 = spec_scalar_ocp(batch=3, xbar=u, s=sl, z=z, mu=mu, eta=eta).to("cuda")
    snap = {k: v.clone() for k, v in b2.it.items()}
    rep2 = m.ipm_solve(b2)
    torch.cuda.synchronize()
    assert torch.all(rep2["status"] == 0) and torch.all(rep2["iters"] == 0)
    for k, v in snap.items():
        assert torch.equal(b2.it[k], v), k
    e = double_integrator_ocp(batch=0).to("cuda")
    m.ipm_solve(e)


def test_mixed_batch_each_instance_as_if_alone():
    """Per-instance convergence masks: a batch interleaving two scalar problems that converge after
    different numbers of iterations gives every instance the status, iteration count and iterate
    bits of its own single-instance solve (the early finisher is frozen while the other keeps
    stepping)."""
    import paper_2509_16370_b200 as m
    from synth.ipm_workloads import spec_equality_qp_ocp, spec_scalar_ocp
    mk = [lambda bb: spec_scalar_ocp(batch=bb, xbar=3.0, s=2.0, z=0.05, mu=0.1, eta=1e4),
          lambda bb: spec_scalar_ocp(batch=bb, xbar=5.0, s=4.0, z=0.025, mu=0.1, eta=1e2)]
    singles = []
    for f in mk:
        b = f(1).to("cuda")
        r = m.ipm_solve(b)
        singles.append((b, r))
    torch.cuda.synchronize()
    # interleave the two problems in one batch of 6
    parts = [mk[i % 2](1) for i in range(6)]
    from synth.ipm_workloads import IPMBatch
    cat = IPMBatch(1, 1, 1, 1, 0, 0, 0, 0,
                   {k: (parts[0].data[k] if k == "model_params" else torch.cat([p.data[k] for p in parts]))
                    for k in parts[0].data},
                   {k: torch.cat([p.it[k] for p in parts]) for k in parts[0].it}).to("cuda")
    rc = m.ipm_solve(cat)
    torch.cuda.synchronize()
    assert int(singles[0][1]["iters"][0]) != int(singles[1][1]["iters"][0])
    for i in range(6):
        b, r = singles[i % 2]
        assert int(rc["iters"][i]) == int(r["iters"][0]) and int(rc["status"][i]) == int(r["status"][0])
        for k in ("u", "s", "z", "x", "y"):
            assert torch.equal(cat.it[k][i], b.it[k][0]), (i, k)


@pytest.mark.parametrize("case", ["ineq_eta1e4", "ineq_eta1e2", "eq_m1", "eq_m3"])
def test_spec_end_to_end_examples(case):
    """min x² s.t. x ≥ 1 from x = 3 → (x, z) = (1, 2); min ½‖x‖² s.t. x₁ = 1 from 0 →
    x = e₁, y = −1; within 1e-6 on the GPU, with the oracle loop's status and iteration count."""
    from synth.ipm_workloads import spec_equality_qp_ocp, spec_scalar_ocp
    b = {"ineq_eta1e4": lambda: spec_scalar_ocp(batch=4, xbar=3.0, s=2.0, z=0.05, mu=0.1, eta=1e4),
         "ineq_eta1e2": lambda: spec_scalar_ocp(batch=4, xbar=3.0, s=2.0, z=0.05, mu=0.1, eta=1e2),
         "eq_m1": lambda: spec_equality_qp_ocp(batch=4, m=1),
         "eq_m3": lambda: spec_equality_qp_ocp(batch=4, m=3)}[case]()
    it_g, rep_g, it_o, rep_o = run_both(b)
    check(it_g, rep_g, it_o, rep_o, keys=("x", "u", "s", "z", "y", "lam"))
    assert np.all(rep_g["status"] == 0)
    if case.startswith("ineq"):
        assert np.all(np.abs(it_g["u"][:, 0, 0] - 1.0) <= 1e-6) and np.all(np.abs(it_g["z"][:, 0, 0] - 2.0) <= 1e-6)
    else:
        m = b.nu
        e1 = np.zeros(m)
        e1[0] = 1.0
        assert np.all(np.abs(it_g["u"][:, 0] - e1) <= 1e-6) and np.all(np.abs(it_g["lam"][:, 0, 0] + 1.0) <= 1e-6)


@pytest.mark.parametrize("iters", [1, 4])
def test_quadrotor_first_iterations(iters):
    """Quadrotor model (analytic Jacobians re-evaluated at every iterate) over the first iterations."""
    b = quadrotor_ipm(24, N=20)
    it_g, rep_g, it_o, rep_o = run_both(b, max_iters=iters)
    check(it_g, rep_g, it_o, rep_o)


def test_quadrotor_solve_converges():
    """The quadrotor hover problems converge (oracle: 18-34 iterations): same status and iteration
    count as the oracle loop, iterate within the 1e-9 bar."""
    b = quadrotor_ipm(6, N=20)
    it_g, rep_g, it_o, rep_o = run_both(b)
    assert np.all(rep_o["status"] == 0)
    check(it_g, rep_g, it_o, rep_o)
    assert np.all(np.maximum(np.maximum(rep_g["r_stat"], rep_g["r_feas"]), rep_g["r_comp"]) <= 1e-6)


def test_cartpole_swing_up_converges_with_linearised_merit():
    """C4 swing-up end to end: with the step's trial merits on the linearised dynamics
    (reading R22, settings linear_merit) every instance reaches the KKT tolerance and the upright
    goal on the GPU and in the oracle, with the same status.  Over 110-200 nonlinear iterations the
    two trajectories differ by accumulated rounding, so the iteration counts are compared within 2
    and the converged iterates at the solution accuracy the loop certifies (tol_kkt = 1e-6, reading
    R22 in DESIGN.md), not at the 1e-9 single-step bar."""
    b = cartpole_c4(8, N=100)
    it_g, rep_g, it_o, rep_o = run_both(b, linear_merit=True, max_iters=300)
    assert np.all(rep_o["status"] == 0), rep_o["status"]
    assert np.array_equal(rep_g["status"], rep_o["status"]), (rep_g["status"], rep_o["status"])
    assert np.all(np.abs(rep_g["iters"].astype(int) - rep_o["iters"].astype(int)) <= 2), (rep_g["iters"], rep_o["iters"])
    assert np.all(np.maximum(np.maximum(rep_g["r_stat"], rep_g["r_feas"]), rep_g["r_comp"]) <= 1e-6)
    xN = it_g["x"][:, -1]
    assert np.all(np.abs(xN[:, 1] - np.pi) < 0.05), xN       # pole upright at the horizon end
    assert np.all(np.abs(it_g["x"][..., 0]) <= 0.5 + 1e-6)     # cart inside the track
    assert np.all(np.abs(it_g["u"]) <= 3.0 + 1e-6)             # force bound
    assert rel(it_g["x"], it_o["x"]) <= 1e-5 and rel(it_g["u"], it_o["u"]) <= 1e-4, (rel(it_g["x"], it_o["x"]), rel(it_g["u"], it_o["u"]))


def test_linear_merit_first_iterations_match_oracle():
    """linear_merit over the first iterations of the swing-up: the 1e-9 bar and bit-exact counts."""
    b = cartpole_c4(8, N=100)
    it_g, rep_g, it_o, rep_o = run_both(b, linear_merit=True, max_iters=6)
    check(it_g, rep_g, it_o, rep_o)
