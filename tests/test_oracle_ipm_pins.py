"""Pins of the IPM-step oracle run THROUGH ITS OWN C CODE (oracle/ipm_oracle.c: orc_ipm_step,
orc_ipm_merit), on SPEC's worked examples encoded as optimal-control instances
(synth.ipm_workloads.spec_scalar_ocp / spec_equality_qp_ocp: N = 1, the state pinned at 0, the
static decision variable = the stage-0 control).  CPU only.

* S:234 exact scalar step: (Δx, Δs, Δz) = (−33/32, −15/16, 15/16), D = −99/32, α = 1,
  𝒜(0) = 4, 𝒜(1) = 3.848760597239781 (P:61-66 merit, Eq.(4×4), P:126-219 Theorem).
* S:215-217 (barrier Lagrangian) and S:224-226 (augmented) merit values, with every term of 𝒜
  (f̄, −μΣlog s, yᵀc on the initial-state and dynamics rows, λᵀc_e, zᵀ(g+s), η/2‖·‖²) placed in a
  case of its own, so an α-independent error in any of them fails a value pin.
* S:248 "largest α": on C4-LS the ladder point before the accepted one violates Armijo, and the
  accepted one satisfies it, both evaluated with orc_ipm_merit.
* S:269-270 end-to-end examples through the oracle loop (oracle/ipm_solve.py around orc_ipm_step).
"""
import math

import numpy as np
import pytest

from oracle.ipm import DIR_SHAPES, ipm_merit_oracle, ipm_step_oracle
from oracle.ipm_solve import SolveSettings, ipm_solve_oracle
from synth.ipm_workloads import cartpole_c4, spec_equality_qp_ocp, spec_scalar_ocp


def zero_dir(b):
    return {k: np.zeros(tuple(b.it[v].shape)) for k, v in DIR_SHAPES.items()}


def merit0(b, i=0):
    """𝒜 at the iterate itself (α = 0), from orc_ipm_merit."""
    return ipm_merit_oracle(b, zero_dir(b), i, 0.0)


# ----------------------------------------------------------------------------- S:234 exact step
def test_scalar_step_exact_through_orc_ipm_step():
    b = spec_scalar_ocp()                       # x = 2, s = 1, z = 1, μ = 1, η = 10
    res, it = ipm_step_oracle(b)
    assert res["status"][0] == 0
    # every quantity below is a dyadic rational or the S:234 decimal: exact in FP64 up to one rounding
    assert res["du"][0, 0, 0] == -33 / 32
    assert res["ds"][0, 0, 0] == -15 / 16
    assert res["dz"][0, 0, 0] == 15 / 16
    assert np.all(res["dx"][0] == 0.0) and np.all(res["dy"][0] == 0.0)   # pinned state rows stay put
    assert res["D"][0] == -99 / 32 and res["D_closed"][0] == -99 / 32
    assert res["alpha_p"][0] == 1.0 and res["n_backtracks"][0] == 0
    assert res["merit0"][0] == 4.0
    assert abs(res["merit_acc"][0] - 3.848760597239781) <= 4e-16 * 3.85
    # α_d: Δz > 0 → no dual cap (S:252 rule on z)
    assert res["alpha_d"][0] == 1.0
    # the update moved (x, s, z) by the full step
    assert it["u"][0, 0, 0] == 2.0 - 33 / 32 and it["s"][0, 0, 0] == 1 / 16 and it["z"][0, 0, 0] == 1 + 15 / 16
    # orc_ipm_merit along the same direction reproduces 𝒜(0) and 𝒜(1)
    assert ipm_merit_oracle(b, res, 0, 0.0) == 4.0
    assert abs(ipm_merit_oracle(b, res, 0, 1.0) - 3.848760597239781) <= 4e-16 * 3.85


def test_scalar_step_fraction_to_boundary_and_backtracking():
    """The same problem from x = 2, s = 0.5, z = 0.1, μ = 0.01: Δs = −1.3375 < −s, so α_max < 1 is
    the fraction-to-boundary cap τ s / (−Δs), and Armijo holds at the accepted
    ladder point."""
    b = spec_scalar_ocp(s=0.5, z=0.1, mu=0.01)
    res, _ = ipm_step_oracle(b)
    ds = res["ds"][0, 0, 0]
    assert res["status"][0] == 0 and ds < 0
    amax = min(1.0, 0.995 * 0.5 / -ds)
    assert amax < 1.0
    assert res["alpha_p"][0] == amax * 0.5 ** res["n_backtracks"][0]
    a = res["alpha_p"][0]
    assert ipm_merit_oracle(b, res, 0, a) <= res["merit0"][0] + 1e-4 * a * res["D"][0]


# ----------------------------------------------------------------------------- S:215-226 merit values
def test_merit_barrier_lagrangian_trivial_zero():
    """f = 0, c = 0, g + s = 0, μ = 1, s = all ones → 0; and the augmented value at a
    feasible point equals it for any η."""
    for eta in (0.0, 10.0, 1e6):
        b = spec_scalar_ocp(xbar=2.0, s=1.0, z=0.7, mu=1.0, eta=eta)
        b.data["fval"].fill_(0.0)          # f = 0; g = 1 − 2 = −1, s = 1 → g + s = 0; log 1 = 0
        assert merit0(b) == 0.0


def test_merit_linear_terms_each_row():
    """f = 2, y = [1], c = [3], no inequalities → 5 (η = 0: the barrier Lagrangian), and
    S:225: c = [3], η = 2 → L + 9.  The residual c is placed in turn on the initial-state row
    (c_0 = s_0 − x̄_0), on the dynamics row (c_1 = d_0 − x̄_1) and on a stage equality (c_e, λ)."""
    for where in ("initial", "dynamics", "stage_eq"):
        for eta, expect in ((0.0, 5.0), (2.0, 14.0)):
            b = spec_equality_qp_ocp(m=1, mu=0.3, eta=eta)   # nc = 1, no inequalities
            b.data["fval"].fill_(2.0)
            b.data["ce"].fill_(0.0)
            if where == "initial":
                b.data["s0"].fill_(3.0)
                b.it["y"][:, 0] = 1.0
            elif where == "dynamics":
                b.data["dres"].fill_(3.0)
                b.it["y"][:, 1] = 1.0
            else:
                b.data["ce"].fill_(3.0)
                b.it["lam"].fill_(1.0)
            assert merit0(b) == expect, (where, eta)


def test_merit_scalar_qp_values():
    """scalar QP (f = x², x = 2, g = 1 − x, s = 1, z = 1, μ = 0.1) → 4; the same with
    g + s = 0.2 (s = 1.2) and η = 10 → L + 0.2 with L = 4 − 0.1·log 1.2 + 1·0.2 (direct substitution)."""
    b = spec_scalar_ocp(xbar=2.0, s=1.0, z=1.0, mu=0.1, eta=0.0)
    assert merit0(b) == 4.0
    b = spec_scalar_ocp(xbar=2.0, s=1.2, z=1.0, mu=0.1, eta=0.0)
    L = merit0(b)
    assert abs(L - (4.0 - 0.1 * math.log(1.2) + 0.2)) <= 1e-15 * 4
    b.it["eta"].fill_(10.0)
    assert abs(merit0(b) - (L + 0.2)) <= 1e-15 * 4


def test_merit_barrier_sign_and_weight():
    """The barrier term is −μΣlog s: at s = e (g = −e, so g + s = 0), f = 0, μ = 0.25 → 𝒜 = −0.25,
    and at s = e² → −2μ = −0.5."""
    for s, expect in ((math.e, -0.25), (math.e ** 2, -0.5)):
        b = spec_scalar_ocp(xbar=1.0 + s, s=s, z=3.0, mu=0.25, eta=7.0)
        b.data["fval"].fill_(0.0)
        assert abs(merit0(b) - expect) <= 1e-14   # g = 1 − (1 + s) rounds: g + s ≈ 1e-15


def test_merit_along_direction_quadratic_cost_term():
    """𝒜(α) − 𝒜(0) on an unconstrained-in-u instance is α∇fᵀΔ + ½α²ΔᵀPΔ plus the exact penalty and
    barrier changes: on S:234's direction at α = 1/2 the value is the closed-form substitution
    f = (2 − 33/64)², s = 1 − 15/32, g = 1 − (2 − 33/64)."""
    b = spec_scalar_ocp()
    res, _ = ipm_step_oracle(b)
    x, s = 2 - 33 / 64, 1 - 15 / 32
    g = 1 - x
    expect = x * x - 1.0 * math.log(s) + 1.0 * (g + s) + 10 / 2 * (g + s) ** 2
    assert abs(ipm_merit_oracle(b, res, 0, 0.5) - expect) <= 1e-15 * abs(expect)


# ----------------------------------------------------------------------------- S:248 largest α
def test_c4_ls_accepted_alpha_is_the_largest_ladder_point():
    p = cartpole_c4(24, seed=2511, N=20, variant="C4-LS")
    res, _ = ipm_step_oracle(p)
    assert np.all(res["status"] == 0)
    checked = 0
    for b in range(p.batch):
        a, k, D, A0 = res["alpha_p"][b], res["n_backtracks"][b], res["D"][b], res["merit0"][b]
        Aa = ipm_merit_oracle(p, res, b, a)
        assert Aa == res["merit_acc"][b]
        assert Aa <= A0 + 1e-4 * a * D                     # Armijo at the accepted point
        if k >= 1:                                         # ... and fails one rung higher
            prev = a / 0.5
            Ap = ipm_merit_oracle(p, res, b, prev)
            assert np.isnan(Ap) or Ap > A0 + 1e-4 * prev * D, (b, k)
            checked += 1
    assert checked >= 12


# ----------------------------------------------------------------------------- S:269-270 end to end
def test_spec_end_to_end_inequality_scalar():
    """min x² s.t. x ≥ 1 (g = 1 − x), start x = 3 → x* = 1, z* = 2 within 1e-6."""
    for eta in (1e2, 1e4):
        b = spec_scalar_ocp(xbar=3.0, s=2.0, z=0.05, mu=0.1, eta=eta)   # s = max(−g, 1e-2), z = μ/s
        it, rep = ipm_solve_oracle(b, SolveSettings())
        assert rep["status"][0] == 0
        assert abs(it["u"][0, 0, 0] - 1.0) <= 1e-6 and abs(it["z"][0, 0, 0] - 2.0) <= 1e-6


def test_spec_end_to_end_equality_qp():
    """min ½‖x‖² s.t. x₁ = 1, start 0 → x* = (1, 0, …), y* = −1 within 1e-6 (y is λ here)."""
    for m, eta in ((1, 1e4), (3, 1e4), (3, 1e2)):
        b = spec_equality_qp_ocp(m=m, eta=eta)
        it, rep = ipm_solve_oracle(b, SolveSettings())
        assert rep["status"][0] == 0
        e1 = np.zeros(m)
        e1[0] = 1.0
        assert np.max(np.abs(it["u"][0, 0] - e1)) <= 1e-6
        assert abs(it["lam"][0, 0, 0] + 1.0) <= 1e-6
