"""Pins of the regularized-IPM step oracle: Eq.(4×4) dense definition, the Lemma, the descent
Theorem (closed form and finite differences), SPEC's exact scalar example, elimination
equivalence of the structured chain (condense → T2 → expand), line-search rules.  CPU only."""
import math

import numpy as np
import pytest
import torch

import synth
from oracle.ipm import DIR_SHAPES, cartpole_step_oracle, ipm_merit_oracle, ipm_step_oracle
from oracle.ipm_dense import kkt4x4, solve4x4, solve_shifted, split_X
from synth.ipm_workloads import cartpole_c4, cartpole_step_torch, random_lq_ocp


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if b.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def scalar_nlp():
    """min x², g(x) = 1 − x ≤ 0, at x = 2, s = 1, z = 1, μ = 1, η = 10."""
    return dict(P=np.array([[2.0]]), grad=np.array([4.0]), X=np.array([2.0]), C=np.zeros((0, 1)),
                c=np.zeros(0), y=np.zeros(0), G=np.array([[-1.0]]), g=np.array([-1.0]),
                s=np.array([1.0]), z=np.array([1.0]), mu=1.0, eta=10.0)


def dense_merit(nlp, x, s):
    """𝒜 for the scalar problem."""
    g = 1.0 - x
    return x * x - nlp["mu"] * math.log(s) + 1.0 * (g + s) + nlp["eta"] / 2 * (g + s) ** 2


def test_scalar_example_exact_rationals():
    nlp = scalar_nlp()
    K, gL, off = kkt4x4(nlp)
    sol = np.linalg.solve(K, -np.concatenate(gL))
    dx, ds, dz = sol[0], sol[1], sol[2]
    assert abs(dx - (-33 / 32)) < 1e-15 and abs(ds - (-15 / 16)) < 1e-15 and abs(dz - 15 / 16) < 1e-15
    # Theorem closed form: D = −ΔxᵀPΔx − ΔsᵀS⁻¹ZΔs − η‖GΔx + Δs‖²
    D = -2 * dx * dx - ds * ds - 10 * (-dx + ds) ** 2
    assert abs(D - (-99 / 32)) < 1e-14
    # ∇𝒜·d: ∇ₓ𝒜 = 2x + Gᵀ(z + η(g+s)), ∇ₛ𝒜 = −μ/s + z + η(g+s)
    gs = -1.0 + 1.0
    Dgrad = (4.0 - (1.0 + 10 * gs)) * dx + (-1.0 + 1.0 + 10 * gs) * ds
    assert abs(Dgrad - D) < 1e-14
    # fraction to boundary: Δs = −15/16 > −s/τ → α_max = 1; Armijo at α = 1
    A0, A1 = dense_merit(nlp, 2.0, 1.0), dense_merit(nlp, 2.0 + dx, 1.0 + ds)
    assert A0 == 4.0 and abs(A1 - 3.848760597239781) < 1e-14
    assert A1 <= A0 + 1e-4 * 1.0 * D


def test_fraction_to_boundary_spec_example():
    """s = 1, Δs = −2 → τ_max = 0.995 · 1/2."""
    s, ds, tau = 1.0, -2.0, 0.995
    assert min(1.0, tau * s / (-ds)) == pytest.approx(0.4975, abs=1e-16)


@pytest.mark.parametrize("eta", [1e2, 1e4, 1e6])
def test_structured_chain_equals_dense_4x4(eta):
    """condense → T2 → expand equals the dense Eq.(4×4) solve (1e-8 relative)."""
    for seed, (n, m, N, ng, ngN, nc, ncN) in enumerate([(2, 1, 3, 2, 1, 1, 1), (3, 2, 4, 3, 2, 1, 1),
                                                        (4, 1, 5, 4, 2, 0, 0), (1, 1, 2, 1, 1, 1, 0)]):
        p = random_lq_ocp(n, m, N, 2, seed=40 + seed, ng=ng, ngN=ngN, nc=nc, ncN=ncN, eta=eta)
        res, _ = ipm_step_oracle(p)
        for b in range(2):
            d = solve4x4(p, b)
            nlp = d["nlp"]
            x, u = split_X(nlp, d["dX"])
            assert rel(res["dx"][b], x) < 1e-8 and rel(res["du"][b], u) < 1e-8
            ndyn = nlp["n_dyn"]
            assert rel(res["dy"][b].ravel(), d["dy"][:ndyn]) < 1e-8
            lam = np.concatenate([res["dlam"][b].ravel(), res["dlamN"][b].ravel()])
            assert rel(lam, d["dy"][ndyn:]) < 1e-8
            ds = np.concatenate([res["ds"][b].ravel(), res["dsN"][b].ravel()])
            dz = np.concatenate([res["dz"][b].ravel(), res["dzN"][b].ravel()])
            assert rel(ds, d["ds"]) < 1e-8 and rel(dz, d["dz"]) < 1e-8


def test_lemma_shifted_system():
    """Lemma: same (Δx, Δs); duals shifted by ηc and η(g+s)."""
    for seed in range(10):
        p = random_lq_ocp(3, 2, 4, 2, seed=70 + seed, ng=2, ngN=1, nc=1, ncN=1, eta=10.0 ** (1 + seed % 4))
        for b in range(2):
            a = solve4x4(p, b)
            sh = solve_shifted(p, b)
            nlp = a["nlp"]
            eta = nlp["eta"]
            assert np.max(np.abs(a["dX"] - sh["dX"])) <= 1e-9 * (1 + np.max(np.abs(a["dX"])))
            assert np.max(np.abs(a["ds"] - sh["ds"])) <= 1e-9 * (1 + np.max(np.abs(a["ds"])))
            scale = 1 + np.max(np.abs(a["dy"]))
            assert np.max(np.abs((a["dy"] - eta * nlp["c"]) - sh["dy_shift"])) <= 1e-9 * scale * eta
            scale = 1 + np.max(np.abs(a["dz"]))
            assert np.max(np.abs((a["dz"] - eta * (nlp["g"] + nlp["s"])) - sh["dz_shift"])) <= 1e-9 * scale * eta


def test_descent_theorem_lq():
    """Theorem: D < 0, D = closed form, D = central FD slope of 𝒜."""
    p = random_lq_ocp(3, 2, 6, 4, seed=5, ng=2, ngN=1, nc=1, ncN=1, eta=1e3)
    res, _ = ipm_step_oracle(p)
    for b in range(4):
        D, Dc = res["D"][b], res["D_closed"][b]
        assert D < 0 and abs(D - Dc) <= 1e-9 * abs(Dc)
        h = 1e-6
        fd = (ipm_merit_oracle(p, res, b, h) - ipm_merit_oracle(p, res, b, -h)) / (2 * h)
        assert abs(fd - D) <= max(1e-6, 1e-4 * abs(D)), (fd, D)


def test_descent_theorem_cartpole_and_model_pins():
    """C4 recipe at N=20: D < 0 equals the closed form and the FD slope of 𝒜 evaluated with the
    nonlinear cart-pole dynamics (so the generator's Jacobians are the model's)."""
    p = cartpole_c4(6, seed=2511, N=20)
    res, _ = ipm_step_oracle(p)
    assert np.all(res["status"] == 0)
    for b in range(6):
        D = res["D"][b]
        assert D < 0 and abs(D - res["D_closed"][b]) <= 1e-8 * abs(D)
        h = 1e-6
        fd = (ipm_merit_oracle(p, res, b, h) - ipm_merit_oracle(p, res, b, -h)) / (2 * h)
        assert abs(fd - D) <= max(1e-6, 1e-4 * abs(D)), (fd, D)


def test_cartpole_model_two_implementations_agree():
    prm = synth.ipm_workloads.cartpole_params().numpy()
    rng = np.random.default_rng(1)
    for _ in range(20):
        x = rng.uniform(-3, 3, 4)
        u = rng.uniform(-5, 5, 1)
        a = cartpole_step_oracle(prm, x, u)
        b = cartpole_step_torch(torch.from_numpy(prm), torch.from_numpy(x), torch.from_numpy(u)).numpy()
        assert np.max(np.abs(a - b)) <= 1e-14 * (1 + np.max(np.abs(a)))


def test_cartpole_jacobians_central_fd():
    """Jacobians A_i, B_i of the C4 generator equal central finite differences."""
    p = cartpole_c4(2, seed=3, N=5)
    prm = p.data["model_params"]
    for b in range(2):
        for i in range(5):
            x = p.it["x"][b, i].clone()
            u = p.it["u"][b, i].clone()
            A = p.data["A"][b, i].reshape(4, 4).T
            B = p.data["B"][b, i].reshape(1, 4).T
            h = 1e-6
            for j in range(4):
                e = torch.zeros(4, dtype=torch.float64); e[j] = h
                col = (cartpole_step_torch(prm, x + e, u) - cartpole_step_torch(prm, x - e, u)) / (2 * h)
                assert torch.max(torch.abs(col - A[:, j])) < 1e-5
            e = torch.tensor([h], dtype=torch.float64)
            col = (cartpole_step_torch(prm, x, u + e) - cartpole_step_torch(prm, x, u - e)) / (2 * h)
            assert torch.max(torch.abs(col - B[:, 0])) < 1e-5


def test_line_search_rules_and_positivity():
    """α_p = α_max β^k with α_max the fraction-to-boundary cap; s, z stay positive
    (S:277); merit decreases."""
    p = cartpole_c4(8, seed=9, N=20)
    res, it = ipm_step_oracle(p)
    for b in range(8):
        ds = np.concatenate([res["ds"][b].ravel(), res["dsN"][b].ravel()])
        s = np.concatenate([p.it["s"][b].numpy().ravel(), p.it["sN"][b].numpy().ravel()])
        neg = ds < 0
        amax = min(1.0, np.min(0.995 * s[neg] / -ds[neg])) if neg.any() else 1.0
        assert res["alpha_p"][b] == pytest.approx(amax * 0.5 ** res["n_backtracks"][b], rel=1e-15)
        assert res["merit_acc"][b] < res["merit0"][b]
        assert np.all(it["s"][b] > 0) and np.all(it["z"][b] > 0) and np.all(it["sN"][b] > 0)


def test_c4_ls_variant_backtracks():
    """C4-LS exercises backtracking: several backtracks per step."""
    p = cartpole_c4(16, seed=2511, N=20, variant="C4-LS")
    res, _ = ipm_step_oracle(p)
    assert np.all(res["status"] == 0)
    assert np.all(res["D"] < 0)
    assert np.max(res["n_backtracks"]) >= 2


def test_kkt_point_gives_zero_direction():
    """at an exact barrier-KKT point the step is zero (zero rhs)."""
    p = random_lq_ocp(2, 1, 3, 1, seed=2, ng=1, ngN=1, nc=0, ncN=0, eta=100.0)
    n, m, N = 2, 1, 3
    d = solve4x4(p, 0)
    nlp = d["nlp"]
    # move the iterate to the Newton point of the (linear-quadratic) barrier problem is not
    # closed-form; instead construct a KKT point: c = 0, g + s = 0, sz = μ, ∇ₓL = 0.
    D = p.data
    It = p.it
    D["dres"].zero_()
    D["s0"][0] = It["x"][0, 0]
    It["s"][0] = -D["gv"][0]
    It["sN"][0] = -D["gvN"][0]
    It["s"][0].clamp_(min=0.1)
    It["sN"][0].clamp_(min=0.1)
    D["gv"][0] = -It["s"][0]
    D["gvN"][0] = -It["sN"][0]
    It["z"][0] = It["mu"][0] / It["s"][0]
    It["zN"][0] = It["mu"][0] / It["sN"][0]
    nlp = solve4x4(p, 0)["nlp"]
    _, (gx, _, _, _), _ = kkt4x4(nlp)
    # choose the gradient so that ∇ₓL = 0
    w = n + m
    g_new = nlp["grad"] - gx
    for i in range(N):
        D["gradf"][0, i] = torch.from_numpy(g_new[i * w:(i + 1) * w])
    D["gradfN"][0] = torch.from_numpy(g_new[N * w:])
    res, _ = ipm_step_oracle(p.select(slice(0, 1)))
    for k in ("dx", "du", "dy", "ds", "dz"):
        assert np.max(np.abs(res[k][0])) < 1e-10, k


def test_dense_4x4_ldlt_equals_lu():
    """North star (a): the full 4×4-block KKT system (Eq.(4×4)) solved by the dense
    Bunch-Kaufman LDLᵀ equals the LU solution and the structured chain condense → T2 → expand."""
    for seed, kw in ((4, dict(ng=2, ngN=1, nc=1, ncN=1)), (5, dict(ng=3, ngN=2, nc=0, ncN=0))):
        p = random_lq_ocp(3, 2, 5, 2, seed=seed, **kw)
        res, _ = ipm_step_oracle(p)
        for b in range(2):
            lu = solve4x4(p, b)
            ld = solve4x4(p, b, method="ldl")
            for k in ("dX", "ds", "dy", "dz"):
                if lu[k].size:
                    assert rel(ld[k], lu[k]) <= 1e-10, k
            N = p.N  # the chain's (Δx, Δu) in the dense ordering (x_0, u_0, ..., x_N)
            dx = np.concatenate([np.concatenate([res["dx"][b][i], res["du"][b][i]]) for i in range(N)]
                                + [res["dx"][b][N]])
            assert rel(dx, ld["dX"]) <= 1e-8
