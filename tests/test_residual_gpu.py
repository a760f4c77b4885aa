"""GPU parity of rr_residual (the paper's residual callback) against the oracle's block
residual (pinned to the dense definition K[x; y] + [s; c]), and iterative refinement through
rr_residual + rr_solve(RR_FLAG_ACCUMULATE)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
TOL = 1e-9


def rr():
    import paper_2509_16370_b200 as m
    return m


def rel(g, o):
    g = np.asarray(g).reshape(g.shape[0], -1)
    o = np.asarray(o).reshape(o.shape[0], -1)
    if g.size == 0:
        return 0.0
    return float(np.max(np.max(np.abs(g - o), axis=1) / np.maximum(np.max(np.abs(o), axis=1), 1e-300)))


@pytest.mark.parametrize("nx,nu,N,batch", [(12, 4, 9, 37), (4, 1, 13, 33), (2, 1, 10, 17), (3, 2, 6, 21),
                                           (7, 6, 4, 11), (16, 16, 3, 5), (12, 4, 0, 4)])
@pytest.mark.parametrize("delta", [0.0, 1e-4, 1.0])
def test_residual_parity_random_candidate(nx, nu, N, batch, delta):
    p = synth.random_stable_lqr(nx, nu, N, batch, seed=nx + nu + N, delta=delta)
    g = torch.Generator().manual_seed(3)
    sol = {"x": torch.rand(batch, N + 1, nx, generator=g, dtype=torch.float64) * 2 - 1,
           "u": torch.rand(batch, N, nu, generator=g, dtype=torch.float64) * 2 - 1,
           "y": torch.rand(batch, N + 1, nx, generator=g, dtype=torch.float64) * 2 - 1}
    res, norms = rr().rr_residual(p.to("cuda"), {k: v.cuda() for k, v in sol.items()})
    torch.cuda.synchronize()
    o = oracle.residual_blocks(p, sol["x"].numpy(), sol["u"].numpy(), sol["y"].numpy())
    for k in ("q", "r", "c", "qN", "c0"):
        assert rel(res[k].cpu().numpy(), o["r" + k]) <= TOL, k
    assert rel(norms.cpu().numpy(), o["norms"]) <= TOL


def test_residual_of_solution_and_refinement():
    m = rr()
    p = synth.random_stable_lqr(12, 4, 40, 64, seed=8, delta=1e-4).to("cuda")
    F, st = m.rr_factor(p)
    sol = m.rr_solve(p, F)
    _, n0 = m.rr_residual(p, sol)
    torch.cuda.synchronize()
    scale = max(float(p.q.abs().max()), float(p.c0.abs().max()), 1.0)
    assert float(n0.max()) < 1e-11 * scale * 100
    ref = {k: sol[k].clone() for k in ("x", "u", "y")}
    # perturb, then one refinement step must restore the solution (exact linear correction)
    gen = torch.Generator(device="cuda").manual_seed(0)
    for k in ("x", "u", "y"):
        sol[k] += 1e-3 * torch.randn(sol[k].shape, generator=gen, device="cuda", dtype=torch.float64)
    norms = m.rr_refine(p, F, sol, iters=2)
    torch.cuda.synchronize()
    for k in ("x", "u", "y"):
        assert rel(sol[k].cpu().numpy(), ref[k].cpu().numpy()) <= 1e-10, k
    assert float(norms.max()) < 1e-9


def test_accumulate_flag_adds():
    m = rr()
    p = synth.random_stable_lqr(4, 1, 7, 9, seed=2, delta=1e-3).to("cuda")
    F, _ = m.rr_factor(p)
    a = m.rr_solve(p, F)
    b = {k: v.clone() for k, v in a.items()}
    m.rr_solve(p, F, out=b, accumulate=True)
    torch.cuda.synchronize()
    for k in ("x", "u", "y"):
        assert torch.allclose(b[k], 2 * a[k], rtol=1e-14, atol=0)


def test_residual_nonfinite_norm():
    m = rr()
    p = synth.random_stable_lqr(12, 4, 5, 6, seed=1).to("cuda")
    F, _ = m.rr_factor(p)
    sol = m.rr_solve(p, F)
    sol["x"][2, 3, 1] = float("nan")
    _, norms = m.rr_residual(p, sol)
    nrm = norms.cpu().numpy()
    assert np.all(np.isnan(nrm[2])) and np.all(np.isfinite(np.delete(nrm, 2, axis=0)))
