"""GPU checks of the caller-evaluated line search (ipm_direction + ipm_merit + ipm_update; SURVEY §8(f4):
user models): the direction equals ipm_step's (same kernel up to the line search), ipm_merit at
caller-evaluated trial values equals the oracle's merit at the same values, and a line search run
by the caller through ipm_merit + ipm_update reproduces ipm_step's iterate."""
import numpy as np
import pytest
import torch

from oracle.ipm_solve import evaluate, merit_at_values
from synth.ipm_workloads import cartpole_c4, random_lq_ocp

pytestmark = pytest.mark.gpu


def rr():
    import paper_2509_16370_b200 as m
    return m


def trial_values(b_cpu, res, alpha):
    a = alpha[:, None, None]
    x = b_cpu.it["x"].numpy() + a * res["dx"]
    u = b_cpu.it["u"].numpy() + a * res["du"]
    d = evaluate(b_cpu, x, u)
    return {k: d[k] for k in ("fval", "dres", "ce", "ceN", "gv", "gvN")}


@pytest.mark.parametrize("make", [lambda: random_lq_ocp(4, 2, 12, 16, seed=3, ng=2, ngN=1, nc=1, ncN=1, eta=1e4),
                                  lambda: cartpole_c4(16, N=30)])
def test_direction_merit_update_reproduce_ipm_step(make):
    m = rr()
    b = make()
    g1 = b.to("cuda")
    g2 = b.to("cuda")
    ref = m.ipm_step(g1)                           # built-in line search
    res = m.ipm_direction(g2)                      # rows a1-a7 only
    torch.cuda.synchronize()
    for k in ("dx", "du", "ds", "dy", "dz", "D", "merit0"):
        assert torch.equal(res[k], ref[k]), k
    assert torch.equal(g2.it["x"], b.it["x"].cuda())  # iterate untouched
    resn = {k: v.cpu().numpy() for k, v in res.items()}
    # the caller's Armijo ladder with its own model evaluation (reading R12 constants)
    alpha = resn["alpha_p"].copy()
    accepted = np.zeros(b.batch, dtype=bool)
    for _ in range(51):
        tv = trial_values(b, resn, alpha)
        merit = m.ipm_merit(g2, res, torch.as_tensor(alpha, device="cuda"),
                            {k: torch.as_tensor(v, device="cuda").contiguous() for k, v in tv.items()}).cpu().numpy()
        want = merit_at_values(b, resn, alpha, tv)
        fin = np.isfinite(want)
        assert np.array_equal(fin, np.isfinite(merit))
        assert np.all(np.abs(merit[fin] - want[fin]) <= 1e-10 * np.maximum(1.0, np.abs(want[fin])))
        ok = fin & (merit <= resn["merit0"] + 1e-4 * alpha * resn["D"]) & ~accepted
        accepted |= ok
        if accepted.all():
            break
        alpha = np.where(accepted, alpha, 0.5 * alpha)
    assert accepted.all()
    m.ipm_update(g2, res, torch.as_tensor(alpha, device="cuda"), res["alpha_d"])
    torch.cuda.synchronize()
    assert np.allclose(alpha, ref["alpha_p"].cpu().numpy(), rtol=0, atol=0)
    for k in ("x", "u", "s", "z", "y"):
        a_, b_ = g2.it[k].cpu().numpy(), g1.it[k].cpu().numpy()
        assert np.max(np.abs(a_ - b_)) <= 1e-12 * max(1.0, np.max(np.abs(b_))), k
