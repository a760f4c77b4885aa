"""Diagnostic: actual GPU-vs-oracle errors of ipm_solve (f1) per workload and iteration budget.
Prints one line per case: status/iters agreement and the normwise relative error of each block."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2509_16370_b200 as m
from oracle.ipm_solve import SolveSettings, ipm_solve_oracle
from synth.ipm_workloads import cartpole_c4, double_integrator_ocp, quadrotor_ipm, random_lq_ocp


def rel(g, o):
    g = np.asarray(g, dtype=np.float64).reshape(len(g), -1)
    o = np.asarray(o, dtype=np.float64).reshape(len(o), -1)
    if g.size == 0:
        return 0.0
    return float(np.max(np.max(np.abs(g - o), axis=1) / np.maximum(np.max(np.abs(o), axis=1), 1e-300)))


cases = [("dblint", lambda: double_integrator_ocp(batch=3), {})]
for (nx, nu, ng, ngN, nc, ncN) in [(4, 2, 2, 1, 0, 0), (4, 1, 3, 2, 0, 0), (3, 2, 2, 1, 1, 1), (8, 3, 4, 2, 2, 1), (12, 4, 6, 2, 2, 0)]:
    cases.append((f"lq{nx}{nu}{ng}{ngN}{nc}{ncN}",
                  lambda nx=nx, nu=nu, ng=ng, ngN=ngN, nc=nc, ncN=ncN: random_lq_ocp(nx, nu, 12, 24, seed=nx * 7 + ng, ng=ng, ngN=ngN, nc=nc, ncN=ncN, eta=1e4), {}))
for it in (1, 2, 3, 4, 6, 10, 20):
    cases.append((f"cartpole_it{it}", lambda: cartpole_c4(16, N=40), dict(max_iters=it)))
for it in (1, 2, 4, 8):
    cases.append((f"quad_it{it}", lambda: quadrotor_ipm(24, N=20), dict(max_iters=it)))
cases.append(("quad_conv", lambda: quadrotor_ipm(6, N=20), {}))
for name, mk, S in cases:
    b = mk()
    bg = b.to("cuda")
    rep = m.ipm_solve(bg, **S)
    torch.cuda.synchronize()
    it_o, rep_o = ipm_solve_oracle(b, SolveSettings(**S))
    rg = {k: v.cpu().numpy() for k, v in rep.items()}
    ig = {k: v.cpu().numpy() for k, v in bg.it.items()}
    errs = {k: rel(ig[k], it_o[k]) for k in ("x", "u", "s", "z", "y", "lam") if it_o[k].size}
    print(name, "status_eq", np.array_equal(rg["status"], rep_o["status"]), "iters_eq", np.array_equal(rg["iters"], rep_o["iters"]),
          "iters", rep_o["iters"].min(), rep_o["iters"].max(), "mu", rel(rg["mu"], rep_o["mu"]), "eta", rel(rg["eta"], rep_o["eta"]),
          " ".join(f"{k}={v:.2e}" for k, v in errs.items()), flush=True)
