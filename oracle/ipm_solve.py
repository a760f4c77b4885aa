"""Full batched regularized-IPM solve -- TEST INFRASTRUCTURE ONLY.

Repeats the one-step oracle (ipm.py: condense -> T2 -> expand -> merit/D -> line search)
inside the outer loop of the regularized interior point method of §1.2.  The paper fixes the step
 but not the outer loop ("how/when μ and η change", SPEC Open Questions); this loop is
SPEC's ipm_solve / update_parameters and DESIGN.md reading R21:

  for k = 0 .. max_iters-1, per instance (converged / failed instances are frozen):
    1. evaluate the problem data at the iterate (model: quadratic cost with Hessian P and linear
       constraints, both exact from the reference data; dynamics linear (LQ) or the cart-pole
       model with its Jacobians)
    2. residuals  r_stat = ||∇ₓL||∞ (∇ₓL = ∇f + Cᵀy + C_eᵀλ + Gᵀz),
                  r_feas = max(||c||∞, ||c_e||∞, ||g + s||∞)   (c: initial-state and dynamics rows),
                  r_comp = ||S z − μ e||∞,  r_comp0 = ||S z||∞
    3. converged  if max(r_stat, r_feas, r_comp0) <= tol_kkt and μ <= 10 mu_min
    4. μ update   if max(r_stat, r_feas, r_comp) <= kappa μ:  μ <- max(mu_min, min(kappa_mu μ, μ^theta_mu))
    5. η update   if k >= 5 and r_feas > tol_kkt and r_feas > 0.9 r_feas(k-5):  η <- min(eta_max, kappa_eta η)
    6. one IPM step at (data(x_k), μ, η); a line-search failure ends the instance (status 5);
     with settings.linear_merit the step's trial merits use the linearised dynamics (reading R22)
  instances still running after max_iters end with status MAXITER (6).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch

from .ipm import ipm_step_oracle

ST_CONVERGED, ST_LS_FAILED, ST_MAXITER = 0, 5, 6


@dataclasses.dataclass
class SolveSettings:
    mu_min: float = 1e-9
    kappa: float = 10.0
    kappa_mu: float = 0.2
    theta_mu: float = 1.5
    eta_max: float = 1e8
    kappa_eta: float = 10.0
    tol_kkt: float = 1e-6
    max_iters: int = 100
    tau: float = 0.995
    armijo_c: float = 1e-4
    beta: float = 0.5
    max_backtracks: int = 50
    linear_merit: bool = False   # reading R22: the step's trial merits on the linearised dynamics


def _unpack(P, n):
    F = np.zeros(P.shape[:-1] + (n, n))
    k = 0
    for c in range(n):
        for r in range(c, n):
            F[..., r, c] = P[..., k]
            F[..., c, r] = P[..., k]
            k += 1
    return F


def _cm(a, rows, cols):
    return np.swapaxes(a.reshape(a.shape[:-1] + (cols, rows)), -1, -2)


def evaluate(ref, x, u):
    """Problem data at (x, u) from the reference batch `ref` (an IPMBatch on CPU whose data were
    evaluated at ref.it x, u).  Returns a dict with the IPMBatch data layout."""
    n, m, N = ref.nx, ref.nu, ref.N
    d = {k: v.detach().cpu().numpy().astype(np.float64).copy() for k, v in ref.data.items()}
    xr = ref.it["x"].cpu().numpy()
    ur = ref.it["u"].cpu().numpy()
    b = xr.shape[0]
    dx, du = x - xr, u - ur
    dz = np.concatenate([dx[:, :N], du], axis=-1)                   # [b, N, n+m]
    dN = dx[:, N]
    P = np.zeros((b, N, n + m, n + m))
    P[..., :n, :n] = _unpack(d["Q"], n)
    P[..., :n, n:] = _cm(d["M"], n, m)
    P[..., n:, :n] = np.swapaxes(_cm(d["M"], n, m), -1, -2)
    P[..., n:, n:] = _unpack(d["R"], m)
    PN = _unpack(d["QN"], n)
    Pdz = np.einsum("bisr,bir->bis", P, dz)
    PNd = np.einsum("bsr,br->bs", PN, dN)
    out = dict(d)
    out["fval"] = (d["fval"] + (d["gradf"] * dz).sum((-1, -2)) + 0.5 * (dz * Pdz).sum((-1, -2))
                   + (d["gradfN"] * dN).sum(-1) + 0.5 * (dN * PNd).sum(-1))
    out["gradf"] = d["gradf"] + Pdz
    out["gradfN"] = d["gradfN"] + PNd
    w = n + m
    if ref.ng:
        out["gv"] = d["gv"] + np.einsum("bikr,bir->bik", _cm(d["Gj"], ref.ng, w), dz)
    if ref.ngN:
        out["gvN"] = d["gvN"] + np.einsum("bkr,br->bk", _cm(d["GjN"], ref.ngN, n), dN)
    if ref.nc:
        out["ce"] = d["ce"] + np.einsum("bikr,bir->bik", _cm(d["Ce"], ref.nc, w), dz)
    if ref.ncN:
        out["ceN"] = d["ceN"] + np.einsum("bkr,br->bk", _cm(d["CeN"], ref.ncN, n), dN)
    if ref.model == 0:   # linear dynamics: d(x, u) - x_{i+1} exact from the reference
        A, B = _cm(d["A"], n, n), _cm(d["B"], n, m)
        out["dres"] = (d["dres"] + np.einsum("bisr,bir->bis", A, dx[:, :N]) + np.einsum("bisr,bir->bis", B, du)
                       - dx[:, 1:])
    else:                # cart-pole / quadrotor (the workload definitions, synth/ipm_workloads.py)
        from synth.ipm_workloads import cartpole_step_torch, quadrotor_step_torch
        step = cartpole_step_torch if ref.model == 1 else quadrotor_step_torch
        prm = torch.as_tensor(d["model_params"])
        xi = torch.as_tensor(x[:, :N].reshape(-1, n))
        ui = torch.as_tensor(u.reshape(-1, m))
        fx = step(prm, xi, ui).numpy().reshape(b, N, n)
        out["dres"] = fx - x[:, 1:]
        jac = torch.func.vmap(torch.func.jacrev(lambda xx, uu: step(prm, xx, uu), argnums=(0, 1)))
        Jx, Ju = jac(xi, ui)
        out["A"] = np.swapaxes(Jx.numpy(), -1, -2).reshape(b, N, n * n)   # column-major
        out["B"] = np.swapaxes(Ju.numpy(), -1, -2).reshape(b, N, n * m)
    return out


def residuals(ref, d, it, mu):
    """(r_stat, r_feas, r_comp, r_comp0) per instance at iterate `it` with data `d` (numpy)."""
    n, m, N, ng, ngN, nc, ncN = ref.nx, ref.nu, ref.N, ref.ng, ref.ngN, ref.nc, ref.ncN
    w = n + m
    x, u, y = it["x"], it["u"], it["y"]
    A, B = _cm(d["A"], n, n), _cm(d["B"], n, m)
    gx = d["gradf"][..., :n] - y[:, :N] + np.einsum("bisr,bis->bir", A, y[:, 1:])
    gu = d["gradf"][..., n:] + np.einsum("bisr,bis->bir", B, y[:, 1:])
    gN = d["gradfN"] - y[:, N]
    g = np.concatenate([gx, gu], axis=-1)
    feas = [np.abs(d["s0"] - x[:, 0]).max(-1), np.abs(d["dres"]).reshape(x.shape[0], -1).max(-1, initial=0.0)]
    comp = [np.zeros(x.shape[0])]
    comp0 = [np.zeros(x.shape[0])]
    if ng:
        g = g + np.einsum("bikr,bik->bir", _cm(d["Gj"], ng, w), it["z"])
        feas.append(np.abs(d["gv"] + it["s"]).reshape(x.shape[0], -1).max(-1))
        sz = it["s"] * it["z"]
        comp.append(np.abs(sz - mu[:, None, None]).reshape(x.shape[0], -1).max(-1))
        comp0.append(np.abs(sz).reshape(x.shape[0], -1).max(-1))
    if ngN:
        gN = gN + np.einsum("bkr,bk->br", _cm(d["GjN"], ngN, n), it["zN"])
        feas.append(np.abs(d["gvN"] + it["sN"]).max(-1))
        szN = it["sN"] * it["zN"]
        comp.append(np.abs(szN - mu[:, None]).max(-1))
        comp0.append(np.abs(szN).max(-1))
    if nc:
        g = g + np.einsum("bikr,bik->bir", _cm(d["Ce"], nc, w), it["lam"])
        feas.append(np.abs(d["ce"]).reshape(x.shape[0], -1).max(-1))
    if ncN:
        gN = gN + np.einsum("bkr,bk->br", _cm(d["CeN"], ncN, n), it["lamN"])
        feas.append(np.abs(d["ceN"]).max(-1))
    r_stat = np.maximum(np.abs(g).reshape(x.shape[0], -1).max(-1, initial=0.0), np.abs(gN).max(-1))
    return r_stat, np.max(feas, axis=0), np.max(comp, axis=0), np.max(comp0, axis=0)


def ipm_solve_oracle(batch, settings: SolveSettings = SolveSettings(), nthreads=8, record=False):
    """Solve every instance of `batch` (an IPMBatch, CPU) from its iterate.  Returns
    (final iterate dict, report dict: status, iters, mu, eta, r_stat, r_feas, r_comp0 [+ history])."""
    from synth.ipm_workloads import IPMBatch, MODEL_LQ
    ref = batch
    it = {k: v.detach().cpu().numpy().astype(np.float64).copy() for k, v in batch.it.items()}
    b = batch.batch
    S = settings
    status = np.full(b, -1, dtype=np.int32)          # -1 = running
    iters = np.zeros(b, dtype=np.int32)
    hist = np.zeros((b, 5))
    rep = {k: np.zeros(b) for k in ("r_stat", "r_feas", "r_comp0")}
    trace = []
    for k in range(S.max_iters + 1):
        act = status < 0
        if not act.any():
            break
        d = evaluate(ref, it["x"], it["u"])
        rs, rf, rc, rc0 = residuals(ref, d, it, it["mu"])
        for key, val in (("r_stat", rs), ("r_feas", rf), ("r_comp0", rc0)):
            rep[key][act] = val[act]
        conv = act & (np.maximum(np.maximum(rs, rf), rc0) <= S.tol_kkt) & (it["mu"] <= 10 * S.mu_min)
        status[conv] = ST_CONVERGED
        act &= ~conv
        if k == S.max_iters:
            status[act] = ST_MAXITER
            break
        dec = act & (np.maximum(np.maximum(rs, rf), rc) <= S.kappa * it["mu"])
        new_mu = np.maximum(S.mu_min, np.minimum(S.kappa_mu * it["mu"], it["mu"] ** S.theta_mu))
        it["mu"] = np.where(dec, new_mu, it["mu"])
        stag = act & (k >= 5) & (rf > S.tol_kkt) & (rf > 0.9 * hist[:, k % 5])
        it["eta"] = np.where(stag, np.minimum(S.eta_max, S.kappa_eta * it["eta"]), it["eta"])
        hist[:, k % 5] = np.where(act, rf, hist[:, k % 5])
        idx = np.nonzero(act)[0]
        # reading R22: with linear_merit the step's line search evaluates 𝒜 at the trial
        # points through the linearisation at the iterate (the LQ merit on the re-evaluated data)
        cur = IPMBatch(ref.nx, ref.nu, ref.N, ref.ng, ref.ngN, ref.nc, ref.ncN,
                       MODEL_LQ if S.linear_merit else ref.model,
                       {kk: torch.as_tensor(v[idx] if kk != "model_params" else v) for kk, v in d.items()},
                       {kk: torch.as_tensor(v[idx]) for kk, v in it.items()})
        res, it2 = ipm_step_oracle(cur, tau=S.tau, armijo_c=S.armijo_c, beta=S.beta,
                                   max_backtracks=S.max_backtracks, nthreads=nthreads)
        st = res["status"]
        for kk, v in it2.items():
            it[kk][idx] = np.where(np.reshape(st == 0, (-1,) + (1,) * (v.ndim - 1)), v, it[kk][idx])
        status[idx[st != 0]] = st[st != 0]
        iters[idx] += 1
        if record:
            trace.append(dict(k=k, active=idx.copy(), alpha_p=res["alpha_p"].copy(), mu=it["mu"].copy(),
                              eta=it["eta"].copy(), r=(rs.copy(), rf.copy(), rc.copy())))
    rep.update(status=status, iters=iters, mu=it["mu"].copy(), eta=it["eta"].copy())
    if record:
        rep["trace"] = trace
    return it, rep


def merit_at_values(batch, res, alpha, trial):
    """𝒜(x̄ + αΔx, s + αΔs; y, λ, z, μ, η) from caller-evaluated values at the trial point (P:61-66,
    reading R14): f − μΣlog(s+αΔs) + yᵀc + λᵀc_e + zᵀ(g+s+αΔs) + η/2(‖c‖² + ‖c_e‖² + ‖g+s+αΔs‖²),
    c = (s_0 − x_0 − αΔx_0, d_i(trial) − x_{i+1}(trial)).  Every argument numpy; returns [b]."""
    it = {k: np.asarray(v.detach().cpu().numpy() if hasattr(v, "detach") else v, dtype=np.float64)
          for k, v in batch.it.items()}
    s0 = np.asarray(batch.data["s0"].cpu().numpy() if hasattr(batch.data["s0"], "cpu") else batch.data["s0"])
    b = it["mu"].shape[0]
    al = np.asarray(alpha, dtype=np.float64)
    out = np.zeros(b)
    for k in range(b):
        a = al[k]
        terms_lin, terms_pen, bar = 0.0, 0.0, 0.0
        ok = True
        for sk, dk, zk, gk in (("s", "ds", "z", "gv"), ("sN", "dsN", "zN", "gvN")):
            if it[sk].size == 0:
                continue
            sa = it[sk][k] + a * res[dk][k]
            if np.any(sa <= 0):
                ok = False
            ga = trial[gk][k] + sa
            bar += np.sum(np.log(np.where(sa > 0, sa, 1.0)))
            terms_lin += np.sum(it[zk][k] * ga)
            terms_pen += np.sum(ga * ga)
        for lk, ck in (("lam", "ce"), ("lamN", "ceN")):
            if it[lk].size == 0:
                continue
            terms_lin += np.sum(it[lk][k] * trial[ck][k])
            terms_pen += np.sum(trial[ck][k] ** 2)
        c0 = s0[k] - (it["x"][k, 0] + a * res["dx"][k, 0])
        cd = trial["dres"][k]
        terms_lin += np.sum(it["y"][k, 0] * c0) + np.sum(it["y"][k, 1:] * cd)
        terms_pen += np.sum(c0 * c0) + np.sum(cd * cd)
        out[k] = (trial["fval"][k] - it["mu"][k] * bar + terms_lin + 0.5 * it["eta"][k] * terms_pen) if ok else np.nan
    return out
