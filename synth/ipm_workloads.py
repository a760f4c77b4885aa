"""Seeded synthetic regularized-IPM workloads (inputs only; no method arithmetic).

An IPMBatch holds, per instance, the stagewise OCP data of §1.1 evaluated at the current iterate
(cost gradient, a positive-definite Hessian approximation P, dynamics Jacobians and
residuals, equality/inequality values and Jacobians) plus the iterate (x, s, y, z, μ, η) of
§1.2, in the C-ABI layout of include/rr.h (ipm_* structs).  Model ids: 0 = LQ (linear dynamics
and constraints, quadratic cost), 1 = cart-pole (C4), 2 = quadrotor (the C5 model of §8(d)).

The cart-pole dynamics below are the workload DEFINITION used to produce iterates and their
Jacobians (torch autograd); the oracle and the CUDA library each carry their own copy of the
same equations for evaluating trial points of the line search.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict

import torch

from .workloads import OP_A, OP_B, OP_L, colmajor, from_colmajor, pack_lower, quadrotor_f, sym_size, uniform

MODEL_LQ, MODEL_CARTPOLE, MODEL_QUADROTOR = 0, 1, 2
N_MODEL_PARAMS = 8

DATA_FIELDS = ("s0", "fval", "gradf", "gradfN", "Q", "M", "R", "QN", "A", "B", "dres",
               "ce", "Ce", "ceN", "CeN", "gv", "Gj", "gvN", "GjN", "model_params")
ITER_FIELDS = ("x", "u", "s", "z", "sN", "zN", "y", "lam", "lamN", "mu", "eta")

# extra operand ids for the counter-based generator
OP_X, OP_U, OP_S0, OP_G, OP_GV, OP_CE, OP_CV, OP_Y, OP_LAM, OP_DRES, OP_P = range(16, 27)


@dataclasses.dataclass
class IPMBatch:
    nx: int
    nu: int
    N: int
    ng: int
    ngN: int
    nc: int
    ncN: int
    model: int
    data: Dict[str, torch.Tensor]
    it: Dict[str, torch.Tensor]

    @property
    def batch(self) -> int:
        return self.it["mu"].shape[0]

    def to(self, device) -> "IPMBatch":
        return IPMBatch(self.nx, self.nu, self.N, self.ng, self.ngN, self.nc, self.ncN, self.model,
                        {k: v.to(device) for k, v in self.data.items()},
                        {k: v.to(device) for k, v in self.it.items()})

    def clone(self) -> "IPMBatch":
        return IPMBatch(self.nx, self.nu, self.N, self.ng, self.ngN, self.nc, self.ncN, self.model,
                        {k: v.clone() for k, v in self.data.items()},
                        {k: v.clone() for k, v in self.it.items()})

    def select(self, idx) -> "IPMBatch":
        d = {k: (v if k == "model_params" else v[idx].contiguous()) for k, v in self.data.items()}
        i = {k: v[idx].contiguous() for k, v in self.it.items()}
        return IPMBatch(self.nx, self.nu, self.N, self.ng, self.ngN, self.nc, self.ncN, self.model, d, i)


def _zeros(*s, device="cpu"):
    return torch.zeros(*s, dtype=torch.float64, device=device)


def random_lq_ocp(nx, nu, N, batch, seed, ng=2, ngN=1, nc=1, ncN=1, mu=0.1, eta=1e3,
                  first=0, device="cpu") -> IPMBatch:
    """A batch of linear-quadratic OCP iterates with stage equalities and inequalities (model LQ).
    P_i = L Lᵀ/(n+m) + blkdiag(0.1 I, I) (PD, as P:88 requires), A_i stable, random iterate with
    s = max(-g, 1e-2) and z = μ/s."""
    dev = torch.device(device)
    inst = torch.arange(first, first + batch, dtype=torch.int64, device=dev)
    st = torch.arange(N, dtype=torch.int64, device=dev)
    n, m, k = nx, nu, nx + nu
    Ah = uniform(seed, inst, st, OP_A, n * n)
    A = 0.95 * Ah / torch.linalg.vector_norm(Ah, dim=-1, keepdim=True)
    B = uniform(seed, inst, st, OP_B, n * m) / math.sqrt(n)
    Lf = from_colmajor(uniform(seed, inst, st, OP_L, k * k), k, k)
    P = Lf @ Lf.transpose(-1, -2) / k
    P[..., :n, :n] += 0.1 * torch.eye(n, dtype=P.dtype, device=dev)
    P[..., n:, n:] += torch.eye(m, dtype=P.dtype, device=dev)
    LN = from_colmajor(uniform(seed, inst, 0, OP_L + 8, n * n), n, n)
    PN = LN @ LN.transpose(-1, -2) / n + torch.eye(n, dtype=torch.float64, device=dev)
    x = uniform(seed, inst, torch.arange(N + 1, device=dev), OP_X, n)
    u = uniform(seed, inst, st, OP_U, m)
    z_st = torch.cat([x[:, :N], u], dim=-1)                       # [b, N, n+m]
    p_lin = uniform(seed, inst, st, OP_P, k)
    pN_lin = uniform(seed, inst, N, OP_P, n)
    gradf = (P @ z_st.unsqueeze(-1)).squeeze(-1) + p_lin
    gradfN = (PN @ x[:, N].unsqueeze(-1)).squeeze(-1) + pN_lin
    fval = (0.5 * (z_st * (P @ z_st.unsqueeze(-1)).squeeze(-1)).sum((-1, -2)) + (p_lin * z_st).sum((-1, -2))
            + 0.5 * (x[:, N] * (PN @ x[:, N].unsqueeze(-1)).squeeze(-1)).sum(-1) + (pN_lin * x[:, N]).sum(-1))
    dres = 0.1 * uniform(seed, inst, st, OP_DRES, n)
    s0 = x[:, 0] + 0.1 * uniform(seed, inst, 0, OP_S0, n)
    Gj = uniform(seed, inst, st, OP_G, ng * k)
    gv = uniform(seed, inst, st, OP_GV, ng) * 0.6 - 0.4
    GjN = uniform(seed, inst, N, OP_G, ngN * n)
    gvN = uniform(seed, inst, N, OP_GV, ngN) * 0.6 - 0.4
    Ce = uniform(seed, inst, st, OP_CE, nc * k)
    ce = 0.1 * uniform(seed, inst, st, OP_CV, nc)
    CeN = uniform(seed, inst, N, OP_CE, ncN * n)
    ceN = 0.1 * uniform(seed, inst, N, OP_CV, ncN)
    s = torch.clamp(-gv, min=1e-2)
    sN = torch.clamp(-gvN, min=1e-2)
    mu_t = torch.full((batch,), float(mu), dtype=torch.float64, device=dev)
    eta_t = torch.full((batch,), float(eta), dtype=torch.float64, device=dev)
    data = dict(s0=s0, fval=fval, gradf=gradf, gradfN=gradfN, Q=pack_lower(P[..., :n, :n]),
                M=colmajor(P[..., :n, n:].contiguous()), R=pack_lower(P[..., n:, n:]), QN=pack_lower(PN),
                A=A, B=B, dres=dres, ce=ce, Ce=Ce, ceN=ceN, CeN=CeN, gv=gv, Gj=Gj, gvN=gvN, GjN=GjN,
                model_params=_zeros(N_MODEL_PARAMS, device=dev))
    it = dict(x=x, u=u, s=s, z=mu / s, sN=sN, zN=mu / sN, y=0.1 * uniform(seed, inst, torch.arange(N + 1, device=dev), OP_Y, n),
              lam=0.1 * uniform(seed, inst, st, OP_LAM, nc), lamN=0.1 * uniform(seed, inst, N, OP_LAM, ncN),
              mu=mu_t, eta=eta_t)
    data = {k2: v.contiguous() for k2, v in data.items()}
    it = {k2: v.contiguous() for k2, v in it.items()}
    return IPMBatch(nx, nu, N, ng, ngN, nc, ncN, MODEL_LQ, data, it)


# ----------------------------------------------------------------------------- cart-pole (C4)
def cartpole_params(dt=0.05, mc=1.0, mp=0.1, l=0.5, g=9.81, device="cpu"):
    p = _zeros(N_MODEL_PARAMS, device=device)
    p[:5] = torch.tensor([dt, mc, mp, l, g], dtype=torch.float64)
    return p


def cartpole_step_torch(prm, x, u):
    """Explicit-Euler cart-pole; x = (p, θ, ṗ, θ̇) with θ from the hanging position (φ = θ − π
    from upright enters the classic equations); u = (F,)."""
    dt, mc, mp, l, g = (prm[i] for i in range(5))
    phi = x[..., 1] - math.pi
    sp, cp = torch.sin(phi), torch.cos(phi)
    thd, F = x[..., 3], u[..., 0]
    mt = mc + mp
    tmp = (F + mp * l * thd * thd * sp) / mt
    thdd = (g * sp - cp * tmp) / (l * (4.0 / 3.0 - mp * cp * cp / mt))
    pdd = tmp - mp * l * thdd * cp / mt
    return torch.stack([x[..., 0] + dt * x[..., 2], x[..., 1] + dt * x[..., 3],
                        x[..., 2] + dt * pdd, x[..., 3] + dt * thdd], dim=-1)


def cartpole_c4(batch, seed=2511, N=100, variant="C4", mu=0.1, eta=1e4, first=0, device="cpu") -> IPMBatch:
    """C4 (BASELINE configs[3]): cart-pole swing-up iterates, n=4, m=1, N=100,
    dt=0.05, cost ½(x−x_g)ᵀdiag(1,1,.1,.1)(x−x_g) + ½·0.01u², Q_N = 100 I, x_g = (0, π, 0, 0);
    inequalities u ≤ 3, −u ≤ 3, p ≤ 0.5, −p ≤ 0.5 (n_g = 4) and terminal ±p ≤ 0.5 (2).
    Iterate: s_0 = (0.5U, 0.3U, 0, 0); x̄ = rollout of ū = 5U with defects 1e-3U;
    s = max(−g, 1e-2), z = μ/s, y = 0.1U, μ = 0.1, η = 1e4.
    variant "C4-LS" (line-search stress): dt = 0.2, bounds ±100, s_0 = (0.5U, 3U, 2U, 8U), defects 0.5U."""
    dev = torch.device(device)
    n, m, k = 4, 1, 5
    ls = variant == "C4-LS"
    dt = 0.2 if ls else 0.05
    ub, pb = (100.0, 100.0) if ls else (3.0, 0.5)
    prm = cartpole_params(dt=dt, device=dev)
    inst = torch.arange(first, first + batch, dtype=torch.int64, device=dev)
    st = torch.arange(N, dtype=torch.int64, device=dev)
    U0 = uniform(seed, inst, 0, OP_S0, n)
    scale = torch.tensor([0.5, 3.0, 2.0, 8.0] if ls else [0.5, 0.3, 0.0, 0.0], dtype=torch.float64, device=dev)
    s0 = U0 * scale
    ubar = 5.0 * uniform(seed, inst, st, OP_U, m)
    defect = (0.5 if ls else 1e-3) * uniform(seed, inst, torch.arange(N + 1, device=dev), OP_DRES, n)
    xs = [s0 + defect[:, 0]]
    for i in range(N):
        xs.append(cartpole_step_torch(prm, xs[-1], ubar[:, i]) + defect[:, i + 1])
    xbar = torch.stack(xs, dim=1)                                  # [b, N+1, n]
    # dynamics residuals and Jacobians at the iterate (autograd; workload definition only)
    xi = xbar[:, :N].reshape(-1, n)
    ui = ubar.reshape(-1, m)
    dxu = cartpole_step_torch(prm, xi, ui)
    dres = (dxu.reshape(batch, N, n) - xbar[:, 1:])
    jac = torch.func.vmap(torch.func.jacrev(lambda xx, uu: cartpole_step_torch(prm, xx, uu), argnums=(0, 1)))
    Jx, Ju = jac(xi, ui)                                           # [bN, n, n], [bN, n, m]
    A = colmajor(Jx).reshape(batch, N, n * n)
    B = colmajor(Ju).reshape(batch, N, n * m)
    xg = torch.tensor([0.0, math.pi, 0.0, 0.0], dtype=torch.float64, device=dev)
    qd = torch.tensor([1.0, 1.0, 0.1, 0.1], dtype=torch.float64, device=dev)
    rw = 0.01
    dx = xbar - xg
    gradf = torch.cat([qd * dx[:, :N], rw * ubar], dim=-1)
    gradfN = 100.0 * dx[:, N]
    fval = 0.5 * (qd * dx[:, :N] ** 2).sum((-1, -2)) + 0.5 * rw * (ubar ** 2).sum((-1, -2)) + 50.0 * (dx[:, N] ** 2).sum(-1)
    Pst = torch.diag(torch.cat([qd, torch.tensor([rw], dtype=torch.float64, device=dev)]))
    Q = pack_lower(Pst[:n, :n]).expand(batch, N, sym_size(n)).contiguous()
    M = _zeros(batch, N, n * m, device=dev)
    R = torch.full((batch, N, 1), rw, dtype=torch.float64, device=dev)
    QN = pack_lower(100.0 * torch.eye(n, dtype=torch.float64, device=dev)).expand(batch, sym_size(n)).contiguous()
    # inequalities g(x,u) ≤ 0: [u − ub, −u − ub, p − pb, −p − pb]; Jacobian rows over (x, u)
    G = _zeros(4, k, device=dev)
    G[0, 4], G[1, 4], G[2, 0], G[3, 0] = 1.0, -1.0, 1.0, -1.0
    Gj = colmajor(G).expand(batch, N, 4 * k).contiguous()
    pos, uu = xbar[:, :N, 0], ubar[..., 0]
    gv = torch.stack([uu - ub, -uu - ub, pos - pb, -pos - pb], dim=-1)
    GN = _zeros(2, n, device=dev)
    GN[0, 0], GN[1, 0] = 1.0, -1.0
    GjN = colmajor(GN).expand(batch, 2 * n).contiguous()
    gvN = torch.stack([xbar[:, N, 0] - pb, -xbar[:, N, 0] - pb], dim=-1)
    s = torch.clamp(-gv, min=1e-2)
    sN = torch.clamp(-gvN, min=1e-2)
    yv = 0.1 * uniform(seed, inst, torch.arange(N + 1, device=dev), OP_Y, n)
    data = dict(s0=s0, fval=fval, gradf=gradf, gradfN=gradfN, Q=Q, M=M, R=R, QN=QN, A=A, B=B, dres=dres,
                ce=_zeros(batch, N, 0, device=dev), Ce=_zeros(batch, N, 0, device=dev),
                ceN=_zeros(batch, 0, device=dev), CeN=_zeros(batch, 0, device=dev),
                gv=gv, Gj=Gj, gvN=gvN, GjN=GjN, model_params=prm)
    it = dict(x=xbar, u=ubar, s=s, z=mu / s, sN=sN, zN=mu / sN, y=yv,
              lam=_zeros(batch, N, 0, device=dev), lamN=_zeros(batch, 0, device=dev),
              mu=torch.full((batch,), float(mu), dtype=torch.float64, device=dev),
              eta=torch.full((batch,), float(eta), dtype=torch.float64, device=dev))
    data = {k2: v.contiguous() for k2, v in data.items()}
    it = {k2: v.contiguous() for k2, v in it.items()}
    return IPMBatch(n, m, N, 4, 2, 0, 0, MODEL_CARTPOLE, data, it)


# ----------------------------------------------------------------------------- double integrator OCP
def double_integrator_ocp(batch=1, N=20, h=0.1, x0=(5.0, 0.0), umax=1.0, q=1.0, r=0.1, qN=10.0, mu=0.1, eta=1e4,
                          device="cpu") -> IPMBatch:
    """SPEC's end-to-end OCP example (acceptance 6): double integrator A = [[1,h],[0,1]],
    B = [h²/2, h], N = 20, h = 0.1, x₀ = (5, 0), |u| <= umax as u − umax <= 0, −u − umax <= 0,
    cost ½ Σ (q|x_i|² + r u_i²) + ½ qN |x_N|² (model LQ).  Iterate x̄ = 0, ū = 0, s = max(−g, 1e-2),
    z = μ/s, y = 0, μ₀ = 0.1 (SPEC Design Decisions); η₀ = 1e4 as in C1/C4 (SPEC's 1e2 needs ~100
    iterations under its own η rule: DESIGN.md reading R21).  All instances identical."""
    dev = torch.device(device)
    n, m, k = 2, 1, 3
    A = torch.tensor([[1.0, h], [0.0, 1.0]], dtype=torch.float64, device=dev)
    B = torch.tensor([[h * h / 2], [h]], dtype=torch.float64, device=dev)
    P = torch.diag(torch.tensor([q, q, r], dtype=torch.float64, device=dev))
    G = torch.tensor([[0.0, 0.0, 1.0], [0.0, 0.0, -1.0]], dtype=torch.float64, device=dev)
    rep = lambda t, *s: t.reshape(-1).expand(*s, t.numel()).contiguous()
    gv = torch.full((batch, N, 2), -umax, dtype=torch.float64, device=dev)
    s = torch.clamp(-gv, min=1e-2)
    data = dict(s0=torch.tensor(x0, dtype=torch.float64, device=dev).expand(batch, n).contiguous(),
                fval=_zeros(batch, device=dev), gradf=_zeros(batch, N, k, device=dev), gradfN=_zeros(batch, n, device=dev),
                Q=rep(pack_lower(P[:n, :n]), batch, N), M=_zeros(batch, N, n * m, device=dev),
                R=rep(pack_lower(P[n:, n:]), batch, N), QN=rep(pack_lower(qN * torch.eye(n, dtype=torch.float64, device=dev)), batch),
                A=rep(colmajor(A), batch, N), B=rep(colmajor(B), batch, N), dres=_zeros(batch, N, n, device=dev),
                ce=_zeros(batch, N, 0, device=dev), Ce=_zeros(batch, N, 0, device=dev),
                ceN=_zeros(batch, 0, device=dev), CeN=_zeros(batch, 0, device=dev),
                gv=gv, Gj=rep(colmajor(G), batch, N), gvN=_zeros(batch, 0, device=dev), GjN=_zeros(batch, 0, device=dev),
                model_params=_zeros(N_MODEL_PARAMS, device=dev))
    it = dict(x=_zeros(batch, N + 1, n, device=dev), u=_zeros(batch, N, m, device=dev), s=s, z=mu / s,
              sN=_zeros(batch, 0, device=dev), zN=_zeros(batch, 0, device=dev), y=_zeros(batch, N + 1, n, device=dev),
              lam=_zeros(batch, N, 0, device=dev), lamN=_zeros(batch, 0, device=dev),
              mu=torch.full((batch,), float(mu), dtype=torch.float64, device=dev),
              eta=torch.full((batch,), float(eta), dtype=torch.float64, device=dev))
    return IPMBatch(n, m, N, 2, 0, 0, 0, MODEL_LQ, data, it)


def quadrotor_params(dt=0.02, mass=0.5, J=(2.32e-3, 2.32e-3, 4e-3), g=9.81, device="cpu"):
    p = _zeros(N_MODEL_PARAMS, device=device)
    p[:6] = torch.tensor([dt, mass, J[0], J[1], J[2], g], dtype=torch.float64)
    return p


def quadrotor_step_torch(prm, x, u):
    """Explicit Euler x + dt f(x, u) of the C5 quadrotor (workload definition, synth.workloads.quadrotor_f)."""
    dt, mass = prm[0], prm[1]
    return x + dt * quadrotor_f(x, u, mass=mass, J=(prm[2], prm[3], prm[4]), g=prm[5])


def quadrotor_ipm(batch, seed=2513, N=50, mu=0.1, eta=1e4, first=0, device="cpu") -> IPMBatch:
    """Quadrotor IPM iterates (model 2; a test workload, not a BASELINE config): n = 12, m = 4, the C5
    model and weights (§8(d): Q = diag(10,10,10,1,…,.1), R = diag(.1,1,1,1), Q_N = 10Q, dt = 0.02),
    cost ½xᵀQx + ½(u − u_h)ᵀR(u − u_h) with hover thrust u_h = (mg, 0, 0, 0); inequalities
    T ≤ 2mg, −T ≤ −0.2mg, τ_x ≤ 0.05, −τ_x ≤ 0.05 (n_g = 4, none terminal).
    Iterate: s_0 = (U, 0.3U, U, 0.5U) by block; ū = (mg(1 + 0.1U), 0.01U); x̄ = rollout of ū with
    defects 1e-3U; s = max(−g, 1e-2), z = μ/s, y = 0.1U."""
    dev = torch.device(device)
    n, m, k = 12, 4, 16
    prm = quadrotor_params(device=dev)
    mass, grav = 0.5, 9.81
    inst = torch.arange(first, first + batch, dtype=torch.int64, device=dev)
    st = torch.arange(N, dtype=torch.int64, device=dev)
    scale = torch.tensor([1, 1, 1, .3, .3, .3, 1, 1, 1, .5, .5, .5], dtype=torch.float64, device=dev)
    s0 = uniform(seed, inst, 0, OP_S0, n) * scale
    Uu = uniform(seed, inst, st, OP_U, m)
    ubar = torch.cat([mass * grav * (1 + 0.1 * Uu[..., :1]), 0.01 * Uu[..., 1:]], dim=-1)
    defect = 1e-3 * uniform(seed, inst, torch.arange(N + 1, device=dev), OP_DRES, n)
    xs = [s0 + defect[:, 0]]
    for i in range(N):
        xs.append(quadrotor_step_torch(prm, xs[-1], ubar[:, i]) + defect[:, i + 1])
    xbar = torch.stack(xs, dim=1)
    xi = xbar[:, :N].reshape(-1, n)
    ui = ubar.reshape(-1, m)
    dres = quadrotor_step_torch(prm, xi, ui).reshape(batch, N, n) - xbar[:, 1:]
    jac = torch.func.vmap(torch.func.jacrev(lambda xx, uu: quadrotor_step_torch(prm, xx, uu), argnums=(0, 1)))
    Jx, Ju = jac(xi, ui)
    A = colmajor(Jx).reshape(batch, N, n * n)
    B = colmajor(Ju).reshape(batch, N, n * m)
    qd = torch.tensor([10, 10, 10, 1, 1, 1, 1, 1, 1, .1, .1, .1], dtype=torch.float64, device=dev)
    rd = torch.tensor([0.1, 1, 1, 1], dtype=torch.float64, device=dev)
    uh = torch.tensor([mass * grav, 0, 0, 0], dtype=torch.float64, device=dev)
    du_ = ubar - uh
    gradf = torch.cat([qd * xbar[:, :N], rd * du_], dim=-1)
    gradfN = 10.0 * qd * xbar[:, N]
    fval = 0.5 * (qd * xbar[:, :N] ** 2).sum((-1, -2)) + 0.5 * (rd * du_ ** 2).sum((-1, -2)) \
        + 5.0 * (qd * xbar[:, N] ** 2).sum(-1)
    Q = pack_lower(torch.diag(qd)).expand(batch, N, sym_size(n)).contiguous()
    M = _zeros(batch, N, n * m, device=dev)
    R = pack_lower(torch.diag(rd)).expand(batch, N, sym_size(m)).contiguous()
    QN = pack_lower(torch.diag(10.0 * qd)).expand(batch, sym_size(n)).contiguous()
    G = _zeros(4, k, device=dev)
    G[0, 12], G[1, 12], G[2, 13], G[3, 13] = 1.0, -1.0, 1.0, -1.0
    Gj = colmajor(G).expand(batch, N, 4 * k).contiguous()
    T, tx = ubar[..., 0], ubar[..., 1]
    gv = torch.stack([T - 2 * mass * grav, -T + 0.2 * mass * grav, tx - 0.05, -tx - 0.05], dim=-1)
    s = torch.clamp(-gv, min=1e-2)
    yv = 0.1 * uniform(seed, inst, torch.arange(N + 1, device=dev), OP_Y, n)
    data = dict(s0=s0, fval=fval, gradf=gradf, gradfN=gradfN, Q=Q, M=M, R=R, QN=QN, A=A, B=B, dres=dres,
                ce=_zeros(batch, N, 0, device=dev), Ce=_zeros(batch, N, 0, device=dev),
                ceN=_zeros(batch, 0, device=dev), CeN=_zeros(batch, 0, device=dev),
                gv=gv, Gj=Gj, gvN=_zeros(batch, 0, device=dev), GjN=_zeros(batch, 0, device=dev), model_params=prm)
    it = dict(x=xbar, u=ubar, s=s, z=mu / s, sN=_zeros(batch, 0, device=dev), zN=_zeros(batch, 0, device=dev), y=yv,
              lam=_zeros(batch, N, 0, device=dev), lamN=_zeros(batch, 0, device=dev),
              mu=torch.full((batch,), float(mu), dtype=torch.float64, device=dev),
              eta=torch.full((batch,), float(eta), dtype=torch.float64, device=dev))
    data = {k2: v.contiguous() for k2, v in data.items()}
    it = {k2: v.contiguous() for k2, v in it.items()}
    return IPMBatch(n, m, N, 4, 0, 0, 0, MODEL_QUADROTOR, data, it)


# ----------------------------------------------------------------------------- SPEC's scalar examples
def _scalar_shell(batch, m, ng, nc, mu, eta, device):
    """n = 1, N = 1 shell whose state is pinned at 0 (x̄_0 = x̄_1 = s_0 = 0, A = 1, B = 0, Q = Q_N = 1):
    the decision variable of a static NLP becomes the stage-0 control u_0 (P:27-37 with N = 1)."""
    dev = torch.device(device)
    n, k = 1, 1 + m
    z0 = lambda *s: _zeros(batch, *s, device=dev)
    data = dict(s0=z0(1), fval=z0(), gradf=z0(1, k), gradfN=z0(1),
                Q=torch.ones(batch, 1, 1, dtype=torch.float64, device=dev), M=z0(1, m),
                R=z0(1, sym_size(m)), QN=torch.ones(batch, 1, dtype=torch.float64, device=dev),
                A=torch.ones(batch, 1, 1, dtype=torch.float64, device=dev), B=z0(1, m), dres=z0(1, 1),
                ce=z0(1, nc), Ce=z0(1, nc * k), ceN=z0(0), CeN=z0(0),
                gv=z0(1, ng), Gj=z0(1, ng * k), gvN=z0(0), GjN=z0(0),
                model_params=_zeros(N_MODEL_PARAMS, device=dev))
    it = dict(x=z0(2, 1), u=z0(1, m), s=z0(1, ng), z=z0(1, ng), sN=z0(0), zN=z0(0), y=z0(2, 1),
              lam=z0(1, nc), lamN=z0(0),
              mu=torch.full((batch,), float(mu), dtype=torch.float64, device=dev),
              eta=torch.full((batch,), float(eta), dtype=torch.float64, device=dev))
    return data, it


def spec_scalar_ocp(batch=1, xbar=2.0, s=1.0, z=1.0, mu=1.0, eta=10.0, device="cpu") -> IPMBatch:
    """SPEC's scalar NLP min x² s.t. g(x) = 1 − x ≤ 0 as an OCP with
    N = 1, n = m = 1 (model LQ): x = u_0, f = u_0² (R = 2, ∇f_u = 2ū, f̄ = ū²), g = 1 − u_0
    (G = [0, −1] over (x_0, u_0)), slack s, multiplier z.  The defaults are S:234's iterate
    (x = 2, s = 1, z = 1, μ = 1, η = 10)."""
    data, it = _scalar_shell(batch, 1, 1, 0, mu, eta, device)
    data["R"].fill_(2.0)
    data["fval"].fill_(xbar * xbar)
    data["gradf"][..., 1] = 2.0 * xbar
    data["gv"].fill_(1.0 - xbar)
    data["Gj"][..., 1] = -1.0
    it["u"].fill_(xbar)
    it["s"].fill_(s)
    it["z"].fill_(z)
    return IPMBatch(1, 1, 1, 1, 0, 0, 0, MODEL_LQ, {k: v.contiguous() for k, v in data.items()},
                    {k: v.contiguous() for k, v in it.items()})


def spec_equality_qp_ocp(batch=1, m=3, mu=0.1, eta=1e4, device="cpu") -> IPMBatch:
    """min ½‖x‖² s.t. x₁ = 1, start x = 0, as an OCP with N = 1, n = 1: x = u_0 ∈ R^m,
    f = ½‖u_0‖² (R = I), one stage equality c_e = u_0[0] − 1 (C_e = [0, 1, 0, …]) with
    multiplier λ; no inequalities."""
    data, it = _scalar_shell(batch, m, 0, 1, mu, eta, device)
    data["R"][...] = pack_lower(torch.eye(m, dtype=torch.float64, device=data["R"].device))
    data["ce"].fill_(-1.0)
    data["Ce"][..., 1] = 1.0
    return IPMBatch(1, m, 1, 0, 0, 1, 0, MODEL_LQ, {k: v.contiguous() for k, v in data.items()},
                    {k: v.contiguous() for k, v in it.items()})
