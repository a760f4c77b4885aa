"""Tier T1 for the IPM step: the DEFINITION, Eq.(4×4), assembled densely for one
instance of the stagewise OCP and solved with LAPACK.  TEST INFRASTRUCTURE ONLY.

NLP view of §1.1: variables X = (x_0, u_0, ..., x_{N-1}, u_{N-1}, x_N); equality
constraints c(X) = (s_0 − x_0, d_i(x_i,u_i) − x_{i+1} (i<N), c_e stage equalities); inequalities
g(X) ≤ 0 with slacks s; multipliers y (all equalities) and z.  P = the given positive-definite
Hessian approximation (block diagonal), C = J(c), G = J(g)."""
from __future__ import annotations

import numpy as np

from .dense import _cm, _np, _sym


def assemble_nlp(prob, b=0):
    n, m, N = prob.nx, prob.nu, prob.N
    ng, ngN, nc, ncN = prob.ng, prob.ngN, prob.nc, prob.ncN
    D = {k: _np(v) for k, v in prob.data.items()}
    I = {k: _np(v) for k, v in prob.it.items()}
    w = n + m
    nX = N * w + n
    xo = lambda i: i * w
    P = np.zeros((nX, nX))
    grad = np.zeros(nX)
    X = np.zeros(nX)
    for i in range(N):
        Q, M, R = _sym(D["Q"][b, i], n), _cm(D["M"][b, i], n, m), _sym(D["R"][b, i], m)
        P[xo(i):xo(i) + w, xo(i):xo(i) + w] = np.block([[Q, M], [M.T, R]])
        grad[xo(i):xo(i) + w] = D["gradf"][b, i]
        X[xo(i):xo(i) + n] = I["x"][b, i]
        X[xo(i) + n:xo(i) + w] = I["u"][b, i]
    P[xo(N):, xo(N):] = _sym(D["QN"][b], n)
    grad[xo(N):] = D["gradfN"][b]
    X[xo(N):] = I["x"][b, N]
    # equalities: initial, dynamics, stage equalities, terminal equalities
    rows_c, vals_c, mult = [], [], []
    Cinit = np.zeros((n, nX)); Cinit[:, 0:n] = -np.eye(n)
    rows_c.append(Cinit); vals_c.append(D["s0"][b] - I["x"][b, 0]); mult.append(I["y"][b, 0])
    for i in range(N):
        Ci = np.zeros((n, nX))
        Ci[:, xo(i):xo(i) + n] = _cm(D["A"][b, i], n, n)
        Ci[:, xo(i) + n:xo(i) + w] = _cm(D["B"][b, i], n, m)
        Ci[:, xo(i + 1):xo(i + 1) + n] = -np.eye(n)
        rows_c.append(Ci); vals_c.append(D["dres"][b, i]); mult.append(I["y"][b, i + 1])
    n_dyn = (N + 1) * n
    for i in range(N):
        if nc:
            Ce = np.zeros((nc, nX)); Ce[:, xo(i):xo(i) + w] = _cm(D["Ce"][b, i], nc, w)
            rows_c.append(Ce); vals_c.append(D["ce"][b, i]); mult.append(I["lam"][b, i])
    if ncN:
        Ce = np.zeros((ncN, nX)); Ce[:, xo(N):] = _cm(D["CeN"][b], ncN, n)
        rows_c.append(Ce); vals_c.append(D["ceN"][b]); mult.append(I["lamN"][b])
    C = np.vstack(rows_c); cval = np.concatenate(vals_c); y = np.concatenate(mult)
    rows_g, vals_g, s, z = [], [], [], []
    for i in range(N):
        if ng:
            G = np.zeros((ng, nX)); G[:, xo(i):xo(i) + w] = _cm(D["Gj"][b, i], ng, w)
            rows_g.append(G); vals_g.append(D["gv"][b, i]); s.append(I["s"][b, i]); z.append(I["z"][b, i])
    if ngN:
        G = np.zeros((ngN, nX)); G[:, xo(N):] = _cm(D["GjN"][b], ngN, n)
        rows_g.append(G); vals_g.append(D["gvN"][b]); s.append(I["sN"][b]); z.append(I["zN"][b])
    if rows_g:
        G = np.vstack(rows_g); gval = np.concatenate(vals_g); s = np.concatenate(s); z = np.concatenate(z)
    else:
        G = np.zeros((0, nX)); gval = np.zeros(0); s = np.zeros(0); z = np.zeros(0)
    return dict(P=P, grad=grad, X=X, C=C, c=cval, y=y, G=G, g=gval, s=s, z=z, n_dyn=n_dyn,
                mu=float(I["mu"][b]), eta=float(I["eta"][b]), n=n, m=m, N=N, nX=nX)


def kkt4x4(nlp):
    """The 4×4 matrix of Eq.(4×4) and the blocks of ∇L."""
    P, C, G, s, z, mu, eta = nlp["P"], nlp["C"], nlp["G"], nlp["s"], nlp["z"], nlp["mu"], nlp["eta"]
    nX, ne, ni = P.shape[0], C.shape[0], G.shape[0]
    K = np.zeros((nX + 2 * ni + ne,) * 2)
    ox, os_, oy, oz = 0, nX, nX + ni, nX + ni + ne
    K[ox:os_, ox:os_] = P
    K[ox:os_, oy:oz] = C.T
    K[ox:os_, oz:] = G.T
    K[os_:oy, os_:oy] = np.diag(z / s)
    K[os_:oy, oz:] = np.eye(ni)
    K[oy:oz, ox:os_] = C
    K[oy:oz, oy:oz] = -np.eye(ne) / eta
    K[oz:, ox:os_] = G
    K[oz:, os_:oy] = np.eye(ni)
    K[oz:, oz:] = -np.eye(ni) / eta
    gL_x = nlp["grad"] + C.T @ nlp["y"] + G.T @ z
    gL_s = -mu / s + z
    gL_y = nlp["c"]
    gL_z = nlp["g"] + s
    return K, (gL_x, gL_s, gL_y, gL_z), (ox, os_, oy, oz)


def solve4x4(prob, b=0, method="lu"):
    nlp = assemble_nlp(prob, b)
    K, gL, off = kkt4x4(nlp)
    if method == "ldl":
        from .dense import ldl_solve
        sol = ldl_solve(K, -np.concatenate(gL))
    else:
        sol = np.linalg.solve(K, -np.concatenate(gL))
    ox, os_, oy, oz = off
    return dict(dX=sol[ox:os_], ds=sol[os_:oy], dy=sol[oy:oz], dz=sol[oz:], nlp=nlp, K=K, gL=gL)


def solve_shifted(prob, b=0):
    """The Lemma's system: same matrix, rhs −[∇ₓ𝒜; ∇ₛ𝒜; 0; 0] with
    ∇ₓ𝒜 = ∇ₓL + ηCᵀc + ηGᵀ(g+s), ∇ₛ𝒜 = ∇ₛL + η(g+s)."""
    nlp = assemble_nlp(prob, b)
    K, (gx, gs, gy, gz), off = kkt4x4(nlp)
    eta = nlp["eta"]
    gA_x = gx + eta * nlp["C"].T @ nlp["c"] + eta * nlp["G"].T @ (nlp["g"] + nlp["s"])
    gA_s = gs + eta * (nlp["g"] + nlp["s"])
    rhs = -np.concatenate([gA_x, gA_s, np.zeros_like(gy), np.zeros_like(gz)])
    sol = np.linalg.solve(K, rhs)
    ox, os_, oy, oz = off
    return dict(dX=sol[ox:os_], ds=sol[os_:oy], dy_shift=sol[oy:oz], dz_shift=sol[oz:], nlp=nlp)


def split_X(nlp, dX):
    n, m, N = nlp["n"], nlp["m"], nlp["N"]
    w = n + m
    x = np.stack([dX[i * w:i * w + n] for i in range(N + 1)])
    u = np.stack([dX[i * w + n:(i + 1) * w] for i in range(N)]) if N else np.zeros((0, m))
    return x, u
