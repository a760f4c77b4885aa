"""Tier T1: the DEFINITION of the regularized LQR solution.  TEST INFRASTRUCTURE ONLY.

The regularized LQR problem is the linear system (§1.4)

    [ P   C^T ] [x]     [s]
    [ C  -δ I ] [y] = - [c]

with P = blkdiag(P_0..P_{N-1}, Q_N), P_i = [[Q_i, M_i], [M_i^T, R_i]],
C banded with block rows  -x_0  and  A_i x_i + B_i u_i - x_{i+1},
s = (q_0, r_0, ..., q_{N-1}, r_{N-1}, q_N), c = (c_0, ..., c_N) (reading R1:
N+1 blocks), x = (x_0, u_0, ..., x_N), y = (y_0, ..., y_N).
It is assembled densely and solved with LAPACK, a library primitive; no structure is exploited:
numpy.linalg.solve (LU), or `ldl_solve` -- the symmetric-indefinite Bunch-Kaufman LDLᵀ
factorisation (LAPACK sytrf via scipy.linalg.ldl) followed by the two triangular solves and the
1×1 / 2×2 block-diagonal solve; both are pinned against each other in tests/test_oracle_rr.py.
"""
from __future__ import annotations

import numpy as np


def _np(t):
    try:
        import torch
        if isinstance(t, torch.Tensor):
            return t.detach().cpu().numpy().astype(np.float64)
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(t, dtype=np.float64)


def _cm(v, rows, cols):
    """column-major flat -> [rows, cols]"""
    return np.asarray(v, dtype=np.float64).reshape(cols, rows).T


def _sym(p, n):
    """LAPACK 'L' packed lower -> full symmetric"""
    F = np.zeros((n, n))
    k = 0
    for c in range(n):
        for r in range(c, n):
            F[r, c] = p[k]
            F[c, r] = p[k]
            k += 1
    return F


def instance_blocks(prob, b):
    """Host copies of instance b's blocks as full matrices (A_i, B_i, Q_i, M_i, R_i, ...)."""
    n, m, N = prob.nx, prob.nu, prob.N
    g = {f: _np(getattr(prob, f))[b] for f in ("A", "B", "Q", "M", "R", "q", "r", "c", "QN", "qN", "c0", "delta")}
    return dict(
        A=[_cm(g["A"][i], n, n) for i in range(N)], B=[_cm(g["B"][i], n, m) for i in range(N)],
        Q=[_sym(g["Q"][i], n) for i in range(N)], M=[_cm(g["M"][i], n, m) for i in range(N)],
        R=[_sym(g["R"][i], m) for i in range(N)], q=[g["q"][i] for i in range(N)],
        r=[g["r"][i] for i in range(N)], c=[g["c"][i] for i in range(N)],
        QN=_sym(g["QN"], n), qN=g["qN"], c0=g["c0"], delta=float(g["delta"]), n=n, m=m, N=N)


def assemble_reglqr(blk):
    """Dense K = [[P, C^T], [C, -δI]] and rhs = -[s; c] for one instance."""
    n, m, N = blk["n"], blk["m"], blk["N"]
    nz = N * (n + m) + n
    ny = (N + 1) * n
    K = np.zeros((nz + ny, nz + ny))
    rhs = np.zeros(nz + ny)
    xo = lambda i: i * (n + m)          # offset of x_i in z
    uo = lambda i: i * (n + m) + n      # offset of u_i in z
    for i in range(N):
        K[xo(i):xo(i) + n, xo(i):xo(i) + n] = blk["Q"][i]
        K[xo(i):xo(i) + n, uo(i):uo(i) + m] = blk["M"][i]
        K[uo(i):uo(i) + m, xo(i):xo(i) + n] = blk["M"][i].T
        K[uo(i):uo(i) + m, uo(i):uo(i) + m] = blk["R"][i]
        rhs[xo(i):xo(i) + n] = -blk["q"][i]
        rhs[uo(i):uo(i) + m] = -blk["r"][i]
    K[xo(N):xo(N) + n, xo(N):xo(N) + n] = blk["QN"]
    rhs[xo(N):xo(N) + n] = -blk["qN"]
    C = np.zeros((ny, nz))
    C[0:n, xo(0):xo(0) + n] = -np.eye(n)
    for i in range(N):
        C[(i + 1) * n:(i + 2) * n, xo(i):xo(i) + n] = blk["A"][i]
        C[(i + 1) * n:(i + 2) * n, uo(i):uo(i) + m] = blk["B"][i]
        C[(i + 1) * n:(i + 2) * n, xo(i + 1):xo(i + 1) + n] = -np.eye(n)
    K[nz:, :nz] = C
    K[:nz, nz:] = C.T
    K[nz:, nz:] = -blk["delta"] * np.eye(ny)
    rhs[nz:nz + n] = -blk["c0"]
    for i in range(N):
        rhs[nz + (i + 1) * n:nz + (i + 2) * n] = -blk["c"][i]
    return K, rhs, C


def unpack_solution(sol, n, m, N):
    nz = N * (n + m) + n
    z, yv = sol[:nz], sol[nz:]
    x = np.stack([z[i * (n + m):i * (n + m) + n] for i in range(N + 1)])
    u = np.stack([z[i * (n + m) + n:(i + 1) * (n + m)] for i in range(N)]) if N > 0 else np.zeros((0, m))
    y = yv.reshape(N + 1, n)
    return x, u, y


def ldl_solve(K, rhs):
    """Solve K z = rhs for symmetric (indefinite) K by Bunch-Kaufman LDLᵀ: P K Pᵀ = L D Lᵀ with D
    block diagonal (1×1 and 2×2 pivots).  scipy returns K = lu·D·luᵀ with lu[perm] lower triangular."""
    import scipy.linalg as sl
    lu, D, perm = sl.ldl(K, lower=True)
    L = lu[perm]                                                        # unit lower triangular
    w = sl.solve_triangular(L, np.asarray(rhs, dtype=np.float64)[perm], lower=True, unit_diagonal=True)
    v = np.zeros_like(w)
    i, nn = 0, K.shape[0]
    while i < nn:                                                       # D w' = w, block by block
        if i + 1 < nn and D[i + 1, i] != 0.0:
            v[i:i + 2] = np.linalg.solve(D[i:i + 2, i:i + 2], w[i:i + 2])
            i += 2
        else:
            v[i] = w[i] / D[i, i]
            i += 1
    z = np.empty_like(v)
    z[perm] = sl.solve_triangular(L.T, v, lower=False, unit_diagonal=True)
    return z


def rr_solve_dense(prob, b=0, method="lu"):
    """T1 solve of instance b (method "lu" or "ldl").  Returns dict(x [N+1,n], u [N,m], y [N+1,n],
    K, rhs, C)."""
    blk = instance_blocks(prob, b)
    K, rhs, C = assemble_reglqr(blk)
    sol = ldl_solve(K, rhs) if method == "ldl" else np.linalg.solve(K, rhs)
    x, u, y = unpack_solution(sol, blk["n"], blk["m"], blk["N"])
    return dict(x=x, u=u, y=y, K=K, rhs=rhs, C=C, blk=blk, sol=sol)
