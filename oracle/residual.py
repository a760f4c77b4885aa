"""KKT residual of the regularized LQR system (the paper's third callback, "a KKT system residual
computation callback").  TEST INFRASTRUCTURE ONLY.

For the system of §1.4

    K [x; y] = -[s; c],   K = [[P, C^T], [C, -δI]],

the residual of a candidate (x, u, y) is r = K [x; y] + [s; c].  Written out block by block from
the definitions of P, C, s and c (reading R1):

    stationarity, x_i (i < N):  Q_i x_i + M_i u_i + q_i - y_i + A_i^T y_{i+1}
    stationarity, u_i:          M_i^T x_i + R_i u_i + r_i + B_i^T y_{i+1}
    stationarity, x_N:          Q_N x_N + q_N - y_N
    primal, row 0:              -x_0 - δ y_0 + c_0
    primal, row i+1:            A_i x_i + B_i u_i - x_{i+1} - δ y_{i+1} + c_{i+1}

`residual_dense` is the definition itself (dense K times the stacked vector, oracle/dense.py);
`residual_blocks` is the block form above in plain numpy, pinned to it in tests.
"""
from __future__ import annotations

import numpy as np

from .dense import _cm, _np, _sym, assemble_reglqr, instance_blocks


def residual_dense(prob, b, x, u, y):
    """r = K [z; y] - rhs for instance b (dense definition).  Returns (r_stat [nz], r_prim [ny])."""
    blk = instance_blocks(prob, b)
    K, rhs, _ = assemble_reglqr(blk)
    n, m, N = blk["n"], blk["m"], blk["N"]
    z = np.zeros(N * (n + m) + n)
    for i in range(N):
        z[i * (n + m):i * (n + m) + n] = x[i]
        z[i * (n + m) + n:(i + 1) * (n + m)] = u[i]
    z[N * (n + m):] = x[N]
    r = K @ np.concatenate([z, np.asarray(y).reshape(-1)]) - rhs
    return r[:z.size], r[z.size:]


def residual_blocks(prob, x, u, y):
    """Block residual for every instance.  x [b,N+1,n], u [b,N,m], y [b,N+1,n] (numpy).
    Returns dict rq [b,N,n], rr [b,N,m], rqN [b,n] (stationarity) and rc0 [b,n], rc [b,N,n]
    (primal rows 0 and i+1) -- the right-hand-side slots of rr_problem -- plus
    norms [b,2] = (max |stationarity|, max |primal|)."""
    n, m, N = prob.nx, prob.nu, prob.N
    g = {f: _np(getattr(prob, f)) for f in ("A", "B", "Q", "M", "R", "q", "r", "c", "QN", "qN", "c0", "delta")}
    bt = g["delta"].shape[0]
    rq = np.zeros((bt, N, n))
    rr = np.zeros((bt, N, m))
    rc = np.zeros((bt, N, n))
    rqN = np.zeros((bt, n))
    rc0 = np.zeros((bt, n))
    for b in range(bt):
        d = g["delta"][b]
        for i in range(N):
            A, B = _cm(g["A"][b, i], n, n), _cm(g["B"][b, i], n, m)
            Q, M, R = _sym(g["Q"][b, i], n), _cm(g["M"][b, i], n, m), _sym(g["R"][b, i], m)
            rq[b, i] = Q @ x[b, i] + M @ u[b, i] + g["q"][b, i] - y[b, i] + A.T @ y[b, i + 1]
            rr[b, i] = M.T @ x[b, i] + R @ u[b, i] + g["r"][b, i] + B.T @ y[b, i + 1]
            rc[b, i] = A @ x[b, i] + B @ u[b, i] - x[b, i + 1] - d * y[b, i + 1] + g["c"][b, i]
        rqN[b] = _sym(g["QN"][b], n) @ x[b, N] + g["qN"][b] - y[b, N]
        rc0[b] = -x[b, 0] - d * y[b, 0] + g["c0"][b]
    stat = np.concatenate([rq.reshape(bt, -1), rr.reshape(bt, -1), rqN], axis=1)
    prim = np.concatenate([rc0, rc.reshape(bt, -1)], axis=1)
    norms = np.stack([np.abs(stat).max(axis=1), np.abs(prim).max(axis=1)], axis=1)
    return dict(rq=rq, rr=rr, rc=rc, rqN=rqN, rc0=rc0, norms=norms)
