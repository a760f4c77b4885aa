"""ctypes wrapper of the IPM-step oracle (ipm_oracle.c).  TEST INFRASTRUCTURE ONLY."""
from __future__ import annotations

import ctypes

import numpy as np

from .rr import _np, load_oracle

_D = ctypes.c_void_p


class orc_ipm_args(ctypes.Structure):
    _fields_ = ([(f, ctypes.c_int) for f in ("nx", "nu", "N", "ng", "ngN", "nc", "ncN", "model")]
                + [("batch", ctypes.c_int64)]
                + [(f, _D) for f in ("s0", "fval", "gradf", "gradfN", "Q", "M", "R", "QN", "A", "B", "dres",
                                     "ce", "Ce", "ceN", "CeN", "gv", "Gj", "gvN", "GjN", "model_params")]
                + [(f, _D) for f in ("x", "u", "s", "z", "sN", "zN", "y", "lam", "lamN", "mu", "eta")]
                + [("tau", ctypes.c_double), ("armijo_c", ctypes.c_double), ("beta", ctypes.c_double),
                   ("max_backtracks", ctypes.c_int)]
                + [(f, _D) for f in ("dx", "du", "ds", "dsN", "dy", "dlam", "dlamN", "dz", "dzN",
                                     "alpha_p", "alpha_d", "D", "D_closed", "merit0", "merit_acc",
                                     "n_backtracks", "status")])


DIR_SHAPES = dict(dx="x", du="u", ds="s", dsN="sN", dy="y", dlam="lam", dlamN="lamN", dz="z", dzN="zN")


def _prep(prob, tau, c1, beta, max_bt):
    """Host copies of the batch (the iterate copies are updated in place by the oracle)."""
    data = {k: _np(v) for k, v in prob.data.items()}
    it = {k: _np(v).copy() for k, v in prob.it.items()}
    b = prob.batch
    res = {k: np.zeros(it[v].shape) for k, v in DIR_SHAPES.items()}
    for k in ("alpha_p", "alpha_d", "D", "D_closed", "merit0", "merit_acc"):
        res[k] = np.zeros(b)
    res["n_backtracks"] = np.zeros(b, dtype=np.int32)
    res["status"] = np.zeros(b, dtype=np.int32)
    ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    args = orc_ipm_args(prob.nx, prob.nu, prob.N, prob.ng, prob.ngN, prob.nc, prob.ncN, prob.model, b,
                        *[ptr(data[f]) for f in ("s0", "fval", "gradf", "gradfN", "Q", "M", "R", "QN", "A", "B",
                                                 "dres", "ce", "Ce", "ceN", "CeN", "gv", "Gj", "gvN", "GjN",
                                                 "model_params")],
                        *[ptr(it[f]) for f in ("x", "u", "s", "z", "sN", "zN", "y", "lam", "lamN", "mu", "eta")],
                        tau, c1, beta, max_bt,
                        *[ptr(res[f]) for f in ("dx", "du", "ds", "dsN", "dy", "dlam", "dlamN", "dz", "dzN",
                                                "alpha_p", "alpha_d", "D", "D_closed", "merit0", "merit_acc",
                                                "n_backtracks", "status")])
    return args, data, it, res


def ipm_step_oracle(prob, tau=0.995, armijo_c=1e-4, beta=0.5, max_backtracks=50, nthreads=1):
    """One regularized-IPM step per instance (condense → T2 → expand → merit/D → line search).
    Returns (result dict, updated iterate dict) as numpy arrays; the input batch is untouched."""
    lib = load_oracle()
    args, data, it, res = _prep(prob, tau, armijo_c, beta, max_backtracks)
    f = lib.orc_ipm_step
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.POINTER(orc_ipm_args), ctypes.c_int]
    rc = f(ctypes.byref(args), int(nthreads))
    if rc != 0:
        raise ValueError("orc_ipm_step rejected its arguments")
    return res, it


def ipm_merit_oracle(prob, direction, b, alpha):
    """𝒜 at (x̄ + αΔx, s + αΔs) for instance b with a given direction (dict like the result)."""
    lib = load_oracle()
    args, data, it, res = _prep(prob, 0.995, 1e-4, 0.5, 50)
    for k in DIR_SHAPES:
        res[k][...] = direction[k]
    f = lib.orc_ipm_merit
    f.restype = ctypes.c_double
    f.argtypes = [ctypes.POINTER(orc_ipm_args), ctypes.c_int64, ctypes.c_double]
    return float(f(ctypes.byref(args), int(b), float(alpha)))


def cartpole_step_oracle(prm, x, u):
    lib = load_oracle()
    f = lib.orc_cartpole_step
    f.argtypes = [ctypes.c_void_p] * 4
    p = np.ascontiguousarray(prm, dtype=np.float64)
    xx = np.ascontiguousarray(x, dtype=np.float64)
    uu = np.ascontiguousarray(u, dtype=np.float64)
    out = np.zeros(4)
    f(p.ctypes.data, xx.ctypes.data, uu.ctypes.data, out.ctypes.data)
    return out


def quadrotor_step_oracle(prm, x, u):
    """x⁺ = x + dt f(x, u) of the C oracle's quadrotor (SURVEY §8(d) C5 model)."""
    lib = load_oracle()
    f = lib.orc_quadrotor_step
    f.argtypes = [ctypes.c_void_p] * 4
    p = np.ascontiguousarray(prm, dtype=np.float64)
    xx = np.ascontiguousarray(x, dtype=np.float64)
    uu = np.ascontiguousarray(u, dtype=np.float64)
    out = np.zeros(12)
    f(p.ctypes.data, xx.ctypes.data, uu.ctypes.data, out.ctypes.data)
    return out
