"""Binding of ipm_step (include/rr.h): one batched regularized-IPM step, rows a1-a8.
Argument marshalling only; all arithmetic runs in librr_b200.so."""
from __future__ import annotations

import ctypes

import torch

from ._lib import (IPM_DATA_FIELDS, IPM_ITER_FIELDS, IPM_RES_FIELDS, RRError, check, ipm_dims, ipm_iterate,
                   ipm_params, ipm_result, ipm_solve_report, ipm_solve_settings, ipm_stage_data, ipm_trial_values, lib)

RES_SHAPE_OF = dict(dx="x", du="u", ds="s", dsN="sN", dy="y", dlam="lam", dlamN="lamN", dz="z", dzN="zN")


INT_FIELDS = ("status", "n_backtracks", "iters")


def _p(t, name=""):
    """Device pointer of a contiguous CUDA tensor: int32 for status / n_backtracks / iters, float64
    otherwise (NULL for an empty tensor)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise RRError("ipm_step needs CUDA tensors (no CPU fallback)")
    dt = torch.int32 if name in INT_FIELDS else torch.float64
    if t.dtype != dt:
        raise RRError("%s: expected %s, got %s" % (name or "tensor", dt, t.dtype))
    if not t.is_contiguous():
        raise RRError("tensor must be contiguous")
    return ctypes.c_void_p(t.data_ptr()) if t.numel() > 0 else None


def _sizes(b):
    """Element counts the dims imply for every data / iterate / result field (include/rr.h ipm_*)."""
    B, N, n, m, ng, ngN, nc, ncN = b.batch, b.N, b.nx, b.nu, b.ng, b.ngN, b.nc, b.ncN
    w, sy = n + m, (lambda k: k * (k + 1) // 2)
    z = dict(s0=B * n, fval=B, gradf=B * N * w, gradfN=B * n, Q=B * N * sy(n), M=B * N * n * m, R=B * N * sy(m),
             QN=B * sy(n), A=B * N * n * n, B=B * N * n * m, dres=B * N * n, ce=B * N * nc, Ce=B * N * nc * w,
             ceN=B * ncN, CeN=B * ncN * n, gv=B * N * ng, Gj=B * N * ng * w, gvN=B * ngN, GjN=B * ngN * n,
             x=B * (N + 1) * n, u=B * N * m, s=B * N * ng, z=B * N * ng, sN=B * ngN, zN=B * ngN,
             y=B * (N + 1) * n, lam=B * N * nc, lamN=B * ncN, mu=B, eta=B)
    for r, it in RES_SHAPE_OF.items():
        z[r] = z[it]
    for k in ("alpha_p", "alpha_d", "D", "merit0", "merit_acc", "n_backtracks", "status", "iters"):
        z[k] = B
    return z


def check_batch(b, res=None):
    """Dtype, device and size of every tensor of the IPMBatch (and result dict) against its dims."""
    dev = b.it["mu"].device
    want = _sizes(b)
    for group in (b.data, b.it, res or {}):
        for k, t in group.items():
            if t is None or k not in want:
                continue
            _p(t, k)
            if t.device != dev:
                raise RRError("%s on %s, the batch is on %s" % (k, t.device, dev))
            if t.numel() != want[k]:
                raise RRError("%s: %d elements, the dims need %d" % (k, t.numel(), want[k]))
    mp = b.data.get("model_params")
    if mp is not None and (mp.dtype != torch.float64 or mp.device != dev or mp.numel() < 8):
        raise RRError("model_params: expected >= 8 float64 on %s" % dev)


def dims_of(b) -> ipm_dims:
    return ipm_dims(b.nx, b.nu, b.N, b.ng, b.ngN, b.nc, b.ncN, b.model, b.batch)


def workspace_bytes(b) -> int:
    nb = lib().ipm_workspace_bytes(ctypes.byref(dims_of(b)))
    if nb < 0:
        raise RRError("no ipm_step kernel compiled for these dims/model")
    return int(nb)


def alloc_result(b):
    dev = b.it["mu"].device
    res = {k: torch.empty_like(b.it[v]) for k, v in RES_SHAPE_OF.items()}
    for k in ("alpha_p", "alpha_d", "D", "merit0", "merit_acc"):
        res[k] = torch.empty(b.batch, dtype=torch.float64, device=dev)
    res["n_backtracks"] = torch.empty(b.batch, dtype=torch.int32, device=dev)
    res["status"] = torch.empty(b.batch, dtype=torch.int32, device=dev)
    return res


class IpmCall:
    """Pre-marshalled ipm_step launch on fixed buffers (iterate updated in place)."""

    def __init__(self, b, res=None, ws=None, tau=0.995, armijo_c=1e-4, beta=0.5, max_backtracks=50):
        self.b = b
        self.res = res if res is not None else alloc_result(b)
        nb = workspace_bytes(b)
        self.ws = ws if ws is not None else torch.empty((nb + 7) // 8, dtype=torch.float64, device=b.it["mu"].device)
        self.d = dims_of(b)
        check_batch(b, self.res)
        self.data = ipm_stage_data(*[_p(b.data[f], f) for f in IPM_DATA_FIELDS])
        self.it = ipm_iterate(*[_p(b.it[f], f) for f in IPM_ITER_FIELDS])
        self.prm = ipm_params(tau, armijo_c, beta, max_backtracks, 0)
        self.r = ipm_result(*[_p(self.res[f], f) for f in IPM_RES_FIELDS])
        self.st = _p(self.res["status"], "status")
        self.wsp, self.wsb = _p(self.ws), self.ws.numel() * 8

    def launch(self, stream=None, direction_only=False):
        s = stream if stream is not None else torch.cuda.current_stream(self.b.it["mu"].device)
        fn = lib().ipm_direction if direction_only else lib().ipm_step
        rc = fn(ctypes.byref(self.d), ctypes.byref(self.data), ctypes.byref(self.it),
                ctypes.byref(self.prm), ctypes.byref(self.r), self.wsp, self.wsb, self.st,
                ctypes.c_void_p(s.cuda_stream))
        check(rc, "ipm_direction" if direction_only else "ipm_step")
        return self.res


def ipm_step(b, tau=0.995, armijo_c=1e-4, beta=0.5, max_backtracks=50, stream=None):
    """One regularized-IPM step for every instance of the IPMBatch `b` (CUDA tensors); the iterate
    b.it is updated in place.  Returns the result dict (direction, α_p, α_d, D, 𝒜(0), 𝒜(α), k, status)."""
    return IpmCall(b, tau=tau, armijo_c=armijo_c, beta=beta, max_backtracks=max_backtracks).launch(stream)


SOLVE_DEFAULTS = dict(mu_min=1e-9, kappa=10.0, kappa_mu=0.2, theta_mu=1.5, eta_max=1e8, kappa_eta=10.0,
                      tol_kkt=1e-6, max_iters=100, tau=0.995, armijo_c=1e-4, beta=0.5, max_backtracks=50,
                      linear_merit=False)
REPORT_FIELDS = ("status", "iters", "mu", "eta", "r_stat", "r_feas", "r_comp")


class IpmSolveCall:
    """Pre-marshalled ipm_solve launch (the batched IPM loop) on fixed buffers.
    b.data is the evaluation at the initial iterate (the model reference); b.it is updated in place."""

    def __init__(self, b, ws=None, **settings):
        S = dict(SOLVE_DEFAULTS)
        S.update(settings)
        self.b = b
        dev = b.it["mu"].device
        self.d = dims_of(b)
        nb = lib().ipm_solve_workspace_bytes(ctypes.byref(self.d))
        if nb < 0:
            raise RRError("no ipm_solve kernel compiled for these dims/model")
        self.ws = ws if ws is not None else torch.empty((nb + 7) // 8, dtype=torch.float64, device=dev)
        check_batch(b)
        self.data = ipm_stage_data(*[_p(b.data[f], f) for f in IPM_DATA_FIELDS])
        self.it = ipm_iterate(*[_p(b.it[f], f) for f in IPM_ITER_FIELDS])
        self.S = ipm_solve_settings(S["mu_min"], S["kappa"], S["kappa_mu"], S["theta_mu"], S["eta_max"],
                                    S["kappa_eta"], S["tol_kkt"], int(S["max_iters"]), int(bool(S["linear_merit"])),
                                    ipm_params(S["tau"], S["armijo_c"], S["beta"], int(S["max_backtracks"]), 0))
        self.rep = {k: torch.empty(b.batch, dtype=torch.int32 if k in ("status", "iters") else torch.float64, device=dev)
                    for k in REPORT_FIELDS}
        self.r = ipm_solve_report(*[_p(self.rep[k], k) for k in REPORT_FIELDS])
        self.wsp, self.wsb = _p(self.ws), self.ws.numel() * 8

    def launch(self, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream(self.b.it["mu"].device)
        rc = lib().ipm_solve(ctypes.byref(self.d), ctypes.byref(self.data), ctypes.byref(self.it), ctypes.byref(self.S),
                             ctypes.byref(self.r), self.wsp, self.wsb, ctypes.c_void_p(s.cuda_stream))
        check(rc, "ipm_solve")
        return self.rep


def ipm_solve(b, stream=None, **settings):
    """Solve every instance of the IPMBatch `b` (CUDA tensors; data evaluated at the initial
    iterate) with the batched regularized IPM; b.it is updated in place.  Returns the report
    (status, iters, mu, eta, r_stat, r_feas, r_comp)."""
    return IpmSolveCall(b, **settings).launch(stream)


def ipm_direction(b, tau=0.995, armijo_c=1e-4, beta=0.5, max_backtracks=50, stream=None):
    """Rows a1-a7 of the step for every instance of `b` (user models): the direction,
    D, 𝒜(0) (merit0), α_max (alpha_p) and the dual cap α_d (alpha_d); the iterate is not modified."""
    return IpmCall(b, tau=tau, armijo_c=armijo_c, beta=beta, max_backtracks=max_backtracks).launch(
        stream, direction_only=True)


TRIAL_FIELDS = ("fval", "dres", "ce", "ceN", "gv", "gvN")


def ipm_merit(b, res, alpha, trial, out=None, stream=None):
    """𝒜 at the trial points x̄ + αΔx, s + αΔs from the caller's model values there (`trial`: dict
    fval, dres, ce, ceN, gv, gvN in the IPMBatch data layouts); alpha: [batch] CUDA tensor."""
    dev = b.it["mu"].device
    merit = out if out is not None else torch.empty(b.batch, dtype=torch.float64, device=dev)
    check_batch(b, {k: v for k, v in res.items() if k in IPM_RES_FIELDS})
    tv = ipm_trial_values(*[_p(trial.get(f), f) for f in TRIAL_FIELDS])
    rc = lib().ipm_merit(ctypes.byref(dims_of(b)), ctypes.byref(ipm_stage_data(*[_p(b.data[f], f) for f in IPM_DATA_FIELDS])),
                         ctypes.byref(ipm_iterate(*[_p(b.it[f], f) for f in IPM_ITER_FIELDS])),
                         ctypes.byref(ipm_result(*[_p(res.get(f), f) for f in IPM_RES_FIELDS])), _p(alpha),
                         ctypes.byref(tv), _p(merit),
                         ctypes.c_void_p((stream or torch.cuda.current_stream(dev)).cuda_stream))
    check(rc, "ipm_merit")
    return merit


def ipm_update(b, res, alpha_p, alpha_d, stream=None):
    """x, u, s, y, λ += α_p Δ and z += α_d Δz in place (per-instance [batch] CUDA tensors)."""
    dev = b.it["mu"].device
    check_batch(b, {k: v for k, v in res.items() if k in IPM_RES_FIELDS})
    rc = lib().ipm_update(ctypes.byref(dims_of(b)), ctypes.byref(ipm_iterate(*[_p(b.it[f], f) for f in IPM_ITER_FIELDS])),
                          ctypes.byref(ipm_result(*[_p(res.get(f), f) for f in IPM_RES_FIELDS])), _p(alpha_p), _p(alpha_d),
                          ctypes.c_void_p((stream or torch.cuda.current_stream(dev)).cuda_stream))
    check(rc, "ipm_update")
