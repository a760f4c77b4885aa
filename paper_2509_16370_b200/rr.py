"""Thin Python binding of the C-ABI (include/rr.h): argument marshalling only.

Tensors are torch CUDA float64 tensors in the C-ABI layout (synth.RRProblem documents it);
every step of the method runs in librr_b200.so.  torch supplies device memory and streams."""
from __future__ import annotations

import ctypes
from typing import Optional

import torch

from ._lib import (RR_FLAG_ACCUMULATE, RR_FLAG_FACTOR_FP32, RRError, check, lib, rr_dims, rr_factor_buf, rr_problem, rr_residual_buf,
                   rr_solution)

PROBLEM_FIELDS = ("A", "B", "Q", "M", "R", "q", "r", "c", "QN", "qN", "c0", "delta")


def _p(t: Optional[torch.Tensor], dtype=torch.float64):
    """Device pointer of a contiguous CUDA tensor of exactly `dtype` (float64 data, int32 status)."""
    if t is None:
        return None
    if not t.is_cuda or t.dtype != dtype:
        raise RRError("expected a CUDA %s tensor, got %s on %s" % (dtype, t.dtype, t.device))
    if not t.is_contiguous():
        raise RRError("tensor must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _sym(k: int) -> int:
    return k * (k + 1) // 2


def check_problem(prob, sol=None):
    """Dtype / device / size of every problem (and solution) tensor against the dims, before any
    pointer reaches the library (a float32 or short tensor would otherwise be read out of bounds)."""
    b, N, n, m = prob.batch, prob.N, prob.nx, prob.nu
    fl = shared_flags(prob)
    bD = 1 if fl & RR_FLAG_SHARED_DYN else b
    bP = 1 if fl & RR_FLAG_SHARED_COST else b
    nD = 1 if fl & RR_FLAG_STAGE_INVARIANT_DYN else N
    nP = 1 if fl & RR_FLAG_STAGE_INVARIANT_COST else N
    want = dict(A=bD * nD * n * n, B=bD * nD * n * m, Q=bP * nP * _sym(n), M=bP * nP * n * m, R=bP * nP * _sym(m),
                q=b * N * n, r=b * N * m, c=b * N * n, QN=bP * _sym(n), qN=b * n, c0=b * n, delta=b)
    dev = prob.delta.device
    for f in PROBLEM_FIELDS:
        t = getattr(prob, f)
        if t is None:
            continue
        if t.dtype != torch.float64 or t.device != dev:
            raise RRError("problem.%s: expected float64 on %s, got %s on %s" % (f, dev, t.dtype, t.device))
        if t.numel() != want[f]:
            raise RRError("problem.%s: %d elements, the dims need %d" % (f, t.numel(), want[f]))
    if sol is not None:
        for f, k in (("x", b * (N + 1) * n), ("u", b * N * m), ("y", b * (N + 1) * n), ("status", b)):
            t = sol.get(f)
            if t is None:
                continue
            dt = torch.int32 if f == "status" else torch.float64
            if t.dtype != dt or t.device != dev or t.numel() != k:
                raise RRError("solution.%s: expected %d %s on %s, got %d %s on %s"
                              % (f, k, dt, dev, t.numel(), t.dtype, t.device))


RR_FLAG_SHARED_DYN, RR_FLAG_SHARED_COST = 2, 4
RR_FLAG_STAGE_INVARIANT_DYN, RR_FLAG_STAGE_INVARIANT_COST = 16, 32


def _layout(t, N: int, name: str):
    """(batch_shared, stage_invariant) of a stage operand from its shape: [b, N, e] per instance and
    stage; [N, e] batch-shared; [b, 1, e] stage-invariant (N > 1); [1, e] both (N > 1)."""
    if t.dim() == 3:
        return False, (t.shape[1] == 1 and N > 1)
    if t.dim() == 2:
        return True, (t.shape[0] == 1 and N > 1)
    raise RRError("problem.%s: expected [batch, N, elems], [N, elems], [batch, 1, elems] or [1, elems]" % name)


def shared_flags(prob) -> int:
    """Operand-layout flags (include/rr.h RR_FLAG_SHARED_* / RR_FLAG_STAGE_INVARIANT_*) from the tensor
    shapes: A, B (and Q, M, R with Q_N) without a batch dimension are batch-shared; with a stage
    dimension of 1 (N > 1) they are stage-invariant (LTI)."""
    f = 0
    dA, dB = _layout(prob.A, prob.N, "A"), _layout(prob.B, prob.N, "B")
    if dA != dB:
        raise RRError("A and B must have the same layout (batch-shared / stage-invariant)")
    f |= (RR_FLAG_SHARED_DYN if dA[0] else 0) | (RR_FLAG_STAGE_INVARIANT_DYN if dA[1] else 0)
    cQ, cM, cR = (_layout(getattr(prob, k), prob.N, k) for k in ("Q", "M", "R"))
    if not (cQ == cM == cR):
        raise RRError("Q, M and R must have the same layout (batch-shared / stage-invariant)")
    if cQ[0] != (prob.QN.dim() == 1):
        raise RRError("Q_N must be batch-shared ([elems]) exactly when Q, M, R are")
    f |= (RR_FLAG_SHARED_COST if cQ[0] else 0) | (RR_FLAG_STAGE_INVARIANT_COST if cQ[1] else 0)
    return f


def dims_of(prob) -> rr_dims:
    return rr_dims(prob.nx, prob.nu, prob.N, shared_flags(prob), prob.batch)


def workspace_bytes(nx: int, nu: int, N: int, batch: int, flags: int = 0) -> int:
    d = rr_dims(nx, nu, N, flags, batch)
    nb = lib().rr_workspace_bytes(ctypes.byref(d))
    if nb < 0:
        raise RRError("no kernel compiled for nx=%d nu=%d" % (nx, nu))
    return int(nb)


def alloc_solution(prob, device=None):
    device = device or prob.delta.device
    b, N, n, m = prob.batch, prob.N, prob.nx, prob.nu
    kw = dict(dtype=torch.float64, device=device)
    return dict(x=torch.empty(b, N + 1, n, **kw), u=torch.empty(b, N, m, **kw),
                y=torch.empty(b, N + 1, n, **kw), status=torch.empty(b, dtype=torch.int32, device=device))


def alloc_factor(prob, device=None):
    device = device or prob.delta.device
    b, N, n, m = prob.batch, prob.N, prob.nx, prob.nu
    kw = dict(dtype=torch.float64, device=device)
    return dict(V=torch.empty(b, N + 1, n * (n + 1) // 2, **kw), v=torch.empty(b, N + 1, n, **kw),
                K=torch.empty(b, N, m * n, **kw), k=torch.empty(b, N, m, **kw))


def alloc_workspace(prob, device=None) -> torch.Tensor:
    device = device or prob.delta.device
    nb = workspace_bytes(prob.nx, prob.nu, prob.N, prob.batch, shared_flags(prob))
    return torch.empty((nb + 7) // 8, dtype=torch.float64, device=device)


class Marshalled:
    """Pre-built ctypes argument structs for repeated launches on fixed buffers (bench loop)."""

    def __init__(self, prob, sol, fac=None, ws=None):
        self.prob, self.sol, self.fac = prob, sol, fac
        check_problem(prob, sol)
        self.ws = ws if ws is not None else alloc_workspace(prob)
        self.d = dims_of(prob)
        self.p = rr_problem(*[_p(getattr(prob, f)) for f in PROBLEM_FIELDS])
        self.f = rr_factor_buf(*[_p(fac[k]) if fac is not None else None for k in ("V", "v", "K", "k")])
        self.s = rr_solution(_p(sol["x"]), _p(sol["u"]), _p(sol["y"]))
        self.st = _p(sol["status"], torch.int32)
        self.wsp = _p(self.ws)
        self.wsb = self.ws.numel() * 8

    def launch(self, stream: Optional[torch.cuda.Stream] = None):
        s = stream if stream is not None else torch.cuda.current_stream(self.prob.delta.device)
        rc = lib().rr_factor_solve(ctypes.byref(self.d), ctypes.byref(self.p), ctypes.byref(self.f),
                                   ctypes.byref(self.s), self.wsp, self.wsb, self.st,
                                   ctypes.c_void_p(s.cuda_stream))
        check(rc, "rr_factor_solve")


def rr_factor_solve(prob, want_factor: bool = False, out=None, fac=None, workspace=None, stream=None):
    """Fused factor + solve of every instance (rows a2-a5).  Returns dict x, u, y, status
    (+ V, v, K, k when want_factor).  Asynchronous on `stream` (default: current stream)."""
    if not prob.delta.is_cuda:
        raise RRError("rr_factor_solve needs CUDA tensors (no CPU fallback)")
    sol = out if out is not None else alloc_solution(prob)
    if want_factor and fac is None:
        fac = alloc_factor(prob)
    Marshalled(prob, sol, fac, workspace).launch(stream)
    res = dict(sol)
    if fac is not None:
        res.update(fac)
    return res


def factor_record_doubles(nx: int, nu: int) -> int:
    """Doubles per factor record (include/rr.h rr_factor_record_doubles)."""
    return (nx * (nx + 1) + nx * nu + nu * (nu + 1) // 2 + 1) & ~1


def factor_bytes(nx: int, nu: int, N: int, batch: int, fp32: bool = False) -> int:
    nb = lib().rr_factor_bytes(ctypes.byref(rr_dims(nx, nu, N, RR_FLAG_FACTOR_FP32 if fp32 else 0, batch)))
    if nb < 0:
        raise RRError("rr_factor: no kernel compiled for nx=%d nu=%d%s" % (nx, nu, " (FP32 records)" if fp32 else ""))
    return int(nb)


def solve_workspace_bytes(nx: int, nu: int, N: int, batch: int) -> int:
    nb = lib().rr_solve_workspace_bytes(ctypes.byref(rr_dims(nx, nu, N, 0, batch)))
    if nb < 0:
        raise RRError("rr_solve: no kernel compiled for nx=%d nu=%d" % (nx, nu))
    return int(nb)


def _stream(stream, device):
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return ctypes.c_void_p(s.cuda_stream)


def rr_factor(prob, factor=None, fac=None, status=None, stream=None, fp32=False):
    """Row a2 (matrix half of Eq.(RR)): returns (factor, status), factor a CUDA float64 tensor
    [batch, N+1, rr_factor_record_doubles] in the include/rr.h record layout
    (V_i | S_i^-1 | K_i | G_i^-1).  fac: optional dict with V / K tensors to receive copies.
    fp32: FP32 records (RR_FLAG_FACTOR_FP32, 12 x 4): a float32 tensor [batch, N+1, R32]."""
    if not prob.delta.is_cuda:
        raise RRError("rr_factor needs CUDA tensors (no CPU fallback)")
    dev = prob.delta.device
    nb = factor_bytes(prob.nx, prob.nu, prob.N, prob.batch, fp32)  # raises if no kernel covers the shape
    if factor is None:
        if fp32:
            factor = torch.empty(prob.batch, prob.N + 1, (factor_record_doubles(prob.nx, prob.nu) + 3) & ~3,
                                 dtype=torch.float32, device=dev)
        else:
            factor = torch.empty(prob.batch, prob.N + 1, factor_record_doubles(prob.nx, prob.nu),
                                 dtype=torch.float64, device=dev)
    if (factor.dtype == torch.float32) != bool(fp32) or factor.numel() * factor.element_size() < nb:
        raise RRError("rr_factor: factor tensor dtype / size does not match fp32=%s" % fp32)
    if status is None:
        status = torch.empty(prob.batch, dtype=torch.int32, device=dev)
    check_problem(prob, dict(status=status))
    p = rr_problem(*[_p(getattr(prob, f)) for f in PROBLEM_FIELDS])
    f = rr_factor_buf(*[_p(fac.get(k)) if fac is not None else None for k in ("V", "v", "K", "k")])
    d = dims_of(prob)
    if fp32:
        d.flags |= RR_FLAG_FACTOR_FP32
    rc = lib().rr_factor(ctypes.byref(d), ctypes.byref(p), _p(factor, factor.dtype), factor.numel() * factor.element_size(),
                         ctypes.byref(f), _p(status, torch.int32), _stream(stream, dev))
    check(rc, "rr_factor")
    return factor, status


def rr_solve(prob, factor, out=None, fac=None, workspace=None, stream=None, accumulate=False):
    """Rows a3-a5 for the right-hand side (q, r, c, qN, c0) of `prob` with rr_factor's records.
    Returns dict x, u, y, status (status: 0 or RR_ST_NONFINITE).  accumulate: add the solution
    to `out` (RR_FLAG_ACCUMULATE, the refinement update) instead of overwriting it."""
    if not prob.delta.is_cuda:
        raise RRError("rr_solve needs CUDA tensors (no CPU fallback)")
    dev = prob.delta.device
    sol = out if out is not None else alloc_solution(prob)
    if workspace is None:
        nb = solve_workspace_bytes(prob.nx, prob.nu, prob.N, prob.batch)
        workspace = torch.empty((nb + 7) // 8, dtype=torch.float64, device=dev)
    check_problem(prob, sol)
    p = rr_problem(*[_p(getattr(prob, f)) for f in PROBLEM_FIELDS])
    f = rr_factor_buf(*[_p(fac.get(k)) if fac is not None else None for k in ("V", "v", "K", "k")])
    s = rr_solution(_p(sol["x"]), _p(sol["u"]), _p(sol["y"]))
    d = dims_of(prob)
    if accumulate:
        if out is None:
            raise RRError("rr_solve(accumulate=True) needs `out` (the solution to update)")
        d.flags |= RR_FLAG_ACCUMULATE
    if factor.dtype == torch.float32:  # FP32 records of rr_factor(fp32=True)
        d.flags |= RR_FLAG_FACTOR_FP32
    elif factor.dtype != torch.float64:
        raise RRError("rr_solve: factor must be float64 (or float32 records of rr_factor(fp32=True))")
    rc = lib().rr_solve(ctypes.byref(d), ctypes.byref(p), _p(factor, factor.dtype), factor.numel() * factor.element_size(),
                        ctypes.byref(f), ctypes.byref(s), _p(workspace), workspace.numel() * 8,
                        _p(sol["status"], torch.int32), _stream(stream, dev))
    check(rc, "rr_solve")
    return sol


def rr_factor_solve_pit(prob, out=None, workspace=None, stream=None):
    """Parallel-in-time solve: the same x, u, y, status as rr_factor_solve, with
    O(log N) depth (block cyclic reduction on the δ-reduced state system); needs δ > 0."""
    if not prob.delta.is_cuda:
        raise RRError("rr_factor_solve_pit needs CUDA tensors (no CPU fallback)")
    dev = prob.delta.device
    sol = out if out is not None else alloc_solution(prob)
    d = dims_of(prob)
    if workspace is None:
        nb = lib().rr_pit_workspace_bytes(ctypes.byref(d))
        if nb < 0:
            raise RRError("rr_factor_solve_pit: nx, nu must be <= 16")
        workspace = torch.empty((nb + 7) // 8, dtype=torch.float64, device=dev)
    check_problem(prob, sol)
    p = rr_problem(*[_p(getattr(prob, f)) for f in PROBLEM_FIELDS])
    s = rr_solution(_p(sol["x"]), _p(sol["u"]), _p(sol["y"]))
    rc = lib().rr_factor_solve_pit(ctypes.byref(d), ctypes.byref(p), ctypes.byref(s), _p(workspace),
                                   workspace.numel() * 8, _p(sol["status"], torch.int32), _stream(stream, dev))
    check(rc, "rr_factor_solve_pit")
    return sol


RESIDUAL_FIELDS = ("q", "r", "c", "qN", "c0")


def rr_residual(prob, sol, res=None, norms=None, stream=None):
    """KKT residual r = K[x; y] + [s; c] (the paper's residual callback) of `sol` (dict x, u, y).
    Returns (res, norms): res a dict q, r, c, qN, c0 in the right-hand-side layouts of `prob`,
    norms [batch, 2] = (max |stationarity|, max |primal|)."""
    if not prob.delta.is_cuda:
        raise RRError("rr_residual needs CUDA tensors (no CPU fallback)")
    dev = prob.delta.device
    if res is None:
        res = {f: torch.empty_like(getattr(prob, f)) for f in RESIDUAL_FIELDS}
    if norms is None:
        norms = torch.empty(prob.batch, 2, dtype=torch.float64, device=dev)
    check_problem(prob, sol)
    p = rr_problem(*[_p(getattr(prob, f)) for f in PROBLEM_FIELDS])
    s = rr_solution(_p(sol["x"]), _p(sol["u"]), _p(sol["y"]))
    r = rr_residual_buf(*[_p(res.get(f)) for f in RESIDUAL_FIELDS])
    rc = lib().rr_residual(ctypes.byref(dims_of(prob)), ctypes.byref(p), ctypes.byref(s), ctypes.byref(r),
                           _p(norms), _stream(stream, dev))
    check(rc, "rr_residual")
    return res, norms


def rr_refine(prob, factor, sol, iters: int = 1, workspace=None, stream=None):
    """Iterative refinement of `sol` in place: iters x (rr_residual -> rr_solve(accumulate)).
    The correction system has the same matrix (A, B, Q, M, R, Q_N, δ -- the factor) and the
    residual as its right-hand side.  Returns the norms of the residual before the last update."""
    norms = None
    res = None
    for _ in range(iters):
        res, norms = rr_residual(prob, sol, res=res, stream=stream)
        corr = type(prob)(prob.nx, prob.nu, prob.N, **{f: (res[f] if f in res else getattr(prob, f))
                                                      for f in PROBLEM_FIELDS})
        rr_solve(corr, factor, out=sol, workspace=workspace, stream=stream, accumulate=True)
    return norms


def version() -> str:
    return lib().rr_version().decode()


class HostMarshalled:
    """End-to-end path through rr_factor_solve_host: problem in (pinned) host tensors, result
    copied back to host tensors; device staging buffers are allocated once by the caller."""

    def __init__(self, prob_host, sol_host, prob_dev, sol_dev, ws=None):
        for t in (prob_host.delta, sol_host["x"]):
            if t.is_cuda:
                raise RRError("host buffers expected")
        check_problem(prob_dev, sol_dev)
        self.keep = (prob_host, sol_host, prob_dev, sol_dev)
        self.d = dims_of(prob_host)
        hp = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
        self.ph = rr_problem(*[hp(getattr(prob_host, f)) for f in PROBLEM_FIELDS])
        self.sh = rr_solution(hp(sol_host["x"]), hp(sol_host["u"]), hp(sol_host["y"]))
        self.sth = hp(sol_host["status"])
        self.pd = rr_problem(*[_p(getattr(prob_dev, f)) for f in PROBLEM_FIELDS])
        self.sd = rr_solution(_p(sol_dev["x"]), _p(sol_dev["u"]), _p(sol_dev["y"]))
        self.std = _p(sol_dev["status"], torch.int32)
        self.ws = ws if ws is not None else alloc_workspace(prob_dev)
        self.wsp, self.wsb = _p(self.ws), self.ws.numel() * 8
        self.h2d_bytes = sum(getattr(prob_host, f).numel() * 8 for f in PROBLEM_FIELDS)
        self.d2h_bytes = sum(sol_host[k].numel() * 8 for k in ("x", "u", "y")) + sol_host["status"].numel() * 4

    def launch(self, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream()
        rc = lib().rr_factor_solve_host(ctypes.byref(self.d), ctypes.byref(self.ph), ctypes.byref(self.sh),
                                        self.sth, ctypes.byref(self.pd), ctypes.byref(self.sd), self.std,
                                        self.wsp, self.wsb, ctypes.c_void_p(s.cuda_stream))
        check(rc, "rr_factor_solve_host")

    def pipelined_workspace_bytes(self, nchunks: int) -> int:
        """Workspace rr_factor_solve_host_pipelined needs for `nchunks` chunks."""
        b, tot = self.d.batch, 0
        nc = min(nchunks, b)
        for c in range(nc):
            cb = b * (c + 1) // nc - b * c // nc
            w = lib().rr_workspace_bytes(ctypes.byref(rr_dims(self.d.nx, self.d.nu, self.d.N, self.d.flags, cb)))
            tot += (w + 255) & ~255
        return tot

    def launch_pipelined(self, streams, nchunks: int = 8, ws=None):
        """rr_factor_solve_host_pipelined: chunks round-robin over `streams` (torch.cuda.Stream list;
        streams[0] is the completion stream).  ws: a workspace of pipelined_workspace_bytes(nchunks)."""
        if ws is None:
            ws = self.ws
        arr = (ctypes.c_void_p * len(streams))(*[s_.cuda_stream for s_ in streams])
        rc = lib().rr_factor_solve_host_pipelined(ctypes.byref(self.d), ctypes.byref(self.ph), ctypes.byref(self.sh),
                                                  self.sth, ctypes.byref(self.pd), ctypes.byref(self.sd), self.std,
                                                  _p(ws), ws.numel() * 8, int(nchunks), arr, len(streams))
        check(rc, "rr_factor_solve_host_pipelined")
