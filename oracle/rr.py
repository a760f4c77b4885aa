"""ctypes wrapper of the plain-C oracle (rr_oracle.c).  TEST INFRASTRUCTURE ONLY."""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = [os.path.join(_HERE, "rr_oracle.c"), os.path.join(_HERE, "ipm_oracle.c")]
_HDR = [os.path.join(_HERE, "orc.h")]
_LIB = os.path.join(_HERE, "liborc.so")
_lock = threading.Lock()
_lib = None


def build_oracle(force: bool = False) -> str:
    """Compile the C oracle with plain -O2 (no BLAS, no intrinsics, no fast-math)."""
    srcs = [s for s in _SRC if os.path.exists(s)]
    newest = max(os.path.getmtime(s) for s in srcs + [h for h in _HDR if os.path.exists(h)])
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-ffp-contract=off",
                               "-o", tmp] + srcs + ["-lm", "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


def load_oracle():
    global _lib
    with _lock:
        if _lib is None:
            build_oracle()
            _lib = ctypes.CDLL(_LIB)
    return _lib


def _ptr(a):
    if a is None:
        return None
    assert a.dtype in (np.float64, np.int32) and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def _np(t):
    """torch tensor or array -> contiguous float64 numpy on host."""
    try:
        import torch
        if isinstance(t, torch.Tensor):
            return np.ascontiguousarray(t.detach().cpu().numpy(), dtype=np.float64)
    except ImportError:  # pragma: no cover
        pass
    return np.ascontiguousarray(t, dtype=np.float64)


def rr_solve_t2(prob, nthreads: int = 1, want_policy: bool = False):
    """Solve every instance of `prob` (synth.RRProblem, any device) with the T2 oracle.

    Returns dict with x [b,N+1,n], u [b,N,m], y [b,N+1,n], status [b] (and V, v, K, k
    in the ABI layout when want_policy)."""
    lib = load_oracle()
    n, m, N, b = prob.nx, prob.nu, prob.N, prob.batch
    arrs = [_np(getattr(prob, f)) for f in ("A", "B", "Q", "M", "R", "q", "r", "c", "QN", "qN", "c0", "delta")]
    x = np.zeros((b, N + 1, n))
    u = np.zeros((b, N, m))
    y = np.zeros((b, N + 1, n))
    st = np.zeros((b,), dtype=np.int32)
    V = v = K = k = None
    if want_policy:
        V = np.zeros((b, N + 1, n * (n + 1) // 2))
        v = np.zeros((b, N + 1, n))
        K = np.zeros((b, N, m * n))
        k = np.zeros((b, N, m))
    f = lib.orc_rr_solve
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int] + [ctypes.c_void_p] * 20
    rc = f(n, m, N, b, max(1, int(nthreads)), *[_ptr(a) for a in arrs], _ptr(x), _ptr(u), _ptr(y),
           _ptr(V), _ptr(v), _ptr(K), _ptr(k), _ptr(st))
    if rc != 0:
        raise ValueError("orc_rr_solve rejected its arguments (rc=%d)" % rc)
    out = dict(x=x, u=u, y=y, status=st)
    if want_policy:
        out.update(V=V, v=v, K=K, k=k)
    return out
