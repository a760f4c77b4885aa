"""Loads the in-tree CUDA library librr_b200.so (built by build.py).  No CPU fallback: if the
library is missing or cannot be loaded, every entry point raises."""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librr_b200.so")
_lock = threading.Lock()
_lib = None


class RRError(RuntimeError):
    pass


class rr_dims(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("nu", ctypes.c_int32), ("N", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("batch", ctypes.c_int64)]


class rr_problem(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in ("A", "B", "Q", "M", "R", "q", "r", "c", "QN", "qN", "c0", "delta")]


class rr_factor_buf(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in ("V", "v", "K", "k")]


class rr_solution(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in ("x", "u", "y")]


def lib():
    """The loaded library (raises RRError if librr_b200.so is absent)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RRError("librr_b200.so not built: run `python -m paper_2509_16370_b200.build` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
            L = ctypes.CDLL(LIB_PATH)
            L.rr_last_error.restype = ctypes.c_char_p
            L.rr_version.restype = ctypes.c_char_p
            L.rr_workspace_bytes.restype = ctypes.c_int64
            L.rr_workspace_bytes.argtypes = [ctypes.POINTER(rr_dims)]
            L.rr_factor_solve.restype = ctypes.c_int32
            L.rr_factor_solve.argtypes = [ctypes.POINTER(rr_dims), ctypes.POINTER(rr_problem),
                                          ctypes.POINTER(rr_factor_buf), ctypes.POINTER(rr_solution),
                                          ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
            L.rr_factor_solve_host.restype = ctypes.c_int32
            L.rr_factor_solve_host.argtypes = [ctypes.POINTER(rr_dims), ctypes.POINTER(rr_problem),
                                               ctypes.POINTER(rr_solution), ctypes.c_void_p,
                                               ctypes.POINTER(rr_problem), ctypes.POINTER(rr_solution),
                                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
            _lib = L
    return _lib


def check(rc: int, what: str):
    if rc != 0:
        msg = lib().rr_last_error().decode(errors="replace")
        raise RRError("%s failed (rc=%d): %s" % (what, rc, msg))
