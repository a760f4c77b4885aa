"""Loads the in-tree CUDA library librr_b200.so (built by build.py).  No CPU fallback: if the
library is missing or cannot be loaded, every entry point raises."""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# RR_B200_LIB: alternate in-tree build of the same library (kernel A/B experiments only)
LIB_PATH = os.environ.get("RR_B200_LIB") or os.path.join(HERE, "librr_b200.so")
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


class rr_residual_buf(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in ("q", "r", "c", "qN", "c0")]


RR_FLAG_ACCUMULATE = 1
RR_FLAG_FACTOR_FP32 = 8


class ipm_dims(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in ("nx", "nu", "N", "ng", "ngN", "nc", "ncN", "model")] + \
               [("batch", ctypes.c_int64)]


IPM_DATA_FIELDS = ("s0", "fval", "gradf", "gradfN", "Q", "M", "R", "QN", "A", "B", "dres",
                   "ce", "Ce", "ceN", "CeN", "gv", "Gj", "gvN", "GjN", "model_params")
IPM_ITER_FIELDS = ("x", "u", "s", "z", "sN", "zN", "y", "lam", "lamN", "mu", "eta")
IPM_RES_FIELDS = ("dx", "du", "ds", "dsN", "dy", "dlam", "dlamN", "dz", "dzN",
                  "alpha_p", "alpha_d", "D", "merit0", "merit_acc", "n_backtracks")


class ipm_stage_data(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in IPM_DATA_FIELDS]


class ipm_iterate(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in IPM_ITER_FIELDS]


class ipm_params(ctypes.Structure):
    _fields_ = [("tau", ctypes.c_double), ("armijo_c", ctypes.c_double), ("beta", ctypes.c_double),
                ("max_backtracks", ctypes.c_int32), ("pad", ctypes.c_int32)]


class ipm_solve_settings(ctypes.Structure):
    _fields_ = [(f, ctypes.c_double) for f in ("mu_min", "kappa", "kappa_mu", "theta_mu", "eta_max", "kappa_eta",
                                               "tol_kkt")] + \
               [("max_iters", ctypes.c_int32), ("linear_merit", ctypes.c_int32), ("step", ipm_params)]


class ipm_solve_report(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in ("status", "iters", "mu", "eta", "r_stat", "r_feas", "r_comp")]


class ipm_trial_values(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in ("fval", "dres", "ce", "ceN", "gv", "gvN")]


class ipm_result(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in IPM_RES_FIELDS]


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
            L.rr_factor_solve_host_pipelined.restype = ctypes.c_int32
            L.rr_factor_solve_host_pipelined.argtypes = [ctypes.POINTER(rr_dims), ctypes.POINTER(rr_problem),
                                                         ctypes.POINTER(rr_solution), ctypes.c_void_p,
                                                         ctypes.POINTER(rr_problem), ctypes.POINTER(rr_solution),
                                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                                         ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32]
            L.rr_factor_bytes.restype = ctypes.c_int64
            L.rr_factor_bytes.argtypes = [ctypes.POINTER(rr_dims)]
            L.rr_solve_workspace_bytes.restype = ctypes.c_int64
            L.rr_solve_workspace_bytes.argtypes = [ctypes.POINTER(rr_dims)]
            L.rr_factor.restype = ctypes.c_int32
            L.rr_factor.argtypes = [ctypes.POINTER(rr_dims), ctypes.POINTER(rr_problem), ctypes.c_void_p,
                                    ctypes.c_int64, ctypes.POINTER(rr_factor_buf), ctypes.c_void_p, ctypes.c_void_p]
            L.rr_solve.restype = ctypes.c_int32
            L.rr_solve.argtypes = [ctypes.POINTER(rr_dims), ctypes.POINTER(rr_problem), ctypes.c_void_p,
                                   ctypes.c_int64, ctypes.POINTER(rr_factor_buf), ctypes.POINTER(rr_solution),
                                   ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
            L.rr_pit_workspace_bytes.restype = ctypes.c_int64
            L.rr_pit_workspace_bytes.argtypes = [ctypes.POINTER(rr_dims)]
            L.rr_factor_solve_pit.restype = ctypes.c_int32
            L.rr_factor_solve_pit.argtypes = [ctypes.POINTER(rr_dims), ctypes.POINTER(rr_problem), ctypes.POINTER(rr_solution),
                                              ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
            L.rr_residual.restype = ctypes.c_int32
            L.rr_residual.argtypes = [ctypes.POINTER(rr_dims), ctypes.POINTER(rr_problem), ctypes.POINTER(rr_solution),
                                      ctypes.POINTER(rr_residual_buf), ctypes.c_void_p, ctypes.c_void_p]
            L.ipm_workspace_bytes.restype = ctypes.c_int64
            L.ipm_workspace_bytes.argtypes = [ctypes.POINTER(ipm_dims)]
            L.ipm_solve_workspace_bytes.restype = ctypes.c_int64
            L.ipm_solve_workspace_bytes.argtypes = [ctypes.POINTER(ipm_dims)]
            L.ipm_solve.restype = ctypes.c_int32
            L.ipm_solve.argtypes = [ctypes.POINTER(ipm_dims), ctypes.POINTER(ipm_stage_data), ctypes.POINTER(ipm_iterate),
                                    ctypes.POINTER(ipm_solve_settings), ctypes.POINTER(ipm_solve_report),
                                    ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
            L.ipm_direction.restype = ctypes.c_int32
            L.ipm_direction.argtypes = [ctypes.POINTER(ipm_dims), ctypes.POINTER(ipm_stage_data),
                                        ctypes.POINTER(ipm_iterate), ctypes.POINTER(ipm_params),
                                        ctypes.POINTER(ipm_result), ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_void_p, ctypes.c_void_p]
            L.ipm_merit.restype = ctypes.c_int32
            L.ipm_merit.argtypes = [ctypes.POINTER(ipm_dims), ctypes.POINTER(ipm_stage_data), ctypes.POINTER(ipm_iterate),
                                    ctypes.POINTER(ipm_result), ctypes.c_void_p, ctypes.POINTER(ipm_trial_values),
                                    ctypes.c_void_p, ctypes.c_void_p]
            L.ipm_update.restype = ctypes.c_int32
            L.ipm_update.argtypes = [ctypes.POINTER(ipm_dims), ctypes.POINTER(ipm_iterate), ctypes.POINTER(ipm_result),
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
            L.ipm_step.restype = ctypes.c_int32
            L.ipm_step.argtypes = [ctypes.POINTER(ipm_dims), ctypes.POINTER(ipm_stage_data),
                                   ctypes.POINTER(ipm_iterate), ctypes.POINTER(ipm_params),
                                   ctypes.POINTER(ipm_result), ctypes.c_void_p, ctypes.c_int64,
                                   ctypes.c_void_p, ctypes.c_void_p]
            _lib = L
    return _lib


def check(rc: int, what: str):
    if rc != 0:
        msg = lib().rr_last_error().decode(errors="replace")
        raise RRError("%s failed (rc=%d): %s" % (what, rc, msg))
