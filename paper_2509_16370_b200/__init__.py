"""B200-native (sm_100a) batched regularized Riccati recursion and regularized-IPM step of
arXiv 2509.16370.  All compute runs in the in-tree CUDA library librr_b200.so (include/rr.h);
this package only marshals torch CUDA tensors into the C-ABI.  There is no CPU fallback."""
from ._lib import RRError, LIB_PATH  # noqa: F401
from .rr import (rr_factor_solve, alloc_solution, alloc_factor, alloc_workspace,  # noqa: F401
                 workspace_bytes, Marshalled, HostMarshalled, version,
                 rr_factor, rr_solve, factor_bytes, factor_record_doubles, solve_workspace_bytes,
                 rr_residual, rr_refine, rr_factor_solve_pit, shared_flags)

from .ipm import ipm_step, IpmCall, ipm_solve, IpmSolveCall, ipm_direction, ipm_merit, ipm_update  # noqa: F401,E402

__version__ = "0.1"
