"""CPU ORACLE for arXiv 2509.16370 -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import this package.  The product path (paper_2509_16370_b200) never
imports it; it shares no code with the CUDA path.

Tiers:
  T1 (dense.py)      the DEFINITION: assemble the regularized LQR KKT matrix of §1.4
                      / Eq.(4x4) densely and solve it with LAPACK.
  T2 (rr_oracle.c)   the paper's recursion Eq.(RR), forward pass and dual
                     recovery, literally, in plain C loops;
                     pinned to T1 and to the textbook pins in tests/.
  R  (residual.py)   the KKT residual K[x; y] + [s; c] (the paper's third callback).
  IPM (ipm.py)       condense -> T2 -> expand, merit,
                     directional derivative, line search (P:221-222 + reading R12).
"""
from .rr import build_oracle, rr_solve_t2, load_oracle  # noqa: F401
from .dense import assemble_reglqr, rr_solve_dense, unpack_solution  # noqa: F401
from .residual import residual_dense, residual_blocks  # noqa: F401,E402
