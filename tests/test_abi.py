"""CPU checks of the boundary: the C-ABI library builds, loads without a GPU, and exports every
function include/*.h declares; the binding fails loudly without CUDA tensors (no CPU fallback)."""
import ctypes
import glob
import os
import re

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        txt = open(h).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        for mm in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*([a-z_][a-z0-9_]*)\s*\(", txt, re.M):
            names.add(mm.group(1))
    return names


def test_library_exports_every_declared_symbol():
    from paper_2509_16370_b200 import build
    path = build.build()
    lib = ctypes.CDLL(path)
    names = declared_functions()
    assert {"rr_factor_solve", "rr_workspace_bytes", "rr_last_error", "rr_version"} <= names
    for nm in names:
        assert hasattr(lib, nm), nm


def test_workspace_query_and_version():
    import paper_2509_16370_b200 as m
    assert "sm_100a" in m.version()
    assert m.workspace_bytes(12, 4, 100, 65536) > 0
    with pytest.raises(m.RRError):
        m.workspace_bytes(40, 30, 10, 4)   # no compiled kernel


def test_binding_rejects_cpu_tensors():
    import paper_2509_16370_b200 as m
    import synth
    p = synth.random_stable_lqr(4, 1, 3, 2, seed=0)
    with pytest.raises(m.RRError):
        m.rr_factor_solve(p)


def test_fp32_factor_record_size_query():
    """RR_FLAG_FACTOR_FP32 (include/rr.h): FP32 records for 12 x 4 only, R rounded up to 4 floats."""
    import paper_2509_16370_b200 as m
    R = m.factor_record_doubles(12, 4)
    assert R == 214
    assert m.factor_bytes(12, 4, 100, 8, fp32=True) == 8 * 101 * 216 * 4
    assert m.factor_bytes(12, 4, 100, 8) == 8 * 101 * R * 8
    with pytest.raises(m.RRError):
        m.factor_bytes(4, 1, 10, 8, fp32=True)   # no FP32 kernel for this shape


def test_operand_layout_flags_from_shapes():
    """include/rr.h RR_FLAG_SHARED_* / RR_FLAG_STAGE_INVARIANT_*: the binding infers them from the
    operand shapes ([b, N, e] | [N, e] batch-shared | [b, 1, e] stage-invariant | [1, e] both)."""
    import paper_2509_16370_b200 as m
    import synth
    R = m.rr
    assert m.shared_flags(synth.random_stable_lqr(4, 1, 5, 3, seed=0)) == 0
    assert m.shared_flags(synth.lti_problem(4, 1, 5, 3, seed=0)) == R.RR_FLAG_SHARED_DYN | R.RR_FLAG_SHARED_COST
    assert m.shared_flags(synth.lti_invariant_problem(4, 1, 5, 3, seed=0)) == \
        R.RR_FLAG_STAGE_INVARIANT_DYN | R.RR_FLAG_STAGE_INVARIANT_COST
    assert m.shared_flags(synth.lti_invariant_problem(4, 1, 5, 3, seed=0, shared=True)) == \
        R.RR_FLAG_SHARED_DYN | R.RR_FLAG_SHARED_COST | R.RR_FLAG_STAGE_INVARIANT_DYN | R.RR_FLAG_STAGE_INVARIANT_COST
    p = synth.lti_invariant_problem(4, 1, 5, 3, seed=0)
    p.B = p.B.expand(3, 5, 4).contiguous()                 # A stage-invariant, B not: refused
    with pytest.raises(m.RRError):
        m.shared_flags(p)
    e = synth.lti_invariant_problem(4, 1, 5, 3, seed=0, shared=True).expanded()
    assert e.A.shape == (3, 5, 16) and e.QN.shape == (3, 10) and m.shared_flags(e) == 0
