"""GPU parity of the thread-per-instance ipm_step kernel for the C4 shape (csrc/ipm_c4t.cu: n = 4,
m = 1, n_g = 4, n_c = 0; an A/B variant selected by RR_IPM_C4T=1 -- measured slower than the default
lane-group kernel) against the CPU oracle and against the lane-group kernel, through the
C-ABI.  Bar: blockwise relative
≤ 1e-9, status words and backtrack counts exact."""
import numpy as np
import pytest
import torch

from oracle.ipm import ipm_step_oracle
from synth.ipm_workloads import cartpole_c4, random_lq_ocp
from test_ipm_gpu import TOL, assert_ipm_parity, rel_blocks, run

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _c4t(monkeypatch):
    monkeypatch.setenv("RR_IPM_C4T", "1")


def both_kernels(p, monkeypatch, **kw):
    import paper_2509_16370_b200 as rr
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("RR_IPM_C4T", flag)
        dev = p.to("cuda")
        res = rr.ipm_step(dev, **kw)
        torch.cuda.synchronize()
        out[flag] = ({k: v.cpu().numpy() for k, v in res.items()}, {k: v.cpu().numpy() for k, v in dev.it.items()})
    return out["1"], out["0"]


@pytest.mark.parametrize("batch,N,ngN", [(1, 1, 0), (33, 7, 2), (70, 20, 4), (333, 12, 1)])
def test_c4t_lq_matches_oracle(batch, N, ngN):
    """C4-shaped LQ problems (model LQ), partial warps, every terminal constraint count."""
    p = random_lq_ocp(4, 1, N, batch, seed=400 + N, ng=4, ngN=ngN, nc=0, ncN=0, eta=1e4)
    assert_ipm_parity(*run(p))


@pytest.mark.parametrize("batch,N,variant", [(97, 100, "C4"), (45, 30, "C4-LS")])
def test_c4t_cartpole_matches_oracle_and_lane_kernel(batch, N, variant, monkeypatch):
    p = cartpole_c4(batch, seed=31, N=N, variant=variant)
    (g1, it1), (g0, it0) = both_kernels(p, monkeypatch)
    o, oit = ipm_step_oracle(p, nthreads=8)
    assert_ipm_parity(g1, it1, o, oit)
    assert np.array_equal(g1["status"], g0["status"]) and np.array_equal(g1["n_backtracks"], g0["n_backtracks"])
    for k in ("dx", "du", "dy", "ds", "dz", "dsN", "dzN"):
        assert rel_blocks(g1[k], g0[k]) <= TOL, k
    for k in ("x", "u", "y", "s", "z", "sN", "zN"):
        assert rel_blocks(it1[k], it0[k]) <= TOL, k


def test_c4t_nonpositive_slack_and_ls_failure():
    p = random_lq_ocp(4, 1, 9, 40, seed=5, ng=4, ngN=2, nc=0, ncN=0, eta=1e4)
    p.it["s"][7, 4, 2] = -1e-3
    p.it["zN"][11, 1] = 0.0
    g, git, o, oit = run(p)
    assert g["status"][7] == (4 | (4 << 8)) and g["status"][11] == (4 | (9 << 8))
    assert np.all(np.isnan(g["dx"][7])) and np.all(np.isnan(g["dsN"][11]))
    np.testing.assert_array_equal(git["x"][7], p.it["x"][7].numpy())
    assert_ipm_parity(g, git, o, oit)
    q = cartpole_c4(40, seed=7, N=20, variant="C4-LS")
    g, git, o, oit = run(q, max_backtracks=0)
    assert np.any(g["status"] == 5)
    assert_ipm_parity(g, git, o, oit)


def test_c4t_direction_only_matches_lane_kernel(monkeypatch):
    """ipm_direction (rows a1-a7: no line search, iterate untouched) on both kernels."""
    import paper_2509_16370_b200 as rr
    p = cartpole_c4(50, seed=3, N=25)
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("RR_IPM_C4T", flag)
        dev = p.to("cuda")
        res = rr.ipm_direction(dev)
        torch.cuda.synchronize()
        out[flag] = {k: v.cpu().numpy() for k, v in res.items()}
        for k in ("x", "s", "z", "y"):
            assert torch.equal(dev.it[k].cpu(), p.it[k]), k
    a, b = out["1"], out["0"]
    assert np.array_equal(a["status"], b["status"])
    for k in ("dx", "du", "dy", "ds", "dz"):
        assert rel_blocks(a[k], b[k]) <= TOL, k
    for k in ("alpha_p", "alpha_d", "D", "merit0"):
        assert np.all(np.abs(a[k] - b[k]) <= TOL * np.maximum(np.abs(b[k]), 1.0)), k
