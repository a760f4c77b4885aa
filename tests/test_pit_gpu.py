"""GPU parity of the parallel-in-time solve (rr_factor_solve_pit, the paper's future
work P:688-691) against the oracle T2: the same unique solution of the regularized system, computed
by block cyclic reduction on the δ_s-reduced state system, δ_s = max(δ, 1e-4), followed by iterated
refinement on the caller's δ (δ = 0, classic LQR, included).  FP64 bar 1e-9."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


def rr():
    import paper_2509_16370_b200 as m
    return m


def rel(g, o):
    g = np.asarray(g).reshape(len(g), -1)
    o = np.asarray(o).reshape(len(o), -1)
    if g.size == 0:
        return 0.0
    return float(np.max(np.max(np.abs(g - o), axis=1) / np.maximum(np.max(np.abs(o), axis=1), 1e-300)))


@pytest.mark.parametrize("nx,nu,N,batch", [(12, 4, 100, 3), (12, 4, 1, 4), (12, 4, 2, 2), (4, 1, 37, 5),
                                           (2, 1, 10, 1), (3, 2, 64, 2), (16, 16, 9, 2), (5, 3, 0, 2),
                                           (7, 6, 129, 2)])
@pytest.mark.parametrize("delta", [0.0, 1e-8, 1e-6, 1e-4, 1e-2, 1.0])
def test_pit_parity(nx, nu, N, batch, delta):
    p = synth.random_stable_lqr(nx, nu, N, batch, seed=nx * 13 + N, delta=delta)
    out = rr().rr_factor_solve_pit(p.to("cuda"))
    torch.cuda.synchronize()
    o = oracle.rr_solve_t2(p)
    assert np.all(out["status"].cpu().numpy() == 0)
    for k in ("x", "u", "y"):
        assert rel(out[k].cpu().numpy(), o[k]) <= 1e-9, (k, rel(out[k].cpu().numpy(), o[k]))


def test_pit_c1_golden_and_long_horizon():
    m = rr()
    p = synth.double_integrator_c1()
    out = m.rr_factor_solve_pit(p.to("cuda"))
    o = oracle.rr_solve_t2(p)
    for k in ("x", "u", "y"):
        assert rel(out[k].cpu().numpy(), o[k]) <= 1e-9
    q = synth.random_stable_lqr(12, 4, 2048, 1, seed=5, delta=1e-4)
    a = m.rr_factor_solve_pit(q.to("cuda"))
    b = m.rr_factor_solve(q.to("cuda"))
    torch.cuda.synchronize()
    for k in ("x", "u", "y"):
        assert rel(a[k].cpu().numpy(), b[k].cpu().numpy()) <= 1e-9


def test_pit_shared_and_failure():
    m = rr()
    p = synth.lti_problem(12, 4, 33, 3, seed=2, delta=1e-3)
    out = m.rr_factor_solve_pit(p.to("cuda"))
    o = oracle.rr_solve_t2(p.expanded())
    for k in ("x", "u", "y"):
        assert rel(out[k].cpu().numpy(), o[k]) <= 1e-9
    z = synth.random_stable_lqr(4, 1, 6, 3, seed=4).with_delta(0.0)   # δ = 0: classic LQR, by refinement
    zo = m.rr_factor_solve_pit(z.to("cuda"))
    oz = oracle.rr_solve_t2(z)
    assert np.all(zo["status"].cpu().numpy() == 0)
    for k in ("x", "u", "y"):
        assert rel(zo[k].cpu().numpy(), oz[k]) <= 1e-9
    bad_p = synth.random_stable_lqr(4, 1, 6, 3, seed=4)
    bad_p.R[1, 2] = -1e6                                                  # R_i not PD in instance 1: no solution
    bad = m.rr_factor_solve_pit(bad_p.to("cuda"))
    st = bad["status"].cpu().numpy()
    assert st[1] != 0 and st[0] == 0 and st[2] == 0


def test_cuda_graph_capture_replay():
    """The C-ABI calls are stream-ordered with no host synchronisation, so they can be captured in a
    CUDA graph and replayed (the latency path for the multi-launch parallel-in-time solve)."""
    m = rr()
    p = synth.random_stable_lqr(12, 4, 200, 2, seed=8, delta=1e-3).to("cuda")
    ref_pit = m.rr_factor_solve_pit(p)
    ref_seq = m.rr_factor_solve(p)
    torch.cuda.synchronize()
    out_pit = m.alloc_solution(p)
    nb = m._lib.lib().rr_pit_workspace_bytes(__import__("ctypes").byref(m.rr.dims_of(p)))
    ws = torch.empty((nb + 7) // 8, dtype=torch.float64, device="cuda")
    call = m.Marshalled(p, m.alloc_solution(p))
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):   # warm-up outside the capture
        m.rr_factor_solve_pit(p, out=out_pit, workspace=ws, stream=s)
        call.launch(s)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        m.rr_factor_solve_pit(p, out=out_pit, workspace=ws, stream=torch.cuda.current_stream())
        call.launch(torch.cuda.current_stream())
    for k in ("x", "u", "y"):
        out_pit[k].zero_()
        call.sol[k].zero_()
    g.replay()
    torch.cuda.synchronize()
    for k in ("x", "u", "y"):
        assert torch.equal(out_pit[k], ref_pit[k]) and torch.equal(call.sol[k], ref_seq[k]), k


@pytest.mark.parametrize("nx,nu,N,batch,delta", [(12, 4, 64, 1, 1e-4), (4, 1, 30, 9, 0.0), (5, 3, 17, 6, 1e-2)])
def test_pit_single_launch_equals_step_launches(nx, nu, N, batch, delta, monkeypatch):
    """Up to 2,048 items per step the whole solve runs as one cooperative launch (grid barrier
    between steps); RR_PIT_STEPS=1 forces one launch per step.  Each item does the same arithmetic in
    both, so the results are bitwise equal (and at the parity bar against the oracle)."""
    p = synth.random_stable_lqr(nx, nu, N, batch, seed=900 + N, delta=delta)
    outs = []
    for flag in ("0", "1"):
        monkeypatch.setenv("RR_PIT_STEPS", flag)
        o = rr().rr_factor_solve_pit(p.to("cuda"))
        torch.cuda.synchronize()
        outs.append({k: v.cpu() for k, v in o.items()})
    for k in ("x", "u", "y", "status"):
        assert torch.equal(outs[0][k], outs[1][k]), k
    ref = oracle.rr_solve_t2(p, nthreads=4)
    g = {k: outs[0][k].numpy() for k in ("x", "u", "y", "status")}
    assert np.array_equal(g["status"], ref["status"])
    for k in ("x", "u", "y"):
        num = np.abs(g[k] - ref[k]).reshape(batch, -1).max(1)
        den = np.maximum(np.abs(ref[k]).reshape(batch, -1).max(1), 1e-300)
        assert float((num / den).max()) <= 1e-9, k
