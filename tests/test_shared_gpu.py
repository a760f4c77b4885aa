"""Batch-shared operands (RR_FLAG_SHARED_DYN / RR_FLAG_SHARED_COST, LTI / fleet MPC):
one [N][...] copy of A, B (and/or Q, M, R, Q_N) serves every instance.  The kernels read the same
values as for the broadcast per-instance problem, so results must be bitwise identical to the
expanded problem, and within 1e-9 of the oracle."""
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
    return float(np.max(np.max(np.abs(g - o), axis=1) / np.maximum(np.max(np.abs(o), axis=1), 1e-300)))


@pytest.mark.parametrize("nx,nu,N,batch", [(12, 4, 20, 37), (4, 1, 15, 33), (3, 2, 7, 9), (16, 16, 4, 5)])
@pytest.mark.parametrize("dyn,cost", [(True, True), (True, False), (False, True)])
def test_shared_equals_expanded(nx, nu, N, batch, dyn, cost):
    m = rr()
    p = synth.lti_problem(nx, nu, N, batch, seed=nx + N, delta=1e-3, shared_dyn=dyn, shared_cost=cost)
    e = p.expanded()
    ps, pe = p.to("cuda"), e.to("cuda")
    a = m.rr_factor_solve(ps)
    b = m.rr_factor_solve(pe)
    Fs, _ = m.rr_factor(ps)
    Fe, _ = m.rr_factor(pe)
    ss = m.rr_solve(ps, Fs)
    se = m.rr_solve(pe, Fe)
    rs, ns = m.rr_residual(ps, ss)
    re_, ne = m.rr_residual(pe, se)
    torch.cuda.synchronize()
    for k in ("x", "u", "y", "status"):
        assert torch.equal(a[k], b[k]), k
        assert torch.equal(ss[k], se[k]), k
    sn = nx * (nx + 1) // 2
    used = 2 * sn + nx * nu + nu * (nu + 1) // 2   # record padding and record N's K / G⁻¹ are unused
    assert torch.equal(Fs[:, :N, :used], Fe[:, :N, :used]) and torch.equal(Fs[:, N, :2 * sn], Fe[:, N, :2 * sn])
    assert torch.equal(ns, ne)
    o = oracle.rr_solve_t2(e)
    for k in ("x", "u", "y"):
        assert rel(a[k].cpu().numpy(), o[k]) <= 1e-9


def test_shared_host_path():
    m = rr()
    p = synth.lti_problem(12, 4, 10, 16, seed=3)
    hp = synth.RRProblem(p.nx, p.nu, p.N, **{f: getattr(p, f).pin_memory() for f in p.FIELDS})
    dp = p.to("cuda")
    hs = {k: torch.empty(v.shape, dtype=v.dtype).pin_memory() for k, v in m.alloc_solution(dp).items()}
    ds = m.alloc_solution(dp)
    call = m.HostMarshalled(hp, hs, dp, ds)
    call.launch()
    torch.cuda.synchronize()
    o = oracle.rr_solve_t2(p.expanded())
    for k in ("x", "u", "y"):
        assert rel(hs[k].numpy(), o[k]) <= 1e-9
    assert call.h2d_bytes < p.expanded().nbytes() / 2


def test_shared_large_shape_unsupported():
    m = rr()
    p = synth.lti_problem(40, 20, 3, 2, seed=1).to("cuda")
    with pytest.raises(m.RRError):
        m.rr_factor_solve(p)


@pytest.mark.parametrize("shared,nchunks,nstreams", [(False, 7, 3), (False, 1, 1), (True, 5, 2), (False, 50, 3)])
def test_host_pipelined_equals_serial(shared, nchunks, nstreams):
    """rr_factor_solve_host_pipelined (chunks round-robin over streams, copies overlapped with the
    solve) gives bitwise the results of rr_factor_solve_host, per-instance and batch-shared operands,
    more chunks than instances included."""
    m = rr()
    if shared:
        p = synth.lti_problem(12, 4, 10, 23, seed=5)
    else:
        p = synth.random_stable_lqr(12, 4, 10, 23 if nchunks < 50 else 13, seed=5, delta=1e-4)
    hp = synth.RRProblem(p.nx, p.nu, p.N, **{f: getattr(p, f).pin_memory() for f in p.FIELDS})
    dp = p.to("cuda")
    out = []
    for pipelined in (False, True):
        hs = {k: torch.full(v.shape, float("nan"), dtype=v.dtype).pin_memory() if v.is_floating_point()
              else torch.zeros(v.shape, dtype=v.dtype).pin_memory() for k, v in m.alloc_solution(dp).items()}
        ds = m.alloc_solution(dp)
        call = m.HostMarshalled(hp, hs, dp, ds)
        if pipelined:
            streams = [torch.cuda.current_stream()] + [torch.cuda.Stream() for _ in range(nstreams - 1)]
            ws = torch.empty((call.pipelined_workspace_bytes(nchunks) + 7) // 8, dtype=torch.float64, device="cuda")
            call.launch_pipelined(streams, nchunks, ws)
            streams[0].synchronize()
        else:
            call.launch()
        torch.cuda.synchronize()
        out.append(hs)
    for k in ("x", "u", "y", "status"):
        assert torch.equal(out[0][k], out[1][k]), k
    o = oracle.rr_solve_t2(p.expanded() if shared else p)
    for k in ("x", "u", "y"):
        assert rel(out[1][k].numpy(), o[k]) <= 1e-9


@pytest.mark.parametrize("nx,nu,N,batch", [(12, 4, 20, 37), (4, 1, 15, 33), (3, 2, 7, 9), (16, 16, 4, 5)])
@pytest.mark.parametrize("shared", [False, True])
def test_stage_invariant_equals_expanded(nx, nu, N, batch, shared):
    """RR_FLAG_STAGE_INVARIANT_DYN | _COST (LTI MPC): one stage block of A, B, Q, M, R per
    instance (or, with shared, for the whole batch) serves every stage.  rr_factor_solve, the split
    API, rr_residual and the parallel-in-time solve give bitwise the results of the expanded problem,
    and the oracle's within 1e-9."""
    m = rr()
    p = synth.lti_invariant_problem(nx, nu, N, batch, seed=nx + N, delta=1e-3, shared=shared)
    e = p.expanded()
    assert m.shared_flags(p) & (m.rr.RR_FLAG_STAGE_INVARIANT_DYN | m.rr.RR_FLAG_STAGE_INVARIANT_COST)
    ps, pe = p.to("cuda"), e.to("cuda")
    a, b = m.rr_factor_solve(ps), m.rr_factor_solve(pe)
    Fs, _ = m.rr_factor(ps)
    Fe, _ = m.rr_factor(pe)
    ss, se = m.rr_solve(ps, Fs), m.rr_solve(pe, Fe)
    rs, ns = m.rr_residual(ps, ss)
    re_, ne = m.rr_residual(pe, se)
    pa, pb = m.rr_factor_solve_pit(ps), m.rr_factor_solve_pit(pe)
    torch.cuda.synchronize()
    for k in ("x", "u", "y", "status"):
        assert torch.equal(a[k], b[k]), k
        assert torch.equal(ss[k], se[k]), k
        assert torch.equal(pa[k], pb[k]), k
    sn = nx * (nx + 1) // 2
    used = 2 * sn + nx * nu + nu * (nu + 1) // 2
    assert torch.equal(Fs[:, :N, :used], Fe[:, :N, :used]) and torch.equal(Fs[:, N, :2 * sn], Fe[:, N, :2 * sn])
    assert torch.equal(ns, ne)
    o = oracle.rr_solve_t2(e)
    for k in ("x", "u", "y"):
        assert rel(a[k].cpu().numpy(), o[k]) <= 1e-9


def test_stage_invariant_host_paths():
    m = rr()
    p = synth.lti_invariant_problem(12, 4, 10, 16, seed=3)
    hp = synth.RRProblem(p.nx, p.nu, p.N, **{f: getattr(p, f).pin_memory() for f in p.FIELDS})
    dp = p.to("cuda")
    o = oracle.rr_solve_t2(p.expanded())
    for pipelined in (False, True):
        hs = {k: torch.empty(v.shape, dtype=v.dtype).pin_memory() for k, v in m.alloc_solution(dp).items()}
        call = m.HostMarshalled(hp, hs, dp, m.alloc_solution(dp))
        if pipelined:
            ws = torch.empty((call.pipelined_workspace_bytes(3) + 7) // 8, dtype=torch.float64, device="cuda")
            call.launch_pipelined([torch.cuda.current_stream(), torch.cuda.Stream()], 3, ws)
        else:
            call.launch()
        torch.cuda.synchronize()
        for k in ("x", "u", "y"):
            assert rel(hs[k].numpy(), o[k]) <= 1e-9, (pipelined, k)
    assert call.h2d_bytes < p.expanded().nbytes() / 4
