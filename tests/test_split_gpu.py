"""GPU parity of the factorization / solve split (rr_factor, rr_solve; the paper's factorization and
solve callbacks) through the C-ABI against the CPU oracle T2.

Bar (BASELINE north_star): per instance and output block, normwise relative error <= 1e-9 (FP64);
status words bit-exact.  The factor records are checked against the oracle's V_i, K_i and against
the defining identities of S_i^-1 = (I + δV_i)^-1 and G_i^-1 = (B_iᵀ W_i B_i + R_i)^-1."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL = 1e-9


def rr():
    import paper_2509_16370_b200 as m
    return m


def blockwise_rel(g, o):
    g = np.asarray(g).reshape(g.shape[0], -1)
    o = np.asarray(o).reshape(o.shape[0], -1)
    if g.shape[1] == 0 or g.shape[0] == 0:
        return 0.0
    num = np.max(np.abs(g - o), axis=1)
    den = np.maximum(np.max(np.abs(o), axis=1), 1e-300)
    return float(np.max(num / den))


def with_rhs(p, seed):
    """Same matrices (A, B, Q, M, R, Q_N, δ), a fresh right-hand side (q, r, c, q_N, c_0)."""
    g = torch.Generator().manual_seed(seed)
    kw = {f: getattr(p, f).clone() for f in p.FIELDS}
    for f in ("q", "r", "c", "qN", "c0"):
        kw[f] = torch.rand(kw[f].shape, generator=g, dtype=torch.float64) * 2 - 1
    return synth.RRProblem(p.nx, p.nu, p.N, **kw)


def factor_solve(p):
    m = rr()
    dev = p.to("cuda")
    fac = m.alloc_factor(dev)
    F, st_f = m.rr_factor(dev, fac=fac)
    sol = m.rr_solve(dev, F, fac=fac)
    torch.cuda.synchronize()
    out = {k: v.cpu().numpy() for k, v in sol.items()}
    out.update({k: v.cpu().numpy() for k, v in fac.items()})
    out["status_f"] = st_f.cpu().numpy()
    out["F"] = F.cpu().numpy()
    return out


def unpack(P, n):
    F = np.zeros(P.shape[:-1] + (n, n))
    k = 0
    for c in range(n):
        for r in range(c, n):
            F[..., r, c] = P[..., k]
            F[..., c, r] = P[..., k]
            k += 1
    return F


@pytest.mark.parametrize("nx,nu,N,batch", [
    (12, 4, 9, 37),      # exact C2 shape, ragged batch
    (12, 4, 1, 5),
    (4, 1, 13, 33),      # exact C4-core shape
    (2, 1, 10, 17),      # exact C1 shape
    (1, 1, 5, 9),        # padded kernels
    (3, 2, 6, 21),
    (7, 6, 4, 11),
    (16, 16, 3, 5),
    (10, 9, 4, 6),
])
@pytest.mark.parametrize("delta", [0.0, 1e-8, 1e-4, 1.0])
def test_split_parity(nx, nu, N, batch, delta):
    p = synth.random_stable_lqr(nx, nu, N, batch, seed=nx * 100 + nu * 10 + N + 7, delta=delta)
    g = factor_solve(p)
    o = oracle.rr_solve_t2(p, nthreads=8, want_policy=True)
    assert np.array_equal(g["status_f"], o["status"])
    assert np.all(g["status"] == 0)
    for k in ("x", "u", "y", "V", "v", "K", "k"):
        assert blockwise_rel(g[k], o[k]) <= TOL, k


def test_factor_records_identities():
    """Record i = [V_i | S_i^-1 | K_i | G_i^-1]: V, K equal the oracle's; S^-1 (I + δV) = I;
    G_i^-1 (B_iᵀ W_i B_i + R_i) = I with W_i = S_{i+1}^-1 V_{i+1} from the oracle's V."""
    n, m, N, b, delta = 12, 4, 6, 9, 1e-2
    p = synth.random_stable_lqr(n, m, N, b, seed=31, delta=delta)
    g = factor_solve(p)
    o = oracle.rr_solve_t2(p, want_policy=True)
    s = n * (n + 1) // 2
    F = g["F"]
    assert F.shape == (b, N + 1, rr().factor_record_doubles(n, m))
    assert blockwise_rel(F[:, :, :s], o["V"]) <= TOL
    assert blockwise_rel(F[:, :N, 2 * s:2 * s + n * m], o["K"]) <= TOL
    V = unpack(o["V"], n)
    Sinv = unpack(F[:, :, s:2 * s], n)
    eye = np.eye(n)
    assert np.max(np.abs(Sinv @ (eye + delta * V) - eye)) < 1e-12
    Ginv = unpack(F[:, :N, 2 * s + n * m:2 * s + n * m + m * (m + 1) // 2], m)
    Bm = p.B.numpy().reshape(b, N, m, n).transpose(0, 1, 3, 2)
    Rm = unpack(p.R.numpy(), m)
    W = np.linalg.solve(eye + delta * V[:, 1:], V[:, 1:])
    G = np.swapaxes(Bm, -1, -2) @ W @ Bm + Rm
    assert np.max(np.abs(Ginv @ G - np.eye(m))) < 1e-11


@pytest.mark.parametrize("nx,nu", [(12, 4), (4, 1), (5, 3)])
def test_one_factor_many_rhs(nx, nu):
    """One rr_factor serves several rr_solve calls with different right-hand sides."""
    m = rr()
    p = synth.random_stable_lqr(nx, nu, 15, 23, seed=5, delta=1e-4)
    dev = p.to("cuda")
    F, st = m.rr_factor(dev)
    for seed in (1, 2, 3):
        p2 = with_rhs(p, seed)
        sol = m.rr_solve(p2.to("cuda"), F)
        torch.cuda.synchronize()
        o = oracle.rr_solve_t2(p2)
        assert np.all(sol["status"].cpu().numpy() == 0)
        for k in ("x", "u", "y"):
            assert blockwise_rel(sol[k].cpu().numpy(), o[k]) <= TOL, (seed, k)


def test_split_equals_fused():
    p = synth.random_stable_lqr(12, 4, 30, 40, seed=9, delta=1e-4).to("cuda")
    a = rr().rr_factor_solve(p)
    F, _ = rr().rr_factor(p)
    b = rr().rr_solve(p, F)
    torch.cuda.synchronize()
    for k in ("x", "u", "y"):
        assert blockwise_rel(a[k].cpu().numpy(), b[k].cpu().numpy()) <= TOL


def test_horizon_zero_split():
    p = synth.random_stable_lqr(12, 4, 0, 3, seed=3, delta=1e-2)
    g = factor_solve(p)
    o = oracle.rr_solve_t2(p)
    for k in ("x", "y"):
        assert blockwise_rel(g[k], o[k]) <= TOL


def test_split_failed_factor_status():
    p = synth.random_stable_lqr(12, 4, 6, 10, seed=4, delta=1e-3)
    p.R[3, 2] = torch.tensor([-50.0, 0, 0, 0, -50.0, 0, 0, -50.0, 0, -50.0], dtype=torch.float64)
    g = factor_solve(p)
    o = oracle.rr_solve_t2(p)
    assert g["status_f"][3] == o["status"][3] == (1 | (2 << 8))
    assert g["status"][3] == 3 and np.all(np.isnan(g["x"][3]))
    ok = np.arange(10) != 3
    assert np.all(g["status"][ok] == 0)
    for k in ("x", "u", "y"):
        assert blockwise_rel(g[k][ok], o[k][ok]) <= TOL


def test_split_unsupported_and_empty():
    m = rr()
    p = synth.random_stable_lqr(40, 20, 2, 2, seed=1).to("cuda")
    with pytest.raises(m.RRError):
        m.rr_factor(p)
    e = synth.random_stable_lqr(12, 4, 5, 0, seed=1).to("cuda")
    F, st = m.rr_factor(e)
    sol = m.rr_solve(e, F)
    assert sol["x"].numel() == 0


def test_split_c2_full_size_sampled_parity():
    """rr_factor + rr_solve (+ rr_residual) in the configuration `bench.py --workload split` times:
    65,536 C2 instances; sampled instances against the oracle, all residual norms small."""
    m = rr()
    p = synth.random_stable_lqr_chunked(12, 4, 100, 65536, seed=2509, delta=1e-4, device="cuda")
    F, st = m.rr_factor(p)
    sol = m.rr_solve(p, F)
    _, norms = m.rr_residual(p, sol)
    torch.cuda.synchronize()
    assert int(st.abs().sum()) == 0 and int(sol["status"].abs().sum()) == 0
    assert float(norms.max()) < 1e-9
    idx = torch.tensor(sorted(set(np.random.default_rng(5).integers(0, 65536, 128).tolist()) | {0, 65535}), device="cuda")
    sub = p.select(idx)
    o = oracle.rr_solve_t2(sub.to("cpu"), nthreads=8)
    for k in ("x", "u", "y"):
        assert blockwise_rel(sol[k][idx].cpu().numpy(), o[k]) <= TOL, k


@pytest.mark.parametrize("delta", [0.0, 1e-4, 1.0])
def test_fp32_factor_record_and_refinement(delta):
    """rr_factor with FP32 records (RR_FLAG_FACTOR_FP32) + rr_solve carries the FP32
    rounding of the factor (error well above the FP64 path, far below 1); rr_residual +
    rr_solve(ACCUMULATE) refinement contracts it by ~1e-6 per step: within the 1e-9 bar of
    the oracle after two steps, and the records equal the FP64 records rounded to float."""
    m = rr()
    p = synth.random_stable_lqr(12, 4, 30, 64, seed=77, delta=delta)
    o = oracle.rr_solve_t2(p)
    dev = p.to("cuda")
    F32, st = m.rr_factor(dev, fp32=True)
    F64, st64 = m.rr_factor(dev)
    sol = m.rr_solve(dev, F32)
    torch.cuda.synchronize()
    assert int(st.abs().sum()) == 0 and int(sol["status"].abs().sum()) == 0
    assert F32.dtype == torch.float32 and F32.shape[-1] == 216
    f32, f64 = F32.cpu().numpy(), F64.cpu().numpy().astype(np.float32)
    np.testing.assert_array_equal(f32[:, :-1, :214], f64[:, :-1])      # records 0..N-1
    np.testing.assert_array_equal(f32[:, -1, :156], f64[:, -1, :156])  # record N: V_N, S_N⁻¹ (K, G⁻¹ unused)
    e0 = max(blockwise_rel(sol[k].cpu().numpy(), o[k]) for k in ("x", "u", "y"))
    assert 1e-12 < e0 < 1e-3, e0
    errs = [e0]
    for _ in range(2):
        m.rr_refine(dev, F32, sol, iters=1)
        torch.cuda.synchronize()
        errs.append(max(blockwise_rel(sol[k].cpu().numpy(), o[k]) for k in ("x", "u", "y")))
    assert errs[1] < errs[0] * 1e-3 and errs[2] <= TOL, errs


def test_fp32_factor_record_unsupported_shape():
    m = rr()
    p = synth.random_stable_lqr(4, 1, 5, 4, seed=1).to("cuda")
    with pytest.raises(m.RRError):
        m.rr_factor(p, fp32=True)
