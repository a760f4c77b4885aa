"""GPU parity of ipm_step (rows a1-a8, librr_b200.so through the C-ABI) against the CPU oracle
(condense -> T2 -> expand -> merit/D -> Armijo line search -> update), on the same input bits.
Bar: per instance and block, normwise relative error ≤ 1e-9 (FP64); status and the accepted
backtracking index k bit-exact (no Armijo ties: margins ≥ 5e-6 relative)."""
import numpy as np
import pytest
import torch

from oracle.ipm import ipm_step_oracle
from synth.ipm_workloads import cartpole_c4, quadrotor_ipm, random_lq_ocp

pytestmark = pytest.mark.gpu
TOL = 1e-9


def rel_blocks(g, o):
    if np.asarray(g).size == 0:
        return 0.0
    g = np.asarray(g).reshape(g.shape[0], -1)
    o = np.asarray(o).reshape(o.shape[0], -1)
    if g.shape[1] == 0:
        return 0.0
    return float(np.max(np.max(np.abs(g - o), axis=1) / np.maximum(np.max(np.abs(o), axis=1), 1e-300)))


def run(p, **kw):
    import paper_2509_16370_b200 as rr
    dev = p.to("cuda")
    res = rr.ipm_step(dev, **kw)
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in res.items()}
    git = {k: v.cpu().numpy() for k, v in dev.it.items()}
    o, oit = ipm_step_oracle(p, nthreads=8, **kw)
    return g, git, o, oit


def assert_ipm_parity(g, git, o, oit):
    assert np.array_equal(g["status"], o["status"]), (g["status"], o["status"])
    ok = o["status"] == 0
    assert np.array_equal(g["n_backtracks"][ok], o["n_backtracks"][ok])
    for k in ("dx", "du", "dy", "ds", "dsN", "dz", "dzN", "dlam", "dlamN"):
        assert rel_blocks(g[k][ok], o[k][ok]) <= TOL, k
    for k in ("alpha_p", "alpha_d"):
        assert np.max(np.abs(g[k] - o[k]) / np.maximum(np.abs(o[k]), 1e-300)) <= 1e-12, k
    for k in ("D", "merit0", "merit_acc"):
        a, b = g[k][ok], o[k][ok]
        assert np.all(np.abs(a - b) <= TOL * np.maximum(np.abs(b), 1.0)), (k, np.max(np.abs(a - b)))
    for k in ("x", "u", "y", "s", "z", "sN", "zN", "lam", "lamN"):
        assert rel_blocks(git[k][ok], oit[k][ok]) <= TOL, k


@pytest.mark.parametrize("n,m,N,ng,ngN,nc,ncN,eta", [
    (3, 2, 6, 2, 1, 1, 1, 1e3),
    (4, 1, 10, 4, 2, 0, 0, 1e4),
    (2, 2, 5, 3, 2, 2, 1, 1e2),
    (6, 3, 7, 5, 3, 2, 2, 1e4),
    (12, 4, 8, 8, 4, 3, 2, 1e4),
    (4, 4, 3, 8, 8, 4, 4, 1e6),
])
def test_ipm_parity_random_lq(n, m, N, ng, ngN, nc, ncN, eta):
    p = random_lq_ocp(n, m, N, 37, seed=n * 31 + N, ng=ng, ngN=ngN, nc=nc, ncN=ncN, eta=eta)
    assert_ipm_parity(*run(p))


def test_ipm_parity_c4_cartpole():
    p = cartpole_c4(300, seed=2511, N=100)
    g, git, o, oit = run(p)
    assert np.all(o["status"] == 0)
    assert_ipm_parity(g, git, o, oit)


def test_ipm_parity_c4_ls_backtracking():
    p = cartpole_c4(200, seed=7, N=30, variant="C4-LS")
    g, git, o, oit = run(p)
    assert np.max(o["n_backtracks"]) >= 2
    assert_ipm_parity(g, git, o, oit)


def test_ipm_nonpositive_slack_status():
    p = random_lq_ocp(3, 2, 5, 6, seed=3, ng=2, ngN=1, nc=1, ncN=1)
    p.it["s"][2, 3, 1] = -1e-3
    g, git, o, oit = run(p)
    assert o["status"][2] == (4 | (3 << 8)) and g["status"][2] == o["status"][2]
    assert np.all(np.isnan(g["dx"][2]))
    np.testing.assert_array_equal(git["x"][2], p.it["x"][2].numpy())  # untouched
    assert_ipm_parity(g, git, o, oit)


def test_ipm_c4_full_batch_sampled():
    """BASELINE configs[3] at full size: 16,384 cart-pole instances, N = 100; 128 sampled
    instances recomputed by the oracle."""
    import paper_2509_16370_b200 as rr
    p = cartpole_c4(16384, seed=2511, N=100, device="cuda")
    host = p.to("cpu")
    res = rr.ipm_step(p)
    torch.cuda.synchronize()
    assert int((res["status"] != 0).sum()) == 0
    idx = np.sort(np.random.default_rng(1).choice(16384, 128, replace=False))
    sub = host.select(torch.from_numpy(idx))
    o, oit = ipm_step_oracle(sub, nthreads=8)
    g = {k: v[torch.from_numpy(idx).cuda()].cpu().numpy() for k, v in res.items()}
    git = {k: v[torch.from_numpy(idx).cuda()].cpu().numpy() for k, v in p.it.items()}
    assert_ipm_parity(g, git, o, oit)


def test_ipm_line_search_failure_status():
    """RR_ST_LS_FAILED: with max_backtracks = 0 the C4-LS instances that need backtracking fail,
    keep their iterate, report α_p = 0 -- exactly as the oracle."""
    p = cartpole_c4(64, seed=7, N=20, variant="C4-LS")
    g, git, o, oit = run(p, max_backtracks=0)
    assert np.any(o["status"] == 5) and np.array_equal(g["status"], o["status"])
    failed = o["status"] == 5
    assert np.all(g["alpha_p"][failed] == 0.0)
    np.testing.assert_array_equal(git["x"][failed], p.it["x"][failed].numpy())
    assert_ipm_parity(g, git, o, oit)


def test_ipm_horizon_zero_and_empty_batch():
    import paper_2509_16370_b200 as rr
    p = random_lq_ocp(3, 2, 0, 4, seed=8, ng=2, ngN=2, nc=1, ncN=1)
    assert_ipm_parity(*run(p))
    e = random_lq_ocp(3, 2, 4, 0, seed=8).to("cuda")
    res = rr.ipm_step(e)
    assert res["status"].numel() == 0


def test_ipm_invalid_parameters_rejected():
    import paper_2509_16370_b200 as rr
    p = random_lq_ocp(3, 2, 4, 2, seed=9).to("cuda")
    with pytest.raises(rr.RRError):
        rr.ipm_step(p, tau=1.5)
    with pytest.raises(rr.RRError):
        rr.ipm_step(p, beta=0.0)


@pytest.mark.parametrize("batch,N,seed", [(37, 20, 2513), (300, 50, 11)])
def test_ipm_parity_quadrotor_model(batch, N, seed):
    """IPM_MODEL_QUADROTOR: trial merits through the C5 quadrotor dynamics (n = 12, m = 4)."""
    p = quadrotor_ipm(batch, seed=seed, N=N)
    g, git, o, oit = run(p)
    assert np.all(o["status"] == 0) and np.any(o["alpha_p"] < 1.0)
    assert_ipm_parity(g, git, o, oit)


def test_quadrotor_model_rules():
    """The quadrotor model needs n = 12, m = 4."""
    import paper_2509_16370_b200 as rr
    bad = random_lq_ocp(4, 1, 5, 3, seed=1, ng=2)
    bad.model = 2
    with pytest.raises(rr.RRError):
        rr.ipm_step(bad.to("cuda"))


def test_spec_scalar_step_exact_on_gpu():
    """S:234 through the CUDA ipm_step (padded 4×1 kernel): (Δu, Δs, Δz) = (−33/32, −15/16, 15/16),
    D = −99/32, α = 1, 𝒜(0) = 4, 𝒜(1) = 3.848760597239781, for a batch of identical instances."""
    from synth.ipm_workloads import spec_scalar_ocp
    p = spec_scalar_ocp(batch=37)
    g, git, o, oit = run(p)
    assert_ipm_parity(g, git, o, oit)
    assert np.all(g["status"] == 0) and np.all(g["n_backtracks"] == 0)
    for k, v in (("du", -33 / 32), ("ds", -15 / 16), ("dz", 15 / 16)):
        assert np.all(np.abs(g[k] - v) <= 2e-16), k
    assert np.all(np.abs(g["D"] + 99 / 32) <= 1e-15) and np.all(g["alpha_p"] == 1.0)
    assert np.all(np.abs(g["merit0"] - 4.0) <= 1e-15)
    assert np.all(np.abs(g["merit_acc"] - 3.848760597239781) <= 2e-15)


def test_ipm_c4_unaligned_operands_equal_aligned(monkeypatch):
    """The exact C4 lane-group kernel copies the stage data with a static plan of 16-byte LDGSTS when
    every copied operand base is 16-byte aligned, else with the generic 8-byte copies (ipm_launch
    decides): an 8-byte-offset view of A and of the iterate x gives bitwise the aligned results.
    (RR_IPM_C4T=0 pins the lane-group kernel: the thread-per-instance A/B variant, RR_IPM_C4T=1, only
    takes aligned inputs.)"""
    import paper_2509_16370_b200 as rr
    monkeypatch.setenv("RR_IPM_C4T", "0")
    b = cartpole_c4(24, N=30).to("cuda")
    c = b.clone()

    def offset_view(t):  # same values, base address shifted by 8 bytes
        buf = torch.empty(t.numel() + 1, dtype=t.dtype, device=t.device)
        v = buf[1:].view(t.shape)
        v.copy_(t)
        assert v.data_ptr() % 16 == 8
        return v
    c.data["A"] = offset_view(c.data["A"])
    c.it["x"] = offset_view(c.it["x"])
    ra, rc = rr.ipm_step(b), rr.ipm_step(c)
    torch.cuda.synchronize()
    for k in ("status", "dx", "du", "ds", "dz", "dy", "alpha_p", "D", "merit0", "merit_acc"):
        assert torch.equal(ra[k], rc[k]), k
    for k in ("x", "u", "s", "z", "y"):
        assert torch.equal(b.it[k], c.it[k]), k
