"""GPU parity of the two C3 (n_x = 64, n_u = 32) kernels against the CPU oracle: K4b (two instances
per SM, the default) and K4 (one instance per SM, RR_B200_CTA=1), both through the C-ABI.

Bar: per instance and output block, normwise relative error ≤ 1e-9 in FP64; status
words bit-exact (S_NOT_PD / G_NOT_PD stages included)."""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from test_rr_gpu import assert_parity, blockwise_rel

pytestmark = pytest.mark.gpu


def solve(p, kernel, want_factor=False):
    import paper_2509_16370_b200 as m
    old = os.environ.get("RR_B200_CTA")
    os.environ["RR_B200_CTA"] = "1" if kernel == "k4" else "0"
    try:
        out = m.rr_factor_solve(p.to("cuda"), want_factor=want_factor)
        torch.cuda.synchronize()
    finally:
        if old is None:
            os.environ.pop("RR_B200_CTA", None)
        else:
            os.environ["RR_B200_CTA"] = old
    return {k: v.cpu().numpy() for k, v in out.items()}


@pytest.mark.parametrize("kernel", ["k4b", "k4"])
@pytest.mark.parametrize("N,batch,delta", [(1, 3, 1e-4), (2, 2, 0.0), (7, 5, 1e-8), (12, 4, 1e-4), (5, 3, 1.0)])
def test_c3_kernels_match_oracle(kernel, N, batch, delta):
    p = synth.random_stable_lqr(64, 32, N, batch, seed=6400 + N, delta=delta)
    g = solve(p, kernel, want_factor=True)
    o = oracle.rr_solve_t2(p, nthreads=8, want_policy=True)
    assert_parity(g, o, keys=("x", "u", "y", "V", "v", "K", "k"))


def test_c3_horizon_zero_and_single_instance():
    for N, batch in ((0, 3), (3, 1)):
        p = synth.random_stable_lqr(64, 32, N, batch, seed=11 + N, delta=1e-3)
        g = solve(p, "k4b")
        o = oracle.rr_solve_t2(p, nthreads=4)
        assert_parity(g, o, keys=("x", "y") if N == 0 else ("x", "u", "y"))


@pytest.mark.parametrize("kernel", ["k4b", "k4"])
def test_c3_status_words(kernel):
    """S_NOT_PD (δ < 0 makes I + δV indefinite) and G_NOT_PD (an indefinite R_i) on single instances,
    NaN-filled outputs, the other instances untouched."""
    p = synth.random_stable_lqr(64, 32, 6, 4, seed=17, delta=1e-4)
    p.delta[1] = -5.0
    R = p.R[2, 3].clone()
    R[0] = -1e3  # R[0][0] of stage 3 of instance 2 (packed 'L': first entry)
    p.R[2, 3] = R
    g = solve(p, kernel)
    o = oracle.rr_solve_t2(p, nthreads=4)
    assert (o["status"][1] & 0xff) == 2 and (o["status"][2] & 0xff) == 1, o["status"]
    assert_parity(g, o)
    assert np.isnan(g["x"][1]).all() and np.isnan(g["u"][2]).all()


def test_c3_k4b_equals_k4_on_a_wave():
    """More instances than one wave of either kernel (148 or 296 resident): K4b and K4 agree to the
    parity bar with each other and with the oracle on sampled instances."""
    p = synth.random_stable_lqr(64, 32, 4, 333, seed=23, delta=1e-4)
    a = solve(p, "k4b")
    b = solve(p, "k4")
    assert np.array_equal(a["status"], b["status"]) and int(np.abs(a["status"]).sum()) == 0
    for k in ("x", "u", "y"):
        assert blockwise_rel(a[k], b[k]) <= 1e-9, k
    idx = torch.tensor([0, 1, 147, 148, 295, 296, 332])
    sub = p.select(idx)
    o = oracle.rr_solve_t2(sub, nthreads=8)
    assert_parity({k: a[k][idx.numpy()] for k in ("x", "u", "y", "status")}, o)
