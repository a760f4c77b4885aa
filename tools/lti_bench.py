"""Timing of the batch-shared (LTI / fleet MPC) paths on the C2 shape: 65,536 instances,
n=12, m=4, N=100, A, B, Q, M, R, Q_N shared; per-instance q, r, c, c_0, q_N.  CUDA events, 3 warm-ups,
10 timed launches each.  Prints one JSON line (an extra measurement, not the driver's bench line)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2509_16370_b200 as rr  # noqa: E402


def timed(fn, steps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    B, N = 65536, 100
    p = synth.lti_problem(12, 4, N, B, seed=2509, device="cuda")
    sol = rr.alloc_solution(p)
    call = rr.Marshalled(p, sol)
    t_fused = timed(lambda: call.launch())
    F, st = rr.rr_factor(p)
    ws = torch.empty((rr.solve_workspace_bytes(12, 4, N, B) + 7) // 8, dtype=torch.float64, device="cuda")
    t_fac = timed(lambda: rr.rr_factor(p, factor=F, status=st))
    t_sol = timed(lambda: rr.rr_solve(p, F, out=sol, workspace=ws))
    assert int((sol["status"] != 0).sum()) == 0
    # algorithmic bytes per (instance, stage) with shared matrices (L2-resident, ~0 per instance):
    # fused: q,r,c in (28 doubles) + policy K,k,V,v out/in (2 x 142) + c re-read (12) + x,u,y out (28)
    # rr_solve: q,r,c,record(214) in, v,k out/in (2 x 16), record(214) + c in, x,u,y out
    alg = {"fused": 8 * (28 + 2 * 142 + 12 + 28), "solve": 8 * (28 + 214 + 16 + 214 + 12 + 16 + 28)}
    peak = 6650.0
    out = {"workload": "LTI C2 shape: 65536 x n12 m4 N100, A,B,Q,M,R,Q_N batch-shared",
           "fused_ms": t_fused, "factor_ms": t_fac, "solve_ms": t_sol,
           "fused_solves_per_s": B / (t_fused / 1e3),
           "fused_hbm_frac": alg["fused"] * B * N / (t_fused / 1e3) / 1e9 / peak,
           "solve_hbm_frac": alg["solve"] * B * N / (t_sol / 1e3) / 1e9 / peak,
           "alg_bytes_per_stage": alg, "peak_gbs": peak}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
