"""Small launches of every kernel, for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2509_16370_b200 as rr  # noqa: E402
import synth  # noqa: E402
from synth.ipm_workloads import cartpole_c4, random_lq_ocp  # noqa: E402

for (n, m, N, b) in [(12, 4, 5, 5), (4, 1, 4, 9), (2, 1, 3, 5), (5, 3, 3, 3), (24, 8, 2, 2)]:
    p = synth.random_stable_lqr(n, m, N, b, seed=1).to("cuda")
    out = rr.rr_factor_solve(p, want_factor=True)
    torch.cuda.synchronize()
    print("rr", n, m, N, b, int(out["status"].abs().sum()))
os.environ["RR_B200_VARIANT"] = "1"
p = synth.random_stable_lqr(12, 4, 5, 5, seed=2).to("cuda")
rr.rr_factor_solve(p)
torch.cuda.synchronize()
os.environ.pop("RR_B200_VARIANT")
b = cartpole_c4(6, seed=3, N=8, device="cuda")
res = rr.ipm_step(b)
torch.cuda.synchronize()
print("ipm c4", res["status"].tolist())
b = random_lq_ocp(3, 2, 4, 5, seed=4, ng=2, ngN=1, nc=1, ncN=1, device="cuda")
res = rr.ipm_step(b)
torch.cuda.synchronize()
print("ipm lq", res["status"].tolist())
# split API, residual, refinement, shared operands, IPM solve
for (n, m, N, b) in [(12, 4, 5, 5), (4, 1, 4, 9), (5, 3, 3, 3)]:
    p = synth.random_stable_lqr(n, m, N, b, seed=5).to("cuda")
    F, st = rr.rr_factor(p)
    sol = rr.rr_solve(p, F)
    rr.rr_refine(p, F, sol, iters=1)
    torch.cuda.synchronize()
    print("split", n, m, N, b, int(st.abs().sum()), int(sol["status"].abs().sum()))
p = synth.lti_problem(12, 4, 6, 5, seed=6).to("cuda")
rr.rr_factor_solve(p)
F, _ = rr.rr_factor(p)
rr.rr_residual(p, rr.rr_solve(p, F))
torch.cuda.synchronize()
print("shared ok")
from synth.ipm_workloads import double_integrator_ocp  # noqa: E402
b = double_integrator_ocp(batch=3, device="cuda")
rep = rr.ipm_solve(b, max_iters=30)
b = cartpole_c4(4, seed=3, N=8, device="cuda")
rep2 = rr.ipm_solve(b, max_iters=3)
torch.cuda.synchronize()
print("ipm_solve", rep["status"].tolist(), rep2["status"].tolist())
# parallel in time, quadrotor model (ipm_step, ipm_solve), user-model line search
p = synth.random_stable_lqr(12, 4, 37, 2, seed=7, delta=1e-3).to("cuda")
rr.rr_factor_solve_pit(p)
from synth.ipm_workloads import quadrotor_ipm  # noqa: E402
q = quadrotor_ipm(3, N=6, device="cuda")
resq = rr.ipm_step(q)
q = quadrotor_ipm(3, N=6, device="cuda")
repq = rr.ipm_solve(q, max_iters=3)
b = random_lq_ocp(3, 2, 4, 5, seed=8, ng=2, ngN=1, nc=1, ncN=1, device="cuda")
d = rr.ipm_direction(b)
torch.cuda.synchronize()
print("pit / quadrotor / direction", resq["status"].tolist(), repq["status"].tolist(), d["status"].tolist())
# round 2: persistent K1-MMA warps with several pairs each (batch > resident slots), the staggered
# (deferred forward) variant, FP32 factor records, the pipelined host path, linear_merit
p = synth.random_stable_lqr(12, 4, 3, 4800, seed=7).to("cuda")
out = rr.rr_factor_solve(p)
os.environ["RR_DEFER_MOD"] = "3"
out2 = rr.rr_factor_solve(p)
os.environ.pop("RR_DEFER_MOD")
torch.cuda.synchronize()
print("persistent", int(out["status"].abs().sum()), bool(torch.equal(out["x"], out2["x"])))
p = synth.random_stable_lqr(12, 4, 4, 6, seed=8).to("cuda")
F32, st = rr.rr_factor(p, fp32=True)
sol = rr.rr_solve(p, F32)
rr.rr_refine(p, F32, sol, iters=1)
torch.cuda.synchronize()
print("fp32", int(st.abs().sum()), int(sol["status"].abs().sum()))
pc = synth.random_stable_lqr(12, 4, 4, 11, seed=9)
hp = synth.RRProblem(pc.nx, pc.nu, pc.N, **{f: getattr(pc, f).pin_memory() for f in pc.FIELDS})
dp = pc.to("cuda")
hs = {k: torch.empty(v.shape, dtype=v.dtype).pin_memory() for k, v in rr.alloc_solution(dp).items()}
call = rr.HostMarshalled(hp, hs, dp, rr.alloc_solution(dp))
ws = torch.empty((call.pipelined_workspace_bytes(4) + 7) // 8, dtype=torch.float64, device="cuda")
call.launch_pipelined([torch.cuda.current_stream(), torch.cuda.Stream()], 4, ws)
torch.cuda.synchronize()
print("pipelined", int(hs["status"].abs().sum()))
b = cartpole_c4(3, seed=3, N=8, device="cuda")
rep3 = rr.ipm_solve(b, max_iters=4, linear_merit=True)
torch.cuda.synchronize()
print("linear_merit", rep3["status"].tolist())
# round 2, session 3: K4b (C3 shape, two CTAs per SM) and K4, the fused cooperative parallel-in-time
# launch (small problems), the thread-per-instance C4 ipm_step (A/B variant)
p = synth.random_stable_lqr(64, 32, 3, 3, seed=10).to("cuda")
o4b = rr.rr_factor_solve(p, want_factor=True)
os.environ["RR_B200_CTA"] = "1"
o4 = rr.rr_factor_solve(p)
os.environ.pop("RR_B200_CTA")
p = synth.random_stable_lqr(12, 4, 9, 3, seed=11, delta=1e-4).to("cuda")
opit = rr.rr_factor_solve_pit(p)
os.environ["RR_IPM_C4T"] = "1"
b = cartpole_c4(37, seed=3, N=8, device="cuda")
rc4t = rr.ipm_step(b)
os.environ.pop("RR_IPM_C4T")
torch.cuda.synchronize()
print("session 3", int(o4b["status"].abs().sum()), int(o4["status"].abs().sum()), int(opit["status"].abs().sum()),
      rc4t["status"].tolist()[:4])
