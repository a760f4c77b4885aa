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
