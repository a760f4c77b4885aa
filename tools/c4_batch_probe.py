"""ipm_step (C4 cart-pole, N = 100) time per step against the batch size: is the kernel wave-bound
(latency) or throughput-bound?  Prints one line per batch: ms, ms per 1,000 instances."""
import copy
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_16370_b200 as rr  # noqa: E402
from synth.ipm_workloads import cartpole_c4  # noqa: E402


def time_batch(B, steps=5):
    b = cartpole_c4(B, seed=2511, N=100, device="cuda")
    call0 = rr.IpmCall(b)

    def fresh():
        bk = copy.copy(b)
        bk.it = {k: v.clone() for k, v in b.it.items()}
        return rr.IpmCall(bk, res=call0.res, ws=call0.ws)
    calls = [fresh() for _ in range(3 + steps)]
    s = torch.cuda.current_stream()
    for k in range(3):
        calls[k].launch(s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for k in range(steps):
        calls[3 + k].launch(s)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


for B in [int(x) for x in (sys.argv[1:] or ["2368", "4736", "7104", "9472", "11840", "14208", "16384"])]:
    ms = time_batch(B)
    print("batch %6d  %.4f ms  %.4f ms per 1k instances" % (B, ms, ms / B * 1e3), flush=True)
