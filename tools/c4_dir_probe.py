import copy, sys
import torch
sys.path.insert(0, ".")
import paper_2509_16370_b200 as rr
from synth.ipm_workloads import cartpole_c4

def timeit(fn, steps=5):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps

for B in (2368, 9472, 16384):
    b = cartpole_c4(B, seed=2511, N=100, device="cuda")
    call = rr.IpmCall(b)
    def step():
        bk = copy.copy(b); bk.it = {k: v.clone() for k, v in b.it.items()}
        rr.IpmCall(bk, res=call.res, ws=call.ws).launch(torch.cuda.current_stream())
    def direction():
        call.launch(torch.cuda.current_stream(), direction_only=True)
    clone_ms = timeit(lambda: {k: v.clone() for k, v in b.it.items()})
    print(B, "step(+clone) %.4f ms, clone %.4f ms, direction only %.4f ms" % (timeit(step), clone_ms, timeit(direction)), flush=True)
