#!/usr/bin/env python
"""bench.py -- batched regularized-LQR solves on B200 (BASELINE.json metric, configs[1] = C2).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--no-cpu-baseline]

One step = one rr_factor_solve over the whole per-GPU batch (all hot-path rows of the fused
solve: stage data in HBM, backward matrix + vector sweep, forward sweep, dual recovery).
C2: 65,536 random stable LQR instances, n_x=12, n_u=4, N=100, δ=1e-4, FP64, per GPU (weak
scaling: rank r solves global instances [r·B, (r+1)·B)).  Inputs (18.7 GB/GPU) exceed the
126 MB L2, so no flush is needed between steps.  Timing: CUDA events on the launching stream,
barrier + synchronize around the timed region, max over ranks.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "regularized-LQR solves/sec & stage-updates/s vs roofline at 1/2/4/8 B200"
NX, NU, HORIZON, BATCH, SEED, DELTA = 12, 4, 100, 65536, 2509, 1e-4
# Algorithmic model per (instance, stage), SURVEY.md §8(d) / DESIGN.md §7 (C2 row):
ALG_BYTES_PER_STAGE = 6976     # fused two-sweep: inputs once + policy write/read + A,B,c re-read + x,u,y
ALG_FLOPS_PER_STAGE = 15769    # 13,077 factor + 864 vector backward + 1,828 forward
FP64_DMMA_TFLOPS = 37.1        # measured on this pool by tools/k0_probe.cu (profiles/r01_k0_fp64_probe.txt)


def measure_dmma_peak():
    """FP64 DMMA peak measured in this run (MEASURED_PEAKS.json has no FP64 entry):
    build and run tools/k0_probe.cu (mma.sync m8n8k4 f64 throughput over every SM), best of its
    repetitions.  Falls back to the recorded pool value if nvcc or the probe is unavailable."""
    import re
    import subprocess
    import tempfile
    src = os.path.join(ROOT, "tools", "k0_probe.cu")
    try:
        with tempfile.TemporaryDirectory() as d:
            exe = os.path.join(d, "k0_probe")
            subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-o", exe, src],
                           check=True, capture_output=True, timeout=240)
            out = subprocess.run([exe], check=True, capture_output=True, text=True, timeout=120).stdout
        vals = [float(v) for v in re.findall(r"DMMA m8n8k4: ([0-9.]+) TFLOP/s", out)]
        if vals:
            return max(vals), "K0 probe (tools/k0_probe.cu, mma.sync m8n8k4 f64) measured in this run"
    except Exception as e:  # noqa: BLE001
        return FP64_DMMA_TFLOPS, "recorded K0 probe value 37.1 (profiles/r01_k0_fp64_probe.txt); in-run probe failed: %s" % str(e)[:80]
    return FP64_DMMA_TFLOPS, "recorded K0 probe value 37.1 (profiles/r01_k0_fp64_probe.txt); in-run probe printed no DMMA line"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=BATCH, help=argparse.SUPPRESS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target oracle sample wall time")
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5", "split", "f32", "c4solve", "c4swing", "pit", "lti"],
                    help="c2 (default, BASELINE configs[1]); c3 = 4,096 dense n64 m32 N50 (configs[2]); "
                         "c4 = ipm_step on 16,384 cart-pole instances (configs[3]); c5 = 1,048,576 "
                         "quadrotor n12 m4 N200 sharded over the ranks, chunks of 65,536 (configs[4]); split = "
                         "rr_factor + rr_solve + rr_residual on the C2 workload, each kernel timed; c4solve = ipm_solve "
                         "(20 IPM iterations) on the C4 cart-pole batch; c1 = single double-integrator instance latency; "
                         "pit = single-instance latency, parallel-in-time vs sequential, long horizons; lti = the C2 shape "
                         "as an LTI fleet (one A, B, Q, M, R for all instances and stages)")
    ap.add_argument("--c5-total", type=int, default=1048576, help=argparse.SUPPRESS)
    ap.add_argument("--ref-seconds", type=float, default=150.0, help=argparse.SUPPRESS)  # reference-arm budget
    ap.add_argument("--no-others", action="store_true",
                    help="default C2 run at N=1: skip the short runs of the other BASELINE configs attached "
                         "to the line (other_workloads)")
    return ap.parse_args()


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)  # one GPU per rank before the communicator exists
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v, ws):
    from paper_2509_16370_b200.shard import max_over_ranks as _m
    import torch
    return _m(v, device=torch.device("cuda", torch.cuda.current_device())) if ws > 1 else v


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic(kernel_key):
    """DRAM bytes per launch of the kernel from the committed ncu --set full capture summary
    (profiles/traffic.json, written by tools/record_traffic.py), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)
        return d.get(kernel_key)
    except (OSError, ValueError):
        return None


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def cpu_baseline(target_s, cores=None):
    """The oracle (plain C T2 recursion, as it stands) on the host cores, on a bounded sample of
    the same C2 workload (same generator, global ids 0..S-1)."""
    import synth
    import oracle
    cores = cores or os.cpu_count() or 1
    cal = synth.random_stable_lqr(NX, NU, HORIZON, 64, SEED, DELTA)
    t0 = time.perf_counter()
    oracle.rr_solve_t2(cal, nthreads=1)
    per_inst = (time.perf_counter() - t0) / 64  # also the 1-thread rate
    S = max(cores, int(target_s * cores / max(per_inst, 1e-6)))
    S = min(S, 65536)
    prob = synth.random_stable_lqr(NX, NU, HORIZON, S, SEED, DELTA)
    t0 = time.perf_counter()
    out = oracle.rr_solve_t2(prob, nthreads=cores)
    dt = time.perf_counter() - t0
    assert int((out["status"] != 0).sum()) == 0
    return {"value": S / dt, "unit": "solves/s", "cores": cores, "kind": "oracle",
            "stage_updates_per_s": S * HORIZON / dt, "one_thread_value": 1.0 / per_inst,
            "cpu_model": cpu_model(),
            "sample": "%d of the %d C2 instances (global ids 0..%d), T2 plain-C oracle, %d threads, %.1f s"
                      % (S, BATCH, S - 1, cores, dt)}


def oracle_rate(make, solve, target_s, total, unit_desc, calib=8, cap=None):
    """Time the oracle as it stands on all host cores on a bounded sample of a workload: `make(k)`
    builds the first k instances (global ids 0..k-1), `solve(batch, threads)` runs the oracle.
    The sample is sized from a 1-thread calibration run so it takes about `target_s` seconds."""
    cores = os.cpu_count() or 1
    cal = make(calib)
    t0 = time.perf_counter()
    solve(cal, 1)
    per_inst = (time.perf_counter() - t0) / calib
    S = max(cores, int(target_s * cores / max(per_inst, 1e-6)))
    S = min(S, cap or total, total)
    prob = make(S)
    t0 = time.perf_counter()
    solve(prob, cores)
    dt = time.perf_counter() - t0
    return {"value": S / dt, "unit": "solves/s", "cores": cores, "kind": "oracle",
            "one_thread_value": 1.0 / per_inst, "cpu_model": cpu_model(),
            "sample": "%d of the %d %s (global ids 0..%d), %d threads, %.1f s" % (S, total, unit_desc, S - 1, cores, dt)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(a, ws, rank):
    """--impl reference: the oracle (this tier's reference arm) on the host cores, rank 0 only."""
    if rank != 0:
        return
    import synth
    import oracle
    cores = os.cpu_count() or 1
    cal = synth.random_stable_lqr(NX, NU, HORIZON, 16, SEED, DELTA)
    t0 = time.perf_counter()
    oracle.rr_solve_t2(cal, nthreads=1)
    per_inst = (time.perf_counter() - t0) / 16
    # each step: a bounded sample sized so warmup+steps finish in ~2-3 minutes
    budget = a.ref_seconds / max(1, a.steps + a.warmup)
    S = max(cores, min(BATCH, int(budget * cores / max(per_inst, 1e-6))))
    prob = synth.random_stable_lqr(NX, NU, HORIZON, S, SEED, DELTA)
    for _ in range(a.warmup):
        oracle.rr_solve_t2(prob, nthreads=cores)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        oracle.rr_solve_t2(prob, nthreads=cores)
    dt = (time.perf_counter() - t0) / a.steps
    val = S / dt
    line = {"metric": METRIC, "value": val, "unit": "solves/s", "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "C2: random stable regularized LQR n_x=12 n_u=4 N=100 delta=1e-4 (oracle sample)",
                       "global_batch": S, "seq_len": HORIZON, "parallelism": "host threads"},
            "stage_updates_per_s": val * HORIZON,
            "cpu_baseline": {"value": val, "unit": "solves/s", "cores": cores, "kind": "oracle",
                             "sample": "%d of %d C2 instances per step, T2 plain-C oracle" % (S, BATCH)},
            "e2e": {"value": val, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    if a.impl == "reference":  # the oracle on host cores: rank 0 alone, no process group needed
        ws, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
        a.gpus = max(a.gpus, ws)
        run_reference(a, ws, rank)
        return
    ws, rank, local = dist_init()
    import torch
    import synth
    import paper_2509_16370_b200 as rr

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if a.workload == "c4":
        return run_c4(a, ws, rank, local)
    if a.workload == "c5":
        return run_c5(a, ws, rank, local)
    if a.workload == "split":
        return run_split(a, ws, rank, local)
    if a.workload == "c4solve":
        return run_c4solve(a, ws, rank, local)
    if a.workload == "c4swing":
        return run_c4solve(a, ws, rank, local, swing=True)
    if a.workload == "f32":
        return run_f32(a, ws, rank, local)
    if a.workload == "c1":
        return run_c1(a, ws, rank, local)
    if a.workload == "pit":
        return run_pit(a, ws, rank, local)
    global NX, NU, HORIZON, BATCH, SEED, ALG_BYTES_PER_STAGE, ALG_FLOPS_PER_STAGE
    if a.workload == "c3":
        # 206,208 B and 2.42M flop per stage (algorithmic)
        NX, NU, HORIZON, BATCH, SEED = 64, 32, 50, 4096, 2510
        ALG_BYTES_PER_STAGE, ALG_FLOPS_PER_STAGE = 206208, 2420000
        if a.batch == 65536:
            a.batch = BATCH
    lti = a.workload == "lti"
    if lti:
        # LTI fleet MPC on the C2 shape: ONE stage block of A, B, Q, M, R (and Q_N) for
        # the whole batch and every stage (RR_FLAG_SHARED_* | RR_FLAG_STAGE_INVARIANT_*), per-instance
        # q, r, c per stage, q_N, c_0, δ.  Per (instance, stage) the fused sweep then reads 20 input
        # doubles; model: q, r, c once 160 + policy written and read 2 x 1,136 + c re-read 96 +
        # x, u, y 224 = 2,752 B (the stage is compute / shared-memory bound at this intensity)
        ALG_BYTES_PER_STAGE = 2752
    B = a.batch
    first = rank * B  # weak scaling: every rank owns B instances (global ids [rB, (r+1)B))
    # ---- inputs resident in HBM (generation excluded from timing) ----
    if lti:
        prob = synth.lti_invariant_problem(NX, NU, HORIZON, B, SEED, DELTA, shared=True, device=dev)
    else:
        prob = synth.empty_problem(NX, NU, HORIZON, B, device=dev)
        gchunk = 4096 if NX <= 16 else 256
        for s in range(0, B, gchunk):
            e = min(B, s + gchunk)
            p = synth.random_stable_lqr(NX, NU, HORIZON, e - s, SEED, DELTA, first=first + s, device=dev)
            for f in synth.RRProblem.FIELDS:
                getattr(prob, f)[s:e].copy_(getattr(p, f))
            del p
    sol = rr.alloc_solution(prob)
    call = rr.Marshalled(prob, sol)   # fac = NULL: outputs x, u, y (policy stays in the workspace)
    stream = torch.cuda.current_stream(dev)
    for _ in range(max(3, a.warmup)):
        call.launch(stream)
    torch.cuda.synchronize()
    if not os.environ.get("RR_B200_LIB"):  # A/B probe builds (tools/ab.sh) may compute garbage on purpose
        assert int((sol["status"] != 0).sum()) == 0, "instance failures in the bench batch"

    clocks = ClockSampler(local)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    per_launch = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(a.steps)]
    clocks.start()
    time.sleep(0.3)
    barrier(ws)
    torch.cuda.synchronize()
    ev0.record(stream)
    for k in range(a.steps):
        per_launch[k][0].record(stream)
        call.launch(stream)
        per_launch[k][1].record(stream)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    clk = clocks.stop()
    t_ms = ev0.elapsed_time(ev1)
    t_ms = max_over_ranks(t_ms, ws)
    ms_step = t_ms / a.steps
    kern_ms = statistics.mean(s.elapsed_time(e) for s, e in per_launch)
    solves = B * ws / (ms_step / 1e3)

    # ---- end to end: pinned host inputs -> H2D -> kernel -> D2H of x, u, y, status ----
    e2e = None
    if not a.no_e2e:
        # N = 1: the whole batch; N > 1: 16,384 instances per rank (the pinned host copies of the full
        # batch would be ~20 GB per rank; end-to-end throughput is PCIe-bound and per-instance constant)
        EB = B if ws == 1 else min(B, 16384)
        if lti:  # same (shared / stage-invariant) layouts on the host and in the staging buffers
            EB = B
            hp = synth.RRProblem(NX, NU, HORIZON, **{f: getattr(prob, f).cpu().pin_memory() for f in synth.RRProblem.FIELDS})
        else:
            hp = synth.empty_problem(NX, NU, HORIZON, EB, device="cpu", pin_memory=True)
            for f in synth.RRProblem.FIELDS:
                getattr(hp, f).copy_(getattr(prob, f)[:EB])
        hs = {k: torch.empty((EB,) + tuple(v.shape[1:]), dtype=v.dtype, pin_memory=True) for k, v in sol.items()}
        stage_p = (synth.RRProblem(NX, NU, HORIZON, **{f: torch.empty_like(getattr(prob, f)) for f in synth.RRProblem.FIELDS})
                   if lti else synth.empty_problem(NX, NU, HORIZON, EB, device=dev))
        stage_s = rr.alloc_solution(stage_p)
        hcall = rr.HostMarshalled(hp, hs, stage_p, stage_s, ws=call.ws)
        # pipelined: 16 chunks round-robin over 3 streams (H2D of one chunk, the solve of another and
        # the D2H of a third overlap on the two copy engines and the SMs)
        NCH = 16
        pstreams = [stream, torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
        pws = torch.empty((hcall.pipelined_workspace_bytes(NCH) + 7) // 8, dtype=torch.float64, device=dev)
        hcall.launch(stream)
        hcall.launch_pipelined(pstreams, NCH, pws)
        torch.cuda.synchronize()
        barrier(ws)
        e_steps = max(1, min(a.steps, 5))

        def e2e_time(fn):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(e_steps):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            barrier(ws)
            return max_over_ranks(e0.elapsed_time(e1) / e_steps, ws)
        e_serial = e2e_time(lambda: hcall.launch(stream))
        e_ms = e2e_time(lambda: hcall.launch_pipelined(pstreams, NCH, pws))
        assert int((hs["status"] != 0).sum()) == 0
        e2e = {"value": EB * ws / (e_ms / 1e3), "unit": "solves/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": hcall.h2d_bytes * ws, "d2h_bytes_per_step": hcall.d2h_bytes * ws,
               "instances_per_rank": EB,
               "path": "rr_factor_solve_host_pipelined (C-ABI, pinned host buffers, %d chunks over 3 streams)" % NCH,
               "serial_ms_per_step": e_serial, "serial_path": "rr_factor_solve_host (one stream)",
               "h2d_gbs": hcall.h2d_bytes / (e_ms / 1e3) / 1e9}
        del hp, hs, stage_p, stage_s, hcall

    if rank != 0:
        barrier(ws)
        return
    peak, peak_src = measured_peaks()
    alg_bytes = ALG_BYTES_PER_STAGE * B * HORIZON
    achieved = alg_bytes / (kern_ms / 1e3) / 1e9
    fp64_tflops = ALG_FLOPS_PER_STAGE * B * HORIZON / (kern_ms / 1e3) / 1e12
    c3 = a.workload == "c3"
    if c3:  # FP64 contraction-bound backward sweep: roofline against the DMMA peak
        dmma_peak, dmma_src = measure_dmma_peak()
        roof = {"bound": "tensor", "achieved": fp64_tflops, "peak": dmma_peak, "unit": "TFLOP/s",
                "frac": fp64_tflops / dmma_peak, "traffic": ncu_traffic("rr_cta_c3"),
                "kernel": ("rr_cta_kernel<64,32> (K4, one instance per SM)" if os.environ.get("RR_B200_CTA") == "1"
                           else "rr_cta2_kernel<64,32> (K4b, two instances per SM)"),
                "kernel_ms": kern_ms, "dtype_peak": "fp64 DMMA",
                "alg_flops_per_stage": ALG_FLOPS_PER_STAGE, "peak_source": dmma_src,
                "hbm_gbs_alg": achieved}
    else:
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None if lti else ncu_traffic("rr_fused_c2"),
                "kernel": "rr_fused_mma_kernel<12,4> (DMMA stage, TMA loads)", "kernel_ms": kern_ms,
                "alg_bytes_per_stage": ALG_BYTES_PER_STAGE, "peak_source": peak_src,
                "fp64_alg_tflops": fp64_tflops}
    line = {
        "metric": METRIC, "value": solves, "unit": "solves/s", "n_gpus": ws, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": ("LTI fleet (C2 shape, one A, B, Q, M, R for all instances and stages; per-instance "
                                 "q, r, c, q_N, c_0): %d regularized LQR per GPU, n_x=%d n_u=%d N=%d delta=%g, FP64"
                                 % (B, NX, NU, HORIZON, DELTA)) if lti else
                               ("%s: %d random stable regularized LQR per GPU, n_x=%d n_u=%d N=%d delta=%g, FP64"
                                % ("C3" if c3 else "C2", B, NX, NU, HORIZON, DELTA)),
                   "global_batch": B * ws, "seq_len": HORIZON, "parallelism": "batch-shard x%d" % ws,
                   "l2": "inputs %.1f GB/GPU > 126 MB L2 (no flush needed)" % (prob.nbytes() / 1e9)},
        "stage_updates_per_s": solves * HORIZON,
        "roofline": roof,
        "clocks": clk,
        "e2e": e2e,
        "gpu_launches": a.steps,
    }
    if not a.no_cpu_baseline and ws == 1:
        if c3:
            import oracle
            line["cpu_baseline"] = oracle_rate(
                lambda k: synth.random_stable_lqr(NX, NU, HORIZON, k, SEED, DELTA),
                lambda p, t: oracle.rr_solve_t2(p, nthreads=t), a.cpu_seconds, BATCH,
                "C3 instances, T2 plain-C oracle", calib=2, cap=512)
        else:
            line["cpu_baseline"] = cpu_baseline(a.cpu_seconds)
            if lti:
                line["cpu_baseline"]["note"] = ("sampled on C2 instances: the plain-C oracle does the same "
                                                "work per instance whatever the operand layout")
    if ws == 1 and a.workload == "c2" and not a.no_others:
        # the other BASELINE configs (C3, C4, C5) and the split / IPM-solve paths, each a short run of
        # this script in its own process (own timing, own roofline), summarised on this line so that
        # every config has a number in the driver's bench record
        del prob, sol, call
        torch.cuda.empty_cache()
        line["other_workloads"] = other_workloads(a)
    print(json.dumps(line), flush=True)
    barrier(ws)


def other_workloads(a):
    out = {}
    steps = str(max(3, min(a.steps, 5)))
    for w in ("c3", "c4", "c5", "split", "c4swing"):
        cmd = [sys.executable, os.path.abspath(__file__), "--workload", w, "--steps", steps, "--warmup", "3",
               "--no-cpu-baseline", "--no-e2e"]
        t0 = time.perf_counter()
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
            d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
            keep = {k: d.get(k) for k in ("metric", "value", "unit", "ms_per_step", "config", "clocks", "status_nonzero",
                                          "status_counts", "iterations", "gpu_launches")
                    if d.get(k) is not None}
            rf = d.get("roofline") or {}
            keep["roofline"] = {k: rf.get(k) for k in ("bound", "achieved", "peak", "unit", "frac", "kernel", "kernels")
                                if rf.get(k) is not None}
            keep["wall_s"] = round(time.perf_counter() - t0, 1)
            out[w] = keep
        except Exception as e:  # noqa: BLE001 -- recorded, never fatal for the headline line
            out[w] = {"error": "%s: %s" % (type(e).__name__, str(e)[:200])}
    return out


def run_c4(a, ws, rank, local):
    """Extra line (not the driver's default): one batched regularized-IPM step (rows a1-a8) on the
    C4 cart-pole workload, 16,384 instances per GPU, N = 100.  ipm_step updates the iterate in place,
    so every step (warm-up and timed) runs on its own device-resident copy of the same initial
    iterate: each timed step is the same first IPM iteration of the C4 recipe."""
    import torch
    import paper_2509_16370_b200 as rr
    from synth.ipm_workloads import cartpole_c4
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    B, Nh = 16384, 100
    import copy
    b = cartpole_c4(B, seed=2511, N=Nh, first=rank * B, device=dev)
    call0 = rr.IpmCall(b)

    def fresh():  # same data / result / workspace buffers, private copy of the initial iterate
        bk = copy.copy(b)
        bk.it = {k: v.clone() for k, v in b.it.items()}
        return rr.IpmCall(bk, res=call0.res, ws=call0.ws)
    nw = max(3, a.warmup)
    calls = [fresh() for _ in range(nw + a.steps)]
    stream = torch.cuda.current_stream(dev)
    for k in range(nw):
        calls[k].launch(stream)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    clocks = ClockSampler(local)
    barrier(ws)
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    for k in range(a.steps):
        ev[k][0].record(stream)
        calls[nw + k].launch(stream)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    clk = clocks.stop()
    ms = max_over_ranks(sum(s_.elapsed_time(e_) for s_, e_ in ev) / a.steps, ws)
    # per-instance IPM summaries (status, α_p, D, 𝒜(0)) gathered to rank 0, timed apart
    from paper_2509_16370_b200.shard import gather_summaries
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    gathered = gather_summaries({k: call0.res[k] for k in ("status", "alpha_p", "D", "merit0")}, rank, ws, B * ws)
    g1.record(stream)
    torch.cuda.synchronize()
    gather_ms = max_over_ranks(g0.elapsed_time(g1), ws)
    st = call0.res["status"]
    if rank == 0:
        alg = 1900 * B * Nh  # ~1.9 KB per (instance, stage)
        peak, src = measured_peaks()
        print(json.dumps({
            "metric": "regularized-IPM steps/s (C4 cart-pole, rows a1-a8)", "value": B * ws / (ms / 1e3),
            "unit": "instance-steps/s", "n_gpus": ws, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C4: %d cart-pole IPM iterates per GPU, N=%d, n_g=4" % (B, Nh),
                       "l2": "stage data %.1f GB/GPU > 126 MB L2 (no flush needed)" % (alg / 1e9)},
            "clocks": clk,
            "status_nonzero": int((gathered["status"] != 0).sum()),
            "summary": {"fields": ["D", "alpha_p", "merit0", "status"], "gathered_to": "rank 0 (dist.gather)",
                        "gather_ms": gather_ms, "D_max": float(gathered["D"].max()),
                        "alpha_p_min": float(gathered["alpha_p"].min())},
            "roofline": {"bound": "hbm", "achieved": alg / (ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": alg / (ms / 1e3) / 1e9 / peak, "traffic": ncu_traffic("ipm_c4"),
                         "alg_bytes_per_stage": 1900, "peak_source": src},
            "cpu_baseline": c4_cpu_baseline(a, B, Nh) if (ws == 1 and not a.no_cpu_baseline) else None,
            "gpu_launches": a.steps}), flush=True)


def c4_cpu_baseline(a, B, Nh):
    from synth.ipm_workloads import cartpole_c4
    from oracle.ipm import ipm_step_oracle
    r = oracle_rate(lambda k: cartpole_c4(k, seed=2511, N=Nh),
                    lambda p, t: ipm_step_oracle(p, nthreads=t), a.cpu_seconds, B,
                    "C4 cart-pole IPM iterates, C oracle ipm_step", calib=64)
    r["unit"] = "instance-steps/s"
    return r


def run_c5(a, ws, rank, local):
    """BASELINE configs[4]: 1,048,576 quadrotor instances (n=12, m=4, N=200) split over the ranks
    (strong scaling: total work fixed), rr_factor_solve in resident chunks of 65,536 instances
    (inputs 37 GB + policy records 31 GB per chunk; the whole batch is ~600 GB of inputs, more than
    one GPU holds).  Every chunk is generated on the device (untimed), then solved W times untimed
    and K times timed with CUDA events; the step time is the sum over the rank's chunks of the
    mean chunk time (each chunk's inputs exceed L2, so re-solving a resident chunk is not cached),
    plus the timed NCCL gather (dist.gather to rank 0) of the per-instance summaries (status, u_0 and
    the KKT residual norms from rr_residual, timed separately as `summary.residual_ms`).  Reported
    time = max over ranks."""
    import torch
    import synth
    import paper_2509_16370_b200 as rr
    from paper_2509_16370_b200.shard import shard_range, gather_summaries
    dev = torch.device("cuda", local)
    n, m, Nh, CH = 12, 4, 200, 65536
    total = a.c5_total
    b0, b1 = shard_range(rank, ws, total)
    mine = b1 - b0
    CH = min(CH, max(mine, 1))
    prob = synth.empty_problem(n, m, Nh, CH, device=dev)
    sol = rr.alloc_solution(prob)
    call = rr.Marshalled(prob, sol)
    stream = torch.cuda.current_stream(dev)
    summ = {"status": torch.empty(mine, dtype=torch.int32, device=dev),
            "u0": torch.empty(mine, m, dtype=torch.float64, device=dev),
            "kkt": torch.empty(mine, 2, dtype=torch.float64, device=dev)}
    chunk_ms, res_ms, gen_s = [], [], 0.0
    clocks = ClockSampler(local)
    clocks.start()
    for s in range(b0, b1, CH):
        e = min(b1, s + CH)
        t0 = time.perf_counter()
        if e - s != CH:  # ragged last chunk: its own buffers
            prob = synth.empty_problem(n, m, Nh, e - s, device=dev)
            sol = rr.alloc_solution(prob)
            call = rr.Marshalled(prob, sol, ws=call.ws)
        for g in range(s, e, 4096):
            ge = min(e, g + 4096)
            p = synth.quadrotor_c5(ge - g, first=g, device=dev)
            for f in synth.RRProblem.FIELDS:
                getattr(prob, f)[g - s:ge - s].copy_(getattr(p, f))
            del p
        torch.cuda.synchronize()
        gen_s += time.perf_counter() - t0
        for _ in range(max(3, a.warmup) if s == b0 else 1):
            call.launch(stream)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
        for k in range(a.steps):
            ev[k][0].record(stream)
            call.launch(stream)
            ev[k][1].record(stream)
        torch.cuda.synchronize()
        chunk_ms.append(statistics.mean(x.elapsed_time(y) for x, y in ev))
        summ["status"][s - b0:e - b0].copy_(sol["status"])
        summ["u0"][s - b0:e - b0].copy_(sol["u"][:, 0, :])
        # KKT residual norms of the chunk's solution (rr_residual, the paper's residual callback
        # P:666) for the summary; timed on its own, not part of the solve time
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        _, norms = rr.rr_residual(prob, sol, stream=stream)
        r1.record(stream)
        torch.cuda.synchronize()
        res_ms.append(r0.elapsed_time(r1))
        summ["kkt"][s - b0:e - b0].copy_(norms)
    barrier(ws)
    torch.cuda.synchronize()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    gathered = gather_summaries(summ, rank, ws, total)
    g1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    solve_ms = max_over_ranks(sum(chunk_ms), ws)
    gather_ms = max_over_ranks(g0.elapsed_time(g1), ws)
    res_ms_max = max_over_ranks(sum(res_ms), ws)
    if rank != 0:
        return
    nbad = int((gathered["status"] != 0).sum())
    kkt_max = float(gathered["kkt"].max()) if total else 0.0
    ms = solve_ms + gather_ms
    kern_ms_chunk = statistics.mean(chunk_ms)
    alg = ALG_BYTES_PER_STAGE * total * Nh / ws
    peak, src = measured_peaks()
    ach = alg / (solve_ms / 1e3) / 1e9
    print(json.dumps({
        "metric": METRIC, "value": total / (ms / 1e3), "unit": "solves/s", "n_gpus": ws, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C5: %d quadrotor regularized LQR (n_x=12 n_u=4 N=200 delta=1e-4) over %d GPU(s), "
                               "chunks of %d, FP64" % (total, ws, CH),
                   "global_batch": total, "seq_len": Nh, "parallelism": "batch-shard x%d" % ws,
                   "l2": "chunk inputs 37 GB > 126 MB L2 (no flush needed)",
                   "timing": "sum over the rank's chunks of the mean event-timed rr_factor_solve launch, "
                             "+ summary gather; max over ranks; generation untimed (%.1f s)" % gen_s},
        "stage_updates_per_s": total * Nh / (ms / 1e3), "solve_ms": solve_ms, "gather_ms": gather_ms,
        "chunks_per_rank": len(chunk_ms), "status_nonzero": nbad,
        "summary": {"fields": sorted(summ), "gathered_to": "rank 0 (dist.gather)", "gather_ms": gather_ms,
                    "kkt_residual_max": kkt_max, "residual_ms": res_ms_max},
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                     "traffic": None, "kernel": "rr_fused_mma_kernel<12,4>", "kernel_ms_per_chunk": kern_ms_chunk,
                     "alg_bytes_per_stage": ALG_BYTES_PER_STAGE, "peak_source": src},
        "clocks": clk, "e2e": None, "gpu_launches": a.steps * len(chunk_ms),
        "cpu_baseline": c5_cpu_baseline(a, total) if (ws == 1 and not a.no_cpu_baseline) else None}), flush=True)


def c5_cpu_baseline(a, total):
    import synth
    import oracle
    return oracle_rate(lambda k: synth.quadrotor_c5(k), lambda p, t: oracle.rr_solve_t2(p, nthreads=t),
                       a.cpu_seconds, total, "C5 quadrotor instances, T2 plain-C oracle", calib=8, cap=8192)


def run_split(a, ws, rank, local):
    """Extra line: the factorization / solve / residual callbacks (rr_factor, rr_solve, rr_residual)
    on the C2 workload, one step = factor + solve (the residual timed beside it).  Each kernel is
    timed with CUDA events on the launching stream and reported against its own algorithmic bytes
    per (instance, stage):  rr_factor reads A,B,Q,M,R and writes the record
    (328 + 214 doubles); rr_solve reads A,B,c,q,r + record in the backward sweep, record + A,B,c in
    the forward sweep, writes/reads v,k and writes x,u,y (220+214+16 + 214+204+16+28 doubles);
    rr_residual reads the stage data + x,u,y once and writes the residual (356+28+28 doubles)."""
    import torch
    import synth
    import paper_2509_16370_b200 as rr
    dev = torch.device("cuda", local)
    B = a.batch
    prob = synth.empty_problem(NX, NU, HORIZON, B, device=dev)
    for s in range(0, B, 4096):
        e = min(B, s + 4096)
        p = synth.random_stable_lqr(NX, NU, HORIZON, e - s, SEED, DELTA, first=rank * B + s, device=dev)
        for f in synth.RRProblem.FIELDS:
            getattr(prob, f)[s:e].copy_(getattr(p, f))
        del p
    stream = torch.cuda.current_stream(dev)
    F, st = rr.rr_factor(prob)
    sol = rr.rr_solve(prob, F)
    nbs = rr.solve_workspace_bytes(NX, NU, HORIZON, B)
    wsb = torch.empty((nbs + 7) // 8, dtype=torch.float64, device=dev)
    res, norms = rr.rr_residual(prob, sol)
    for _ in range(max(3, a.warmup)):
        rr.rr_factor(prob, factor=F, status=st)
        rr.rr_solve(prob, F, out=sol, workspace=wsb)
        rr.rr_residual(prob, sol, res=res, norms=norms)
    torch.cuda.synchronize()
    assert int((st != 0).sum()) == 0 and int((sol["status"] != 0).sum()) == 0
    E = lambda: torch.cuda.Event(enable_timing=True)
    ev = {k: [(E(), E()) for _ in range(a.steps)] for k in ("factor", "solve", "residual")}
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier(ws)
    torch.cuda.synchronize()
    t0, t1 = E(), E()
    t0.record(stream)
    for k in range(a.steps):
        ev["factor"][k][0].record(stream)
        rr.rr_factor(prob, factor=F, status=st)
        ev["factor"][k][1].record(stream)
        ev["solve"][k][0].record(stream)
        rr.rr_solve(prob, F, out=sol, workspace=wsb)
        ev["solve"][k][1].record(stream)
    t1.record(stream)
    for k in range(a.steps):
        ev["residual"][k][0].record(stream)
        rr.rr_residual(prob, sol, res=res, norms=norms)
        ev["residual"][k][1].record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    clk = clocks.stop()
    ms = max_over_ranks(t0.elapsed_time(t1) / a.steps, ws)
    kms = {k: statistics.mean(x.elapsed_time(y) for x, y in v) for k, v in ev.items()}
    if rank != 0:
        return
    peak, src = measured_peaks()
    per_stage = {"factor": 8 * (328 + 214), "solve": 8 * (220 + 214 + 16 + 214 + 204 + 16 + 28),
                 "residual": 8 * (356 + 28 + 28)}
    kern = {}
    for k, b in per_stage.items():
        ach = b * B * HORIZON / (kms[k] / 1e3) / 1e9
        kern[k] = {"ms": kms[k], "record_model_bytes_per_stage": b, "achieved_gbs": ach, "frac": ach / peak,
                   "traffic": ncu_traffic("rr_split_%s_c2" % k)}
    # headline: SURVEY §8(d)'s split-API algorithmic bytes (9,680 B/stage: rr_factor writes V, K, L_G;
    # rr_solve's two sweeps re-read them with A, B, q, r, c), not this build's larger record model
    # (per kernel above: the record also carries S⁻¹ and G⁻¹, 11,632 B/stage for the pair)
    SPLIT_ALG = 9680
    tot_b = SPLIT_ALG * B * HORIZON
    ach = tot_b / (ms / 1e3) / 1e9
    print(json.dumps({
        "metric": METRIC + " (split API: rr_factor + rr_solve)", "value": B * ws / (ms / 1e3), "unit": "solves/s",
        "n_gpus": ws, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2 via rr_factor + rr_solve: %d random stable regularized LQR per GPU, n_x=%d n_u=%d "
                               "N=%d delta=%g, FP64" % (B, NX, NU, HORIZON, DELTA),
                   "l2": "inputs %.1f GB/GPU > 126 MB L2 (no flush needed)" % (prob.nbytes() / 1e9)},
        "stage_updates_per_s": B * ws * HORIZON / (ms / 1e3),
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                     "traffic": None, "kernel": "rr_fused_mma_kernel<12,4,FAC> + rr_solve_kernel<12,4>",
                     "alg_bytes_per_stage": SPLIT_ALG, "peak_source": src, "kernels": kern},
        "clocks": clk, "e2e": None, "gpu_launches": 2 * a.steps,
        "cpu_baseline": cpu_baseline(a.cpu_seconds) if (ws == 1 and not a.no_cpu_baseline) else None}), flush=True)


def run_f32(a, ws, rank, local):
    """Extra line: C2 through the FP32 factor record + FP64 iterative refinement --
    rr_factor(RR_FLAG_FACTOR_FP32) + rr_solve + k x (rr_residual + rr_solve(ACCUMULATE)), k the
    smallest refinement count whose per-instance error against the FP64 fused solution is within
    the 1e-9 bar on the whole batch (measured here, 0..4).  The line carries the A/B against the
    FP64 split path (rr_factor + rr_solve) and the fused kernel, each timed on the same stream."""
    import torch
    import synth
    import paper_2509_16370_b200 as rr
    dev = torch.device("cuda", local)
    B = a.batch
    prob = synth.empty_problem(NX, NU, HORIZON, B, device=dev)
    for s0 in range(0, B, 4096):
        e = min(B, s0 + 4096)
        p = synth.random_stable_lqr(NX, NU, HORIZON, e - s0, SEED, DELTA, first=rank * B + s0, device=dev)
        for f in synth.RRProblem.FIELDS:
            getattr(prob, f)[s0:e].copy_(getattr(p, f))
        del p
    stream = torch.cuda.current_stream(dev)
    ref = rr.rr_factor_solve(prob)                        # FP64 fused solution (the parity reference)
    F64, st64 = rr.rr_factor(prob)
    F32, st32 = rr.rr_factor(prob, fp32=True)
    nbs = rr.solve_workspace_bytes(NX, NU, HORIZON, B)
    wsb = torch.empty((nbs + 7) // 8, dtype=torch.float64, device=dev)
    sol = rr.rr_solve(prob, F32, workspace=wsb)
    torch.cuda.synchronize()
    assert int((st32 != 0).sum()) == 0 and int((sol["status"] != 0).sum()) == 0

    def err(s_):
        w = 0.0
        for k in ("x", "u", "y"):
            d = (s_[k] - ref[k]).abs().reshape(B, -1).amax(1) / ref[k].abs().reshape(B, -1).amax(1).clamp_min(1e-300)
            w = max(w, float(d.max()))
        return w
    errs = [err(sol)]
    for _ in range(4):
        rr.rr_refine(prob, F32, sol, iters=1, workspace=wsb)
        torch.cuda.synchronize()
        errs.append(err(sol))
    kref = next((k for k, e_ in enumerate(errs) if e_ <= 1e-9), None)
    E = lambda: torch.cuda.Event(enable_timing=True)

    def timed(fn):
        for _ in range(max(3, a.warmup)):
            fn()
        torch.cuda.synchronize()
        ev = [(E(), E()) for _ in range(a.steps)]
        for k in range(a.steps):
            ev[k][0].record(stream)
            fn()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
        return statistics.mean(x.elapsed_time(y) for x, y in ev)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier(ws)
    kms = {
        "factor_fp32": timed(lambda: rr.rr_factor(prob, factor=F32, status=st32, fp32=True)),
        "solve_fp32": timed(lambda: rr.rr_solve(prob, F32, out=sol, workspace=wsb)),
        "refine_step_fp32": timed(lambda: rr.rr_refine(prob, F32, sol, iters=1, workspace=wsb)),
        "factor_fp64": timed(lambda: rr.rr_factor(prob, factor=F64, status=st64)),
        "solve_fp64": timed(lambda: rr.rr_solve(prob, F64, out=sol, workspace=wsb)),
    }
    call = rr.Marshalled(prob, ref)
    kms["fused_fp64"] = timed(lambda: call.launch(stream))
    barrier(ws)
    clk = clocks.stop()
    kk = kref if kref is not None else 4
    ms = max_over_ranks(kms["factor_fp32"] + kms["solve_fp32"] + kk * kms["refine_step_fp32"], ws)
    if rank != 0:
        return
    peak, src = measured_peaks()
    ach = 6976 * B * HORIZON / (ms / 1e3) / 1e9
    print(json.dumps({
        "metric": METRIC + " (FP32 factor record + FP64 refinement)", "value": B * ws / (ms / 1e3), "unit": "solves/s",
        "n_gpus": ws, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 factor record, f64 arithmetic", "data": "synthetic",
        "config": {"workload": "C2 via rr_factor(FP32 records) + rr_solve + %d x (rr_residual + rr_solve): %d random "
                               "stable regularized LQR per GPU, n_x=%d n_u=%d N=%d delta=%g" % (kk, B, NX, NU, HORIZON, DELTA),
                   "l2": "inputs %.1f GB/GPU > 126 MB L2 (no flush needed)" % (prob.nbytes() / 1e9)},
        "refinement_steps_for_1e-9": kref, "max_rel_err_after_k_refinements": errs,
        "kernels_ms": kms,
        "ab": {"fp32_pipeline_ms": ms, "fp64_split_ms": kms["factor_fp64"] + kms["solve_fp64"],
               "fp64_fused_ms": kms["fused_fp64"]},
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                     "traffic": None, "alg_bytes_per_stage": 6976, "peak_source": src,
                     "note": "against the fused FP64 algorithmic bytes (the work the pipeline replaces)"},
        "clocks": clk, "e2e": None, "gpu_launches": 2 + 2 * kk, "cpu_baseline": None}), flush=True)


def run_c4solve(a, ws, rank, local, swing=False):
    """Extra line: ipm_solve (the batched IPM loop) on the C4 cart-pole batch, 16,384
    instances per GPU, N = 100.
      c4solve: a fixed budget of 20 IPM iterations with the model's trial merits (the swing-up does
        not converge within it, so every instance runs all 20: a fixed amount of work per step);
      c4swing: the whole swing-up to convergence (settings.linear_merit, reading R22; at most 300
        iterations) -- converged instances drop out of the loop's active list.
    Each timed step solves a fresh device copy of the same initial iterate.  Per iteration and
    stage the loop moves the ipm_step bytes (~1.9 KB) plus the evaluation /
    residual passes (~0.9 KB); the roofline uses 2.8 KB per (instance, stage, iteration)."""
    import copy
    import numpy as np
    import torch
    import paper_2509_16370_b200 as rr
    from synth.ipm_workloads import cartpole_c4
    dev = torch.device("cuda", local)
    B, Nh, IT = 16384, 100, (300 if swing else 20)
    S = dict(max_iters=IT, linear_merit=swing)
    b = cartpole_c4(B, seed=2511, N=Nh, first=rank * B, device=dev)
    call0 = rr.IpmSolveCall(b, **S)

    def fresh():
        bk = copy.copy(b)
        bk.it = {k: v.clone() for k, v in b.it.items()}
        return rr.IpmSolveCall(bk, ws=call0.ws, **S)
    nw = max(3, a.warmup)
    calls = [fresh() for _ in range(nw + a.steps)]
    stream = torch.cuda.current_stream(dev)
    for k in range(nw):
        calls[k].launch(stream)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    clocks = ClockSampler(local)
    barrier(ws)
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    for k in range(a.steps):
        ev[k][0].record(stream)
        rep = calls[nw + k].launch(stream)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    clk = clocks.stop()
    ms = max_over_ranks(sum(s_.elapsed_time(e_) for s_, e_ in ev) / a.steps, ws)
    iters = int(rep["iters"].sum())
    nconv = int((rep["status"] == 0).sum())
    if rank == 0:
        alg = 2800 * Nh * iters
        peak, src = measured_peaks()
        if swing:
            metric = "regularized-IPM solve: converged C4 cart-pole swing-ups/s (ipm_solve to tol 1e-6)"
            value, unit = nconv * ws / (ms / 1e3), "solves/s"
        else:
            metric = "regularized-IPM solve: instance-iterations/s (C4 cart-pole, ipm_solve, 20 iterations)"
            value, unit = iters * ws / (ms / 1e3), "instance-iterations/s"
        it_np = rep["iters"].cpu().numpy()
        print(json.dumps({
            "metric": metric, "value": value, "unit": unit, "n_gpus": ws, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C4 ipm_solve: %d cart-pole instances per GPU, N=%d, max_iters=%d%s" % (
                B, Nh, IT, ", linear_merit (reading R22)" if swing else ""),
                       "l2": "stage data 3.1 GB/GPU > 126 MB L2 (no flush needed)"},
            "solves_per_s": B * ws / (ms / 1e3), "iterations_total": iters,
            "instance_iterations_per_s": iters * ws / (ms / 1e3),
            "iterations": {"min": int(it_np.min()), "median": float(np.median(it_np)), "max": int(it_np.max())},
            "status_counts": {str(int(k)): int(v) for k, v in zip(*torch.unique(rep["status"], return_counts=True))},
            "roofline": {"bound": "hbm", "achieved": alg / (ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": alg / (ms / 1e3) / 1e9 / peak, "traffic": None,
                         "alg_bytes_per_stage_iteration": 2800, "peak_source": src},
            "clocks": clk, "gpu_launches": a.steps * (4 * IT + 3),
            "cpu_baseline": c4solve_cpu_baseline(a, B, Nh, IT, swing) if (ws == 1 and not a.no_cpu_baseline) else None}),
              flush=True)


def c4solve_cpu_baseline(a, B, Nh, IT, swing=False):
    """The oracle IPM loop (oracle/ipm_solve.py around the C oracle step) on a bounded sample of the
    same C4 batch and settings; rate in the line's unit (instance-iterations/s, or converged
    solves/s for the swing-up)."""
    from synth.ipm_workloads import cartpole_c4
    from oracle.ipm_solve import SolveSettings, ipm_solve_oracle
    r = oracle_rate(lambda k: cartpole_c4(k, seed=2511, N=Nh),
                    lambda p, t: ipm_solve_oracle(p, SolveSettings(max_iters=IT, linear_merit=swing), nthreads=t),
                    a.cpu_seconds, B,
                    "C4 cart-pole instances, oracle IPM loop (%s)" % ("swing-up to convergence, linear_merit" if swing
                                                                      else "%d iterations" % IT),
                    calib=(2 if swing else 16), cap=(256 if swing else 2048))
    if not swing:
        r["value"] *= IT
        r["one_thread_value"] *= IT
        r["unit"] = "instance-iterations/s"
    else:
        r["unit"] = "solves/s"
    return r


def run_c1(a, ws, rank, local):
    """BASELINE configs[0]: ONE double-integrator instance (n=2, m=1, N=10, terminal equality folded
    with η = 1e4, δ = 1e-4; latency, no roofline claim).  Latency of one
    rr_factor_solve launch (CUDA events around each launch, median of K), the same through the
    host-buffer C-ABI path (H2D + solve + D2H), and the T2 oracle on one host thread (median)."""
    import torch
    import synth
    import oracle
    import paper_2509_16370_b200 as rr
    if rank != 0:
        return
    dev = torch.device("cuda", local)
    p = synth.double_integrator_c1()
    pd = p.to(dev)
    sol = rr.alloc_solution(pd)
    call = rr.Marshalled(pd, sol)
    stream = torch.cuda.current_stream(dev)
    K = max(a.steps, 50)
    for _ in range(max(3, a.warmup)):
        call.launch(stream)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for s_, e_ in ev:
        s_.record(stream)
        call.launch(stream)
        e_.record(stream)
    torch.cuda.synchronize()
    us = statistics.median(s_.elapsed_time(e_) * 1e3 for s_, e_ in ev)
    hp = synth.RRProblem(p.nx, p.nu, p.N, **{f: getattr(p, f).pin_memory() for f in p.FIELDS})
    hs = {k: torch.empty(v.shape, dtype=v.dtype).pin_memory() for k, v in sol.items()}
    hcall = rr.HostMarshalled(hp, hs, pd, rr.alloc_solution(pd), ws=call.ws)
    for _ in range(3):
        hcall.launch(stream)
    torch.cuda.synchronize()
    evh = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for s_, e_ in evh:
        s_.record(stream)
        hcall.launch(stream)
        e_.record(stream)
    torch.cuda.synchronize()
    us_h = statistics.median(s_.elapsed_time(e_) * 1e3 for s_, e_ in evh)
    o = oracle.rr_solve_t2(p)
    err = max(float(abs(hs[k].numpy() - o[k]).max() / abs(o[k]).max()) for k in ("x", "u", "y"))
    t_or = []
    for _ in range(21):
        t0 = time.perf_counter()
        oracle.rr_solve_t2(p, nthreads=1)
        t_or.append(time.perf_counter() - t0)
    print(json.dumps({
        "metric": "regularized-LQR single-instance latency (C1 double integrator)", "value": us, "unit": "us",
        "n_gpus": 1, "steps": K, "warmup": a.warmup, "ms_per_step": us / 1e3, "higher_is_better": False,
        "scaling": "none", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C1: 1 double integrator n_x=2 n_u=1 N=10, terminal equality folded (eta=1e4), delta=1e-4"},
        "kernel": "rr_fused_kernel<2,1> (lane group of 4)",
        "e2e": {"value": us_h, "unit": "us", "h2d_bytes_per_step": hcall.h2d_bytes, "d2h_bytes_per_step": hcall.d2h_bytes,
                "path": "rr_factor_solve_host (C-ABI, pinned host buffers)"},
        "max_rel_err_vs_oracle": err, "roofline": None,
        "cpu_baseline": {"value": statistics.median(t_or) * 1e6, "unit": "us", "cores": 1, "kind": "oracle",
                         "sample": "the C1 instance, T2 plain-C oracle through ctypes, median of 21"},
        "gpu_launches": K}), flush=True)


def run_pit(a, ws, rank, local):
    """Extra line: single-instance latency of the parallel-in-time solve
    (rr_factor_solve_pit: O(log N) levels + one refinement) against the sequential fused recursion
    (rr_factor_solve: N dependent stages) on C2-recipe instances (n=12, m=4, δ=1e-4) with long
    horizons.  CUDA events around each call, median of K."""
    import torch
    import synth
    import paper_2509_16370_b200 as rr
    if rank != 0:
        return
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    K = max(a.steps, 10)

    def lat(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        for s_, e_ in ev:
            s_.record(stream)
            fn()
            e_.record(stream)
        torch.cuda.synchronize()
        return statistics.median(s_.elapsed_time(e_) for s_, e_ in ev)
    rows = []
    for N in (64, 512, 4096):
        p = synth.random_stable_lqr(12, 4, N, 1, SEED, DELTA, device=dev)
        sol = rr.alloc_solution(p)
        call = rr.Marshalled(p, sol)
        t_seq = lat(lambda: call.launch(stream))
        ws_ = torch.empty((rr._lib.lib().rr_pit_workspace_bytes(ctypes_dims(rr, p)) + 7) // 8, dtype=torch.float64,
                          device=dev)
        sol2 = rr.alloc_solution(p)
        t_pit = lat(lambda: rr.rr_factor_solve_pit(p, out=sol2, workspace=ws_, stream=stream))
        err = max(float(((sol2[k] - sol[k]).abs().max() / sol[k].abs().max()).item()) for k in ("x", "u", "y"))
        # the same call captured once in a CUDA graph and replayed (no per-kernel launch overhead)
        gs = torch.cuda.Stream(dev)
        gs.wait_stream(stream)
        with torch.cuda.stream(gs):
            rr.rr_factor_solve_pit(p, out=sol2, workspace=ws_, stream=gs)
        stream.wait_stream(gs)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            rr.rr_factor_solve_pit(p, out=sol2, workspace=ws_, stream=torch.cuda.current_stream())
        t_graph = lat(lambda: graph.replay())
        rows.append({"N": N, "sequential_ms": t_seq, "pit_ms": t_pit, "pit_graph_ms": t_graph,
                     "speedup": t_seq / t_pit, "speedup_graph": t_seq / t_graph, "max_rel_diff": err})
    best = rows[-1]
    # the oracle (T2 plain C, one thread: a single instance) on the same N = 4096 instance
    import oracle
    pc = p.to("cpu")
    t_or = []
    for _ in range(3):
        t0 = time.perf_counter()
        oracle.rr_solve_t2(pc, nthreads=1)
        t_or.append(time.perf_counter() - t0)
    levels = max(1, (rows[-1]["N"]).bit_length())  # strides 1, 2, 4, ... <= N
    per_call = (1 + 1 + 1 + 2 * levels + 1 + levels + 1) + (1 + 1 + 1 + 2 * levels + 1 + levels + 1 + 3) + 1
    print(json.dumps({
        "metric": "regularized-LQR single-instance latency, parallel-in-time vs sequential (n=12 m=4, N=4096)",
        "value": min(best["pit_ms"], best["pit_graph_ms"]) * 1e3, "unit": "us", "n_gpus": 1, "steps": K, "warmup": 3,
        "ms_per_step": min(best["pit_ms"], best["pit_graph_ms"]), "higher_is_better": False, "scaling": "none", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": "1 random stable regularized LQR (C2 recipe) n_x=12 n_u=4 delta=1e-4, N in {64, 512, 4096}"},
        "horizons": rows, "roofline": None, "gpu_launches": per_call * K,
        "cpu_baseline": {"value": statistics.median(t_or) * 1e6, "unit": "us", "cores": 1, "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": "the same N = %d instance, T2 plain-C oracle, 1 thread, median of 3" % rows[-1]["N"]}}),
          flush=True)


def ctypes_dims(rr, p):
    import ctypes
    from paper_2509_16370_b200.rr import dims_of
    return ctypes.byref(dims_of(p))


if __name__ == "__main__":
    main()
