"""Multi-GPU path on CPU (gloo, world size 2): shard ranges partition the batch, every rank's
generated shard is bitwise the unsharded generation of the same global ids, the oracle on the
shards equals the oracle on the whole batch, and the timing reduction is a max over ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_16370_b200.shard import max_over_ranks, shard_range


@pytest.mark.parametrize("world,total", [(1, 10), (2, 65536), (3, 10), (8, 1048576), (8, 5), (4, 0)])
def test_shard_ranges_partition(world, total):
    got = [shard_range(r, world, total) for r in range(world)]
    assert got[0][0] == 0 and got[-1][1] == total
    for (b0, e0), (b1, e1) in zip(got, got[1:]):
        assert e0 == b1
    sizes = [e - b for b, e in got]
    assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    b, e = shard_range(rank, world, total)
    p = synth.random_stable_lqr(5, 2, 6, e - b, seed=99, first=b)
    o = oracle.rr_solve_t2(p)
    # gather results to rank 0 through gloo (test-only check of the sharded outputs)
    xs = [torch.zeros(0)] * world
    obj = [None] * world
    dist.all_gather_object(obj, (b, e, o["x"], p.A.numpy()))
    t = max_over_ranks(float(rank + 1) * 0.5)
    if rank == 0:
        out.put((obj, t))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_shards_equal_unsharded():
    import oracle
    import synth
    total, world = 37, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    obj, tmax = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert tmax == 1.0
    full = synth.random_stable_lqr(5, 2, 6, total, seed=99)
    of = oracle.rr_solve_t2(full)
    for b, e, x, A in obj:
        assert np.array_equal(A, full.A[b:e].numpy())     # generator keyed by global id
        assert np.array_equal(x, of["x"][b:e])


def _gather_worker(rank, world, port, total, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2509_16370_b200.shard import gather_summaries
    b, e = shard_range(rank, world, total)
    ids = torch.arange(b, e, dtype=torch.int64)
    parts = {"status": (ids % 7).to(torch.int32), "u0": torch.stack([ids.double(), -ids.double()], dim=1),
             "kkt": torch.stack([ids.double() * 1e-12, ids.double() * 2e-12], dim=1)}
    # the IPM-step summary set of SURVEY §8(e) from the oracle on this rank's shard of a C4-LS batch
    from oracle.ipm import ipm_step_oracle
    from synth.ipm_workloads import cartpole_c4
    if e > b:
        res, _ = ipm_step_oracle(cartpole_c4(e - b, seed=2511, N=6, variant="C4-LS", first=b))
    else:  # empty shard (world > total)
        res = {k: np.zeros(0) for k in ("alpha_p", "D", "merit0")}
        res["status"] = np.zeros(0, dtype=np.int32)
    for k in ("alpha_p", "D", "merit0"):
        parts[k] = torch.from_numpy(res[k])
    parts["ipm_status"] = torch.from_numpy(res["status"])
    g = gather_summaries(parts, rank, world, total)
    if rank == 0:
        out.put({k: v.numpy() for k, v in g.items()})
    else:
        assert g is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,total", [(2, 11), (3, 10), (3, 2)])
def test_gloo_summary_gather_global_order(world, total):
    """Per-instance summaries of uneven (or empty) shards arrive on rank 0 only, in global-id order
    (row e: dist.gather to rank 0), and the IPM summaries (α_p, D, 𝒜(0), status) gathered from
    the shards equal the oracle on the unsharded batch bitwise."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    g = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    ids = np.arange(total)
    assert np.array_equal(g["status"], (ids % 7).astype(np.int32))
    assert np.array_equal(g["u0"], np.stack([ids, -ids], axis=1).astype(np.float64))
    assert np.array_equal(g["kkt"], np.stack([ids * 1e-12, ids * 2e-12], axis=1))
    from oracle.ipm import ipm_step_oracle
    from synth.ipm_workloads import cartpole_c4
    full, _ = ipm_step_oracle(cartpole_c4(total, seed=2511, N=6, variant="C4-LS"))
    for k in ("alpha_p", "D", "merit0"):
        assert np.array_equal(g[k], full[k]), k
    assert np.array_equal(g["ipm_status"], full["status"])
