"""N>1 path on CPU: replicas over torch.distributed (gloo, world_size 2).

The solver does not shard across GPUs in this tier (replicas
only), so `bench.py --gpus N` runs N independent replicas and combines them
with a barrier, max-over-ranks time and sum-over-ranks work.  This test runs
that exact combination logic (bench.dist_max / dist_sum / barrier) with the
gloo backend and the CPU oracle as the per-rank workload."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                      LOCAL_RANK=str(rank))
    import bench
    import paper_2008_01539_b200 as pkg
    from oracle import Oracle
    dist = bench.init_dist(ws, rank, backend="gloo")
    case = pkg.Case(1, nx=24, ny=24, n_steps=4)
    orc = Oracle(case)
    r = orc.run_case(1, case.init_state(), case.schedule(), case.solver_opts())
    bench.barrier(dist)
    t_local = 1.0 + rank  # synthetic per-rank time: the job time is the max
    t = bench.dist_max(dist, t_local)
    na = bench.dist_sum(dist, float(r["sum_na"]))
    q.put((rank, r["sum_na"], r["iterations"], t, na, r["states"].u.tobytes()))
    dist.destroy_process_group()


def test_replicas_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, na0, it0, t0, tot0, u0), (r1, na1, it1, t1, tot1, u1) = out
    assert na0 == na1 and it0 == it1 and u0 == u1  # identical replicas
    assert t0 == t1 == 2.0  # max over ranks
    assert tot0 == tot1 == na0 + na1  # whole-job work = sum over ranks
