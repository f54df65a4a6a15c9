"""Replica (multi-GPU) host logic on CPU: world_size 2 over gloo, each rank
solving its own systems with the oracle (the GPU path is identical per rank)."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1912_04385_b200 import replicas


def test_assignment_partitions_the_systems():
    for world in (1, 2, 3, 8):
        seen = sorted(i for r in range(world) for i in replicas.assign(11, r, world))
        assert seen == list(range(11))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_1912_04385_b200 import gen
    o = oracle.api()
    iters, secs = 0, 0.0
    for sid in replicas.assign(3, rank, world):
        a, b, xs = gen.generate(gen.make_spec(10 + sid, 8, 4, kappa=1.0, perm_sigma=1.0, band=True, seed=20 + sid))
        r = o.system(a).setup("cptr3-amg", b).solve()
        assert r.converged and np.linalg.norm(r.x - xs) / np.linalg.norm(xs) < 1e-6
        iters += r.total_iterations
        secs += r.wall_time_s + 0.01 * (rank + 1)
    tmax = replicas.reduce_max(secs)
    total = replicas.reduce_sum(iters)
    thr = replicas.whole_job_throughput(iters, secs)
    out[rank] = (iters, secs, tmax, total, thr)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_replicas_over_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    iters = [res[r][0] for r in range(world)]
    secs = [res[r][1] for r in range(world)]
    for r in range(world):
        assert res[r][2] == max(secs)
        assert res[r][3] == sum(iters)
        assert abs(res[r][4] - sum(iters) / max(secs)) < 1e-9
