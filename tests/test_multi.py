"""world_size-2 gloo test of the μ-sharded path: rank-sharded solves gathered on rank 0
equal the single-process solve bit for bit.  The CPU oracle stands in for the device solve (this container has
no GPU); the host logic (split, per-rank solve, final gather — the only collective) is the product code."""

import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import rbns_oracle as oracle
    from paper_1807_11866_b200 import sharding, synthetic

    model = synthetic.config_model(0)
    mu = synthetic.config_mu(0)

    def solve(mu_local):  # per-sample oracle: like the device path, independent of the batch split
        res = [oracle.solve_sample(model, m) for m in mu_local]
        return {"u": np.array([r[0] for r in res]), "p": None, "iters": np.array([r[1] for r in res]),
                "status": np.array([r[2] for r in res]), "last_update": np.array([r[3] for r in res])}

    res = sharding.solve_sharded(mu, world, rank, solve)
    if rank == 0:
        out_q.put({k: v for k, v in res.items() if v is not None})
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_equals_single_process():
    from oracle import rbns_oracle as oracle
    from paper_1807_11866_b200 import synthetic

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world, port = 2, _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    model = synthetic.config_model(0)
    res = [oracle.solve_sample(model, m) for m in synthetic.config_mu(0)]
    u, it, st = (np.array([r[i] for r in res]) for i in range(3))
    np.testing.assert_array_equal(got["u"], u)
    np.testing.assert_array_equal(got["iters"], it)
    np.testing.assert_array_equal(got["status"], st)
