"""Multi-process μ-sharding on the GPU with the CUDA solver, not the oracle.

The box the tests run on has one B200, and NCCL refuses two ranks on one device, so these use the ``gloo``
backend with both ranks on cuda:0.  The ranks' kernels never wait on one another (no collective on the solve
path), so this checks the N > 1 host logic — shard split, per-rank device solve, the final tensor gather, and
bench.py's barrier / max-over-ranks / subset-check path — not scaling.
"""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, nb, out_q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1807_11866_b200 import online, sharding, synthetic

    model = synthetic.config_model(cfg)
    mu = synthetic.config_mu(cfg, nb)
    dm = online.DeviceModel(model, 0)

    def solve(mu_local):  # the product path: host μ in, rbns_solve_host_ex on the device, host arrays out
        r = dm.solve_host(mu_local, pressure=True)
        return {k: r[k] for k in sharding.RESULT_KEYS}

    res = sharding.solve_sharded(mu, world, rank, solve)
    if rank == 0:
        out_q.put({k: v for k, v in res.items() if v is not None})
    dm.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg,nb", [(2, 3001), (4, 2048)])
def test_sharded_device_solve_equals_single_process(cfg, nb):
    """world 2: each rank solves its shard through the C ABI on the device; the gather on rank 0 is bitwise
    the single-process solve of the whole batch (u, p, iteration counts, status, last update)."""
    import torch.multiprocessing as mp

    from paper_1807_11866_b200 import online, synthetic

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world, port = 2, _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, nb, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    model = synthetic.config_model(cfg)
    with online.DeviceModel(model, 0) as dm:
        ref = dm.solve_host(synthetic.config_mu(cfg, nb), pressure=True)
    for k in ("u", "iters", "status", "last_update") + (("p",) if model.n_p else ()):
        np.testing.assert_array_equal(got[k], ref[k], err_msg=k)
    assert (got["status"] == 0).all()


def test_bench_two_ranks_functional():
    """bench.py's N > 1 path under torchrun (gloo, both ranks on cuda:0): one JSON line from rank 0 with
    n_gpus 2, the whole-job value, the bitwise subset check and the functional-check marker."""
    env = dict(os.environ, RBNS_BENCH_BACKEND="gloo", PYTHONPATH=str(ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"),
           "--gpus", "2", "--steps", "1", "--warmup", "3", "--batch", "2048", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = lines[0]
    assert line["n_gpus"] == 2 and line["config"]["global_batch"] == 4096
    assert line["bitwise_subset_check"] is True
    assert line["newton"]["converged"] == 2048
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    assert "functional_check" in line
