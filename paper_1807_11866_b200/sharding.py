"""μ-sharding across GPUs: one process per GPU, no collective on the solve path.

Each rank solves a contiguous, balanced slice of the global μ batch on its own device with its own replica
of the (immutable) operators; the only communication is the final gather of the per-sample results to rank 0
(tensor collectives, no pickling; and, in bench.py, the barrier + max-reduction of the device time).  Per-sample results do not depend on
how the batch is split (each sample's arithmetic is independent of its tile neighbours), so an N-rank run is
bitwise identical to a 1-rank run.

The solve itself is injected (``solve_fn``) so the same host logic runs with the CUDA path on GPU ranks and is
exercised on CPU with the ``gloo`` backend in the tests.
"""

from __future__ import annotations

from typing import Callable, Dict, Optional, Tuple

import numpy as np

RESULT_KEYS = ("u", "p", "iters", "status", "last_update")


def shard_bounds(total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous balanced split: the first ``total % world`` ranks get one extra sample."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(int(total), world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard(mu_all: np.ndarray, world: int, rank: int) -> np.ndarray:
    s, e = shard_bounds(mu_all.shape[0], world, rank)
    return np.ascontiguousarray(mu_all[s:e])


def gather_to_rank0(local: Dict[str, Optional[object]], world: int, rank: int, group=None):
    """Final result gather (the only data collective): every per-sample array is sent as one tensor collective
    (``dist.gather``; shards are padded to the largest shard and trimmed on rank 0), not pickled.  Arrays may be
    numpy (gloo, CPU) or torch tensors (they stay on their device: NCCL gathers over NVLink on a GPU box).
    Returns the concatenated dict on rank 0 (numpy for numpy input, tensors for tensor input), else None."""
    if world == 1:
        return local
    import torch
    import torch.distributed as dist

    first = next(v for v in local.values() if v is not None)
    n_local = int(first.shape[0])
    sizes = [torch.zeros(1, dtype=torch.int64, device=first.device if torch.is_tensor(first) else "cpu")
             for _ in range(world)]
    mine = torch.tensor([n_local], dtype=torch.int64, device=sizes[0].device)
    dist.all_gather(sizes, mine, group=group)
    counts = [int(c.item()) for c in sizes]
    cap = max(counts)
    out = {}
    for k in RESULT_KEYS:
        v = local.get(k)
        present = torch.tensor([v is not None], dtype=torch.int64, device=sizes[0].device)
        dist.all_reduce(present, op=dist.ReduceOp.MIN, group=group)
        if not present.item():
            out[k] = None
            continue
        t = v if torch.is_tensor(v) else torch.from_numpy(np.ascontiguousarray(v))
        buf = torch.zeros((cap,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        buf[:n_local] = t
        parts = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
        dist.gather(buf, parts, dst=0, group=group)
        if rank == 0:
            cat = torch.cat([p[:c] for p, c in zip(parts, counts)])
            out[k] = cat if torch.is_tensor(v) else cat.numpy()
    return out if rank == 0 else None


def solve_sharded(mu_all: np.ndarray, world: int, rank: int,
                  solve_fn: Callable[[np.ndarray], Dict[str, Optional[np.ndarray]]], group=None):
    """Solve this rank's shard with ``solve_fn`` (host arrays in/out) and gather everything on rank 0."""
    local = solve_fn(shard(mu_all, world, rank))
    return gather_to_rank0(local, world, rank, group)
