"""μ-sharding across GPUs: one process per GPU, no collective on the solve path.

Each rank solves a contiguous, balanced slice of the global μ batch on its own device with its own replica
of the (immutable) operators; the only communication is the final gather of the per-sample results to rank 0
(and, in bench.py, the barrier + max-reduction of the device time).  Per-sample results do not depend on
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


def gather_to_rank0(local: Dict[str, Optional[np.ndarray]], world: int, rank: int, group=None):
    """Final result gather (the only data collective).  Returns the concatenated dict on rank 0, else None."""
    if world == 1:
        return local
    import torch.distributed as dist

    parts = [None] * world if rank == 0 else None
    dist.gather_object(local, parts, dst=0, group=group)
    if rank != 0:
        return None
    out = {}
    for k in RESULT_KEYS:
        vals = [p[k] for p in parts if p.get(k) is not None]
        out[k] = np.concatenate(vals) if len(vals) == world else None
    return out


def solve_sharded(mu_all: np.ndarray, world: int, rank: int,
                  solve_fn: Callable[[np.ndarray], Dict[str, Optional[np.ndarray]]], group=None):
    """Solve this rank's shard with ``solve_fn`` (host arrays in/out) and gather everything on rank 0."""
    local = solve_fn(shard(mu_all, world, rank))
    return gather_to_rank0(local, world, rank, group)
