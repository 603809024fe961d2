"""Multi-GPU work assignment for the window sweep.

The unit of work is one (window, restart) swarm; units are independent and
seeded by index only (window w: mix_seed(base, w), calibration.cpp:199;
restart r: base + r), so any assignment reproduces the single-device results
bit for bit and ranks never exchange data on the path.  One process per GPU.
"""
from __future__ import annotations


def partition(n_units: int, world: int, rank: int) -> range:
    """Contiguous, balanced share of n_units for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    q, r = divmod(n_units, world)
    begin = rank * q + min(rank, r)
    return range(begin, begin + q + (1 if rank < r else 0))


def restart_seed(base_seed: int, restart: int) -> int:
    """Base seed of sweep restart `restart` (restart r runs on rank r in bench.py)."""
    return (base_seed + restart) & 0xFFFFFFFFFFFFFFFF


def units(n_windows: int, n_restarts: int) -> list[tuple[int, int]]:
    """All (window, restart) units in canonical order."""
    return [(w, r) for r in range(n_restarts) for w in range(n_windows)]


def merge_by_index(parts: list[list[tuple[int, object]]]) -> list[object]:
    """Merge per-rank [(unit index, result)] lists into unit order (deterministic)."""
    flat = sorted((i, v) for part in parts for i, v in part)
    idx = [i for i, _ in flat]
    if idx != list(range(len(idx))):
        raise ValueError("shards do not cover the units exactly once")
    return [v for _, v in flat]


def run_sharded(n_units: int, compute, group=None, dst: int = 0):
    """Run `n_units` independent units across the ranks of a torch.distributed
    process group (one process per GPU) and merge the results in unit order
    on rank `dst` (None elsewhere).  `compute(indices)` evaluates one rank's
    contiguous share in one call — e.g. one engine plan holding all of the
    rank's swarms — and returns one picklable result per index.  The only
    collective is the final gather of the (small) results: nothing crosses
    GPUs on the compute path.  Without an initialised process group this is
    a single-process run."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return compute(list(range(n_units)))
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    mine = list(partition(n_units, world, rank))
    part = list(zip(mine, compute(mine))) if mine else []
    parts = [None] * world if rank == dst else None
    dist.gather_object(part, parts, dst=dst, group=group)
    return merge_by_index(parts) if rank == dst else None
