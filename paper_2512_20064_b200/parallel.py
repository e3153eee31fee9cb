"""Multi-GPU executors (one process per GPU, torch.distributed for the plumbing).

Data parallel — the reference's ``run_data_parallel`` (parallel.cpp:240-330).  The reference
round-robins macro batches over simulated workers and has worker 0 broadcast every site payload
(parallel.cpp:271-289).  Here every rank keeps the whole compressed MPS resident in its own HBM,
so the data path has *no* collective: each rank sweeps a contiguous global-sample range
(``balanced_partition``, collective.cpp:80-92) and, because draws are keyed by the global sample
index (rng.hpp:7-9), the merged outcome matrix is identical to the serial one.  Only the final
outcome rows are gathered (to rank 0) once.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Tuple

import numpy as np


def balanced_partition(extent: int, parts: int) -> List[Tuple[int, int]]:
    """collective.cpp:80-92: [begin, end) ranges whose sizes differ by at most one."""
    base, rem = divmod(extent, parts)
    out, at = [], 0
    for i in range(parts):
        n = base + (1 if i < rem else 0)
        out.append((at, at + n))
        at += n
    return out


def rank_range(first: int, count: int, rank: int, world: int) -> Tuple[int, int]:
    a, b = balanced_partition(count, world)[rank]
    return first + a, b - a


def run_data_parallel(sample_fn: Callable[[int, int, int], np.ndarray], first: int, count: int,
                      seed: int, num_sites: int, group=None, dst: int = 0) -> Optional[np.ndarray]:
    """Sweep this rank's share of [first, first+count) and gather all rows on rank `dst`.

    sample_fn(first, count, seed) -> (count, num_sites) uint8 is the per-rank sampler (a
    GpuSampler.sample bound method on the B200).  Returns the full (count, M) matrix on `dst`,
    None elsewhere.  Works over any torch.distributed backend (nccl on B200s, gloo for tests)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    f, n = rank_range(first, count, rank, world)
    rows = sample_fn(f, n, seed) if n > 0 else np.zeros((0, num_sites), np.uint8)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    parts = balanced_partition(count, world)
    width = max(b - a for a, b in parts) if parts else 0
    buf = torch.zeros((width, num_sites), dtype=torch.uint8, device=dev)
    if n:
        buf[:n] = torch.from_numpy(np.ascontiguousarray(rows)).to(dev)
    gathered = [torch.zeros_like(buf) for _ in range(world)] if rank == dst else None
    dist.gather(buf, gathered, dst=dst, group=group)
    if rank != dst:
        return None
    out = np.empty((count, num_sites), np.uint8)
    for r, (a, b) in enumerate(parts):
        out[a:b] = gathered[r][: b - a].cpu().numpy()
    return out
