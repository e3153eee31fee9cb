"""Multi-GPU executors (one process per GPU, torch.distributed for the plumbing).

Tensor parallel — the reference's even-site double-site scheme (parallel.cpp:420-443) applied at
every site: each rank of a group of p2 holds the column shard tp_partition(chiR, p2, granule)[rank]
of every Gamma_i (balanced_partition rounded to whole contraction K blocks, so that a sharded
sweep accumulates exactly the unsharded sweep's K blocks and samples bit-identically to it) (so chi >= 4096 chains are split across HBMs), contracts it against the full
environment, exchanges the small per-(sample, outcome) (weight, max) partials and draws the same
outcome on every rank, then all-gathers the environment shards.  The exchange runs inside libmpsg
(NCCL, or an in-process group for ranks sharing a process); ``tp_connect_nccl`` shares the NCCL id
through torch.distributed and ``TensorParallelLocal`` drives p2 ranks from threads of one process.

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


def tp_partition(extent: int, parts: int, granule: int) -> List[Tuple[int, int]]:
    """Column shards of a tensor-parallel group (engine.cu part_range): balanced_partition
    (collective.cpp:80-92) rounded to whole K blocks of `granule` columns (64 for the 3M scheme,
    32 for 4M); every shard but the last holds round_up(ceil(extent / parts), granule) columns,
    trailing shards may be empty."""
    if parts <= 1:
        return [(0, extent)]
    a = -(-(-(-extent // parts)) // granule) * granule
    return [(min(i * a, extent), min(i * a + a, extent)) for i in range(parts)]


def tp_granule(scheme: int) -> int:
    """K block of a handle's contraction scheme (MPSG_SCHEME_3M: 64, MPSG_SCHEME_4M: 32)."""
    return 64 if scheme == 3 else 32


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


def tp_connect_nccl(sampler, group=None) -> None:
    """Share an NCCL unique id over torch.distributed and connect this rank's TP sampler."""
    import torch.distributed as dist

    from .sampler import nccl_unique_id
    obj = [nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    sampler.connect_nccl(obj[0])


class TensorParallelLocal:
    """p2 tensor-parallel ranks in one process (one thread each), e.g. several GPUs without NCCL or
    p2 ranks on a single GPU for testing the sharded path."""

    def __init__(self, mps, p2: int, devices=None, **kw):
        from .sampler import GpuSampler, connect_local
        devices = devices or [0] * p2
        self.ranks = [GpuSampler(mps, devices=[devices[r]], tp_size=p2, tp_rank=r, **kw) for r in range(p2)]
        connect_local(self.ranks)

    def _all(self, fn):
        import threading
        out = [None] * len(self.ranks)
        err = []

        def run(r):
            try:
                out[r] = fn(self.ranks[r])
            except Exception as e:  # pragma: no cover
                err.append(e)

        ts = [threading.Thread(target=run, args=(r,)) for r in range(len(self.ranks))]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if err:
            raise err[0]
        return out

    def sample(self, first: int, count: int, seed: int, mu=None):
        """Returns every rank's rows (they are identical)."""
        return self._all(lambda s: s.sample(first, count, seed, mu=mu))

    def marginals(self, first: int, forced, mu=None):
        return self._all(lambda s: s.marginals(first, forced, mu=mu))

    def decoded_gamma(self, site: int):
        """The full decoded Gamma_i assembled from every rank's column shard."""
        from . import _lib
        from .sampler import _check
        b = self.ranks[0].bond_dims
        full = np.zeros((b[site], b[site + 1], self.ranks[0].phys_dim), np.complex128)
        for r, s in enumerate(self.ranks):
            part = np.zeros_like(full)
            _check(_lib.lib().mpsg_decoded_gamma(s._h, site, part.ctypes.data_as(_lib._pd)))
            gran = tp_granule(_lib.lib().mpsg_scheme(s._h))
            c0, c1 = tp_partition(b[site + 1], len(self.ranks), gran)[r]
            full[:, c0:c1, :] = part[:, c0:c1, :]
        return full

    def close(self):
        for s in self.ranks:
            s.close()
