"""Paths sharded over ranks (one process per GPU), one tiny collective.

The reference's only parallelism is 256-path batches over threads, merged in
batch order (mlmc.hpp:74-110).  Here the unit of sharding is a chunk of
LPMC_CHUNK_PATHS = 2^18 paths (1024 batches): each rank runs a contiguous
chunk range on its own GPU, the per-chunk moment partials (3 x 40 bytes per
chunk) are all-gathered (NCCL over NVLink for cuda tensors, gloo on CPU), and
every rank folds them in chunk order.  Because chunk partials do not depend
on which rank computed them, the result is bitwise identical for any number
of ranks -- including one.
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np

from . import _native as N
from .api import CoupledMoments, fold_partials, level_partials


def shard_chunks(n_chunks: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced chunk range [c0, c1) of `rank` out of `world`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(int(n_chunks), int(world))
    c0 = rank * base + min(rank, extra)
    c1 = c0 + base + (1 if rank < extra else 0)
    return c0, c1


def n_chunks_for(n_paths: int) -> int:
    return (int(n_paths) + N.CHUNK_PATHS - 1) // N.CHUNK_PATHS


def allgather_partials(local: np.ndarray, n_chunks: int, group=None,
                       device: Optional[str] = None) -> np.ndarray:
    """Gather every rank's (k_r, 3, 5) partials into the full (n_chunks, 3, 5)
    array in chunk order.  One all_gather of a padded float64 tensor."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    kmax = max(shard_chunks(n_chunks, r, world)[1] - shard_chunks(n_chunks, r, world)[0]
               for r in range(world))
    buf = np.zeros((max(kmax, 1), 3, 5))
    buf[: local.shape[0]] = local
    t = torch.from_numpy(buf.reshape(-1).copy())
    if device is not None:
        t = t.to(device)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    rows = []
    for r in range(world):
        c0, c1 = shard_chunks(n_chunks, r, world)
        rows.append(out[r].cpu().numpy().reshape(-1, 3, 5)[: c1 - c0])
    return np.concatenate(rows, axis=0)


def sharded_run_coupled_paths(model, level, spec_low, approx, kahan, n_paths, seed, path_base,
                              group=None, device: Optional[str] = None,
                              partials_fn: Callable = level_partials, **ext) -> CoupledMoments:
    """run_coupled_paths with this rank's chunk shard on its own GPU; every
    rank returns the same (bitwise) CoupledMoments."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n_chunks = n_chunks_for(n_paths)
    c0, c1 = shard_chunks(n_chunks, rank, world)
    if c1 > c0:
        local = partials_fn(model, level, spec_low, approx, kahan, n_paths, seed, path_base,
                            c0, c1, **ext)
    else:
        local = np.zeros((0, 3, 5))
    full = allgather_partials(np.asarray(local).reshape(-1, 3, 5), n_chunks, group, device)
    return fold_partials(full)


def _many_partials(model, approx, seed, runs, ranges, **ext):
    from .api import run_coupled_many_partials
    return run_coupled_many_partials(model, approx, seed, runs, ranges, **ext)


def sharded_run_coupled_many(model, approx, seed, runs, group=None, device: Optional[str] = None,
                             partials_fn: Callable = _many_partials, **ext) -> list:
    """run_coupled_many with every run sharded over the ranks: rank r runs its
    contiguous chunk range of each run in ONE concurrent multi-run call
    (lpmc_run_coupled_many_partials), then one all_gather per run and an
    index-order fold.  Every rank returns the same (bitwise) list of
    CoupledMoments, equal to run_coupled_many's on one device."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    runs = list(runs)
    nck = [n_chunks_for(r[3]) for r in runs]
    ranges = [shard_chunks(k, rank, world) for k in nck]
    parts = partials_fn(model, approx, seed, runs, ranges, **ext)
    out = []
    for k, part in zip(nck, parts):
        full = allgather_partials(np.asarray(part).reshape(-1, 3, 5), k, group, device)
        out.append(fold_partials(full))
    return out
