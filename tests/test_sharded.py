"""Multi-rank path sharding (paper_2012_09739_b200/sharded.py) on CPU: two
gloo ranks each compute their chunk shard, one all_gather, every rank folds
in chunk order.  The partials come from the oracle here (the product
computes them on the GPU); what is under test is the shard/gather/fold
logic: the result must be bitwise identical to a single-rank fold and to the
oracle's whole-run tree, for any rank count."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT  # noqa: F401

N_PATHS = 2 * 262144 + 777  # three chunks, the last ragged
LEVEL = 0


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, queue) -> None:
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_2012_09739_b200 as L
    from oracle.bind import Oracle
    from paper_2012_09739_b200.sharded import sharded_run_coupled_paths

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    O = Oracle()
    cfg = O.config(level=LEVEL, mantissa_bits=23, approx="linear:16", kahan=True, seed=3)

    def partials(model, level, spec, approx, kahan, n, seed, base, c0, c1, **_):
        return O.chunk_partials(cfg, n, base, c0, c1)

    m = sharded_run_coupled_paths(L.make_gbm(), LEVEL, L.PrecisionSpec.fp32(), None, True,
                                  N_PATHS, 3, 1000, partials_fn=partials)
    queue.put((rank, [m.d_hat.state(), m.d_bar.state(), m.d_four.state()]))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_chunks_partition():
    from paper_2012_09739_b200.sharded import shard_chunks
    for n in (1, 3, 7, 16, 64):
        for world in (1, 2, 3, 4, 8):
            ranges = [shard_chunks(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
                assert a1 == b0 and a1 >= a0
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1


def test_two_rank_gloo_fold_is_bitwise_single_rank(oracle):
    import paper_2012_09739_b200 as L
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[0] == got[1]
    cfg = oracle.config(level=LEVEL, mantissa_bits=23, approx="linear:16", kahan=True, seed=3)
    single = L.fold_partials(oracle.chunk_partials(cfg, N_PATHS, 1000, 0, 3))
    assert got[0] == [single.d_hat.state(), single.d_bar.state(), single.d_four.state()]
    rc, whole, _ = oracle.run_tree(cfg, N_PATHS, 1000)
    assert rc == 0 and got[0] == whole
