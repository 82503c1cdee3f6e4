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


def _many_worker(rank: int, world: int, port: int, queue) -> None:
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_2012_09739_b200 as L
    from oracle.bind import Oracle
    from paper_2012_09739_b200.sharded import sharded_run_coupled_many

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    O = Oracle()

    def partials(model, approx, seed, runs, ranges, **_):
        out = []
        for (level, spec, kahan, n, base), (c0, c1) in zip(runs, ranges):
            cfg = O.config(level=level, mantissa_bits=spec.mantissa_bits, approx="linear:16",
                           kahan=kahan, seed=seed)
            out.append(O.chunk_partials(cfg, n, base, c0, c1) if c1 > c0 else np.zeros((0, 3, 5)))
        return out

    P = L.PrecisionSpec
    runs = [(0, P.fp32(), True, N_PATHS, 1000), (0, P.fp16(), False, 262144 + 5, 7 << 40),
            (1, P.fp32(), False, 1000, 1 << 40)]
    ms = sharded_run_coupled_many(L.make_gbm(), None, 3, runs, partials_fn=partials)
    queue.put((rank, [[m.d_hat.state(), m.d_bar.state(), m.d_four.state()] for m in ms]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_multi_run_gloo_fold_is_bitwise_single_rank(oracle, world):
    """The bench's e2e path for N > 1: one multi-run partials call per rank
    over its chunk shard of every run (ranks own 0, 1 or 2 chunks of a run)."""
    import paper_2012_09739_b200 as L
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_many_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(1, world):
        assert got[r] == got[0]
    want = []
    for level, m, kahan, n, base in [(0, 23, True, N_PATHS, 1000), (0, 10, False, 262144 + 5, 7 << 40),
                                     (1, 23, False, 1000, 1 << 40)]:
        cfg = oracle.config(level=level, mantissa_bits=m, approx="linear:16", kahan=kahan, seed=3)
        k = (n + 262143) // 262144
        s = L.fold_partials(oracle.chunk_partials(cfg, n, base, 0, k))
        want.append([s.d_hat.state(), s.d_bar.state(), s.d_four.state()])
    assert got[0] == want
