"""Runs sharded over several devices of one process (lpmc_options.devices):
contiguous chunk ranges per listed device, launched concurrently, folded in
chunk order -- bitwise the single-device result.  The box has one GPU, so the
lists repeat device 0 (each entry still gets its own sub-range, stream and
buffers); on an 8-GPU box the same code spreads the sub-ranges over the GPUs.
"""
from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu


def _state(m):
    return [m.d_hat.state(), m.d_bar.state(), m.d_four.state()]


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0], [0, 0, 0, 0, 0, 0, 0, 0]])
@pytest.mark.parametrize("reduce", ["tree", "sequential"])
def test_sharded_run_equals_single_device(gpu, devices, reduce):
    model = gpu.make_gbm()
    tb = gpu.InvCdfApprox.parse("linear:16")
    n = 5 * 262144 + 777  # 6 chunks, ragged
    args = (model, 3, gpu.PrecisionSpec.fp32(), tb, True, n, 4, 3 << 40)
    one = gpu.run_coupled_paths(*args, reduce=reduce)
    many = gpu.run_coupled_paths(*args, reduce=reduce, devices=devices)
    assert _state(many) == _state(one)


def test_sharded_level_stats_and_glibc(gpu):
    model = gpu.make_gbm()
    args = (model, 6, gpu.PrecisionSpec.carrier(), None, False, 1 << 20, 1)
    one = gpu.estimate_level_stats(*args, reduce="sequential", exact_z="glibc")
    many = gpu.estimate_level_stats(*args, reduce="sequential", exact_z="glibc", devices=[0, 0, 0])
    assert many == one
    assert many.mean_hat == float.fromhex("0x1.6bc234c2c6020p-16")  # the reference's C1 checkpoint


def test_sharded_multi_run_and_nested(gpu):
    model = gpu.make_gbm()
    P = gpu.PrecisionSpec
    tb = gpu.InvCdfApprox.parse("linear:16")
    runs = [(l, P.fp16() if l % 2 else P.fp32(), bool(l % 3 == 0), 1000 + 300000 * (l % 4), l << 40)
            for l in range(9)]
    one = gpu.run_coupled_many(model, tb, 2, runs)
    many = gpu.run_coupled_many(model, tb, 2, runs, devices=[0, 0, 0, 0])
    assert [_state(m) for m in many] == [_state(m) for m in one]
    r1 = gpu.run_nested_estimator(model, 5, P.fp16(), tb, False, 1e-3, 1)
    r2 = gpu.run_nested_estimator(model, 5, P.fp16(), tb, False, 1e-3, 1, devices=[0, 0])
    assert r2.value == r1.value and r2.level_contributions == r1.level_contributions


def test_sharded_failures_and_range_fallback(gpu):
    P = gpu.PrecisionSpec
    bad = gpu.make_gbm(1e30, 0.0, 1e300)
    for devices in (None, [0, 0, 0]):
        with pytest.raises(gpu.DomainError, match="non-finite operand") as ei:
            gpu.run_coupled_paths(bad, 4, P.carrier(), None, False, 600000, 1, 0, devices=devices)
        assert ei.value.path_index == 0
    hot = gpu.make_gbm(80.0, 0.2)  # native fp32 legs leave the exact range: emulated re-run
    tb = gpu.InvCdfApprox.parse("linear:16")
    args = (hot, 4, P.fp32(), tb, True, 3 * 262144 + 5, 2, 0)
    assert _state(gpu.run_coupled_paths(*args, devices=[0, 0])) == _state(gpu.run_coupled_paths(*args))
    with pytest.raises(gpu.InvalidArgument):
        gpu.run_coupled_paths(gpu.make_gbm(), 2, P.fp32(), tb, False, 100, 1, 0, devices=[0, 99])


def test_many_partials_equal_level_partials(gpu):
    """lpmc_run_coupled_many_partials (bench.py's e2e call for every N): each
    run's chunk range equals lpmc_level_partials of that range bitwise, and
    folding the ranges of all 'ranks' equals run_coupled_many."""
    import numpy as np

    from paper_2012_09739_b200.sharded import n_chunks_for, shard_chunks
    model = gpu.make_gbm()
    P = gpu.PrecisionSpec
    tb = gpu.InvCdfApprox.parse("linear:16")
    runs = [(l, P.fp16() if l % 2 else P.fp32(), False, 2 * 262144 + 1000 * l, l << 40)
            for l in (0, 3, 7)]
    ext = dict(payoff="call", strike=1.0)
    whole = gpu.run_coupled_many(model, tb, 1, runs, **ext)
    for world in (1, 2, 4):
        shards = []
        for rank in range(world):
            ranges = [shard_chunks(n_chunks_for(r[3]), rank, world) for r in runs]
            parts = gpu.run_coupled_many_partials(model, tb, 1, runs, ranges, **ext)
            for (l, spec, k, n, base), (c0, c1), part in zip(runs, ranges, parts):
                if c1 > c0:
                    one = gpu.level_partials(model, l, spec, tb, k, n, 1, base, c0, c1, **ext)
                    assert np.array_equal(part.view(np.uint64), one.view(np.uint64))
            shards.append(parts)
        for i, m in enumerate(whole):
            full = np.concatenate([s[i] for s in shards], axis=0)
            assert _state(gpu.fold_partials(full)) == _state(m)
