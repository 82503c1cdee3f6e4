"""Pin the C oracle (oracle/lpmc_oracle.c) to the reference before trusting it:
against every golden vector generated from the unmodified reference
(tests/golden/reference_vectors.json) and, where oracle/_ref exists, against
the reference itself on fresh inputs.  CPU only."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import bits, unhex


def test_rng_words_and_uniforms(oracle, golden):
    for seed, path, ctr, w in golden["rng"]["words"]:
        assert oracle.stream_word(seed, path, ctr) == w
    for g in golden["rng"]["uniforms"]:
        u = oracle.uniforms(g["seed"], g["path"], 64)
        assert np.array_equal(bits(u), bits(unhex(g["u"])))


def test_exact_inv_cdf_bitwise(oracle, golden):
    u = unhex(golden["gauss"]["u"])
    z = unhex(golden["gauss"]["z"])
    for x, want in zip(u, z):
        if 0.0 < x < 1.0:
            got = oracle.exact_inv_cdf(x)
            assert bits([got])[0] == bits([want])[0], (x, got, want)
        else:
            with pytest.raises(ValueError):
                oracle.exact_inv_cdf(x)


def test_round_to_precision_bitwise(oracle, golden):
    x = unhex(golden["rounding"]["x"])
    for m, want in golden["rounding"]["by_m"].items():
        got = np.array([oracle.round(v, int(m)) for v in x])
        assert np.array_equal(bits(got), bits(unhex(want))), m


def test_tables_bitwise(oracle, golden):
    u = unhex(golden["tables_u"])
    for name, g in golden["tables"].items():
        t = oracle.table(name)
        assert t.K == g["K"]
        assert t.w_max == float.fromhex(g["w_max"]) and t.step_w == float.fromhex(g["step_w"])
        assert t.tail == float.fromhex(g["tail"])
        assert np.array_equal(bits(t.bp), bits(unhex(g["bp"])))
        assert np.array_equal(bits(t.coeff.reshape(-1)), bits(unhex(g["coeff"])))
        z = np.array([oracle.approx(name, x) for x in u])
        assert np.array_equal(bits(z), bits(unhex(g["z"]))), name


def test_paths_bitwise(oracle, golden):
    for c in golden["paths"]:
        want = unhex(c["out"]).reshape(-1, 4)
        cfg = oracle.config(level=c["level"], mantissa_bits=c["m"], approx=c["approx"],
                            kahan=c["kahan"], seed=c["seed"])
        got, _, fails = oracle.simulate(cfg, c["path_base"], want.shape[0])
        assert not fails
        assert np.array_equal(bits(got), bits(want)), c


def test_moments_bitwise(oracle, golden):
    for c in golden["moments"]:
        if c["n"] > 1 << 16:
            continue  # the 2^20-path checkpoint is covered on the GPU
        cfg = oracle.config(level=c["level"], mantissa_bits=c["m"], approx=c["approx"],
                            kahan=c["kahan"], seed=c["seed"])
        rc, got, _ = oracle.run_sequential(cfg, c["n"], c["path_base"], threads=4)
        assert rc == 0
        want = [(a[0], *unhex(a[1:])) for a in c["acc"]]
        assert got == [tuple(w) for w in want], c


def test_error_cases(oracle):
    cfg = oracle.config(level=4, mantissa_bits=52, mu=1e30, sigma=0.0, x0=1e300)
    rc, _, (fpath, fstep) = oracle.run_sequential(cfg, 8, 0)
    assert rc == 2 and fpath == 0  # non-finite operand on the first path
    cfg = oracle.config(level=-1, mantissa_bits=52)
    rc, got, _ = oracle.run_sequential(cfg, 0, 0)
    assert rc == 0 and got[0][0] == 0


def test_reference_unit_pins(oracle):
    """test_sde.cpp:22-47 known answers through the oracle's op layer."""
    # swamping: fp16 em_step at X=1, z=0, dt=2^-11 leaves X unchanged
    r = oracle.round
    spec = 10
    dt = r(2.0 ** -11, spec)
    a = r(r(0.05, spec) * 1.0, spec)
    drift = r(a * dt, spec)
    assert r(1.0 + r(drift + 0.0, spec), spec) == 1.0
    # Kahan: 4096 adds of 2^-11 recover 3.0 (every plain add ties back to 1.0)
    plain, s, c = 1.0, 1.0, 0.0
    for _ in range(4096):
        plain = r(plain + 2.0 ** -11, spec)
        y = r(2.0 ** -11 - c, spec)
        t = r(s + y, spec)
        c = r(r(t - s, spec) - y, spec)
        s = t
    assert plain == 1.0 and s == 3.0


def test_ieee_half_restatement_is_ieee(oracle):
    """The oracle's binary16 ops are correctly rounded IEEE ops (numpy float16
    rounds each op the same way); subnormals included."""
    rng = np.random.default_rng(0)
    a = rng.standard_normal(20000) * np.exp2(rng.integers(-20, 4, 20000))
    b = rng.standard_normal(20000) * np.exp2(rng.integers(-20, 4, 20000))
    ah, bh = a.astype(np.float16), b.astype(np.float16)
    for x, y in zip(ah[:2000], bh[:2000]):
        assert oracle.lib.orc_to_half(float(x) * float(y)) == float(np.float16(x) * np.float16(y))
        assert oracle.lib.orc_to_half(float(x) + float(y)) == float(np.float16(x) + np.float16(y))
    for v in a[:2000]:
        assert oracle.lib.orc_to_half(v) == float(np.float16(v))


# --- against the unmodified reference (only where oracle/_ref was built) ----
@pytest.mark.parametrize("level", [0, 1, 3, 7])
@pytest.mark.parametrize("m", [52, 23, 10, 7, 16, 3, 26])
@pytest.mark.parametrize("approx", ["exact", "linear:16", "cubic:8", "linear:128"])
def test_oracle_vs_reference_paths(oracle, ref, level, m, approx):
    for kahan in (0, 1):
        rc, msg, want = ref.simulate(level=level, mantissa_bits=m, approx=approx, kahan=kahan,
                                     seed=11, path_base=77, n=20)
        assert rc == 0, msg
        cfg = oracle.config(level=level, mantissa_bits=m, approx=approx, kahan=kahan, seed=11)
        got, _, _ = oracle.simulate(cfg, 77, 20)
        assert np.array_equal(bits(got), bits(want))


def test_oracle_vs_reference_moments_threads(oracle, ref):
    for threads in (1, 3):
        rc, msg, want = ref.run_coupled_paths(level=4, mantissa_bits=10, approx="linear:64", n=1000,
                                              seed=5, threads=threads)
        cfg = oracle.config(level=4, mantissa_bits=10, approx="linear:64", seed=5)
        rc2, got, _ = oracle.run_sequential(cfg, 1000, 0, threads=threads)
        assert rc == rc2 == 0 and got == [tuple(w) for w in want]
