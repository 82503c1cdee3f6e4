"""Host-side logic of the C-ABI library, no GPU needed: the library loads and
exports every symbol include/lpmc_b200.h declares; host numerics (table
build, rounding, moment merges, fold, LevelStats) are bitwise the
reference's; sampling without a device fails loudly (no CPU fallback)."""
from __future__ import annotations

import ctypes as C
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT, bits, unhex


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "lpmc_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(lpmc_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol(lib):
    from paper_2012_09739_b200 import _native as N
    so = N.load()
    declared = header_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(so, name), name
        assert name in N.SIGNATURES, f"{name} not bound in _native.SIGNATURES"
    assert so.lpmc_abi_version() == 3


def test_cpp_api_header_compiles():
    """include/lpmc/*.hpp (the reference-shaped C++ API) compiles and links
    against liblpmc_b200.so."""
    import subprocess
    import tempfile
    from paper_2012_09739_b200 import _native as N
    N.load()
    src = os.path.join(ROOT, "tests", "cpp", "api_smoke.cpp")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "api_smoke")
        subprocess.check_call(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src,
                               "-o", exe, "-L", os.path.dirname(N.LIB_PATH), "-llpmc_b200",
                               "-Wl,-rpath," + os.path.dirname(N.LIB_PATH)])
        out = subprocess.run([exe, "--host-only"], capture_output=True, text=True)
        assert out.returncode == 0, out.stdout + out.stderr
        assert "host-only ok" in out.stdout


def test_tables_bitwise_vs_reference(lib, golden):
    u = unhex(golden["tables_u"])
    for name, g in golden["tables"].items():
        t = lib.InvCdfApprox.parse(name)
        assert t.interval_count() == g["K"]
        assert t.max_value() == float.fromhex(g["tail"])
        assert np.array_equal(bits(t.breakpoints()), bits(unhex(g["bp"])))
        assert np.array_equal(bits(t.coefficients().reshape(-1)), bits(unhex(g["coeff"])))
        sel = u[::7]
        z = np.array([t(x) for x in sel])
        assert np.array_equal(bits(z), bits(unhex(g["z"])[::7])), name


def test_constant_table_is_degree_zero(lib, oracle):
    t = lib.InvCdfApprox.parse("constant:16")
    o = oracle.table("constant:16")
    assert np.all(t.coefficients()[:, 1:] == 0.0)
    assert np.array_equal(bits(t.coefficients()), bits(o.coeff))
    lin = lib.InvCdfApprox.parse("linear:16")
    assert np.array_equal(bits(t.coefficients()[:, 0]), bits(lin.coefficients()[:, 0]))
    assert t.max_value() == t.coefficients()[-1, 0]


def test_table_validation(lib):
    for k in (0, 3, 12):
        with pytest.raises(lib.InvalidArgument):
            lib.InvCdfApprox.build("linear", k)
    with pytest.raises(lib.InvalidArgument):
        lib.InvCdfApprox.parse("spline:8")
    assert lib.InvCdfApprox.parse("cubic:64").degree() == 3
    t = lib.InvCdfApprox.parse("linear:8")
    assert t(0.5) == 0.0
    with pytest.raises(lib.DomainError):
        t(1.0)
    with pytest.raises(lib.DomainError):
        t(0.0)


def test_round_to_precision_bitwise(lib, golden):
    x = unhex(golden["rounding"]["x"])
    for m, want in golden["rounding"]["by_m"].items():
        spec = lib.PrecisionSpec(int(m))
        got = np.array([lib.round_to_precision(v, spec) for v in x])
        assert np.array_equal(bits(got), bits(unhex(want)))
    with pytest.raises(lib.DomainError):
        lib.round_to_precision(float("inf"), lib.PrecisionSpec.fp16())


def test_precision_spec_parse(lib):
    P = lib.PrecisionSpec
    assert P.parse("bf16").mantissa_bits == 7 and P.parse("fp22").mantissa_bits == 16
    assert P.parse("double").is_carrier() and P.parse("custom:12").mantissa_bits == 12
    assert P.parse("fp16-ieee").ieee_half
    for bad in ("fp8", "custom:0", "custom:27", "custom:x"):
        with pytest.raises(lib.InvalidArgument):
            P.parse(bad)
    assert P.fp16().unit_roundoff() == 2.0 ** -11


def test_moments_add_merge_bitwise(lib, oracle, ref):
    rng = np.random.default_rng(99)
    xs = rng.lognormal(0.0, 0.7, 5000)
    a = lib.MomentAccumulator()
    for x in xs:
        a.add(x)
    assert a.state() == ref.moments_add(xs) == oracle.moments_add(xs)
    parts = [xs[:700], xs[700:701], xs[701:]]
    accs = []
    for p in parts:
        m = lib.MomentAccumulator()
        for x in p:
            m.add(x)
        accs.append(m)
    ab = lib.MomentAccumulator(*accs[0].state())
    ab.merge(accs[1])
    ab.merge(accs[2])
    want = oracle.moments_merge(oracle.moments_merge(accs[0].state(), accs[1].state()),
                                accs[2].state())
    assert ab.state() == want
    assert ab.variance() == pytest.approx(np.var(xs, ddof=1), rel=1e-12)
    empty = lib.MomentAccumulator()
    w = lib.MomentAccumulator(*ab.state())
    w.merge(empty)
    assert w.state() == ab.state()


def test_fold_partials_matches_oracle_tree(lib, oracle):
    """The library's index-order fold of chunk partials equals the restated
    tree (oracle) for a multi-chunk, ragged run."""
    rng = np.random.default_rng(3)
    n = 2 * 262144 + 777
    dh = rng.standard_normal(n) * 1e-3
    db = dh + rng.standard_normal(n) * 1e-6
    want = oracle.tree_from_values(dh, db)
    parts = np.stack([np.array(oracle.tree_from_values(dh[s:s + 262144], db[s:s + 262144]))
                      for s in range(0, n, 262144)])
    got = lib.fold_partials(parts)
    assert [got.d_hat.state(), got.d_bar.state(), got.d_four.state()] == want


def test_level_stats_from_moments_matches_reference(lib, ref):
    for level, m, approx, kahan, n, psa in [(3, 52, "exact", 0, 64, 0.25),
                                            (0, 10, "exact", 1, 64, 0.25),
                                            (5, 23, "linear:16", 1, 2048, 0.0)]:
        rc, _, mom = ref.run_coupled_paths(level=level, mantissa_bits=m, approx=approx,
                                           kahan=kahan, n=n)
        rc2, _, want = ref.estimate_level_stats(level=level, mantissa_bits=m, approx=approx,
                                                kahan=kahan, n=n, per_step_arithmetic=psa)
        assert rc == rc2 == 0
        cm = lib.CoupledMoments(*(lib.MomentAccumulator(*a) for a in mom))
        s = lib.level_stats_from_moments(cm, level, lib.PrecisionSpec(m), bool(kahan), n,
                                         lib.CostModel(per_step_arithmetic=psa))
        got = [s.mean_hat, s.v_hat, s.v_hat_stderr, s.mean_bar, s.v_bar, s.v_bar_stderr,
               s.mean_four, s.V_bar, s.V_bar_stderr, s.c_hat, s.c_bar, s.C_bar, s.m_hat,
               s.m_bar, s.M_bar, s.level]
        assert np.array_equal(bits(np.array(got, dtype=np.float64)), bits(want))


def test_sampling_without_device_fails_loudly(lib):
    if lib.device_count() > 0:
        pytest.skip("a device is present")
    with pytest.raises(lib.api.N.NoDevice):
        lib.run_coupled_paths(lib.make_gbm(), 2, lib.PrecisionSpec.fp32(), None, False, 16, 1, 0)
    with pytest.raises(lib.InvalidArgument):
        lib.estimate_level_stats(lib.make_gbm(), 2, lib.PrecisionSpec.fp32(), None, False, 1, 1)
    sde = lib.SdeModel()
    with pytest.raises(lib.InvalidArgument):
        lib.run_coupled_paths(sde, 2, lib.PrecisionSpec.fp32(), None, False, 16, 1, 0)


def test_null_outputs_are_invalid_argument(lib):
    """The C-ABI checks its pointers: a null output is invalid_argument, never
    a crash (host-side entry points; no device needed)."""
    import ctypes as C
    from paper_2012_09739_b200 import _native as N
    so = N.load()
    err = N.Error()
    st = (N.LevelStatsC * 1)()
    assert so.lpmc_predicted_times(st, 1, 0.1, None, None, C.byref(err)) == N.LPMC_INVALID_ARGUMENT
    assert so.lpmc_per_level_speedup(st, None, None, C.byref(err)) == N.LPMC_INVALID_ARGUMENT
    assert so.lpmc_round_to_precision(1.0, 10, None, C.byref(err)) == N.LPMC_INVALID_ARGUMENT
    assert so.lpmc_invcdf_eval(None, 0.3, None, C.byref(err)) == N.LPMC_INVALID_ARGUMENT
    assert b"null" in err.message
