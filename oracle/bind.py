"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the CPU checkers.

* ``Oracle``   -> oracle/liblpmc_oracle.so (the C restatement, lpmc_oracle.c)
* ``Reference``-> oracle/_ref/liblpmc_ref.so (the unmodified reference headers
  behind ref_driver.cpp; built only where /root/reference exists, and then
  shipped as a prebuilt file)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liblpmc_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "liblpmc_ref.so")
REF_INC = "/root/reference/proj/include"

_dp = C.POINTER(C.c_double)
_u64 = C.c_uint64


def build(ref: bool | None = None) -> None:
    """Compile the oracle (always) and oracle/_ref (when the reference exists)."""
    subprocess.check_call(["make", "-s", "-C", HERE, "oracle"])
    if ref is None:
        ref = os.path.isdir(os.path.join(REF_INC, "lpmc"))
    if ref:
        subprocess.check_call(["make", "-s", "-C", HERE, "ref"])


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


class OrcTable(C.Structure):
    _fields_ = [("kind", C.c_int), ("K", C.c_int), ("w_max", C.c_double), ("step_w", C.c_double),
                ("tail", C.c_double), ("bp", _dp), ("coeff", _dp)]


class OrcConfig(C.Structure):
    _fields_ = [("mu", C.c_double), ("sigma", C.c_double), ("x0", C.c_double),
                ("horizon", C.c_double), ("level", C.c_int), ("mantissa_bits", C.c_int),
                ("ieee_half", C.c_int), ("table", C.POINTER(OrcTable)), ("kahan", C.c_int),
                ("seed", _u64), ("legs", C.c_uint), ("payoff", C.c_int), ("strike", C.c_double)]


class OrcMoments(C.Structure):
    _fields_ = [("n", _u64), ("mean", C.c_double), ("m2", C.c_double), ("m3", C.c_double),
                ("m4", C.c_double)]

    def as_tuple(self):
        return (int(self.n), self.mean, self.m2, self.m3, self.m4)


KIND_IDS = {"linear": 0, "cubic": 1, "constant": 2}


@dataclass
class Table:
    """Host copy of an approximation table (kind, K, w_max, step_w, tail, bp, coeff)."""
    kind: str
    K: int
    w_max: float
    step_w: float
    tail: float
    bp: np.ndarray
    coeff: np.ndarray  # (K, 4)

    def orc(self) -> OrcTable:
        self._bp = np.ascontiguousarray(self.bp, dtype=np.float64)
        self._co = np.ascontiguousarray(self.coeff, dtype=np.float64).reshape(-1)
        return OrcTable(KIND_IDS[self.kind], self.K, self.w_max, self.step_w, self.tail,
                        _ptr(self._bp), _ptr(self._co))


def parse_approx(name: str) -> tuple[str, int] | None:
    if name == "exact":
        return None
    kind, k = name.split(":")
    return kind, int(k)


class Oracle:
    """The C restatement."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.orc_mix64.restype = _u64
        L.orc_mix64.argtypes = [_u64]
        L.orc_stream_word.restype = _u64
        L.orc_stream_word.argtypes = [_u64, _u64, _u64]
        L.orc_uniform.restype = C.c_double
        L.orc_uniform.argtypes = [_u64, _u64, _u64]
        L.orc_exact_inv_cdf.argtypes = [C.c_double, _dp]
        L.orc_round.argtypes = [C.c_double, C.c_int, _dp]
        L.orc_table_build.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp]
        L.orc_approx_eval.argtypes = [C.POINTER(OrcTable), C.c_double, _dp]
        L.orc_to_half.restype = C.c_double
        L.orc_to_half.argtypes = [C.c_double]
        L.orc_simulate_coupled.argtypes = [C.POINTER(OrcConfig), _u64, _dp, _dp,
                                           C.POINTER(_u64)]
        L.orc_simulate_coupled_z.argtypes = [C.POINTER(OrcConfig), _u64, _dp, _dp, _dp,
                                             C.POINTER(_u64)]
        L.orc_run_sequential.argtypes = [C.POINTER(OrcConfig), _u64, _u64, C.c_int,
                                         C.POINTER(OrcMoments), C.POINTER(_u64), C.POINTER(_u64)]
        L.orc_run_tree.argtypes = [C.POINTER(OrcConfig), _u64, _u64, C.POINTER(OrcMoments),
                                   C.POINTER(_u64), C.POINTER(_u64)]
        L.orc_tree_from_values.argtypes = [_dp, _dp, _u64, C.c_uint, C.POINTER(OrcMoments)]
        L.orc_replay_hat.argtypes = [C.POINTER(OrcConfig), _dp, _dp]
        L.orc_sequential_from_values.argtypes = [_dp, _dp, _u64, C.POINTER(OrcMoments)]
        L.orc_moments_add.argtypes = [C.POINTER(OrcMoments), C.c_double]
        L.orc_moments_merge.argtypes = [C.POINTER(OrcMoments), C.POINTER(OrcMoments)]
        self._tables: dict[str, Table] = {}

    # -- primitives --------------------------------------------------------
    def stream_word(self, seed, path, ctr):
        return int(self.lib.orc_stream_word(seed, path, ctr))

    def uniforms(self, seed, path, count, ctr0=0):
        return np.array([self.lib.orc_uniform(seed, path, ctr0 + i) for i in range(count)])

    def exact_inv_cdf(self, u: float) -> float:
        z = C.c_double()
        rc = self.lib.orc_exact_inv_cdf(u, C.byref(z))
        if rc:
            raise ValueError("exact_inv_cdf requires u in (0, 1)")
        return z.value

    def round(self, x: float, m: int) -> float:
        out = C.c_double()
        if self.lib.orc_round(x, m, C.byref(out)):
            raise ValueError("non-finite operand")
        return out.value

    def table(self, name: str) -> Table:
        if name in self._tables:
            return self._tables[name]
        kind, K = parse_approx(name)
        bp = np.zeros(K)
        co = np.zeros(4 * K)
        wm, sw, tl = C.c_double(), C.c_double(), C.c_double()
        rc = self.lib.orc_table_build(KIND_IDS[kind], K, _ptr(bp), _ptr(co), C.byref(wm),
                                      C.byref(sw), C.byref(tl))
        if rc:
            raise ValueError("interval count must be a power of two >= 2")
        t = Table(kind, K, wm.value, sw.value, tl.value, bp, co.reshape(K, 4))
        self._tables[name] = t
        return t

    def approx(self, name: str, u: float) -> float:
        t = self.table(name).orc()
        z = C.c_double()
        if self.lib.orc_approx_eval(C.byref(t), u, C.byref(z)):
            raise ValueError("approx_inv_cdf requires u in (0, 1)")
        return z.value

    # -- paths --------------------------------------------------------------
    def config(self, *, level, mantissa_bits, approx="exact", kahan=False, seed=1, mu=0.05,
               sigma=0.2, x0=1.0, horizon=1.0, ieee_half=False, legs=3, payoff=0, strike=1.0):
        tab = None
        keep = None
        if approx != "exact":
            keep = self.table(approx).orc()
            tab = C.pointer(keep)
        cfg = OrcConfig(mu, sigma, x0, horizon, level, mantissa_bits, int(ieee_half), tab,
                        int(kahan), seed, legs, payoff, strike)
        cfg._keep = keep  # the table must outlive the config
        return cfg

    def simulate(self, cfg: OrcConfig, path_base: int, n: int, want_z=False, z_in=None):
        """-> (n,4) terminal values, optional (n, 2^l) Z, list of failures.
        z_in (n, 2^l) replaces the exact Gaussians (replay of device Z)."""
        out = np.zeros((n, 4))
        nz = 1 << max(cfg.level, 0)
        zs = np.zeros((n, nz)) if want_z else None
        fails = []
        r4 = np.zeros(4)
        zrow = np.zeros(nz)
        st = _u64()
        for i in range(n):
            if z_in is not None:
                zi = np.ascontiguousarray(z_in[i], dtype=np.float64)
                rc = self.lib.orc_simulate_coupled_z(C.byref(cfg), path_base + i, _ptr(zi),
                                                     _ptr(r4), None, C.byref(st))
            else:
                rc = self.lib.orc_simulate_coupled(C.byref(cfg), path_base + i, _ptr(r4),
                                                   _ptr(zrow) if want_z else None, C.byref(st))
            if rc:
                fails.append((i, rc, int(st.value)))
                out[i] = np.nan
            else:
                out[i] = r4
            if want_z:
                zs[i] = zrow
        return out, zs, fails

    def run_sequential(self, cfg, n, path_base=0, threads=1):
        out = (OrcMoments * 3)()
        fp, fs = _u64(), _u64()
        rc = self.lib.orc_run_sequential(C.byref(cfg), n, path_base, threads, out, C.byref(fp),
                                         C.byref(fs))
        return rc, [m.as_tuple() for m in out], (int(fp.value), int(fs.value))

    def run_tree(self, cfg, n, path_base=0):
        out = (OrcMoments * 3)()
        fp, fs = _u64(), _u64()
        rc = self.lib.orc_run_tree(C.byref(cfg), n, path_base, out, C.byref(fp), C.byref(fs))
        return rc, [m.as_tuple() for m in out], (int(fp.value), int(fs.value))

    def tree_from_values(self, d_hat: np.ndarray, d_bar: np.ndarray, legs=3):
        d_hat = np.ascontiguousarray(d_hat, dtype=np.float64)
        d_bar = np.ascontiguousarray(d_bar, dtype=np.float64)
        out = (OrcMoments * 3)()
        self.lib.orc_tree_from_values(_ptr(d_hat), _ptr(d_bar), len(d_hat), legs, out)
        return [m.as_tuple() for m in out]

    def replay_hat(self, cfg, z: np.ndarray) -> np.ndarray:
        """(n, 2^l) device Gaussians -> (n, 2) carrier legs (hat_f, hat_c)."""
        z = np.ascontiguousarray(z, dtype=np.float64)
        out = np.zeros((z.shape[0], 2))
        o2 = np.zeros(2)
        for i in range(z.shape[0]):
            row = np.ascontiguousarray(z[i])
            self.lib.orc_replay_hat(C.byref(cfg), _ptr(row), _ptr(o2))
            out[i] = o2
        return out

    def diffs(self, cfg, path_base: int, n: int):
        """Per-path (d_hat, d_bar) of paths path_base .. path_base+n-1."""
        dh = np.zeros(n)
        db = np.zeros(n)
        self.lib.orc_diffs.argtypes = [C.POINTER(OrcConfig), _u64, _u64, _dp, _dp]
        rc = self.lib.orc_diffs(C.byref(cfg), path_base, n, _ptr(dh), _ptr(db))
        if rc:
            raise RuntimeError(f"oracle path failure {rc}")
        return dh, db

    def chunk_partials(self, cfg, n_paths: int, path_base: int, c0: int, c1: int,
                       chunk_paths: int = 262144):
        """(c1-c0, 3, 5) chunk accumulators of the device library's tree."""
        out = []
        for c in range(c0, c1):
            a = c * chunk_paths
            m = min(chunk_paths, n_paths - a)
            dh, db = self.diffs(cfg, path_base + a, m)
            out.append(self.tree_from_values(dh, db, cfg.legs))
        return np.array(out, dtype=np.float64).reshape(-1, 3, 5)

    def sequential_from_values(self, d_hat, d_bar):
        d_hat = np.ascontiguousarray(d_hat, dtype=np.float64)
        d_bar = np.ascontiguousarray(d_bar, dtype=np.float64)
        out = (OrcMoments * 3)()
        self.lib.orc_sequential_from_values(_ptr(d_hat), _ptr(d_bar), len(d_hat), out)
        return [m.as_tuple() for m in out]

    def moments_add(self, xs):
        a = OrcMoments()
        for x in xs:
            self.lib.orc_moments_add(C.byref(a), float(x))
        return a.as_tuple()

    def moments_merge(self, a, b):
        ma, mb = OrcMoments(*a), OrcMoments(*b)
        self.lib.orc_moments_merge(C.byref(ma), C.byref(mb))
        return ma.as_tuple()


class Reference:
    """The unmodified reference behind ref_driver.cpp (oracle/_ref)."""

    ERR = {1: "invalid_argument", 2: "domain_error", 3: "runtime_error", 4: "exception"}

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    def __init__(self, path: str = REF_SO):
        L = self.lib = C.CDLL(path)
        L.ref_stream_word.restype = _u64
        L.ref_stream_word.argtypes = [_u64, _u64, _u64]
        L.ref_uniforms.argtypes = [_u64, _u64, _u64, _u64, _dp]
        L.ref_exact_inv_cdf_many.argtypes = [_dp, _u64, _dp]
        L.ref_round_many.argtypes = [_dp, _u64, C.c_int, _dp]
        L.ref_table.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), _dp, _dp,
                                _dp, _dp, _dp, C.c_int, C.c_char_p, C.c_int]
        L.ref_approx_many.argtypes = [C.c_char_p, _dp, _u64, _dp]
        L.ref_simulate_coupled.argtypes = [C.c_double] * 4 + [C.c_int, C.c_int, C.c_char_p,
                                                              C.c_int, _u64, _u64, _u64, _dp,
                                                              C.c_char_p, C.c_int]
        L.ref_run_coupled_paths.argtypes = [C.c_double] * 4 + [C.c_int, C.c_int, C.c_char_p,
                                                               C.c_int, _u64, _u64, _u64,
                                                               C.c_int, _dp, C.c_char_p,
                                                               C.c_int]
        L.ref_estimate_level_stats.argtypes = [C.c_double] * 4 + [
            C.c_int, C.c_int, C.c_char_p, C.c_int, _u64, _u64, C.c_double, C.c_int, _u64, _dp,
            C.c_char_p, C.c_int]
        L.ref_moments_add.argtypes = [_dp, _u64, _dp]
        L.ref_moments_merge.argtypes = [_dp, _dp, _dp]
        L.ref_hardware_threads.restype = C.c_int
        _pu = C.POINTER(_u64)
        _pi = C.POINTER(C.c_int)
        L.ref_allocate_samples.argtypes = [_dp, _u64, C.c_double, C.c_int, _pu, _pu, _pi,
                                           C.c_char_p, C.c_int]
        L.ref_predicted_times.argtypes = [_dp, _u64, C.c_double, _dp, C.c_char_p, C.c_int]
        L.ref_per_level_speedup.argtypes = [_dp, _dp, _pi, C.c_char_p, C.c_int]
        L.ref_run_nested_estimator.argtypes = [C.c_double] * 4 + [
            C.c_int, C.c_int, C.c_char_p, C.c_int, C.c_double, _u64, _u64, C.c_int, _dp, _dp,
            _dp, _pu, _pu, C.c_char_p, C.c_int]
        L.ref_simulate_two_way.argtypes = [C.c_double] * 4 + [C.c_int, C.c_int, C.c_char_p,
                                                              C.c_int, _u64, _u64, _u64, _dp,
                                                              C.c_char_p, C.c_int]
        L.ref_step_error_probe.argtypes = [C.c_double] * 4 + [C.c_int, C.c_int, C.c_char_p, _u64,
                                                              _u64, _dp, C.c_char_p, C.c_int]
        L.ref_density_report.argtypes = [C.c_char_p, _u64, C.c_int, _u64, C.c_double, _dp,
                                         C.c_int, C.POINTER(C.c_int), C.c_char_p, C.c_int]
        L.ref_two_way_experiment.argtypes = [C.c_double] * 4 + [
            C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_int, _u64, _u64, C.c_int, _dp,
            C.c_char_p, C.c_int]

    def _err(self, rc, msg):
        if rc:
            raise RuntimeError(f"{self.ERR.get(rc, rc)}: {msg.value.decode()}")

    def stream_word(self, seed, path, ctr):
        return int(self.lib.ref_stream_word(seed, path, ctr))

    def uniforms(self, seed, path, count, ctr0=0):
        out = np.zeros(count)
        self.lib.ref_uniforms(seed, path, ctr0, count, _ptr(out))
        return out

    def exact_inv_cdf(self, u: np.ndarray) -> np.ndarray:
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros_like(u)
        self.lib.ref_exact_inv_cdf_many(_ptr(u), len(u), _ptr(out))
        return out

    def round(self, x: np.ndarray, m: int) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros_like(x)
        self.lib.ref_round_many(_ptr(x), len(x), m, _ptr(out))
        return out

    def table(self, name: str) -> Table:
        kind, K = parse_approx(name)
        k, deg = C.c_int(), C.c_int()
        wm, sw, tl = C.c_double(), C.c_double(), C.c_double()
        bp = np.zeros(K)
        co = np.zeros(4 * K)
        msg = C.create_string_buffer(256)
        rc = self.lib.ref_table(name.encode(), C.byref(k), C.byref(deg), C.byref(wm),
                                C.byref(sw), C.byref(tl), _ptr(bp), _ptr(co), K, msg, 256)
        self._err(rc, msg)
        return Table(kind, K, wm.value, sw.value, tl.value, bp, co.reshape(K, 4))

    def approx(self, name: str, u: np.ndarray) -> np.ndarray:
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros_like(u)
        self.lib.ref_approx_many(name.encode(), _ptr(u), len(u), _ptr(out))
        return out

    def simulate(self, *, level, mantissa_bits, approx="exact", kahan=False, seed=1,
                 path_base=0, n=1, mu=0.05, sigma=0.2, x0=1.0, horizon=1.0):
        out = np.zeros((n, 4))
        msg = C.create_string_buffer(256)
        rc = self.lib.ref_simulate_coupled(mu, sigma, x0, horizon, level, mantissa_bits,
                                           approx.encode(), int(kahan), seed, path_base, n,
                                           _ptr(out), msg, 256)
        return rc, msg.value.decode(), out

    def run_coupled_paths(self, *, level, mantissa_bits, approx="exact", kahan=False, n=1000,
                          seed=1, path_base=0, threads=1, mu=0.05, sigma=0.2, x0=1.0,
                          horizon=1.0):
        out = np.zeros(15)
        msg = C.create_string_buffer(256)
        rc = self.lib.ref_run_coupled_paths(mu, sigma, x0, horizon, level, mantissa_bits,
                                            approx.encode(), int(kahan), n, seed, path_base,
                                            threads, _ptr(out), msg, 256)
        moms = [(int(out[5 * k]), *out[5 * k + 1:5 * k + 5]) for k in range(3)]
        return rc, msg.value.decode(), moms

    def estimate_level_stats(self, *, level, mantissa_bits, approx="exact", kahan=False,
                             n=1000, seed=1, per_step_arithmetic=0.0, threads=1, path_base=0,
                             mu=0.05, sigma=0.2, x0=1.0, horizon=1.0):
        out = np.zeros(16)
        msg = C.create_string_buffer(256)
        rc = self.lib.ref_estimate_level_stats(mu, sigma, x0, horizon, level, mantissa_bits,
                                               approx.encode(), int(kahan), n, seed,
                                               per_step_arithmetic, threads, path_base,
                                               _ptr(out), msg, 256)
        return rc, msg.value.decode(), out

    def moments_add(self, xs):
        xs = np.ascontiguousarray(xs, dtype=np.float64)
        out = np.zeros(5)
        self.lib.ref_moments_add(_ptr(xs), len(xs), _ptr(out))
        return (int(out[0]), *out[1:])

    def hardware_threads(self) -> int:
        return int(self.lib.ref_hardware_threads())

    # --------------------------------------- callers (mlmc.hpp:151-285) ----
    STATS_FIELDS = ("mean_hat", "v_hat", "v_hat_stderr", "mean_bar", "v_bar", "v_bar_stderr",
                    "mean_four", "V_bar", "V_bar_stderr", "c_hat", "c_bar", "C_bar", "m_hat",
                    "m_bar", "M_bar", "level")

    @staticmethod
    def _stats16(stats) -> np.ndarray:
        """LevelStats-like objects or dicts -> n x 16 doubles."""
        rows = []
        for st in stats:
            get = st.get if isinstance(st, dict) else (lambda k, st=st: getattr(st, k))
            rows.append([float(get(k)) for k in Reference.STATS_FIELDS])
        return np.ascontiguousarray(np.array(rows, dtype=np.float64).reshape(-1, 16))

    def allocate_samples(self, stats, eps, kind):
        a = self._stats16(stats)
        n = a.shape[0]
        prim = (C.c_uint64 * max(1, n))()
        sec = (C.c_uint64 * max(1, n))()
        deg = C.c_int()
        msg = C.create_string_buffer(256)
        rc = self.lib.ref_allocate_samples(_ptr(a), n, eps, int(kind), prim, sec, C.byref(deg),
                                           msg, 256)
        return rc, msg.value.decode(), ([int(x) for x in prim[:n]], [int(x) for x in sec[:n]],
                                        bool(deg.value))

    def predicted_times(self, stats, eps):
        a = self._stats16(stats)
        out = np.zeros(2)
        msg = C.create_string_buffer(256)
        rc = self.lib.ref_predicted_times(_ptr(a), a.shape[0], eps, _ptr(out), msg, 256)
        return rc, msg.value.decode(), (out[0], out[1])

    def per_level_speedup(self, st):
        a = self._stats16([st])
        v = C.c_double()
        flag = C.c_int()
        msg = C.create_string_buffer(256)
        rc = self.lib.ref_per_level_speedup(_ptr(a), C.byref(v), C.byref(flag), msg, 256)
        return rc, msg.value.decode(), (v.value, bool(flag.value))

    def run_nested_estimator(self, *, max_level, mantissa_bits, approx="exact", kahan=False,
                             eps=1e-2, seed=1, pilot_paths=1000, threads=1, mu=0.05, sigma=0.2,
                             x0=1.0, horizon=1.0):
        L = max(0, max_level) + 1
        out4 = np.zeros(4)
        contrib = np.zeros(L)
        pilot = np.zeros(16 * L)
        prim = (C.c_uint64 * L)()
        sec = (C.c_uint64 * L)()
        msg = C.create_string_buffer(256)
        rc = self.lib.ref_run_nested_estimator(mu, sigma, x0, horizon, max_level, mantissa_bits,
                                               approx.encode(), int(kahan), eps, seed,
                                               pilot_paths, threads, _ptr(out4), _ptr(contrib),
                                               _ptr(pilot), prim, sec, msg, 256)
        return rc, msg.value.decode(), {
            "value": out4[0], "t_hat": out4[1], "t_bar": out4[2], "degenerate": bool(out4[3]),
            "contributions": contrib, "pilot": pilot.reshape(L, 16),
            "primary": [int(x) for x in prim], "secondary": [int(x) for x in sec]}

    def simulate_two_way(self, *, level, mantissa_bits, approx="exact", kahan=False, seed=1,
                         path_base=0, n=1, mu=0.05, sigma=0.2, x0=1.0, horizon=1.0):
        out = np.zeros((n, 2))
        msg = C.create_string_buffer(256)
        rc = self.lib.ref_simulate_two_way(mu, sigma, x0, horizon, level, mantissa_bits,
                                           approx.encode(), int(kahan), seed, path_base, n,
                                           _ptr(out), msg, 256)
        return rc, msg.value.decode(), out

    def two_way_experiment(self, *, precision, approx, kahan, level_min, level_max, paths,
                           seed=1, threads=1, mu=0.05, sigma=0.2, x0=1.0, horizon=1.0):
        rows = level_max - level_min + 1
        out = np.zeros(4 * max(rows, 1))
        msg = C.create_string_buffer(256)
        rc = self.lib.ref_two_way_experiment(mu, sigma, x0, horizon, precision.encode(),
                                             approx.encode(), int(kahan), level_min, level_max,
                                             paths, seed, threads, _ptr(out), msg, 256)
        return rc, msg.value.decode(), out[:4 * rows].reshape(rows, 4)

    def step_error_probe(self, *, level, mantissa_bits, approx="exact", n_samples=10000, seed=1,
                         mu=0.05, sigma=0.2, x0=1.0, horizon=1.0):
        out = np.zeros(5)
        msg = C.create_string_buffer(256)
        rc = self.lib.ref_step_error_probe(mu, sigma, x0, horizon, level, mantissa_bits,
                                           approx.encode(), n_samples, seed, _ptr(out), msg, 256)
        return rc, msg.value.decode(), out

    def density_report(self, *, approx, seed=1, curve_points=2048, hist_samples=1000000,
                       bin_width=0.05, cap=100000):
        out = np.zeros(3 * cap)
        n = C.c_int()
        msg = C.create_string_buffer(256)
        rc = self.lib.ref_density_report(approx.encode(), seed, curve_points, hist_samples,
                                         bin_width, _ptr(out), cap, C.byref(n), msg, 256)
        return rc, msg.value.decode(), out[:3 * n.value].reshape(-1, 3)
