"""Fit the direct piecewise-polynomial table of the fast exact Gaussian
(paper_2012_09739_b200/csrc/lpmc_direct_coef.h) with mpmath at 50 digits.

-Phi^-1 on the lower half (the upper quantile Phi^-1(1 - v) > 0), v =
min(u, 1 - u) in [2^-(B+1), 1/2), is cut the
way the paper cuts its approximate transforms, but to binary64 accuracy:
every binade [2^-(k+1), 2^-k), k = 1..B, into 2^S equal sub-intervals, a
degree-DEG polynomial in t = v - v_c on each (v_c the sub-interval's
midpoint: a double whose bit pattern is v's with the mantissa bits below the
top S replaced by 100...0, so t is one exact subtraction).  The record index
is read off v's high word: (hi >> (20 - S)) - BASE.

A record is ROW doubles, highest power first, c0 split hi + lo:
    c_DEG ... c_1, c0_lo, c0_hi   (+ padding to ROW)
ROW/2 is odd so that records 8 apart are the only ones sharing a
shared-memory bank quad in the flat layout; S = 4, DEG = 8 fills ROW = 10
exactly (five 128-bit loads), and 225 records x 8 lane-private copies
(144 KB) fit the shared memory of one SM (math::LaneDirectTab).  One extra all-zero record serves v == 1/2
(Phi^-1 = 0 exactly, gaussian.hpp:62).

Approximation error (Chebyshev-node interpolant) in units of
eps (v / phi(z) + |z|), eps = 2^-52: <= 1.1e-2 for S = 4, DEG = 8 (the
conditioning of Z on the rounding of u plus one ulp of Z; the same unit as
tests/test_gpu_parity.py).  The evaluation adds 0.5 ulp of Z (the final
c0_hi addition) plus ~0.05 ulp from the polynomial part, |t P(t)| <= 2 % of
|z| away from z = 0.

    python tools/fit_direct.py > paper_2012_09739_b200/csrc/lpmc_direct_coef.h
    python tools/fit_direct.py --check   # evaluation error on random draws
"""
from __future__ import annotations

import os
import sys

import mpmath as mp

mp.mp.dps = 50

B = int(os.environ.get("LPMC_DIRECT_B", "14"))      # binades
S = int(os.environ.get("LPMC_DIRECT_S", "4"))       # log2 sub-intervals per binade
DEG = int(os.environ.get("LPMC_DIRECT_DEG", "8"))
ROW = int(os.environ.get("LPMC_DIRECT_ROW", "10"))  # doubles per record
assert ROW >= DEG + 2 and ROW % 2 == 0 and (ROW // 2) % 2 == 1


def ndtri_lower(v):
    return -mp.sqrt(2) * mp.erfinv(1 - 2 * v)


def table_value(v):
    """What the table stores: -Phi^-1(v) = Phi^-1(1 - v) > 0 for v < 1/2, so
    that the exact and the approximate transform (which evaluates the upper
    half, invcdf_approx.hpp:47-49) flip their signs on the same predicate."""
    return -ndtri_lower(v)


def fit_interval(a, b):
    """Monomial coefficients (ascending, in t = v - (a+b)/2) of the
    interpolant of Phi^-1 at DEG+1 Chebyshev nodes of [a, b]."""
    n = DEG + 1
    mid, half = (a + b) / 2, (b - a) / 2
    xs = [mp.cos(mp.pi * (2 * i + 1) / (2 * n)) for i in range(n)]
    fs = [table_value(mid + half * x) for x in xs]
    V = mp.matrix(n, n)
    for i, x in enumerate(xs):
        for j in range(n):
            V[i, j] = x ** j
    sol = mp.lu_solve(V, mp.matrix(fs))
    return [sol[j] / half ** j for j in range(n)]


def records():
    """Records in index order (increasing v), each a list of ROW mpf/float."""
    out = []
    for k in range(B, 0, -1):
        lo = mp.mpf(2) ** -(k + 1)
        w = lo / 2 ** S
        for sub in range(2 ** S):
            a = lo + sub * w
            c = fit_interval(a, a + w)
            hi = float(c[0])
            lo0 = float(c[0] - mp.mpf(hi))
            rec = [float(c[j]) for j in range(DEG, 0, -1)] + [lo0, hi]
            rec += [0.0] * (ROW - len(rec))
            out.append(rec)
    out.append([0.0] * ROW)  # v == 1/2
    return out


def fl(x):
    return mp.mpf(float(x))


def eval_record(rec, t):
    """The device's evaluation, every operation rounded to binary64."""
    p = mp.mpf(rec[0])
    for j in range(1, DEG):
        p = fl(p * t + mp.mpf(rec[j]))          # DFMA
    r = fl(p * t + mp.mpf(rec[DEG]))            # + c0_lo
    return fl(r + mp.mpf(rec[DEG + 1]))          # + c0_hi


def check(n=20000):
    import random
    random.seed(1)
    recs = records()
    eps = mp.mpf(2) ** -52
    worst, worst_ulp = mp.mpf(0), mp.mpf(0)
    base = (1023 - (B + 1)) << S
    for i in range(n):
        m = random.getrandbits(53)
        u = (mp.mpf(m) + mp.mpf(1) / 2) * mp.mpf(2) ** -53
        u = fl(u)
        v = 1 - u if u > 0.5 else u
        if v < mp.mpf(2) ** -(B + 1):
            continue
        if random.random() < 0.3:  # stress the interval edges
            e = random.randrange(1, B + 1)
            sub = random.randrange(2 ** S)
            v = mp.mpf(2) ** -(e + 1) * (1 + mp.mpf(sub) / 2 ** S)
            v = v + random.choice([0, 1, 2, 3]) * mp.mpf(2) ** -(e + 1 + 52)
        vf = float(v)
        import struct
        hi = struct.unpack("<Q", struct.pack("<d", vf))[0] >> 32
        idx = (hi >> (20 - S)) - base
        hc = (hi & ~((1 << (20 - S)) - 1)) | (1 << (19 - S))
        vc = struct.unpack("<d", struct.pack("<Q", hc << 32))[0]
        t = mp.mpf(vf) - mp.mpf(vc)
        assert t == fl(t)
        z = eval_record(recs[idx], t)
        zt = table_value(mp.mpf(vf))
        phi = mp.exp(-zt * zt / 2) / mp.sqrt(2 * mp.pi)
        unit = eps * (mp.mpf(vf) / phi + abs(zt))
        worst = max(worst, abs(z - zt) / unit)
        worst_ulp = max(worst_ulp, abs(z - zt) / (eps * abs(zt)) if zt != 0 else 0)
    print(f"B={B} S={S} DEG={DEG}: max |dz| = {float(worst):.3f} eps (v/phi + |z|), "
          f"{float(worst_ulp):.3f} eps |z|", file=sys.stderr)


def main():
    recs = records()
    n = len(recs)
    out = ["// Generated by tools/fit_direct.py (mpmath, 50 digits).  Do not edit.",
           "#pragma once", "",
           "// -Phi^-1(v) = Phi^-1(1 - v) >= 0, v in [2^-(B+1), 1/2]: B binades x 2^S sub-intervals, degree DEG in",
           "// t = v - midpoint; record = c_DEG..c_1, c0_lo, c0_hi (+ padding), index order =",
           "// increasing v, last record (all zero) = v == 1/2.",
           f"#define LPMC_DIRECT_B {B}", f"#define LPMC_DIRECT_S {S}",
           f"#define LPMC_DIRECT_DEG {DEG}", f"#define LPMC_DIRECT_ROW {ROW}",
           f"#define LPMC_DIRECT_N {n}",
           "#define LPMC_DIRECT_COEF_LIST \\"]
    lines = []
    for rec in recs:
        lines.append("  " + ", ".join(float(x).hex() for x in rec))
    out.append(",\\\n".join(lines))
    print("\n".join(out))


if __name__ == "__main__":
    if "--check" in sys.argv:
        check()
    else:
        main()
