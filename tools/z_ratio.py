"""Normalised error of the fast-mode exact Gaussians against the reference's
(glibc) on the sampler's grid: r = |z_dev - z_ref| / (eps (v / pdf(z) + |z|)),
v = min(u, 1 - u) -- the conditioning of Z = Phi^-1(u) to a 1-ulp error in
Phi and to a 1-ulp error in z itself.  Prints the max and quantiles over
uniform draws of the reference stream and over the extreme tails (for the
asserted bound in tests/test_gpu_parity.py and DESIGN.md section 7).

    python tools/z_ratio.py
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2012_09739_b200 as L  # noqa: E402
from oracle.bind import Reference  # noqa: E402

EPS = 2.0 ** -52


def ratio(u, zd, zr):
    v = np.minimum(u, 1.0 - u)
    pdf = np.exp(-0.5 * zr * zr) / math.sqrt(2 * math.pi)
    return np.abs(zd - zr) / (EPS * (np.maximum(v, 1e-300) / np.maximum(pdf, 1e-300) + np.abs(zr)))


def main():
    R = Reference()
    u = np.concatenate([R.uniforms(77, p, 4096) for p in range(256)])  # 1M stream draws
    rng = np.random.default_rng(3)
    tails = np.concatenate([rng.uniform(2 ** -54, 1.1e-5, 100000),  # t >= 3: libdevice path
                            np.exp(-rng.uniform(0, 37, 100000))])
    tails = np.concatenate([tails, 1.0 - tails[tails < 0.5]])
    for name, uu in (("stream", u), ("tails", tails)):
        zr = R.exact_inv_cdf(uu)
        zd = L.device_inv_cdf(uu)
        r = ratio(uu, zd, zr)
        ulp = np.abs(zd.view(np.int64) - zr.view(np.int64))
        print(f"{name}: n={len(uu)} bitwise {np.mean(ulp == 0):.4f} max ulp {ulp.max()} "
              f"ratio max {r.max():.3f} p99.99 {np.quantile(r, 0.9999):.3f} "
              f"p99 {np.quantile(r, 0.99):.3f} at u={uu[np.argmax(r)]!r}")


if __name__ == "__main__":
    main()
