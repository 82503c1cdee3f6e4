"""Per-opcode dynamic instruction counts (warp level) from an ncu report's
source page (--import-source / SASS view), optionally diffed against a
second report.

    python tools/sass_hot.py rep.ncu-rep [base.ncu-rep] [--units N]

--units divides the counts (e.g. the warp-steps of the launch) so the
table reads as instructions per unit.
"""
from __future__ import annotations

import collections
import csv
import io
import re
import subprocess
import sys


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, isrc, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
    c = collections.Counter()
    for r in rows[2:]:
        if len(r) <= iex:
            continue
        t = re.sub(r"^@!?U?P\w+\s+", "", r[isrc].strip())
        if not t:
            continue
        c[t.split()[0]] += int(r[iex] or 0)
    return c


args = [a for a in sys.argv[1:] if not a.startswith("--")]
units = 1.0
if "--units" in sys.argv:
    units = float(sys.argv[sys.argv.index("--units") + 1])
    args = [a for a in args if a != sys.argv[sys.argv.index("--units") + 1]]
a = load(args[0])
b = load(args[1]) if len(args) > 1 else None
keys = sorted(set(a) | set(b or {}), key=lambda k: -a.get(k, 0))
print(f"{'opcode':28s} {'this':>10s}" + (f" {'base':>10s} {'delta':>10s}" if b else ""))
for k in keys:
    x = a.get(k, 0) / units
    if b is None:
        if x > 0.05:
            print(f"{k:28s} {x:10.2f}")
    else:
        y = b.get(k, 0) / units
        if abs(x - y) > 0.05 or x > 1:
            print(f"{k:28s} {x:10.2f} {y:10.2f} {x - y:+10.2f}")
print(f"{'total':28s} {sum(a.values()) / units:10.2f}" +
      (f" {sum(b.values()) / units:10.2f}" if b else ""))
