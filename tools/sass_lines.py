"""Dynamic warp-instruction counts of one kernel per source line: joins the
ncu report's SASS page (Instructions Executed per address) with the line
table of the same kernel in the locally built object (deterministic build of
the same sources).

    python tools/sass_lines.py rep.ncu-rep obj.o function-regex [--units N] [--top K] [--stalls]

--stalls: rank lines by warp-stall samples instead, with each line's
dominant stall reasons (ncu source-page stall_* columns).
"""
from __future__ import annotations

import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

args = [a for a in sys.argv[1:] if not a.startswith("--")]
units = float(sys.argv[sys.argv.index("--units") + 1]) if "--units" in sys.argv else 1.0
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 60
args = [a for a in args if a not in (str(units), str(top)) and not re.fullmatch(r"[0-9.e+]+", a)]
rep, obj, fun = args[:3]

if rep.endswith(".csv"):  # the source page exported on the GPU box (tools/ncu_capture.sh)
    with open(rep) as f:
        out = f.read()
else:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, isrc, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
stall_cols = [(i, k[len("stall_"):]) for i, k in enumerate(hdr)
              if k.startswith("stall_") and "Not Issued" not in k]
dyn = []
stalls = {}
for r in rows[2:]:
    if len(r) > iex and r[ia].startswith("0x"):
        a = int(r[ia], 16)
        dyn.append((a, r[isrc].strip(), int(r[iex] or 0)))
        stalls[a] = {name: int(r[i] or 0) for i, name in stall_cols}
base = dyn[0][0]

with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True,
                   capture_output=True)
    cub = glob.glob(os.path.join(d, "*.cubin"))[0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
sec = None
where = {}
cur = "?"
for line in dis.split("\n"):
    m = re.match(r"//-+ \.text\.(\S+) -+", line)
    if m:
        sec = m.group(1)
        continue
    if sec is None or not re.search(fun, sec):
        continue
    m = re.match(r"\s*//## File \"(.*)\", line (\d+)", line)
    if m:
        cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4})\*/\s+(.*?);", line)
    if m:
        where[int(m.group(1), 16)] = cur

per = collections.Counter()
ops = collections.defaultdict(collections.Counter)
why = collections.defaultdict(collections.Counter)
samples = collections.Counter()
miss = 0
for a, src, n in dyn:
    loc = where.get(a - base)
    if loc is None:
        miss += n
        continue
    per[loc] += n
    for k, v in stalls[a].items():
        why[loc][k] += v
        samples[loc] += v
    op = re.sub(r"^@!?U?P\w+\s+", "", src).split()[0] if src else "?"
    ops[loc][op.split(".")[0]] += n
tot = sum(per.values()) + miss
print(f"total {tot / units:.2f} per unit (unmapped {miss / units:.2f})")
if "--stalls" in sys.argv:
    all_s = sum(samples.values()) or 1
    for loc, v in samples.most_common(top):
        reasons = ", ".join(f"{k} {100 * c / v:.0f}%" for k, c in why[loc].most_common(3) if c)
        print(f"{100 * v / all_s:6.2f}%  {loc:28s} exec {per[loc] / units:7.2f}  {reasons}")
    sys.exit(0)
for loc, n in per.most_common(top):
    mix = ", ".join(f"{k} {v / units:.2f}" for k, v in ops[loc].most_common(5))
    print(f"{n / units:8.2f}  {loc:28s} {mix}")
