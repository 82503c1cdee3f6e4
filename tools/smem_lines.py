"""Shared-memory wavefronts (actual vs ideal) per SASS instruction of the
kernel in an ncu report (--set full --import-source on): which loads carry
bank conflicts.  The shared-memory crossbar moves one 128-byte wavefront per
cycle per SM, so wavefronts per path-step bound the kernel like issue slots.

    python tools/smem_lines.py rep.ncu-rep
"""
from __future__ import annotations

import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Address" in r)
ia, isrc = hdr.index("Address"), hdr.index("Source")
iw, iwi = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Ideal")
by_addr = {}
for r in rows[rows.index(hdr) + 1:]:
    if len(r) <= iw or not r[ia].startswith("0x"):
        continue
    w = float(r[iw] or 0)
    if w:
        by_addr[int(r[ia], 16)] = (w, float(r[iwi] or 0), r[isrc].strip())

tot = sum(w for w, _, _ in by_addr.values())
tid = sum(i for _, i, _ in by_addr.values())
print(f"total wavefronts {tot:.4g}, ideal {tid:.4g} (excess {tot / max(tid, 1) - 1:.1%})")
for a, (w, i, s) in sorted(by_addr.items(), key=lambda kv: -kv[1][0])[:40]:
    print(f"  {a:#07x} {w:12.4g} ideal {i:12.4g} x{w / max(i, 1):.2f}  {s}")
