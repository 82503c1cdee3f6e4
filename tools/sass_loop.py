"""Static instruction mix of a kernel's hottest loop (CPU-side proxy for the
issue-slot cost of a change, before spending GPU time on it).

    python tools/sass_loop.py [object-or-so] [function-regex]

Defaults: the C2 level kernel (ArithF32, no Kahan, all legs, table,
no dump) from the in-tree build.  The loop is the outermost backward branch
whose body holds FP64 work; nested loops (the warp-uniform tail pass) are
counted once.
"""
from __future__ import annotations

import collections
import re
import subprocess
import sys

ROOT = __file__.rsplit("/tools/", 1)[0]
ARGS = [a for a in sys.argv[1:] if not a.startswith("--")]
OBJ = ARGS[0] if len(ARGS) > 0 else f"{ROOT}/paper_2012_09739_b200/_build/lpmc_level_f32.cu.o"
FUN = ARGS[1] if len(ARGS) > 1 else r"level_kernelINS0_8ArithF32ELb0ELi3ELi1ELb0ELi0E"

sass = subprocess.run(["cuobjdump", "-sass", OBJ], capture_output=True, text=True, check=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
body = next(f for f in funcs[1:] if re.search(FUN, f.split("\n", 1)[0]))
ins = []
for line in body.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
loops = []
for i, (a, text) in enumerate(ins):
    m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)\s*)?(?:.*?)0x([0-9a-f]+)", text)
    if m and "BRA" in text:
        tgt = int(m.group(1), 16)
        if tgt < a and tgt in addr:
            loops.append((addr[tgt], i))


def opclass(text):
    t = re.sub(r"^@!?U?P\w+\s+", "", text)
    op = t.split()[0]
    return op


if "--list" in sys.argv:
    for lo, hi in sorted(loops):
        c = collections.Counter(opclass(t).split(".")[0] for _, t in ins[lo:hi + 1])
        print(f"{ins[lo][0]:#x}..{ins[hi][0]:#x} {hi - lo + 1:5d} DFMA {c['DFMA']} CALL {c['CALL']} "
              f"LDL {c['LDL']}")
best = None
for lo, hi in loops:
    ops = [opclass(t) for _, t in ins[lo:hi + 1]]
    if any(o.startswith(("DFMA", "DADD", "DMUL")) for o in ops):
        if best is None or hi - lo > best[1] - best[0]:
            best = (lo, hi)
lo, hi = best
ops = [opclass(t) for _, t in ins[lo:hi + 1]]
cnt = collections.Counter(o.split(".")[0] for o in ops)
fp64 = sum(v for k, v in cnt.items() if k in ("DFMA", "DADD", "DMUL", "DSETP", "DMNMX", "F2F", "I2F",
                                              "F2I", "DSET", "MUFU"))
print(f"loop {ins[lo][0]:#x}..{ins[hi][0]:#x}: {hi - lo + 1} instructions")
print("  " + ", ".join(f"{k} {v}" for k, v in cnt.most_common()))
print(f"  DFMA/DADD/DMUL/DSETP {sum(cnt[k] for k in ('DFMA', 'DADD', 'DMUL', 'DSETP'))}, "
      f"conversions+MUFU {sum(cnt[k] for k in ('F2F', 'I2F', 'F2I', 'MUFU'))}")
