#!/usr/bin/env python
"""Instruction-class sequence of one kernel's SASS (run-length compressed):
F = FP64, l = LDS, s = STS, G = LDG, W = STG, | = BAR, y = SYNCS (mbarrier), b = BRA, . = other.
   python tools/sass_shape.py <object-or-so> <mangled-name-substring>"""
import re
import subprocess
import sys

obj, pat = sys.argv[1], sys.argv[2]
txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
cur, ops = None, []
for line in txt.split("\n"):
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    if cur and pat in cur:
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_]+)", line)
        if m:
            ops.append(m.group(1))
cls = {"DADD": "F", "DMUL": "F", "DFMA": "F", "LDS": "l", "STS": "s", "LDG": "G", "STG": "W", "BAR": "|", "SYNCS": "y",
       "BRA": "b"}
st = "".join(cls.get(o, ".") for o in ops)
out, i = [], 0
while i < len(st):
    j = i
    while j < len(st) and st[j] == st[i]:
        j += 1
    out.append(f"{st[i]}{j - i}" if j - i > 1 else st[i])
    i = j
print(len(ops), "instructions")
print(" ".join(out))
