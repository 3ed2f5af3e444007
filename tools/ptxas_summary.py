#!/usr/bin/env python
"""Registers and spill bytes per kernel from a build_ptxas*.log (demangled names).
   python tools/ptxas_summary.py [log] [name-filter]"""
import re
import subprocess
import sys

log = sys.argv[1] if len(sys.argv) > 1 else "paper_2103_16400_b200/build_ptxas.log"
flt = sys.argv[2] if len(sys.argv) > 2 else ""
name, out = None, {}
for line in open(log):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = m.group(1)
        out[name] = [0, 0, 0]
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and name:
        out[name][1:] = [int(m.group(1)), int(m.group(2))]
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        out[name][0] = int(m.group(1))
names = subprocess.run(["c++filt"], input="\n".join(out), capture_output=True, text=True).stdout.split("\n")
for mangled, dem in zip(out, names):
    dem = re.sub(r"\(CUtensorMap.*|\(nk::.*", "", dem).replace("void nk::", "").replace("nk::", "").replace("(bool)", "")
    if flt in dem:
        r = out[mangled]
        print(f"{dem:60s} regs {r[0]:3d}  spill st {r[1]:4d} ld {r[2]:4d}")
