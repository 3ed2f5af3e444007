#!/usr/bin/env python
"""Split a kernel's SASS (ncu --page source, sass view) into regions at
barriers and report where the warp-stall samples fall, plus an opcode mix.

    python tools/ncu_sass_phases.py gpurun_out/x/prof.ncu-rep [kernel-regex] [launch-index]
"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "ntt"
if rep.endswith(".csv") or rep.endswith(".csv.gz"):  # a --page source export (tools/gpu_check.sh)
    import gzip
    import re
    opener = gzip.open if rep.endswith(".gz") else open
    with opener(rep, "rt") as f:
        text = f.read()
    # keep the kernels whose name matches kre
    parts = re.split(r'(?m)^(?="Kernel Name")', text)
    out = "".join(p for p in parts if p.startswith('"Kernel Name"') and re.search(kre, p.splitlines()[0]))
else:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          "regex:" + kre], capture_output=True, text=True).stdout
lines = out.splitlines()
# multiple kernels: blocks start with "Kernel Name"
blocks, cur = [], None
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        cur = [ln]
        blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
which = int(sys.argv[3]) if len(sys.argv) > 3 else None
for bi, b in enumerate(blocks):
    if which is not None and bi != which:
        continue
    name = next(csv.reader([b[0]]))[1]
    rows = list(csv.reader(b[1:]))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = 0
    regions = []
    reg = {"n": 0, "samples": 0, "inst": 0, "first": None, "stalls": collections.Counter()}
    ops = collections.Counter()
    opsamp = collections.Counter()
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]].strip()
        toks = src.split()
        op = toks[0] if toks else ""
        if op.startswith("@"):
            op = toks[1] if len(toks) > 1 else op
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        ie = int(r[ix["Instructions Executed"]] or 0)
        tot += s
        base = op.split(".")[0]
        ops[base] += ie
        opsamp[base] += s
        if reg["first"] is None:
            reg["first"] = src[:50]
        reg["n"] += 1
        reg["samples"] += s
        reg["inst"] += ie
        for c in stall_cols:
            v = r[ix[c]]
            if v and v != "0":
                reg["stalls"][c[6:]] += int(v)
        if base in ("BAR", "SYNCS") and ("SYNC" in op or "ARRIVE" in op or "TRYWAIT" in op):
            regions.append(reg)
            reg = {"n": 0, "samples": 0, "inst": 0, "first": None, "stalls": collections.Counter()}
    regions.append(reg)
    print("==", name[:100], "total samples", tot)
    for i, g in enumerate(regions):
        if g["samples"] == 0:
            continue
        top = ", ".join(f"{k}={v}" for k, v in g["stalls"].most_common(4))
        print(f"  region {i:2d}: {g['n']:5d} sass, inst {g['inst']:10d}, samples {g['samples']:7d} "
              f"({100.0 * g['samples'] / max(1, tot):5.1f}%)  [{top}]  first: {g['first']}")
    itot = sum(ops.values())
    print("  opcode mix (dynamic warp-instr share / sample share):")
    for op, n in ops.most_common(22):
        print(f"    {op:10s} {100.0 * n / itot:5.1f}%  {100.0 * opsamp[op] / max(1, tot):5.1f}%")
