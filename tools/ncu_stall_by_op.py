#!/usr/bin/env python
"""Stall samples per opcode (and per stall reason) for one kernel of an ncu report."""
import collections, csv, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
which = int(sys.argv[3]) if len(sys.argv) > 3 else 0
if rep.endswith(".csv.gz") or rep.endswith(".csv"):  # a --page source export (tools/gpu_check.sh)
    import gzip, re
    txt = (gzip.open(rep, "rt") if rep.endswith(".gz") else open(rep)).read()
    # keep the blocks of kernels matching kre
    parts = txt.split('"Kernel Name"')
    out = "".join('"Kernel Name"' + p for p in parts[1:] if re.search(kre, p.splitlines()[0]))
else:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre],
                         capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = []
        blocks.append(cur)
    elif cur is not None:
        cur.append(r)
b = blocks[which]
hdr = b[0]
ix = {h: i for i, h in enumerate(hdr)}
sc = [h for h in hdr if h.startswith("stall_") and "Not" not in h]
agg = collections.defaultdict(collections.Counter)
tot = collections.Counter()
for r in b[1:]:
    if len(r) != len(hdr):
        continue
    toks = r[ix["Source"]].split()
    op = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "")
    op = op.split(".")[0]
    for h in sc:
        v = r[ix[h]]
        if v and v != "0":
            agg[op][h[6:]] += int(v)
            tot[h[6:]] += int(v)
T = sum(tot.values())
print("all:", ", ".join(f"{k}={100*v/T:.1f}%" for k, v in tot.most_common(10)))
for op, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:14]:
    s = sum(c.values())
    print(f"{op:8s} {100*s/T:5.1f}%  " + ", ".join(f"{k}={100*v/T:.1f}" for k, v in c.most_common(5)))
