#!/usr/bin/env python
"""Summarise an ncu --set full report into profiles/ncu_summary.json (per
kernel: duration, dram bytes, pipe utilisation) for bench.py's `traffic`.

    python tools/ncu_to_json.py gpurun_out/x/prof.ncu-rep profiles/ncu_summary.json "<note>"
"""
import csv, json, re, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
note = sys.argv[3] if len(sys.argv) > 3 else ""
if rep.endswith(".csv"):  # a --page raw --csv export (tools/gpu_check.sh)
    raw = open(rep).read()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
keep = {"gpu__time_duration.sum": "duration", "dram__bytes_read.sum": "dram_bytes_read",
        "dram__bytes_write.sum": "dram_bytes_write",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
        "launch__registers_per_thread": "registers", "launch__grid_size": "grid",
        "sm__cycles_elapsed.avg.per_second": "sm_clock"}
scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "us": 1e-6, "ms": 1e-3, "ns": 1e-9,
         "Ghz": 1e9, "Mhz": 1e6, "hz": 1}
res = {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d.get("Kernel Name", "")
    m = re.search(r"(\w+)<(?:nk::)?(\w+), (?:\(bool\))?(\d)", name)
    m1 = re.search(r"(\w+)<(?:nk::)?(\w+)>", name)  # one template argument (poly_mul14<A>)
    if m and m.group(1) in ("ntt_str14", "ntt_stri14"):  # the direction is in the kernel's name
        key = f"{m.group(1)}<{m.group(2)},{'fwd' if m.group(1) == 'ntt_str14' else 'inv'}>"
    else:
        key = (f"{m.group(1)}<{m.group(2)},{'fwd' if m.group(3) == '1' else 'inv'}>" if m
               else f"{m1.group(1)}<{m1.group(2)}>" if m1 else name[:60])
    e = {}
    for k, short in keep.items():
        if k in d and d[k]:
            v = float(d[k].replace(",", ""))
            u = units[hdr.index(k)]
            e[short] = v * scale.get(u, 1.0)
    res.setdefault(key, e)  # first launch of each kernel
json.dump({"source": rep, "note": note, "kernels": res}, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
