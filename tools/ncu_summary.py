#!/usr/bin/env python
"""Print the key metrics of an ncu report (run here, on the CPU box), or of
its `--page raw --csv` export (tools/gpu_check.sh writes *_raw.csv)."""
import csv, subprocess, sys
rep = sys.argv[1]
if rep.endswith(".csv"):
    out = open(rep).read()
else:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hdr, units = r[0], r[1]
keys = ['Kernel Name', 'gpu__time_duration.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__t_bytes.sum', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'launch__registers_per_thread',
        'smsp__inst_executed.sum', 'launch__grid_size', 'sm__cycles_elapsed.avg.per_second']
for row in r[2:]:
    d = dict(zip(hdr, row))
    for k in keys:
        if k in d:
            print(k[:80].ljust(80), units[hdr.index(k)][:10].ljust(10), d[k][:60])
    st = [(h, float(d[h])) for h in hdr if 'warps_issue_stalled' in h and h.endswith('per_issue_active.ratio') and d[h]]
    st.sort(key=lambda x: -x[1])
    print('stalls:', ', '.join(f"{h.split('stalled_')[1].split('_per')[0]}={v:.2f}" for h, v in st[:8]))
    print()
