#!/bin/bash
# Copies the judged summaries of one tools/gpu_check.sh run (gpurun_out/<tag>) into profiles/
# under the tag's name and regenerates profiles/ncu_summary.json (bench.py's `traffic`).
#   bash tools/collect_profiles.sh r02h
set -e
T=$1; O=gpurun_out/$T; P=profiles
cp $O/bench.json $P/bench_$T.json
cp $O/bench_ref.json $P/bench_ref_$T.json
cp $O/cfgs.jsonl $P/cfgs_$T.jsonl
cp $O/api_latency.txt $P/api_latency_$T.txt
tail -3 $O/pytest_gpu.log > $P/gpu_tests_$T.log
cp $O/launches.csv $P/launches_$T.csv
cp $O/launches_cfg4.csv $P/launches_cfg4_$T.csv
cp $O/launches_cfg5.csv $P/launches_cfg5_$T.csv
cp $O/launches_poly4096.csv $P/launches_poly4096_$T.csv
cp $O/polyblk.jsonl $P/polyblk_$T.jsonl
python tools/ncu_summary.py $O/prof_raw.csv > $P/ncu_${T}_cfg3.txt
python tools/ncu_summary.py $O/prof_poly_raw.csv > $P/ncu_${T}_poly.txt
python tools/ncu_summary.py $O/prof_elt_raw.csv > $P/ncu_${T}_eltwise_steady.txt
python tools/ncu_stall_by_op.py $O/prof_source.csv.gz ntt_str14 > $P/ncu_${T}_fwd_stalls.txt
python tools/ncu_stall_by_op.py $O/prof_source.csv.gz ntt_stri14 > $P/ncu_${T}_inv_stalls.txt
python tools/ncu_stall_by_op.py $O/prof_poly_source.csv.gz poly_ > $P/ncu_${T}_poly_stalls.txt
python - "$T" <<'PY'
import json, subprocess, sys
t = sys.argv[1]
a = json.loads(subprocess.run(["python", "tools/ncu_to_json.py", f"gpurun_out/{t}/prof_raw.csv", "/tmp/_a.json"], capture_output=True, text=True).stdout)
b = json.loads(subprocess.run(["python", "tools/ncu_to_json.py", f"gpurun_out/{t}/prof_poly_raw.csv", "/tmp/_b.json"], capture_output=True, text=True).stdout)
a.update(b)
json.dump({"source": f"gpurun_out/{t}/prof_raw.csv, gpurun_out/{t}/prof_poly_raw.csv",
           "note": f"{t}: ncu --set full of tools/prof_ntt.py (cfg3 shape, forward + inverse; cfg5 shape, poly_mult_mod), per launch",
           "kernels": a}, open("profiles/ncu_summary.json", "w"), indent=1)
print(json.dumps(a, indent=1))
PY
