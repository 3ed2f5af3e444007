#!/bin/bash
# One gpurun call: GPU parity tests, bench line, reference arm, launch lists,
# ncu --set full captures of the cfg3 transforms, of the element-wise
# kernels at steady state and of the single-kernel poly_mult_mod, all-config
# device times.
#   gpurun --timeout 2400 -- bash tools/gpu_check.sh [tag]
TAG=${1:-run}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
# the library is prebuilt here and travels with the snapshot
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest_gpu=$?" | tee -a $O/status
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench=$?" | tee -a $O/status
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "bench_ref=$?" | tee -a $O/status
timeout 300 ./tools/api_latency > $O/api_latency.txt 2>&1; echo "api_latency=$?" | tee -a $O/status
timeout 300 python tools/time_cfgs.py > $O/cfgs.jsonl 2>&1; echo "cfgs=$?" | tee -a $O/status
timeout 300 python tools/polyblk_bench.py > $O/polyblk.jsonl 2>&1; echo "polyblk=$?" | tee -a $O/status
if [ "${SKIP_NCU:-0}" = "0" ]; then
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-configs --no-records > $O/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-configs --no-records > $O/ncu_launch.log 2>&1
  echo "ncu_launch=$?" | tee -a $O/status
  timeout 300 python tools/prof_ntt.py --op both --iters 2 > $O/prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ntt -s 2 -c 2 \
      -o $O/prof python tools/prof_ntt.py --op both --iters 2 > $O/ncu_full.log 2>&1
  echo "ncu_full=$?" | tee -a $O/status
  timeout 120 python tools/prof_eltwise.py --big > $O/prof_elt_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none -k regex:eltwise -s 3 -c 3 \
      -o $O/prof_elt python tools/prof_eltwise.py --big > $O/ncu_elt.log 2>&1
  echo "ncu_elt=$?" | tee -a $O/status
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
      --log-file $O/launches_cfg4.csv python tools/prof_ntt.py --n 65536 --limbs 24 --polys 16 --bits 60 --fin 4 --iters 1 > $O/ncu_cfg4.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $O/launches_cfg5.csv python tools/prof_ntt.py --n 16384 --limbs 16 --polys 128 --op poly --iters 1 > $O/ncu_cfg5.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $O/launches_poly4096.csv python tools/prof_ntt.py --n 4096 --limbs 16 --polys 512 --op poly --iters 1 > $O/ncu_poly4096.log 2>&1
  echo "ncu_cfg45=$?" | tee -a $O/status
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:poly_ -s 1 -c 1 \
      -o $O/prof_poly python tools/prof_ntt.py --n 16384 --limbs 16 --polys 128 --op poly --iters 2 > $O/ncu_poly.log 2>&1
  echo "ncu_poly=$?" | tee -a $O/status
fi
cat $O/status
tail -3 $O/pytest_gpu.log
# keep the merge-back under gpurun's 64 MiB cap: text exports of every report,
# the binary reports only when small
for r in $O/*.ncu-rep; do
  [ -f "$r" ] || continue
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}_raw.csv" 2>/dev/null
  ncu -i "$r" --page details --csv > "${r%.ncu-rep}_details.csv" 2>/dev/null
  ncu -i "$r" --page source --csv --print-source sass > "${r%.ncu-rep}_source.csv" 2>/dev/null
  gzip -f "${r%.ncu-rep}_source.csv"
  [ $(stat -c %s "$r") -gt 15000000 ] && rm -f "$r"
done
du -sh $O
