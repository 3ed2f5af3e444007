#!/bin/bash
# One gpurun call: GPU parity tests, bench line, reference arm, launch list,
# and an ncu --set full capture of the NTT kernels.
#   gpurun --timeout 1500 -- bash tools/gpu_check.sh [tag]
TAG=${1:-run}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
make -s -C paper_2103_16400_b200 > $O/make.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest_gpu=$?" | tee -a $O/status
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench=$?" | tee -a $O/status
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "bench_ref=$?" | tee -a $O/status
if [ "${SKIP_NCU:-0}" = "0" ]; then
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
  echo "ncu_launch=$?" | tee -a $O/status
  timeout 300 python tools/prof_ntt.py --op ${PROF_OP:-both} --iters 2 > $O/prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${PROF_K:-ntt} -s ${PROF_S:-2} -c ${PROF_C:-2} \
      -o $O/prof python tools/prof_ntt.py --op ${PROF_OP:-both} --iters 2 > $O/ncu_full.log 2>&1
  echo "ncu_full=$?" | tee -a $O/status
  timeout 120 python tools/prof_eltwise.py > $O/prof_elt_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:eltwise -s 3 -c 3 \
      -o $O/prof_elt python tools/prof_eltwise.py > $O/ncu_elt.log 2>&1
  echo "ncu_elt=$?" | tee -a $O/status
fi
cat $O/status
tail -3 $O/pytest_gpu.log
cat $O/bench.json $O/bench_ref.json
