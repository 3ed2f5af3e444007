mkdir -p gpurun_out/t1
nvidia-smi > gpurun_out/t1/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t1/pytest.log 2>&1; echo "pytest=$?" >> gpurun_out/t1/status
timeout 300 python bench.py > gpurun_out/t1/bench.json 2> gpurun_out/t1/bench.err; echo "bench=$?" >> gpurun_out/t1/status
timeout 300 python tools/time_cfgs.py > gpurun_out/t1/cfgs.jsonl 2>&1; echo "cfgs=$?" >> gpurun_out/t1/status
cat gpurun_out/t1/status; tail -3 gpurun_out/t1/pytest.log; cat gpurun_out/t1/bench.json
