O=gpurun_out/t7; mkdir -p $O
timeout 300 python tools/kvariants.py --kernels 0,1,2,3 > $O/kv_cfg3.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_ntt.py -x -q -k "block_kernels" > $O/pytest_grp.log 2>&1; echo "pytest=$?" >> $O/status
cat $O/status; cat $O/kv_cfg3.jsonl; tail -2 $O/pytest_grp.log
