#!/bin/bash
# iteration helper: short parity subset + timings (scratch output)
O=gpurun_out/${1:-q}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ntt.py tests/test_gpu_golden.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest=$?"; tail -2 $O/pytest.log
timeout 120 python tools/kvariants.py --reps 30 --kernels 1 2>&1 | tee $O/kv.log
timeout 120 python tools/kvariants.py --reps 30 --kernels 1 --n 65536 --limbs 24 --polys 16 --bits 60 --fin 4 2>&1 | tee -a $O/kv.log
timeout 120 python tools/prof_ntt.py --n 16384 --limbs 16 --polys 128 --op poly --iters 20 2>&1 | tee -a $O/kv.log
