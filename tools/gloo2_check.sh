#!/bin/bash
# Two ranks sharing the one GPU (gloo): the sharded bench path and its reference arm.
#   gpurun -- bash tools/gloo2_check.sh r02i
T=${1:-run}; O=gpurun_out/$T; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 --dist-backend gloo > $O/bench_gloo2.json 2> $O/bench_gloo2.err; echo "gloo2=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 3 --warmup 1 --dist-backend gloo > $O/bench_ref2.json 2> $O/bench_ref2.err; echo "ref2=$?"
