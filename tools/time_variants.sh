#!/bin/bash
# time fwd/inv cfg3 for the default library and each variant given as args
for v in "" "$@"; do
  for op in fwd inv; do
    if [ -z "$v" ]; then lib=paper_2103_16400_b200/libnttkit_b200.so; else lib=paper_2103_16400_b200/libnttkit_b200_$v.so; fi
    echo -n "[${v:-default}] "; NK_LIB_PATH=$lib timeout 60 python tools/prof_ntt.py --op $op --iters 20
  done
done
