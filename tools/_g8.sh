O=gpurun_out/t8; mkdir -p $O
for v in noex noexctw; do NK_LIB_PATH=paper_2103_16400_b200/libnttkit_b200_$v.so timeout 300 python tools/kvariants.py --kernels 2 > $O/kv_$v.jsonl 2>&1; done
cat $O/kv_noex.jsonl $O/kv_noexctw.jsonl
