O=gpurun_out/t9; mkdir -p $O
export NK_LIB_PATH=paper_2103_16400_b200/libnttkit_b200_noexctw.so
timeout 300 python tools/prof_ntt.py --kernel 2 --op inv --iters 2 > $O/plain.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ntt_grp -s 1 -c 1 -o $O/skel_inv python tools/prof_ntt.py --kernel 2 --op inv --iters 2 > $O/ncu_inv.log 2>&1
for r in $O/*.ncu-rep; do ncu -i "$r" --page raw --csv > "${r%.ncu-rep}_raw.csv" 2>/dev/null; done
ls $O
