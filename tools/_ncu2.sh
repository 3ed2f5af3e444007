O=gpurun_out/n2; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ntt_str14 -s 2 -c 1 -o $O/prof python tools/prof_ntt.py --op fwd --iters 3 --kernel 2 > $O/ncu.log 2>&1
echo rc=$?
ncu -i $O/prof.ncu-rep --page raw --csv > $O/raw.csv
ncu -i $O/prof.ncu-rep --page source --csv --print-source sass > $O/source.csv; gzip -f $O/source.csv
rm -f $O/prof.ncu-rep
