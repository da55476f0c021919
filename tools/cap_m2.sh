mkdir -p gpurun_out/ncu /tmp/ncu
for sk in 0 1; do
ncu --set full --clock-control none --import-source on -k regex:merge_m2_kernel -s $sk -c 1 -f -o /tmp/ncu/m2_$sk python tools/prof_run.py C4 1024 > /dev/null 2>&1
ncu -i /tmp/ncu/m2_$sk.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/ncu/m2cur_${sk}_sass.csv.gz
ncu -i /tmp/ncu/m2_$sk.ncu-rep --page raw --csv 2>&1 > gpurun_out/ncu/m2cur_${sk}_raw.csv
done
