# ncu --set full (source attribution) of the tier-M merges at C4 d9 and d6
mkdir -p gpurun_out/ncu /tmp/ncu
cap() {  # name regex skip
  ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -f -o /tmp/ncu/$1 python tools/prof_run.py C4 1024 > gpurun_out/ncu/$1.log 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page raw --csv > gpurun_out/ncu/$1_raw.csv 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/ncu/$1_sass.csv.gz
}
cap m2_d9_C4 merge_m2_kernel 0
cap m2_d6_C4 merge_m2_kernel 3
ls -la gpurun_out/ncu | tail -4
