# ncu --set full captures of the fused tier-L merges (C4 d5, d4, d3) and tier-M d8, d7
mkdir -p gpurun_out/ncu /tmp/ncu
cap() {  # name regex skip
  ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -f -o /tmp/ncu/$1 python tools/prof_run.py C4 1024 > gpurun_out/ncu/$1.log 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page raw --csv > gpurun_out/ncu/$1_raw.csv 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page details --csv > gpurun_out/ncu/$1_details.csv 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/ncu/$1_source_sass.csv.gz
}
cap l_d5_C4 merge_l_kernel 0
cap l_d4_C4 merge_l_kernel 1
cap l_d3_C4 merge_l_kernel 2
cap m2_d8_C4 merge_m2_kernel 1
ls -la gpurun_out/ncu
