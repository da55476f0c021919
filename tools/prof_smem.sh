# source-attributed captures (smem wavefronts) of tier-M d9/d6 and fused tier-L d4 (C4)
mkdir -p gpurun_out/smem /tmp/ncu
cap() {  # name regex skip
  ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -f -o /tmp/ncu/$1 python tools/prof_run.py C4 1024 > gpurun_out/smem/$1.log 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page raw --csv > gpurun_out/smem/$1_raw.csv 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/smem/$1_sass.csv.gz
}
cap m2_d9 merge_m2_kernel 0
cap m2_d6 merge_m2_kernel 3
cap l_d4 merge_l_kernel 1
ls gpurun_out/smem
