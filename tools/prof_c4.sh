# C4 (1024 samples): stage times + phase clocks (tick build: python tools/ab_build.py ticks HDD_PROFILE_TICKS), launch list, ncu --set full of the leaf,
# the first tier-M merge (d9) and the tier-L merge at depth 2; reports exported to CSV
# (raw metrics + source-level SASS hot spots, gzipped) under gpurun_out/ncu/.
mkdir -p gpurun_out/ncu /tmp/ncu
HDD_LIB_PATH=${HDD_LIB_PATH:-build/ab/libhdd_ticks.so} python tools/prof_run.py C4 1024 > gpurun_out/prof_C4.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches_C4_1024.csv python tools/prof_run.py C4 1024 > /dev/null 2>&1
cap() {  # name regex skip
  ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -f -o /tmp/ncu/$1 python tools/prof_run.py C4 1024 > gpurun_out/ncu/$1.log 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page raw --csv > gpurun_out/ncu/$1_raw.csv 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page details --csv > gpurun_out/ncu/$1_details.csv 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/ncu/$1_source_sass.csv.gz
}
cap leaf_C4 leaf2_kernel 0
cap m2_d9_C4 merge_m2_kernel 0
cap m2_d6_C4 merge_m2_kernel 3
cap l_d2_C4 merge_l_kernel 3
cat gpurun_out/prof_C4.txt
ls -la gpurun_out/ncu
