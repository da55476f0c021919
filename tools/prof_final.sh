# Round-2 final captures of the current build (C4, 1024 samples): launch list of the
# driver's bench command (first 400 launches), ncu --set full raw metrics of the top kernels
mkdir -p gpurun_out/final /tmp/ncu
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches_bench_C4.csv python bench.py --steps 1 --warmup 1 --batch 4096 --no-cpu-baseline --no-per-config > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_C4_1024.csv python tools/prof_run.py C4 1024 > /dev/null 2>&1
cap() {  # name regex skip
  ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -f -o /tmp/ncu/$1 python tools/prof_run.py C4 1024 > gpurun_out/final/$1.log 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page raw --csv > gpurun_out/final/$1_raw.csv 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page details --csv > gpurun_out/final/$1_details.csv 2>&1
}
cap leaf_C4 leaf2_kernel 0
cap m2_d9_C4 merge_m2_kernel 0
cap m2_d6_C4 merge_m2_kernel 3
cap l_d4_C4 merge_l_kernel 1
cap l_d2_C4 merge_l_kernel 3
cap schur_l_d2_C4 schur_l_kernel 0
ls -la gpurun_out/final
