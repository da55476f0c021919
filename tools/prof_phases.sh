# C4 and C5 (1024 / 512 samples): stage times + per-phase CTA clocks (ticks build) + a launch list
mkdir -p gpurun_out/ncu
HDD_LIB_PATH=build/ab/libhdd_ticks.so python tools/prof_run.py C4 1024 > gpurun_out/prof_C4.txt 2>&1
HDD_LIB_PATH=build/ab/libhdd_ticks.so python tools/prof_run.py C5 512 > gpurun_out/prof_C5.txt 2>&1
python tools/prof_run.py C4 1024 >> gpurun_out/prof_C4.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches_C4_1024.csv python tools/prof_run.py C4 1024 > /dev/null 2>&1
cat gpurun_out/prof_C4.txt gpurun_out/prof_C5.txt
