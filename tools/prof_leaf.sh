# ncu --set full of the C4 leaf kernel with source attribution
mkdir -p gpurun_out/ncu /tmp/ncu
ncu --set full --clock-control none --import-source on -k regex:leaf2_kernel -c 1 -f -o /tmp/ncu/leaf python tools/prof_run.py C4 1024 > gpurun_out/ncu/leaf.log 2>&1
ncu -i /tmp/ncu/leaf.ncu-rep --page raw --csv > gpurun_out/ncu/leaf_raw.csv 2>&1
ncu -i /tmp/ncu/leaf.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/ncu/leaf_sass.csv.gz
ncu -i /tmp/ncu/leaf.ncu-rep --page source --csv --print-source cuda 2>&1 | gzip > gpurun_out/ncu/leaf_cuda.csv.gz
ls -la gpurun_out/ncu/leaf*
