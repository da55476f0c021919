# full GPU test suite + a source-level (SASS) ncu capture of the C4 leaf kernel
mkdir -p gpurun_out/ncu /tmp/ncu
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log
ncu --set full --clock-control none --import-source on -k regex:leaf2_kernel -c 1 -f -o /tmp/ncu/leaf python tools/prof_run.py C4 1024 > /dev/null 2>&1
ncu -i /tmp/ncu/leaf.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/ncu/leaf_C4_sass_cur.csv.gz
ls -la gpurun_out/ncu | tail -2
