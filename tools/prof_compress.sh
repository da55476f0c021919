# source-attributed capture of compress_kernel and compress_warp_kernel (C5 low-rank, 256 samples)
mkdir -p gpurun_out/lr /tmp/ncu
python tools/prof_run.py C5 256 lr | head -1
cap() {  # name regex skip
  ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -f -o /tmp/ncu/$1 python tools/prof_run.py C5 256 lr > gpurun_out/lr/$1.log 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page raw --csv > gpurun_out/lr/$1_raw.csv 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/lr/$1_sass.csv.gz
}
cap compress_d7 "compress_kernel" 4
cap cwarp_d11 "compress_warp_kernel" 0
ls gpurun_out/lr
