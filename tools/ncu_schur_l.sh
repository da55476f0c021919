mkdir -p gpurun_out/ncu /tmp/ncu
# schur_l launches: d5 32 nodes, d4 16, d3 8, d2 4 (in this order); capture one d5 node and one d2 node
for sk in 0 56; do
ncu --set full --clock-control none -k regex:schur_l_kernel -s $sk -c 1 -f -o /tmp/ncu/sl_$sk python tools/prof_run.py C4 1024 > /dev/null 2>&1
ncu -i /tmp/ncu/sl_$sk.ncu-rep --page details --csv > gpurun_out/ncu/sl_${sk}_details.csv 2>&1
ncu -i /tmp/ncu/sl_$sk.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/ncu/sl_${sk}_sass.csv.gz
done
