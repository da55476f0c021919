# final round-2 evidence: full GPU tests, smoke, driver-style bench, launch list of the same bench command, ncu --set full of the
# dominant kernel at its three depths + leaf + tier-M d9/d7 + schur_l (C4, 1024 samples)
mkdir -p gpurun_out/ncu /tmp/ncu
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
t0=$(date +%s); python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc $? wall $(( $(date +%s) - t0 )) s"
t0=$(date +%s); python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref bench rc $? wall $(( $(date +%s) - t0 )) s"
python bench.py --steps 1 --warmup 1 --batch 2048 --no-per-config --no-cpu-baseline > gpurun_out/bench_2048.json 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu/launches_bench.csv python bench.py --steps 1 --warmup 1 --batch 2048 --no-per-config --no-cpu-baseline > /dev/null 2>&1
python tools/prof_run.py C4 1024 > gpurun_out/prof_C4.txt 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches_C4_1024.csv python tools/prof_run.py C4 1024 > /dev/null 2>&1
cap() {  # name regex skip
  ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -f -o /tmp/ncu/$1 python tools/prof_run.py C4 1024 > gpurun_out/ncu/$1.log 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page raw --csv > gpurun_out/ncu/$1_raw.csv 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page details --csv > gpurun_out/ncu/$1_details.csv 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/ncu/$1_sass.csv.gz
}
# prof_run does 2 forwards: skip the first forward's launches (merge_l_kernel: d5 d4 d3 d2 d1 d0 = 6 per forward)
cap l_d5_C4 merge_l_kernel 6
cap l_d4_C4 merge_l_kernel 7
cap l_d3_C4 merge_l_kernel 8
cap leaf_C4 leaf2_kernel 1
cap m2_d9_C4 merge_m2_kernel 4
cap m2_d7_C4 merge_m2_kernel 6
cap schur_l_d2_C4 schur_l_kernel 6
cat gpurun_out/prof_C4.txt | head -1
ls -la gpurun_out/ncu | tail -30
