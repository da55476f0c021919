# final lib: full GPU tests, smoke, driver-style bench + reference arm, launch list of prof_run
mkdir -p gpurun_out/ncu
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
t0=$(date +%s); python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc $? wall $(( $(date +%s) - t0 )) s"
t0=$(date +%s); python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref bench rc $? wall $(( $(date +%s) - t0 )) s"
python tools/prof_run.py C4 1024 > gpurun_out/prof_C4.txt 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches_C4_1024.csv python tools/prof_run.py C4 1024 > /dev/null 2>&1
head -1 gpurun_out/prof_C4.txt
