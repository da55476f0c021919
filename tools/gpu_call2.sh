# sanitizer probe (one tool, smallest case), phase clocks of C4, low-rank block stats + stage times of C5 low-rank
mkdir -p gpurun_out
python tools/sanitize_run.py c1 > gpurun_out/sanitize_plain_c1.log 2>&1 && \
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_run.py c1 > gpurun_out/sanitizer_memcheck_c1.log 2>&1; echo "memcheck rc $?" >> gpurun_out/sanitizer_memcheck_c1.log
tail -5 gpurun_out/sanitizer_memcheck_c1.log
HDD_LIB_PATH=build/ab/libhdd_ticks.so python tools/prof_run.py C4 1024 > gpurun_out/prof_C4_ticks.txt 2>&1; cat gpurun_out/prof_C4_ticks.txt
python tools/prof_run.py C4 1024 2>&1 | head -1
HDD_LR_STATS=1 python tools/prof_run.py C5 256 lr > gpurun_out/prof_C5_lr.txt 2>&1; head -20 gpurun_out/prof_C5_lr.txt
python tools/prof_run.py C5 512 2>&1 | head -1
python bench.py --steps 1 --warmup 1 --batch 4096 --no-per-config > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err; tail -c 1500 gpurun_out/bench_small.json; tail -3 gpurun_out/bench_small.err
