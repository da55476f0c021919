# the driver's bench command + a launch list of the same program (first 400 launches)
mkdir -p gpurun_out
t0=$(date +%s); python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench wall $(( $(date +%s) - t0 )) s"
tail -c 300 gpurun_out/bench_full.json; tail -3 gpurun_out/bench_full.err
