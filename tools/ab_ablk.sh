timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 900 env HDD_L_ABLK=2 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for cfg in "C4 1024" "C5 512" "C3 2048"; do
  for v in 0 1 2; do echo "ablk=$v $(HDD_L_ABLK=$v python tools/prof_run.py $cfg 2>&1 | head -1)"; done
done
