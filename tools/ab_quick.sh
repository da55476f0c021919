# parity subset (tier-L paths) + C4 1024 / C5 512 stage times for the in-tree library
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py tests/test_gpu_lowrank.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
python tools/prof_run.py C4 1024 2>&1 | head -1
python tools/prof_run.py C5 512 2>&1 | head -1
python tools/prof_run.py C3 2048 2>&1 | head -1
