# full GPU test suite + C4 1024 / C5 512 / C3 2048 / C2 1024 stage times for the in-tree library
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
python tools/prof_run.py C4 1024 2>&1 | head -1
python tools/prof_run.py C5 512 2>&1 | head -1
python tools/prof_run.py C3 2048 2>&1 | head -1
python tools/prof_run.py C2 1024 2>&1 | head -1
