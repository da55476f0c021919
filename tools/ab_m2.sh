for v in 0 3 2; do echo "minb=$v $(HDD_M2_MINB=$v python tools/prof_run.py C4 1024 2>&1 | head -1)"; done
for v in 0 3 2; do echo "minb=$v $(HDD_M2_MINB=$v python tools/prof_run.py C2 1024 2>&1 | head -1)"; done
