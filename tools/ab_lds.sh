timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for cfg in "C4 1024" "C5 512" "C2 1024"; do
  echo "new   $(python tools/prof_run.py $cfg 2>&1 | head -1)"
  echo "old8  $(HDD_PANEL_LD8=1 HDD_LIB_PATH=build/ab/libhdd_old8.so python tools/prof_run.py $cfg 2>&1 | head -1)"
  echo "ld8   $(HDD_PANEL_LD8=1 python tools/prof_run.py $cfg 2>&1 | head -1)"
done
