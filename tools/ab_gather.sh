# split tier L with the son-gathering schur_l epilogue (HDD_SCHUR_GATHER) on every tier-L depth vs the default
timeout 900 env HDD_SCHUR_GATHER=1 HDD_SCHUR_L_MIN_NG=1 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "split or global_panel or C4 or C5" 2>&1 | tail -2
for cfg in "C4 1024" "C5 512"; do
  echo "default  $(python tools/prof_run.py $cfg 2>&1 | head -1)"
  echo "gather   $(HDD_SCHUR_GATHER=1 python tools/prof_run.py $cfg 2>&1 | head -1)"
  echo "gall     $(HDD_SCHUR_GATHER=1 HDD_SCHUR_L_MIN_NG=1 python tools/prof_run.py $cfg 2>&1 | head -1)"
  echo "splitall $(HDD_SCHUR_L_MIN_NG=1 python tools/prof_run.py $cfg 2>&1 | head -1)"
done
