# quick parity subset + A/B stage times (C4 1024, C5 512) for env / library variants
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -4
for cfg in "C4 1024" "C5 512"; do
  for v in "${@:-default}"; do
    case $v in
      default) env="" ;;
      split) env="HDD_SCHUR_L_SPLIT=1" ;;
      split64) env="HDD_SCHUR_L_SPLIT=1 HDD_SCHUR_L_MIN_NG=64" ;;
      *) env="HDD_LIB_PATH=build/ab/libhdd_$v.so" ;;
    esac
    echo "$v $(env $env python tools/prof_run.py $cfg 2>&1 | head -1)"
  done
done
