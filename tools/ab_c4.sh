# A/B of build variants / tuning env on C4 (1024 samples, stage times, 2 runs each)
for v in default noticks tierl150; do
  case $v in
    default) env="" ;;
    noticks) env="HDD_LIB_PATH=build/ab/libhdd_noticks.so" ;;
    tierl150) env="HDD_TIER_L_KB=150" ;;
  esac
  for r in 1 2; do echo "$v: $(env $env python tools/prof_run.py C4 1024 2>&1 | head -1)"; done
done
