# usage: bash tools/ab_libs.sh VARIANT...  (default = in-tree lib; others build/ab/libhdd_V.so): stage times on C4 1024, C5 512, C2 1024
for v in "$@"; do
  if [ $v = default ]; then e=""; else e="HDD_LIB_PATH=build/ab/libhdd_$v.so"; fi
  for c in ${AB_CASES:-"C4 1024" "C5 512" "C2 1024"}; do echo "$v $(env $e python tools/prof_run.py $c 2>&1 | head -1)"; done
done
