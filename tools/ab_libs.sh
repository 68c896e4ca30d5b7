# A/B of library builds on the device-resident quantize: bash tools/ab_libs.sh CONFIG LIB_A LIB_B [rounds]
# (a lib of "cur" = the in-tree build); prints ms/step medians from tools/ab_debug.py (flag 0 only)
CFG=$1; A=$2; B=$3; R=${4:-3}
for i in $(seq $R); do
  for v in $A $B; do
    if [ "$v" = cur ]; then unset CQB_LIB_PATH; else export CQB_LIB_PATH=$PWD/$v; fi
    echo -n "$CFG $v: "; timeout 200 python tools/ab_debug.py $CFG 0 1 2>&1 | head -1
  done
done
