# A/B/C.. of library builds on the device-resident quantize (tools/ab_debug.py, flag 0):
# bash tools/ab_multi.sh "CONFIGS" LIB1 LIB2 ... ("cur" = the in-tree build); 2 alternating rounds
for c in $1; do
  shift_done=0
  for i in 1 2; do
    for v in "${@:2}"; do
      if [ "$v" = cur ]; then unset CQB_LIB_PATH; else export CQB_LIB_PATH=$PWD/$v; fi
      echo -n "$c $v: "; timeout 200 python tools/ab_debug.py $c 0 1 2>&1 | head -1
    done
  done
done
