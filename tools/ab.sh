# A/B of library builds: bash tools/ab.sh CONFIG LIB1 LIB2 ... (a lib of "cur" = the in-tree build)
CFG=$1; shift
for i in 1 2; do
for v in "$@"; do
  if [ "$v" = cur ]; then unset CQB_LIB_PATH; else export CQB_LIB_PATH=$PWD/$v; fi
  echo -n "$CFG $v "; timeout 200 python bench.py --config $CFG --no-cpu-baseline --no-secondary 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['e2e']['value'],2))"
done; done
