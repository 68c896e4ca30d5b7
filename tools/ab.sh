for i in 1 2 3; do
for v in old new; do
  if [ $v = old ]; then export CQB_LIB_PATH=$PWD/build/ab/old.so; else unset CQB_LIB_PATH; fi
  echo -n "$v "; timeout 200 python bench.py --no-cpu-baseline --no-secondary 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'])"
done; done
