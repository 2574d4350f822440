# A/B: the shipped libdsx.so vs build/variants/prev/libdsx.so on a bench config
cfg=${1:-mlp_wide}
cp paper_2502_11058_b200/lib/libdsx.so /tmp/libdsx_cur.so
for round in 1 2; do
for v in cur prev; do
  if [ $v = prev ]; then cp build/variants/prev/libdsx.so paper_2502_11058_b200/lib/libdsx.so; else cp /tmp/libdsx_cur.so paper_2502_11058_b200/lib/libdsx.so; fi
  timeout 300 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$v', '$cfg', d['value'], r.get('achieved'), (r.get('step') or {}).get('achieved'))"
done; done
cp /tmp/libdsx_cur.so paper_2502_11058_b200/lib/libdsx.so
