python tools/kprof.py --config c3 2>&1 | tail -20
for i in 1 2; do timeout 300 python bench.py --config c3 --steps 40 --warmup 5 --cpu-seconds 1 --no-extra 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c3',d['value'],d['ms_per_step'],d['clocks'])"; done
