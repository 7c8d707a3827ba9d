timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/t10_pytest.log 2>&1; tail -2 gpurun_out/t10_pytest.log
python tools/kprof.py --config c3 2>&1 | grep -E "event|k_canon|k_fixup"
python tools/kprof.py --config c5 2>&1 | grep -E "event|k_canon|k_fixup"
for C in c3 c5; do timeout 300 python bench.py --config $C --cpu-seconds 1 --no-extra 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$C',d['value'],d['ms_per_step'],d['roofline']['frac'],d['clocks'])"; done
