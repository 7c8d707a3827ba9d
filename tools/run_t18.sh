timeout 1200 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/t18_pytest.log 2>&1; tail -1 gpurun_out/t18_pytest.log
timeout 600 python bench.py > gpurun_out/t18_bench.json 2> gpurun_out/t18_bench.err; echo rc $?
python - <<'P'
import json
d=json.loads(open('gpurun_out/t18_bench.json').read().strip().splitlines()[-1])
r=d['roofline']
print('c3', round(d['value'],3), round(d['ms_per_step'],4), 'frac', round(r['frac'],4), 'step', round(r['step_frac'],4), 'e2e', d['e2e']['value'], d['clocks'])
print(json.dumps(d['configs']))
print(json.dumps(d['cpu_baseline']))
P
