# round-1 re-entry baseline: GPU tests, smoke, default bench line
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/c0_pytest.log 2>&1; tail -3 gpurun_out/c0_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c0_smoke.log 2>&1; echo smoke rc $?; tail -2 gpurun_out/c0_smoke.log
timeout 900 python bench.py > gpurun_out/c0_bench.json 2> gpurun_out/c0_bench.err; echo bench rc $?
python - <<'P'
import json
d=json.loads(open('gpurun_out/c0_bench.json').read().strip().splitlines()[-1])
r=d['roofline']
print('c3', round(d['value'],3), round(d['ms_per_step'],4), 'frac', round(r['frac'],4), 'step', round(r['step_frac'],4), 'e2e', d['e2e']['value'], d['clocks'])
print(json.dumps(d['configs']))
print(json.dumps(d['cpu_baseline']))
P
