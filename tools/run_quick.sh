# quick check of a kernel change: parity subset + bench line (all configs); $1 = tag
T=${1:-q}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "multitile or full_size or kkt or edge or determinism" > gpurun_out/${T}_pytest.log 2>&1; tail -2 gpurun_out/${T}_pytest.log
timeout 600 python bench.py --steps 100 --cpu-seconds 2 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo bench rc $?
python - "$T" <<'P'
import json,sys
d=json.loads(open('gpurun_out/%s_bench.json'%sys.argv[1]).read().strip().splitlines()[-1])
r=d['roofline']
print('c3 %.3f GDoF/s %.4f ms  dom %.4f ms frac %.4f  step %.4f  clocks %s' % (d['value'], d['ms_per_step'], r['kernel_ms'], r['frac'], r['step_frac'], d['clocks']))
for k,v in d['configs'].items():
    print(k, {a: (round(b,4) if isinstance(b,float) else b) for a,b in v.items()})
P
