timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/t16_pytest.log 2>&1; tail -1 gpurun_out/t16_pytest.log
timeout 300 python bench.py --config c4 --steps 50 --cpu-seconds 0.5 --no-extra 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('c4',round(d['value'],3),round(d['ms_per_step'],4),round(r['step_frac'],4), d['e2e'])"
