timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/t12_pytest.log 2>&1; tail -2 gpurun_out/t12_pytest.log
timeout 600 python bench.py --cpu-seconds 2 > gpurun_out/b12.json 2> gpurun_out/b12.err; tail -2 gpurun_out/b12.err
python -c "import json;d=json.load(open('gpurun_out/b12.json'));print('c3',d['value'],d['ms_per_step'],d['roofline']['frac'],d['clocks'],d['e2e']);print(json.dumps(d['configs']))"
