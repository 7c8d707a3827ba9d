timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/t11_pytest.log 2>&1; tail -2 gpurun_out/t11_pytest.log
timeout 600 python bench.py --cpu-seconds 2 > gpurun_out/b11.json 2> gpurun_out/b11.err; tail -2 gpurun_out/b11.err
python -c "import json;d=json.load(open('gpurun_out/b11.json'));print('c3',d['value'],d['ms_per_step'],d['roofline']['frac'],d['clocks']);print(json.dumps(d['configs']))"
for Q in 1 2 4; do IGALR_QX=$Q timeout 300 python bench.py --config c4 --steps 20 --cpu-seconds 1 --no-extra 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c4 QX=$Q',d['value'],d['ms_per_step'],d['roofline']['frac'])"; done
IGALR_F2_MIN=1 timeout 300 python bench.py --config c2 --steps 50 --cpu-seconds 1 --no-extra 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c2 canon',d['value'],d['ms_per_step'],d['roofline']['frac'])"
