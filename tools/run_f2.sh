timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/f2_pytest.log 2>&1; tail -2 gpurun_out/f2_pytest.log
for c in c3 c2 c4; do timeout 120 python tools/kprof.py --config $c 2>&1 | grep -E "event|k_canon|fixup|combos" | cut -c1-60,150-200; done
bash tools/run_quick.sh f2b 2>&1 | tail -8
