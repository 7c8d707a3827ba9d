timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/exp3_pytest.log 2>&1; tail -3 gpurun_out/exp3_pytest.log
for c in c3 c5; do echo "== $c"; timeout 120 python tools/kprof.py --config $c --reps 10 2>&1 | grep -E "event|k_canon|fixup|rror" | cut -c1-60,120-150; done
