timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "multitile or full_size or kkt or edge or determinism or mass_only" > gpurun_out/f1_pytest.log 2>&1; tail -2 gpurun_out/f1_pytest.log
for c in c3 c4 c2 c5; do timeout 120 python tools/kprof.py --config $c 2>&1 | grep -E "event|k_canon|fixup|combos" | cut -c1-60,150-200; done
for m in 2 4; do echo "minlen $m"; IGALR_MINLEN=$m timeout 120 python tools/kprof.py --config c2 2>&1 | grep -E "event|k_canon|fixup" | cut -c1-60,150-200; done
IGALR_MINLEN=2 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "multitile or c2 or kkt_full" > gpurun_out/f1_pytest_ml2.log 2>&1; tail -2 gpurun_out/f1_pytest_ml2.log
