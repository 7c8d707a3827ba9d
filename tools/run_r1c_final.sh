# round-1 final evidence: default bench line; launch list of the same bench command; full captures
timeout 900 python bench.py > gpurun_out/r01c_bench.json 2> gpurun_out/r01c_bench.err; echo bench rc $?
python bench.py --steps 5 --warmup 3 --no-extra --cpu-seconds 0.5 > gpurun_out/r01c_bench_plain.json 2> gpurun_out/r01c_bench_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01c_launches_bench_c3.csv python bench.py --steps 5 --warmup 3 --no-extra --cpu-seconds 0.5 > gpurun_out/r01c_bench_ncu.log 2>&1; echo launches rc $?
python tools/prof_apply.py --config c3 --reps 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_canon|k_fixup" -c 4 -o gpurun_out/prof_r01c_c3 python tools/prof_apply.py --config c3 --reps 1 > gpurun_out/r01c_ncu_c3.log 2>&1; echo c3 rc $?
python tools/prof_apply.py --config c5 --reps 1 > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:"k_canon|k_fixup" -c 4 -o gpurun_out/prof_r01c_c5 python tools/prof_apply.py --config c5 --reps 1 > gpurun_out/r01c_ncu_c5.log 2>&1; echo c5 rc $?
ls -la gpurun_out/*.ncu-rep
