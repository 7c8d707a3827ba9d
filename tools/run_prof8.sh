# 1) plain bench (no ncu) must exit 0 first; 2) launch list of the same command; 3) full captures
python bench.py --steps 5 --warmup 3 --no-extra --cpu-seconds 0.5 > gpurun_out/p8_bench_plain.json 2> gpurun_out/p8_bench_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p8_launches_c3.csv python bench.py --steps 5 --warmup 3 --no-extra --cpu-seconds 0.5 > gpurun_out/p8_bench_ncu.log 2>&1
python tools/prof_apply.py --config c3 --reps 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_canon -c 2 -o gpurun_out/prof_final_c3 python tools/prof_apply.py --config c3 --reps 1 > /dev/null 2>&1
python tools/prof_apply.py --config c5 --reps 1 > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:k_canon -c 2 -o gpurun_out/prof_final_c5 python tools/prof_apply.py --config c5 --reps 1 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep | tail -3
