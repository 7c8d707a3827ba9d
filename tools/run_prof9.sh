# launch list: the plain command must exit 0 first, then the same command under ncu (one ncu per call)
python bench.py --steps 5 --warmup 3 --no-extra --cpu-seconds 0.5 > gpurun_out/p9_bench_plain.json 2> gpurun_out/p9_bench_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p9_launches_c3.csv python bench.py --steps 5 --warmup 3 --no-extra --cpu-seconds 0.5 > gpurun_out/p9_bench_ncu.log 2>&1
echo rc $?
