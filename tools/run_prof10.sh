# full capture of the canonical kernels at c3 (the plain command must exit 0 first; one ncu per call)
python tools/prof_apply.py --config c3 --reps 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_canon -c 2 -o gpurun_out/prof_r01b_c3 python tools/prof_apply.py --config c3 --reps 1 > gpurun_out/p10_ncu.log 2>&1
echo rc $?
