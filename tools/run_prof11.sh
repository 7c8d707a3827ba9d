# full capture of the canonical kernels at c5 (plain command first; one ncu per call)
python tools/prof_apply.py --config c5 --reps 1 > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:k_canon -c 2 -o gpurun_out/prof_r01b_c5 python tools/prof_apply.py --config c5 --reps 1 > gpurun_out/p11_ncu.log 2>&1
echo rc $?
