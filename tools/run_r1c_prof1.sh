# source-level ncu capture of the c3 stiffness k_canon (one launch), for per-instruction stall analysis
python tools/prof_apply.py --config c3 --reps 1 > /dev/null 2>&1 || { echo plain run failed; exit 1; }
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:ShapeStiff -c 1 -o gpurun_out/prof_c1_c3stiff python tools/prof_apply.py --config c3 --reps 1 > gpurun_out/c1_ncu.log 2>&1
echo ncu rc $?
ncu -i gpurun_out/prof_c1_c3stiff.ncu-rep --page source --csv --print-source sass > gpurun_out/c1_src_sass.csv 2>&1; echo src rc $?
ls -la gpurun_out/
