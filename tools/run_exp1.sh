# experiment: stiffness kernel time with and without staging/sync / TMEM loads / X-stage LDS (results invalid in exp builds)
for v in base nosync notm nox; do
  if [ $v = base ]; then L=""; else L=$PWD/exp/libigalr_$v.so; fi
  echo "== $v"; IGALR_LIB=$L timeout 120 python tools/kprof.py --config c3 --reps 10 2>&1 | grep -E "event|k_canon|rror" | cut -c1-60,120-150
done > gpurun_out/exp1.txt
cat gpurun_out/exp1.txt
