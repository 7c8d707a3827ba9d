for v in base unroll; do
  if [ $v = base ]; then L=""; else L=$PWD/exp/libigalr_$v.so; fi
  for c in c3 c5; do echo "== $v $c"; IGALR_LIB=$L timeout 120 python tools/kprof.py --config $c --reps 10 2>&1 | grep -E "event|k_canon|rror" | cut -c1-60,120-150; done
done
