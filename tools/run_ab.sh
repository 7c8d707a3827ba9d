# A/B timing: default in-tree library vs exp/libigalr_<tag>.so for each tag given
for t in default "$@"; do
  if [ $t = default ]; then L=""; else L=$PWD/exp/libigalr_$t.so; fi
  IGALR_LIB=$L timeout 300 python tools/ab_time.py c3 c5 c4 2>&1 | grep -v Warning
done
