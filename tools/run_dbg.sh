for args in "c2 64 m" "c2 64 s" "c3 128 s" "c3 128 m" "c2 64 s QX4" "c2 64 s QX1" "c2 64 s Y0" "c3 64 s"; do
  set -- $args
  Q=""; Y=""
  [ "$4" = "QX4" ] && Q=4; [ "$4" = "QX1" ] && Q=1; [ "$4" = "Y0" ] && Y=0
  IGALR_QX=$Q IGALR_YRES=$Y timeout 60 python tools/dbg_tma.py $1 $2 $3 2>&1 | grep -E "^OK|Error|error" | head -2
done
