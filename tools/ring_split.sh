for d in -1 1 0; do
  echo "== FT_DYN_TAIL=$d"
  if [ $d = -1 ]; then unset FT_DYN_TAIL; else export FT_DYN_TAIL=$d; fi
  FT_DEBUG_GEOMETRY=1 RING_R_MULT=140 RING_GROUPS=1,4,10,14 timeout 600 python tools/ring_groups.py > /tmp/rs.txt 2>&1
  grep "us/frame\|PARITY" /tmp/rs.txt
done
unset FT_DYN_TAIL
timeout 200 python tools/debug_pipe.py | tail -2
