timeout 200 python tools/debug_pipe.py
for pairs in 1 0; do
  echo "== pairs=$pairs"
  FT_STEREO_PAIRS=$pairs RING_R_MULT=140 RING_GROUPS=1,4,10,14 timeout 600 python tools/ring_groups.py 2>&1 | grep "us/frame\|PARITY"
done
for gm in 3 4 5; do
  echo "== G=10 Gm=$gm"
  FT_GEOM_GM=$gm RING_R_MULT=140 RING_GROUPS=10 timeout 300 python tools/ring_groups.py 2>&1 | grep "us/frame\|PARITY"
done
FT_DEBUG_GEOMETRY=1 RING_R_MULT=140 RING_GROUPS=10 timeout 300 python tools/ring_groups.py 2>&1 | grep -o "W=[0-9]* Gs=[0-9]* Gm=[0-9]* smem=[0-9]* grid=[0-9]*" | sort | uniq -c
