for t in 0 1; do
  echo "== tails=$t"
  FT_GEOM_TAILS=$t FT_DEBUG_GEOMETRY=1 RING_R_MULT=140 RING_GROUPS=4,10,14 timeout 600 python tools/ring_groups.py > /tmp/rs.txt 2>&1
  grep "us/frame\|PARITY" /tmp/rs.txt; grep -o "W=[0-9]* Gs=[0-9]* Gm=[0-9]* smem=[0-9]* grid=[0-9]*" /tmp/rs.txt | sort | uniq -c | grep -v "Gs=80"
done
