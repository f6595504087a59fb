for G in 8 14 16; do
  echo "== G=$G model split"
  FT_DEBUG_GEOMETRY=1 RING_GROUPS=$G timeout 300 python tools/ring_groups.py > /tmp/rs.txt 2>&1
  grep "us/frame\|PARITY\|Error" /tmp/rs.txt; grep -o "W=[0-9]* Gs=[0-9]* Gm=[0-9]* smem=[0-9]* grid=[0-9]*" /tmp/rs.txt | sort | uniq -c | grep -v "Gs=80"
done
