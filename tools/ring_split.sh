FT_DEBUG_GEOMETRY=1 RING_R_MULT=140 RING_GROUPS=10,14,20,28,35 timeout 900 python tools/ring_groups.py > /tmp/rs.txt 2>&1
grep "us/frame\|PARITY\|Error" /tmp/rs.txt; grep -o "W=[0-9]* Gs=[0-9]* Gm=[0-9]* smem=[0-9]* grid=[0-9]*" /tmp/rs.txt | sort | uniq -c | grep -v "Gs=80"
