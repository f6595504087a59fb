RING_R_MULT=120 RING_GROUPS=8,10,12 timeout 600 python tools/ring_groups.py 2>&1 | grep "us/frame\|PARITY"
RING_R_MULT=126 RING_GROUPS=7,9,14,18 timeout 600 python tools/ring_groups.py 2>&1 | grep "us/frame\|PARITY"
