RING_R_MULT=140 RING_GROUPS=1,4,10,14 timeout 600 python tools/ring_groups.py 2>&1 | grep "us/frame\|PARITY"
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
