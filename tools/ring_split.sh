RING_R_MULT=140 RING_GROUPS=1,4,10,14 timeout 600 python tools/ring_groups.py 2>&1 | grep "us/frame\|PARITY"
for gm in 3 4; do echo "== G=10 Gm=$gm"; FT_GEOM_GM=$gm RING_R_MULT=140 RING_GROUPS=10 timeout 300 python tools/ring_groups.py 2>&1 | grep "us/frame\|PARITY"; done
for gm in 2 3; do echo "== G=14 Gm=$gm"; FT_GEOM_GM=$gm RING_R_MULT=140 RING_GROUPS=14 timeout 300 python tools/ring_groups.py 2>&1 | grep "us/frame\|PARITY"; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
