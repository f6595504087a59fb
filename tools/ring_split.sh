RING_R_MULT=140 RING_GROUPS=1,2,4,10,14 timeout 600 python tools/ring_groups.py 2>&1 | grep "us/frame\|PARITY"
timeout 600 python -m pytest tests/test_gpu_pipeline.py -x -q -k "ring or persistent" 2>&1 | tail -1
